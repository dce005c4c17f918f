// bfv_kernels.cu -- sm_100a kernels for the batched RNS-BFV cloud phase.
//
// Every kernel covers all RNS limbs of all items of a batch in one launch:
// elementwise kernels put one thread on one coefficient index k of one item
// (coalesced over k for every limb); NTTs run as two-phase tiled kernels.
// Formulas E1..E5 refer to DESIGN.md "Arithmetic spec"; the CPU oracle
// (oracle/bfv_oracle.c) states the same integer formulas.
#include <cstdio>
#include <map>
#include <mutex>
#include <type_traits>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "bfv_kernels.cuh"
#include "ntt.cuh"

namespace cssc {

#define CSSC_CHECK_LAUNCH()                                                            \
    do {                                                                               \
        cudaError_t e_ = cudaGetLastError();                                           \
        if (e_ != cudaSuccess)                                                         \
            throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e_)); \
    } while (0)

constexpr int EW_THREADS = 128;

__device__ __forceinline__ void add128(u64& hi, u64& lo, u64 xhi, u64 xlo) {
    lo += xlo;
    hi += xhi + (lo < xlo);
}

// ---------------------------------------------------------------------------
// ChaCha20 block (RFC 8439 2.3); key = the context's SeedKey (rns_params.hpp)
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 rotl32(u32 v, int n) { return __funnelshift_l(v, v, n); }

#define CSSC_QR(a, b, c, d)                         \
    a += b; d ^= a; d = rotl32(d, 16);              \
    c += d; b ^= c; b = rotl32(b, 12);              \
    a += b; d ^= a; d = rotl32(d, 8);               \
    c += d; b ^= c; b = rotl32(b, 7);

__device__ __forceinline__ void chacha20_block(const SeedKey& seed, u32 ctr, u32 n0, u32 n1, u32 n2, u32 out[16]) {
    const u32 s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                       seed.w[0],   seed.w[1],   seed.w[2],   seed.w[3],
                       seed.w[4],   seed.w[5],   seed.w[6],   seed.w[7],
                       ctr,         n0,          n1,          n2};
    u32 x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = s[i];
#pragma unroll 1
    for (int i = 0; i < 10; ++i) {
        CSSC_QR(x[0], x[4], x[8], x[12]);
        CSSC_QR(x[1], x[5], x[9], x[13]);
        CSSC_QR(x[2], x[6], x[10], x[14]);
        CSSC_QR(x[3], x[7], x[11], x[15]);
        CSSC_QR(x[0], x[5], x[10], x[15]);
        CSSC_QR(x[1], x[6], x[11], x[12]);
        CSSC_QR(x[2], x[7], x[8], x[13]);
        CSSC_QR(x[3], x[4], x[9], x[14]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) out[i] = x[i] + s[i];
}

// The same block computed by an aligned group of 4 lanes, one column each
// (lane i holds x[i], x[4+i], x[8+i], x[12+i]); diagonal rounds rotate rows
// b, c, d across the group with shuffles.  Lane i stores words i, 4+i, 8+i,
// 12+i of the output block.
__device__ __forceinline__ void chacha20_block_x4(const SeedKey& seed, u32 ctr, u32 n0, u32 n1, u32 n2, u32* out) {
    const int i = threadIdx.x & 3;
    const u32 sa = i == 0 ? 0x61707865u : i == 1 ? 0x3320646eu : i == 2 ? 0x79622d32u : 0x6b206574u;
    const u32 sb = i == 0 ? seed.w[0] : i == 1 ? seed.w[1] : i == 2 ? seed.w[2] : seed.w[3];
    const u32 sc = i == 0 ? seed.w[4] : i == 1 ? seed.w[5] : i == 2 ? seed.w[6] : seed.w[7];
    const u32 sd = i == 0 ? ctr : i == 1 ? n0 : i == 2 ? n1 : n2;
    u32 a = sa, b = sb, c = sc, d = sd;
    const unsigned full = 0xffffffffu;
#pragma unroll 1
    for (int r = 0; r < 10; ++r) {
        CSSC_QR(a, b, c, d);
        b = __shfl_sync(full, b, (i + 1) & 3, 4);
        c = __shfl_sync(full, c, (i + 2) & 3, 4);
        d = __shfl_sync(full, d, (i + 3) & 3, 4);
        CSSC_QR(a, b, c, d);
        b = __shfl_sync(full, b, (i + 3) & 3, 4);
        c = __shfl_sync(full, c, (i + 2) & 3, 4);
        d = __shfl_sync(full, d, (i + 1) & 3, 4);
    }
    out[i] = a + sa;
    out[4 + i] = b + sb;
    out[8 + i] = c + sc;
    out[12 + i] = d + sd;
}

__device__ __forceinline__ u64 word64(const u32* blk, int w) {
    return (u64)blk[2 * w] | ((u64)blk[2 * w + 1] << 32);
}
__device__ __forceinline__ int64_t ternary_of(u64 w) { return (int64_t)(w % 3) - 1; }
__device__ __forceinline__ int64_t cbd_of(u64 w) {
    return (int64_t)__popcll(w & 0x1FFFFFull) - (int64_t)__popcll((w >> 21) & 0x1FFFFFull);
}
__device__ __forceinline__ u64 lift_signed(int64_t v, u64 q) {
    return v >= 0 ? (u64)v : q - (u64)(-v);
}

// ---------------------------------------------------------------------------
// NTT: two-phase kernels (see ntt.cuh)
// ---------------------------------------------------------------------------
__device__ __forceinline__ const u64* job_src(const NttJob& job, int item, int j, int n) {
    return job.src_items ? job.src_items[item] + (size_t)(job.src_limb_offset + j) * n
                         : job.src + ((size_t)item * job.limbs + j) * n;
}
__device__ __forceinline__ u64* job_dst(const NttJob& job, int item, int j, int n) {
    return job.dst_items ? job.dst_items[item] + (size_t)j * n : job.dst + ((size_t)item * job.limbs + j) * n;
}

// Column phase: LN strided columns of R1 elements per CTA (LN = 16, or 8 for
// launches too small to fill the GPU: twice the CTAs, half the serial work
// each).  Forward: first phase (src -> dst).  Inverse: last phase (dst ->
// dst), applies N^-1, canonical.
template <int LOGN, bool INV, int LN = 16>
__global__ void __launch_bounds__(Ntt2<LOGN>::TC, 256 / Ntt2<LOGN>::TC * 3) k_ntt_cols(const DevConsts* __restrict__ dc, NttJob job) {
    using G = Ntt2<LOGN>;
    constexpr int T = G::TC;
    constexpr int CTAS = G::R2 / LN;     // column tiles per limb
    constexpr int SEG = LN / 2;          // 16-byte copies per row
    extern __shared__ u64 smem[];
    u64* tile = smem;                    // [R1][LN]
    u64* tws = smem + LN * G::R1;        // [R1] pairs
    const int tileid = blockIdx.x % CTAS;
    const int lj = blockIdx.x / CTAS;
    const int item = lj / job.limbs, j = lj - item * job.limbs;
    const int prime = job.pidx[j];
    const u64 q = dc->mod[prime].q;
    const u64* tw = INV ? dc->tw[prime].inv : dc->tw[prime].fwd;
    const u64* src = INV ? job_dst(job, item, j, G::N) : job_src(job, item, j, G::N);
    u64* dst = job_dst(job, item, j, G::N);
    const int col0 = tileid * LN;
    // twiddles W[0 .. R1) and the tile (rows of LN consecutive words, SEG
    // threads x 16 B per row) via async copies: every load in flight at once
    for (int i = threadIdx.x; i < G::R1; i += T) cp_async16(tws + 2 * i, tw + 2 * i);
#pragma unroll
    for (int r = 0; r < G::R1 * SEG / T; ++r) {
        const int i = threadIdx.x + T * r, c = i / SEG, h = i % SEG;
        cp_async16(tile + c * LN + 2 * h, src + (size_t)c * G::R2 + col0 + 2 * h);
    }
    cp_async_wait_all();
    __syncthreads();
    if (INV && job.add_items) {
        const u64* ad = job.add_items[item];
        if (ad) {
            ad += (size_t)j * G::N;
            const u64 q2 = 2 * q;
#pragma unroll
            for (int r = 0; r < G::R1 * SEG / T; ++r) {
                const int i = threadIdx.x + T * r, c = i / SEG, h = i % SEG;
                const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(ad + (size_t)c * G::R2 + col0 + 2 * h);
                u64 s0 = tile[c * LN + 2 * h] + x.x, s1 = tile[c * LN + 2 * h + 1] + x.y;
                tile[c * LN + 2 * h] = s0 >= q2 ? s0 - q2 : s0;
                tile[c * LN + 2 * h + 1] = s1 >= q2 ? s1 - q2 : s1;
            }
            __syncthreads();
        }
    }
    auto addr = [](int l, int pos) { return pos * LN + l; };
    auto twf = [&](int sl, int, int blk) {
        const int k = (1 << sl) + blk;
        return make_ulonglong2(tws[2 * k], tws[2 * k + 1]);
    };
    // radix-8 passes (3 CTAs per SM); 4-column tiles: radix-4, one group per thread
    // ciphertext primes are = 1 mod 2^32 (cheaper product); the plaintext modulus is not
    if ((u32)q == 1u)
        line_ntt_v<G::A, 0, INV, (LN >= 8 ? 3 : 2), LN>(tile, SpecQ{q}, addr, twf, whole_cta());
    else
        line_ntt_v<G::A, 0, INV, (LN >= 8 ? 3 : 2), LN>(tile, ConstQ{q}, addr, twf, whole_cta());
    const u64 ni = dc->ninv[prime], nish = dc->ninv_sh[prime];
    const bool scale = INV && !job.lazy_out;
#pragma unroll
    for (int r = 0; r < G::R1 * SEG / T; ++r) {
        const int i = threadIdx.x + T * r, c = i / SEG, h = i % SEG;
        u64 a0 = tile[c * LN + 2 * h], a1 = tile[c * LN + 2 * h + 1];
        if (scale) {  // ciphertext primes (= 1 mod 2^32): the cheaper quotient correction, same words
            a0 = (u32)q == 1u ? shoup_q(a0, ni, nish, q) : shoup(a0, ni, nish, q);
            a1 = (u32)q == 1u ? shoup_q(a1, ni, nish, q) : shoup(a1, ni, nish, q);
        }
        *reinterpret_cast<ulonglong2*>(dst + (size_t)c * G::R2 + col0 + 2 * h) = make_ulonglong2(a0, a1);
    }
}

// Column-tile width: 8 columns only when twice the CTAs still fit one wave
// (3 CTAs per SM, register-bound).  A wave-quantisation model that also
// picked 8 columns for 1-2 waves (C2's 144-limb launch) measured 6 % slower:
// an 8-column CTA costs well over half a 16-column one.  CSSC_COLS_LN=8|16
// forces a width.
static int cols_forced() {
    static const int forced = [] {
        const char* e = std::getenv("CSSC_COLS_LN");
        return e ? std::atoi(e) : 0;
    }();
    return forced;
}

bool cols_use_ln8(long ctas16, bool allowed) {
    if (!allowed) return false;
    const int forced = cols_forced();
    if (forced == 8 || forced == 4) return true;
    if (forced == 16) return false;
    return 2 * ctas16 <= 3L * 148;
}

bool blocks_use_ln8(long ctas16) {
    static const long lim = [] {
        const char* e = std::getenv("CSSC_BLOCKS_LN8_MAX");
        return e ? std::atol(e) : 2L * 148;
    }();
    static const int forced = [] {
        const char* e = std::getenv("CSSC_BLOCKS_LN");
        return e ? std::atoi(e) : 0;
    }();
    if (forced) return forced == 8;
    return ctas16 < lim;
}

// 4-column tiles (radix-4 passes, 4 words per thread) for launches whose
// 8-column CTAs fill less than half a wave (a lone rotation's key switch):
// the CTA's serial chain halves, the CTA count doubles.
bool cols_use_ln4(long ctas16, bool allowed) {
    if (!allowed) return false;
    const int forced = cols_forced();
    if (forced) return forced == 4;
    return 4 * ctas16 <= 3L * 148;
}

template <int LOGN, bool INV>
static void launch_cols(const DevConsts* dc, const NttJob& job, int limbs, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    // 4-column tiles for launches under a quarter wave (CSSC_COLS_SMALL4=0 keeps 8)
    static const bool small4 = [] {
        const char* e = std::getenv("CSSC_COLS_SMALL4");
        return !e || std::atoi(e) != 0;
    }();
    if ((small4 || cols_forced() == 4) && cols_use_ln4((long)limbs * G::CTAS_C, G::R2 >= 16 && G::R1 >= G::TC)) {
        constexpr int LN = 4;
        k_ntt_cols<LOGN, INV, LN><<<limbs * (G::R2 / LN), G::TC, (LN * G::R1 + 2 * G::R1) * 8, st>>>(dc, job);
    } else if (cols_use_ln8((long)limbs * G::CTAS_C, G::R2 >= 16 && G::R1 * 4 >= G::TC)) {
        constexpr int LN = 8;
        k_ntt_cols<LOGN, INV, LN><<<limbs * (G::R2 / LN), G::TC, (LN * G::R1 + 2 * G::R1) * 8, st>>>(dc, job);
    } else {
        k_ntt_cols<LOGN, INV><<<limbs * G::CTAS_C, G::TC, G::SMEM_C, st>>>(dc, job);
    }
}

// Block phase: 16 contiguous blocks of R2 elements.  Forward: last phase
// (dst -> dst, canonical output).  Inverse: first phase (src -> dst).
// The twiddles of a block tile (~2x the tile's bytes) depend only on the
// prime and the tile, so one CTA handles the same tile of `ipc` items that
// share limb index j (same prime): twiddles staged once, tiles double-buffered
// (the next item's cp.async load overlaps the current item's butterflies).
template <int LOGN, bool INV>
__global__ void __launch_bounds__(128) k_ntt_blocks(const DevConsts* __restrict__ dc, NttJob job, int items,
                                                    int ipc) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TILE = G::LINES * PITCH;
    const int tileid = blockIdx.x % G::CTAS_B;
    const int rest = blockIdx.x / G::CTAS_B;
    const int j = rest % job.limbs, grp = rest / job.limbs;
    const int it0 = grp * ipc, it1 = min(items, it0 + ipc);
    const int prime = job.pidx[j];
    const u64 q = dc->mod[prime].q;
    const u64* tw = INV ? dc->tw[prime].inv : dc->tw[prime].fwd;
    const int blk0 = tileid * G::LINES;
    const size_t base = (size_t)blk0 * G::R2;
    u64* tws = smem + 2 * TILE;
    auto src_of = [&](int it) { return INV ? job_src(job, it, j, G::N) : job_dst(job, it, j, G::N); };
    auto issue_load = [&](int it, u64* buf) {
        const u64* src = src_of(it) + base;
#pragma unroll
        for (int r = 0; r < G::LINES * G::R2 / 128; ++r) {
            const int x = threadIdx.x + 128 * r, b = x >> G::B, c = x & (G::R2 - 1);
            cp_async8(buf + b * PITCH + c, src + x);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    issue_load(it0, smem);
    load_block_twiddles<LOGN>(tws, tw, blk0);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl, int l, int blk) { return block_tw<LOGN>(tws, sl, l, blk); };
    const Modulus md = dc->mod[prime];
#pragma unroll 1
    for (int it = it0; it < it1; ++it) {
        u64* cur = smem + ((it - it0) & 1) * TILE;
        if (it + 1 < it1) {
            issue_load(it + 1, smem + ((it + 1 - it0) & 1) * TILE);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        if ((u32)q == 1u)
            line_ntt_q<G::B, 0, INV>(cur, q, addr, twf);
        else
            line_ntt<G::B, 0, INV>(cur, q, addr, twf);
        u64* dst = job_dst(job, it, j, G::N) + base;
#pragma unroll
        for (int r = 0; r < G::LINES * G::R2 / 256; ++r) {
            const int x = 2 * (threadIdx.x + 128 * r), b = x >> G::B, c = x & (G::R2 - 1);
            u64 a0 = cur[b * PITCH + c], a1 = cur[b * PITCH + c + 1];
            if (!INV) {  // forward output < 31q -> canonical
                a0 = (u32)q == 1u ? reduce_small_quot_q(a0, md) : reduce_small_quot(a0, md);
                a1 = (u32)q == 1u ? reduce_small_quot_q(a1, md) : reduce_small_quot(a1, md);
            }
            *reinterpret_cast<ulonglong2*>(dst + x) = make_ulonglong2(a0, a1);
        }
        __syncthreads();  // `cur` is reloaded two items later
    }
}

// items per block-phase CTA: amortise twiddle staging while keeping >= ~2 waves
static int blocks_ipc(int items, int limbs_per_item, int ctas_per_limb) {
    static const int forced = [] {
        const char* e = std::getenv("CSSC_BLOCKS_IPC");
        return e ? std::atoi(e) : 0;
    }();
    if (forced > 0) return std::min(forced, std::max(items, 1));
    // largest power of two <= 8 that still leaves >= 3 CTAs per SM (measured:
    // 144 limbs of 2^14 run 6% faster at ipc 4 than at 1; 1152 limbs saturate at 8)
    int ipc = 1;
    while (ipc < 8 && ipc < items && (long)items * limbs_per_item * ctas_per_limb / (2 * ipc) >= 148 * 3) ipc *= 2;
    return ipc;
}

template <int LOGN, bool INV>
static void launch_blocks(const DevConsts* dc, const NttJob& job, int items, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int ipc = blocks_ipc(items, job.limbs, G::CTAS_B);
    const int groups = (items + ipc - 1) / ipc;
    k_ntt_blocks<LOGN, INV><<<groups * job.limbs * G::CTAS_B, 128, G::SMEM_B, st>>>(dc, job, items, ipc);
}

size_t ntt_smem_bytes(int logn) { return (size_t)8 << logn; }

void smem_optin(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes opted in
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "get device");
    std::lock_guard<std::mutex> lk(mu);
    int& have = done[{fn, dev}];
    if (bytes <= have) return;
    cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), "smem opt-in");
    have = bytes;
}

static thread_local std::vector<KernelMark>* g_kmarks = nullptr;
void kmarks_install(std::vector<KernelMark>* marks) { g_kmarks = marks; }
void kmark(const char* name, cudaStream_t st) {
    if (!g_kmarks) return;
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "event");
    cuda_check(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal), "event record");
    g_kmarks->push_back({name, e});
}

template <int LOGN>
static void launch_ntt_t(const DevConsts* dc, bool inv, const NttJob& job, int items,
                         cudaStream_t st) {
    using G = Ntt2<LOGN>;
    smem_optin_k(k_ntt_cols<LOGN, false>, G::SMEM_C);
    smem_optin_k(k_ntt_cols<LOGN, true>, G::SMEM_C);
    smem_optin_k(k_ntt_blocks<LOGN, false>, G::SMEM_B);
    smem_optin_k(k_ntt_blocks<LOGN, true>, G::SMEM_B);
    const int limbs = items * job.limbs;
    if (limbs == 0) return;
    if (!inv) {
        launch_cols<LOGN, false>(dc, job, limbs, st);
        CSSC_CHECK_LAUNCH();
        launch_blocks<LOGN, false>(dc, job, items, st);
    } else {
        launch_blocks<LOGN, true>(dc, job, items, st);
        CSSC_CHECK_LAUNCH();
        launch_cols<LOGN, true>(dc, job, limbs, st);
    }
    CSSC_CHECK_LAUNCH();
}

template <int LOGN>
static void launch_phase_t(const DevConsts* dc, bool inv, bool cols, const NttJob& job, int items,
                           cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int limbs = items * job.limbs;
    if (limbs == 0) return;
    if (cols) {
        if (inv)
            launch_cols<LOGN, true>(dc, job, limbs, st);
        else
            launch_cols<LOGN, false>(dc, job, limbs, st);
    } else {
        if (inv)
            launch_blocks<LOGN, true>(dc, job, items, st);
        else
            launch_blocks<LOGN, false>(dc, job, items, st);
    }
    CSSC_CHECK_LAUNCH();
}

// One phase only (used by fused pipelines).  Column phase of an inverse
// transform reads and writes job.dst in place, like the second half of
// launch_ntt.
void launch_ntt_phase(const DevConsts* dc, int logn, bool inverse, bool cols, const NttJob& job,
                      int items, cudaStream_t st) {
    switch (logn) {
        case 10: launch_ntt_t<10>(dc, inverse, job, 0, st); launch_phase_t<10>(dc, inverse, cols, job, items, st); break;
        case 11: launch_ntt_t<11>(dc, inverse, job, 0, st); launch_phase_t<11>(dc, inverse, cols, job, items, st); break;
        case 12: launch_ntt_t<12>(dc, inverse, job, 0, st); launch_phase_t<12>(dc, inverse, cols, job, items, st); break;
        case 13: launch_ntt_t<13>(dc, inverse, job, 0, st); launch_phase_t<13>(dc, inverse, cols, job, items, st); break;
        case 14: launch_ntt_t<14>(dc, inverse, job, 0, st); launch_phase_t<14>(dc, inverse, cols, job, items, st); break;
        case 15: launch_ntt_t<15>(dc, inverse, job, 0, st); launch_phase_t<15>(dc, inverse, cols, job, items, st); break;
        default: throw std::invalid_argument("NTT: unsupported logn " + std::to_string(logn));
    }
}

void launch_ntt(const DevConsts* dc, int logn, bool inverse, const NttJob& job, int items,
                cudaStream_t st) {
    switch (logn) {
        case 10: launch_ntt_t<10>(dc, inverse, job, items, st); break;
        case 11: launch_ntt_t<11>(dc, inverse, job, items, st); break;
        case 12: launch_ntt_t<12>(dc, inverse, job, items, st); break;
        case 13: launch_ntt_t<13>(dc, inverse, job, items, st); break;
        case 14: launch_ntt_t<14>(dc, inverse, job, items, st); break;
        case 15: launch_ntt_t<15>(dc, inverse, job, items, st); break;
        default: throw std::invalid_argument("NTT: unsupported logn " + std::to_string(logn));
    }
}

static dim3 ew_grid(int n, int items) { return dim3((unsigned)(n / EW_THREADS), (unsigned)items); }

// Compile-time RNS shapes (L data primes, K special primes, alpha primes per
// digit) of the supported parameter sets; 0 = read from DevConsts at run time.
// With a fixed shape every per-coefficient residue array lives in registers.
template <class F>
static void dispatch_shape(const RnsParams& P, F&& f) {
    const auto& c = P.cfg;
    using std::integral_constant;
    if (c.L == 2 && c.K == 2 && c.alpha == 2)
        f(integral_constant<int, 2>{}, integral_constant<int, 2>{}, integral_constant<int, 2>{});
    else if (c.L == 4 && c.K == 4 && c.alpha == 4)
        f(integral_constant<int, 4>{}, integral_constant<int, 4>{}, integral_constant<int, 4>{});
    else
        f(integral_constant<int, 0>{}, integral_constant<int, 0>{}, integral_constant<int, 0>{});
}
#define SHAPE_ARGS decltype(l_)::value, decltype(k_)::value, decltype(a_)::value

// ---------------------------------------------------------------------------
// E1: exact centred basis extension of one coefficient (X residues -> Y)
// ---------------------------------------------------------------------------
template <int NXT, int NYT>
__device__ __forceinline__ void extend_exact(const DevConsts* __restrict__ dc,
                                             const ExtConsts& e, const u64* x, u64* out) {
    const int nx = NXT ? NXT : e.nx, ny = NYT ? NYT : e.ny;
    u64 y[MAXB];
    u64 shi = 0, slo = 0;
#pragma unroll
    for (int i = 0; i < nx; ++i) {
        const u64 qi = dc->mod[e.xi[i]].q;
        y[i] = shoup_q(x[i], e.xhat_inv[i], e.xhat_inv_sh[i], qi);
        add128(shi, slo, 0, frac64(y[i], e.R1[i], e.R0[i]));
    }
    const u64 v = shi + (slo >> 63);
#pragma unroll
    for (int j = 0; j < ny; ++j) {
        const u64 p = dc->mod[e.yi[j]].q;
        // lazy sum: nx <= 16 terms < 2p each stay below 2^(k+5) -> one reduction
        u64 acc = 0;
#pragma unroll
        for (int i = 0; i < nx; ++i) acc += shoup_lazy_q(y[i], e.xhat_y[i][j], e.xhat_y_sh[i][j], p);
        acc = reduce_small_quot_q(acc, dc->mod[e.yi[j]]);
        out[j] = sub_mod(acc, shoup_q(v, e.X_y[j], e.X_y_sh[j], p), p);
    }
}

// ---------------------------------------------------------------------------
// Kernel-parameter copies of the RNS constants (fixed shapes).  A
// __grid_constant__ parameter lives in the constant bank, so the modmul IMADs
// take the constants as operands: no LDG per constant and no load latency
// on the E1/E2/E4 chains (k_mul_scale issued ~180 constant LDGs per
// coefficient when it read them through the DevConsts pointer).
// ---------------------------------------------------------------------------
template <int NX, int NY>
struct ExtK {
    u64 xq[NX];
    Modulus ym[NY];
    u64 xhat_inv[NX], xhat_inv_sh[NX], R1[NX], R0[NX];
    W29 w[NX][NY];  // [X/x_i]_{y_j} in 29-bit halves (Dot29)
    W29 nX[NY];     // [-X]_{y_j}
};

static inline u64 host_mulmod(u64 a, u64 b, u64 p) { return (u64)((unsigned __int128)a * b % p); }

template <int NX, int NY>
static void fill_extk(ExtK<NX, NY>& k, const DevConsts& h, const ExtConsts& e) {
    static_assert(NX + 1 <= 15, "Dot29 bound: at most 15 terms");
    for (int i = 0; i < NX; ++i) {
        k.xq[i] = h.mod[e.xi[i]].q;
        k.xhat_inv[i] = e.xhat_inv[i];
        k.xhat_inv_sh[i] = e.xhat_inv_sh[i];
        k.R1[i] = e.R1[i];
        k.R0[i] = e.R0[i];
        for (int j = 0; j < NY; ++j) k.w[i][j] = split29(e.xhat_y[i][j]);
    }
    for (int j = 0; j < NY; ++j) {
        k.ym[j] = h.mod[e.yi[j]];
        const u64 p = k.ym[j].q;
        k.nX[j] = split29((p - e.X_y[j] % p) % p);
    }
}

// extend_exact with the constants from a parameter block: the same value,
// sum_i y_i [X/x_i]_p - v [X]_p mod p, as one Dot29 per target prime
template <int NX, int NY>
__device__ __forceinline__ void extend_k(const ExtK<NX, NY>& e, const u64* x, u64* out) {
    u64 y[NX];
    u64 shi = 0, slo = 0;
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        y[i] = shoup_q(x[i], e.xhat_inv[i], e.xhat_inv_sh[i], e.xq[i]);
        add128(shi, slo, 0, frac64(y[i], e.R1[i], e.R0[i]));
    }
    const u32 v = (u32)(shi + (slo >> 63));  // <= NX
#pragma unroll
    for (int j = 0; j < NY; ++j) {
        Dot29 d;
#pragma unroll
        for (int i = 0; i < NX; ++i) dot29_mac(d, y[i], e.w[i][j]);
        dot29_mac_small(d, v, e.nX[j]);
        out[j] = dot29_reduce_q(d, e.ym[j]);
    }
}

// The over-Q multiply's input conversions (fixed shapes; E6-E8,
// oracle mul_tensor_overq): a's Q limbs are copied and extended Q -> R (E1);
// b is scaled to R, b''_k = sum_i y_i [floor(R/q_i)]_{r_k} + round(sum_i y_i
// theta_i) (E6, y_i = [b_i (Q/q_i)^-1]_{q_i}, theta_i in 64-bit fixed point),
// and b'' extended R -> Q (E1): the Q limbs of b's slot hold ext(b''), not b.
template <int L>
struct ExtendK {
    int n;
    ExtK<L, L> qr;     // Q -> R (its x-side constants give y_i for E6 too)
    ExtK<L, L> rq;     // R -> Q
    u64 theta[L];      // floor(2^64 [R]_{q_i} / q_i)
    W29 omega[L][L];   // [floor(R / q_i)]_{r_k}
};

template <int L>
__device__ __forceinline__ void mul_extend_overq(const ExtendK<L>& c, bool is_b, const u64* x, u64* qo, u64* ro) {
    if (!is_b) {
#pragma unroll
        for (int i = 0; i < L; ++i) qo[i] = x[i];
        extend_k(c.qr, x, ro);
        return;
    }
    u64 y[L];
    u64 shi = 0, slo = 0;
#pragma unroll
    for (int i = 0; i < L; ++i) {
        y[i] = shoup_q(x[i], c.qr.xhat_inv[i], c.qr.xhat_inv_sh[i], c.qr.xq[i]);
        add128(shi, slo, umulhi(y[i], c.theta[i]), y[i] * c.theta[i]);
    }
    const u64 rnd = shi + (slo >> 63);  // < L 2^58: rides in both Dot29 column sums (x 1)
#pragma unroll
    for (int k = 0; k < L; ++k) {
        Dot29 d;
        d.a0 = d.am = rnd;
#pragma unroll
        for (int i = 0; i < L; ++i) dot29_mac(d, y[i], c.omega[i][k]);
        ro[k] = dot29_reduce_q(d, c.qr.ym[k]);
    }
    extend_k(c.rq, ro, qo);
}

template <int L>
__global__ void k_mul_extend_k(const __grid_constant__ ExtendK<L> c, const u64* const* A, const u64* const* B,
                               u64* T) {
    constexpr int M = 2 * L;
    const int n = c.n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const int p = blockIdx.z;
    const u64* src = (p < 2 ? A[item] : B[item]) + (size_t)(p & 1) * L * n;
    u64* dst = T + ((size_t)item * 4 + p) * M * n;
    u64 x[L], qo[L], ro[L];
#pragma unroll
    for (int i = 0; i < L; ++i) x[i] = src[(size_t)i * n + k];
    mul_extend_overq(c, p >= 2, x, qo, ro);
#pragma unroll
    for (int i = 0; i < L; ++i) {
        dst[(size_t)i * n + k] = qo[i];
        dst[(size_t)(L + i) * n + k] = ro[i];
    }
}

// The pipeline's encryption finish fused into the multiply's base
// extension: for one (chunk, polynomial of a or b) and 128 coefficients, the
// ChaCha e draw of k_enc_finish, c = (pk u) + e (+ Delta m for c0) per Q
// limb (the ciphertext words, also stored to the ciphertext), then E1 of
// those words into T.  Same words as k_enc_finish followed by k_mul_extend.

template <int L>
struct ExtendEncK {
    ExtendK<L> x;
    u64 delta[L], delta_sh[L];
};

template <int L>
__global__ void __launch_bounds__(128) k_mul_extend_enc(const __grid_constant__ ExtendEncK<L> c, const EncIn in,
                                                        u64* T) {
    constexpr int M = 2 * L;
    __shared__ u32 blk[16][16];
    const int n = c.x.n;
    const int item = blockIdx.y, p = blockIdx.z, poly = p & 1;
    const int eitem = (p < 2 ? 0 : in.n_chunks) + (in.order ? in.order[item] : item);
    const int kk = threadIdx.x, k = blockIdx.x * 128 + kk;
    int64_t e;
    if (in.E) {  // drawn ahead by k_enc_sample_e (the early graph)
        e = in.E[((size_t)eitem * 2 + poly) * n + k];
    } else {
        const u64 id = in.streams[eitem];
        const int g = threadIdx.x >> 2;
        if (g < 16)
            chacha20_block_x4(in.seed, (u32)(blockIdx.x * 16 + g), poly ? DOM_ENC_E1 : DOM_ENC_E0, (u32)id,
                              (u32)(id >> 32), blk[g]);
        __syncthreads();
        e = cbd_of(word64(blk[kk >> 3], kk & 7));
    }
    const u64* cm = in.CM + (size_t)eitem * in.cstride + (size_t)poly * L * n + k;
    const u64 m = poly ? 0 : in.MSG[(size_t)eitem * in.mstride + k];
    u64* ct = in.OUT[eitem] + (size_t)poly * L * n + k;
    u64* dst = T + ((size_t)item * 4 + p) * M * n + k;
    u64 x[L], qo[L], ro[L];
#pragma unroll
    for (int i = 0; i < L; ++i) {
        const u64 q = c.x.qr.xq[i];
        u64 v = add_mod(cm[(size_t)i * n], lift_signed(e, q), q);
        if (!poly) v = add_mod(v, shoup_q(m, c.delta[i], c.delta_sh[i], q), q);
        x[i] = v;
        ct[(size_t)i * n] = v;
    }
    mul_extend_overq(c.x, p >= 2, x, qo, ro);
#pragma unroll
    for (int i = 0; i < L; ++i) {
        dst[(size_t)i * n] = qo[i];
        dst[(size_t)(L + i) * n] = ro[i];
    }
}

// E8, round(t z / R) mod q_j from z's Q u R residues (the over-Q multiply's
// scale; oracle scale_r_to_q): y_k = [z_k (R/r_k)^-1]_{r_k},
//   out_j = [t R^-1]_{q_j} z_j + sum_k y_k [-t R^-1 R/r_k]_{q_j} + round(sum_k t y_k / r_k)
// as one Dot29 per q_j; the rounding term in E2's fixed point.
template <int L>
struct ScaleK {
    int n;
    u64 r[L], RhatInv[L], RhatInv_sh[L], T1[L], T0[L];  // T = floor(t 2^128 / r_k)
    Modulus qm[L];
    W29 A[L];         // [t R^-1]_{q_j}
    W29 C[L][L];      // [-t R^-1 R/r_k]_{q_j}
    u64 dhi[L], dhi_sh[L];  // ModUp factors [(Q_d / q_i)^-1]_{q_i} (KsY)
};

template <int L>
__global__ void k_mul_scale_k(const __grid_constant__ ScaleK<L> c, const u64* __restrict__ Z, u64* const* OUT,
                              u64* __restrict__ D2, u64* __restrict__ D2Y, u64* const* Y1) {
    constexpr int M = 2 * L;
    const int n = c.n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const int r = blockIdx.z;
    const size_t P = (size_t)M * n;
    const u64* z = Z + ((size_t)item * 3 + r) * P;
    u64 y[L], o[L];
    u64 shi = 0, slo = 0;
#pragma unroll
    for (int kk = 0; kk < L; ++kk) {
        y[kk] = shoup_q(z[(size_t)(L + kk) * n + k], c.RhatInv[kk], c.RhatInv_sh[kk], c.r[kk]);
        add128(shi, slo, umulhi(y[kk], c.T1[kk]), y[kk] * c.T1[kk]);
        add128(shi, slo, 0, umulhi(y[kk], c.T0[kk]));
    }
    const u64 rnd = shi + (slo >> 63);  // < L t + 1
#pragma unroll
    for (int j = 0; j < L; ++j) {
        Dot29 d;
        d.a0 = d.am = rnd;
        u64 zq = z[(size_t)j * n + k];  // lazy (< 2q) when the inverse NTT left N^-1 to A
        zq = zq >= c.qm[j].q ? zq - c.qm[j].q : zq;
        dot29_mac(d, zq, c.A[j]);
#pragma unroll
        for (int kk = 0; kk < L; ++kk) dot29_mac(d, y[kk], c.C[kk][j]);
        o[j] = dot29_reduce_q(d, c.qm[j]);
    }
    u64* dst = r < 2 ? OUT[item] + (size_t)r * L * n : D2 + (size_t)item * L * n;
#pragma unroll
    for (int i = 0; i < L; ++i) dst[(size_t)i * n + k] = o[i];
    // ModUp factors (KsY) of c2 for the relinearisation, and of z1 when the
    // product's c1 is key-switched unrelinearised (the folded level 0)
    u64* yy = r == 2 ? (D2Y ? D2Y + (size_t)item * L * n : nullptr) : (r == 1 && Y1 ? Y1[item] : nullptr);
    if (yy) {
#pragma unroll
        for (int i = 0; i < L; ++i) yy[(size_t)i * n + k] = shoup_q(o[i], c.dhi[i], c.dhi_sh[i], c.qm[i].q);
    }
}

static u64 host_inv(u64 a, u64 q) { return inv_mod_host(a % q, q); }

template <int L>
static ExtendK<L> make_extend_k(const RnsParams& P) {
    const DevConsts& h = P.host;
    ExtendK<L> c{};
    c.n = P.n;
    fill_extk(c.qr, h, h.extQR);
    fill_extk(c.rq, h, h.extRQ);
    for (int i = 0; i < L; ++i) {
        const u64 q = h.mod[i].q;
        u64 Rq = 1;
        for (int kk = 0; kk < L; ++kk) Rq = host_mulmod(Rq, h.mod[h.extQR.yi[kk]].q % q, q);
        c.theta[i] = (u64)(((unsigned __int128)Rq << 64) / q);
        for (int kk = 0; kk < L; ++kk) {  // floor(R/q_i) = (R - [R]_{q_i}) / q_i, R = 0 mod r_k
            const u64 rk = h.mod[h.extQR.yi[kk]].q;
            c.omega[i][kk] = split29(host_mulmod((rk - Rq % rk) % rk, host_inv(q, rk), rk));
        }
    }
    return c;
}

// lazy: Z is the inverse NTT without its final x N^-1 (NttJob::lazy_out); N^-1
// rides in the constants that multiply z ((R/r_k)^-1 for the R limbs, A_j for
// the Q limbs), so y_k and the output words are unchanged
template <int L>
static ScaleK<L> make_scale_k(const RnsParams& P, bool lazy = false) {
    const DevConsts& h = P.host;
    const u64 t = P.cfg.t;
    ScaleK<L> c{};
    c.n = P.n;
    for (int kk = 0; kk < L; ++kk) {
        const int ri = h.extRQ.xi[kk];
        const u64 rk = h.mod[ri].q;
        c.r[kk] = rk;
        c.RhatInv[kk] = lazy ? host_mulmod(h.extRQ.xhat_inv[kk], h.ninv[ri], rk) : h.extRQ.xhat_inv[kk];
        c.RhatInv_sh[kk] = shoup_factor(c.RhatInv[kk], rk);
        // T = floor(t 2^128 / r_k) = t floor(2^128 / r_k) + floor(t [2^128]_{r_k} / r_k)
        using u128 = unsigned __int128;
        u128 Rf = (~(u128)0) / rk, rem = (~(u128)0) % rk + 1;
        if (rem == rk) {
            Rf += 1;
            rem = 0;
        }
        const u128 T = Rf * t + rem * t / rk;
        c.T1[kk] = (u64)(T >> 64);
        c.T0[kk] = (u64)T;
    }
    for (int j = 0; j < L; ++j) {
        c.qm[j] = h.mod[j];
        const u64 q = h.mod[j].q;
        u64 Rq = 1;
        for (int kk = 0; kk < L; ++kk) Rq = host_mulmod(Rq, c.r[kk] % q, q);
        const u64 tRinv = host_mulmod(t % q, host_inv(Rq, q), q);
        c.A[j] = split29(lazy ? host_mulmod(tRinv, h.ninv[j], q) : tRinv);
        for (int kk = 0; kk < L; ++kk) {
            u64 hk = 1;
            for (int m = 0; m < L; ++m)
                if (m != kk) hk = host_mulmod(hk, c.r[m] % q, q);
            c.C[kk][j] = split29((q - host_mulmod(tRinv, hk, q)) % q);
        }
        c.dhi[j] = h.dig_hat_inv[j];
        c.dhi_sh[j] = h.dig_hat_inv_sh[j];
    }
    return c;
}

// T[item][poly 0..3][M][N]: Q limbs copied, B limbs by E1.  polys: a0 a1 b0 b1
template <int LT, int KT, int AT>
__global__ void k_mul_extend(const DevConsts* __restrict__ dc, const u64* const* A,
                             const u64* const* B, u64* T) {
    const int n = dc->n, L = LT ? LT : dc->L, nB = L + 1, M = L + nB;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    u64 x[MAXB], o[MAXB];
    {  // one polynomial per grid z-slice: keeps the E1 constants out of registers
        const int p = blockIdx.z;
        const u64* src = (p < 2 ? A[item] : B[item]) + (size_t)(p & 1) * L * n;
        u64* dst = T + ((size_t)item * 4 + p) * M * n;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            x[i] = src[(size_t)i * n + k];
            dst[(size_t)i * n + k] = x[i];
        }
        extend_exact<LT, LT ? LT + 1 : 0>(dc, dc->extQB, x, o);
#pragma unroll
        for (int j = 0; j < nB; ++j) dst[(size_t)(L + j) * n + k] = o[j];
    }
}

bool fixed_rns_shape(const RnsParams& P) {
    bool fixed = false;
    dispatch_shape(P, [&](auto l_, auto, auto) { fixed = decltype(l_)::value > 0; });
    return fixed;
}

void launch_mul_extend_enc(const DevConsts* dc, const RnsParams& P, const EncIn& in, u64* T, int items,
                           cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        constexpr int LT = decltype(l_)::value;
        if constexpr (LT > 0) {
            ExtendEncK<LT> c{};
            c.x = make_extend_k<LT>(P);
            for (int i = 0; i < LT; ++i) {
                c.delta[i] = P.host.delta[i];
                c.delta_sh[i] = P.host.delta_sh[i];
            }
            dim3 g = ew_grid(P.n, items);
            g.z = 4;
            k_mul_extend_enc<LT><<<g, 128, 0, st>>>(c, in, T);
        } else {
            throw std::invalid_argument("fused encryption + extension needs a fixed RNS shape");
        }
    });
    CSSC_CHECK_LAUNCH();
}

void launch_mul_extend(const DevConsts* dc, const RnsParams& P, const u64* const* A,
                       const u64* const* B, u64* T, int items, cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        constexpr int LT = decltype(l_)::value;
        dim3 g = ew_grid(P.n, items);
        g.z = 4;
        if constexpr (LT > 0)
            k_mul_extend_k<LT><<<g, EW_THREADS, 0, st>>>(make_extend_k<LT>(P), A, B, T);
        else
            k_mul_extend<SHAPE_ARGS><<<g, EW_THREADS, 0, st>>>(dc, A, B, T);
    });
    CSSC_CHECK_LAUNCH();
}

template <int LT, int KT, int AT>
__global__ void k_mul_tensor(const DevConsts* __restrict__ dc, const u64* __restrict__ T,
                             u64* __restrict__ Z) {
    // fixed shapes multiply over Q u R (2L limbs), the others over Q u B (2L + 1)
    const int n = dc->n, L = LT ? LT : dc->L, K = KT ? KT : dc->K, M = LT ? 2 * L : 2 * L + 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const size_t P = (size_t)M * n;
    const u64* t = T + (size_t)item * 4 * P;
    u64* z = Z + (size_t)item * 3 * P;
#pragma unroll
    for (int j = 0; j < M; ++j) {
        const int pi = j < L ? j : K + j;  // B limbs follow P in the prime table
        const Modulus md = dc->mod[pi];
        const size_t o = (size_t)j * n + k;
        const u64 a0 = t[o], a1 = t[P + o], b0 = t[2 * P + o], b1 = t[3 * P + o];
        z[o] = mul_mod(a0, b0, md);
        z[P + o] = add_mod(mul_mod(a0, b1, md), mul_mod(a1, b0, md), md.q);
        z[2 * P + o] = mul_mod(a1, b1, md);
    }
}

void launch_mul_tensor(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items,
                       cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        k_mul_tensor<SHAPE_ARGS><<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, T, Z);
    });
    CSSC_CHECK_LAUNCH();
}

// E2: w = round(t z / Q) in B, then E1 B -> Q.  r = 0,1 -> OUT ct, r = 2 -> D2
template <int LT, int KT, int AT>
__global__ void k_mul_scale(const DevConsts* __restrict__ dc, const u64* __restrict__ Z,
                            u64* const* OUT, u64* __restrict__ D2) {
    const int n = dc->n, L = LT ? LT : dc->L, nB = L + 1, K = KT ? KT : dc->K, M = L + nB;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const size_t P = (size_t)M * n;
    u64 xi[MAXL], w[MAXB], o[MAXB];
    {  // one tensor component per grid z-slice
        const int r = blockIdx.z;
        const u64* z = Z + ((size_t)item * 3 + r) * P;
        u64 shi = 0, slo = 0;
#pragma unroll
        for (int i = 0; i < L; ++i) {
            const u64 qi = dc->mod[i].q;
            xi[i] = shoup(z[(size_t)i * n + k], dc->QhatInv[i], dc->QhatInv_sh[i], qi);
            add128(shi, slo, umulhi(xi[i], dc->T1[i]), xi[i] * dc->T1[i]);
            add128(shi, slo, 0, umulhi(xi[i], dc->T0[i]));
        }
        const u64 rr = shi + (slo >> 63);
#pragma unroll
        for (int j = 0; j < nB; ++j) {
            const u64 bj = dc->mod[L + K + j].q;
            u64 acc = 0;
#pragma unroll
            for (int i = 0; i < L; ++i) acc += shoup_lazy(xi[i], dc->QhatB[i][j], dc->QhatB_sh[i][j], bj);
            acc = reduce_small_quot(acc, dc->mod[L + K + j]);
            const u64 alpha = shoup(sub_mod(acc, z[(size_t)(L + j) * n + k], bj), dc->QinvB[j],
                                    dc->QinvB_sh[j], bj);
            w[j] = sub_mod(rr, shoup(alpha, dc->tB[j], dc->tB_sh[j], bj), bj);
        }
        extend_exact<LT ? LT + 1 : 0, LT>(dc, dc->extBQ, w, o);
        u64* dst = r < 2 ? OUT[item] + (size_t)r * L * n : D2 + (size_t)item * L * n;
#pragma unroll
        for (int i = 0; i < L; ++i) dst[(size_t)i * n + k] = o[i];
    }
}

void launch_mul_scale(const DevConsts* dc, const RnsParams& P, const u64* Z, u64* const* OUT,
                      u64* D2, int items, cudaStream_t st, u64* D2Y, bool lazy_in, u64* const* Y1) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        dim3 g = ew_grid(P.n, items);
        g.z = 3;
        constexpr int LT = decltype(l_)::value;
        if constexpr (LT > 0)
            k_mul_scale_k<LT><<<g, EW_THREADS, 0, st>>>(make_scale_k<LT>(P, lazy_in), Z, OUT, D2, D2Y, Y1);
        else if (lazy_in)
            throw std::invalid_argument("unscaled inverse-NTT input needs a fixed RNS shape");
        else if (D2Y || Y1)
            throw std::invalid_argument("hoisted ModUp factors need a fixed RNS shape");
        else
            k_mul_scale<SHAPE_ARGS><<<g, EW_THREADS, 0, st>>>(dc, Z, OUT, D2);
    });
    CSSC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// hybrid key switching
// ---------------------------------------------------------------------------
__device__ __forceinline__ int automorph_src(u32 ginv, int k, int n, bool& neg) {
    if (ginv == 0) {
        neg = false;
        return k;
    }
    const u32 i0 = (u32)(((unsigned long long)ginv * (unsigned)k) & (unsigned long long)(2 * n - 1));
    neg = i0 >= (u32)n;
    return neg ? (int)(i0 - n) : (int)i0;
}

// E3: DX[item][digit][LK][N] = ModUp of SRC (optionally permuted by X -> X^g)
template <int LT, int KT, int AT>
__global__ void k_ks_modup(const DevConsts* __restrict__ dc, const u64* const* SRC,
                           const u64* SRCC, int src_poly, const u32* ginv, u64* DX) {
    const int n = dc->n, L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int alpha = AT ? AT : dc->alpha, dnum = (L + alpha - 1) / alpha;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64* src = SRC ? SRC[item] + (size_t)src_poly * L * n : SRCC + (size_t)item * L * n;
    bool neg;
    const int idx = automorph_src(ginv ? ginv[item] : 0u, k, n, neg);
    u64 x[MAXL], y[MAXL];
#pragma unroll
    for (int i = 0; i < L; ++i) {  // ModUp of the un-rotated source, phi_g's sign after (DESIGN 2.9)
        const u64 q = dc->mod[i].q;
        x[i] = src[(size_t)i * n + idx];
        y[i] = shoup(x[i], dc->dig_hat_inv[i], dc->dig_hat_inv_sh[i], q);
    }
#pragma unroll
    for (int dg = 0; dg < dnum; ++dg) {
        const int lo = dg * alpha, hi = min(lo + alpha, L);
        u64* out = DX + ((size_t)item * dnum + dg) * LK * n;
#pragma unroll
        for (int j = 0; j < LK; ++j) {
            u64 v;
            if (j >= lo && j < hi) {
                v = x[j];
            } else {
                const u64 m = dc->mod[j].q;
                v = 0;
#pragma unroll
                for (int i = lo; i < hi; ++i) v += shoup_lazy(y[i], dc->dig_hat[i][j], dc->dig_hat_sh[i][j], m);
                v = reduce_small_quot(v, dc->mod[j]);
            }
            out[(size_t)j * n + k] = neg ? neg_mod(v, dc->mod[j].q) : v;
        }
    }
}

void launch_ks_modup(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, int src_poly,
                     const u32* ginv, u64* DX, int items, cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        k_ks_modup<SHAPE_ARGS><<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, SRC, nullptr, src_poly, ginv, DX);
    });
    CSSC_CHECK_LAUNCH();
}

void launch_ks_modup_contig(const DevConsts* dc, const RnsParams& P, const u64* SRC, u64* DX,
                            int items, cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        k_ks_modup<SHAPE_ARGS><<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, nullptr, SRC, 0, nullptr, DX);
    });
    CSSC_CHECK_LAUNCH();
}

// ACC[item][2][LK][N] = sum_digit DX (.) KEY  (NTT domain)
template <int LT, int KT, int AT>
__global__ void k_ks_inner(const DevConsts* __restrict__ dc, const u64* __restrict__ DX,
                           const u64* const* KEY, u64* __restrict__ ACC) {
    const int n = dc->n, L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int alpha = AT ? AT : dc->alpha, dnum = (L + alpha - 1) / alpha;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64* key = KEY[item];
    const size_t PL = (size_t)LK * n;
#pragma unroll
    for (int j = 0; j < LK; ++j) {
        const Modulus md = dc->mod[j];
        u64 a0 = 0, a1 = 0;
#pragma unroll
        for (int dg = 0; dg < dnum; ++dg) {
            const u64 d = DX[((size_t)item * dnum + dg) * PL + (size_t)j * n + k];
            const u64 k0 = __ldg(key + ((size_t)dg * 2 + 0) * PL + (size_t)j * n + k);
            const u64 k1 = __ldg(key + ((size_t)dg * 2 + 1) * PL + (size_t)j * n + k);
            a0 = add_mod(a0, mul_mod(d, k0, md), md.q);
            a1 = add_mod(a1, mul_mod(d, k1, md), md.q);
        }
        ACC[((size_t)item * 2 + 0) * PL + (size_t)j * n + k] = a0;
        ACC[((size_t)item * 2 + 1) * PL + (size_t)j * n + k] = a1;
    }
}

void launch_ks_inner(const DevConsts* dc, const RnsParams& P, const u64* DX,
                     const u64* const* KEY, u64* ACC, int items, cudaStream_t st) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        k_ks_inner<SHAPE_ARGS><<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, DX, KEY, ACC);
    });
    CSSC_CHECK_LAUNCH();
}

// E4 + fused adds: out = BASE[item] + EXTRA[item] + phi_g(RSRC[item].c0) + ModDown(acc);
// per-item BASE / EXTRA entries may be null.  PAIR (nullable): PAIR[item] = j >= 0
// also adds item j's rotation phi_gj(RSRC[j].c0) + ModDown(acc_j) (item j has no
// BASE / EXTRA of its own) and PAIR[j] = -3 - item: item's CTAs write limbs
// [0, L/2) of the merged sum, j's CTAs limbs [L/2, L), both into OUT[item].
// Every sum is exact mod q, so merging two rotations' adds into one pass gives
// the words of the separate rotate and add.
// one polynomial per grid z-slice; the output loop is only partly unrolled so
// the acc/base/extra loads of all limbs are not hoisted into registers at once
template <int LT, int KT, int AT>
__global__ void __launch_bounds__(128, 6) k_ks_moddown(const DevConsts* __restrict__ dc, const u64* __restrict__ ACC,
                             const u64* const* BASE, const u64* const* RSRC, const u32* ginv,
                             u64* const* OUT, const u64* const* EXTRA, const int* PAIR) {
    const int n = dc->n, L = LT ? LT : dc->L, K = KT ? KT : dc->K, LK = L + K;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int pv = PAIR ? PAIR[blockIdx.y] : -1;  // see k_ks_moddown_k
    const int item = pv <= -3 ? -3 - pv : blockIdx.y;
    const int pair = pv <= -3 ? blockIdx.y : pv;
    const int nsrc = pair >= 0 ? 2 : 1;
    const int jlo = pv <= -3 ? L / 2 : 0, jhi = pv >= 0 ? L / 2 : L;
    const size_t PL = (size_t)LK * n;
    const int p = blockIdx.z;
    u64* out = OUT[item] + (size_t)p * L * n;
    const u64* base = BASE ? BASE[item] : nullptr;
    if (base) base += (size_t)p * L * n;
    const u64* ex = EXTRA ? EXTRA[item] : nullptr;
    if (ex) ex += (size_t)p * L * n;
    for (int s = 0; s < nsrc; ++s) {
        const int it = s ? pair : item;
        bool neg = false;
        int ridx = k;
        if (RSRC) ridx = automorph_src(ginv ? ginv[it] : 0u, k, n, neg);
        u64 y[MAXL];
        const u64* acc = ACC + ((size_t)it * 2 + p) * PL;
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const u64 pk = dc->mod[L + kk].q;
            y[kk] = shoup_q(acc[(size_t)(L + kk) * n + k], dc->phat_inv[kk], dc->phat_inv_sh[kk], pk);
        }
        const u64* rs = (RSRC && p == 0) ? RSRC[it] : nullptr;
#pragma unroll 2
        for (int j = jlo; j < jhi; ++j) {
            const u64 q = dc->mod[j].q;
            u64 c = 0;
#pragma unroll
            for (int kk = 0; kk < K; ++kk) c += shoup_lazy_q(y[kk], dc->phat_q[kk][j], dc->phat_q_sh[kk][j], q);
            c = reduce_small_quot_q(c, dc->mod[j]);
            u64 v = shoup_q(sub_mod(acc[(size_t)j * n + k], c, q), dc->Pinv_q[j], dc->Pinv_q_sh[j], q);
            if (s) {
                v = add_mod(v, out[(size_t)j * n + k], q);  // this thread's own first-pass word
            } else {
                if (base) v = add_mod(v, base[(size_t)j * n + k], q);
                if (ex) v = add_mod(v, ex[(size_t)j * n + k], q);
            }
            if (rs) {
                const u64 r = rs[(size_t)j * n + ridx];
                v = add_mod(v, neg ? neg_mod(r, q) : r, q);
            }
            out[(size_t)j * n + k] = v;
        }
    }
}

template <int L, int K>
struct ModDownK {
    int n;
    u64 pk[K], phat_inv[K], phat_inv_sh[K];
    Modulus qm[L];
    // out_j = (acc_j - sum_k y_k [P/p_k]_{q_j}) P^-1 = acc_j Pinv + sum_k y_k E_kj
    W29 E[K][L];  // [-[P/p_k]_{q_j} P^-1]_{q_j} in 29-bit halves
    W29 F[L];     // [P^-1]_{q_j}
    u64 dhi[L], dhi_sh[L];  // ModUp factors of the output's c1 (KsY)
};

// k_ks_moddown with the constants from a parameter block (same values; the
// ModDown of each target limb is one Dot29 of K + 1 terms; same PAIR merge)
template <int L, int K>
__global__ void __launch_bounds__(128, 6) k_ks_moddown_k(const __grid_constant__ ModDownK<L, K> c,
                                                         const u64* __restrict__ ACC, const u64* const* BASE,
                                                         const u64* const* RSRC, const u32* ginv, u64* const* OUT,
                                                         const u64* const* EXTRA, const int* PAIR,
                                                         u64* const* YOUT) {
    constexpr int LK = L + K;
    static_assert(K + 1 <= 15, "Dot29 bound");
    const int n = c.n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    // PAIR: a merged pair (D, O) shares its 2 x L limb outputs: D's CTAs
    // write limbs [0, L/2) of rot_D + rot_O, O's CTAs limbs [L/2, L), both
    // into D's output with D's BASE / EXTRA
    const int pv = PAIR ? PAIR[blockIdx.y] : -1;
    const int item = pv <= -3 ? -3 - pv : blockIdx.y;
    const int pair = pv <= -3 ? blockIdx.y : pv;
    const int p = blockIdx.z;
    u64* out = OUT[item] + (size_t)p * L * n;
    u64* yo = (p == 1 && YOUT) ? YOUT[item] : nullptr;  // ModUp factors of c1 for the next key switch
    const u64* base = BASE ? BASE[item] : nullptr;
    if (base) base += (size_t)p * L * n;
    const u64* ex = EXTRA ? EXTRA[item] : nullptr;
    if (ex) ex += (size_t)p * L * n;
    auto setup = [&](int it, u64* y, const u64*& acc, const u64*& rs, int& ridx, bool& neg) {
        neg = false;
        ridx = k;
        if (RSRC) ridx = automorph_src(ginv ? ginv[it] : 0u, k, n, neg);
        acc = ACC + ((size_t)it * 2 + p) * LK * n;
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
            y[kk] = shoup_q(acc[(size_t)(L + kk) * n + k], c.phat_inv[kk], c.phat_inv_sh[kk], c.pk[kk]);
        rs = (RSRC && p == 0) ? RSRC[it] : nullptr;
    };
    auto term = [&](int j, const u64* y, const u64* acc, const u64* rs, int ridx, bool neg) {
        const u64 q = c.qm[j].q;
        Dot29 d;
        u64 a = acc[(size_t)j * n + k];  // lazy (< 2q) when the inverse NTT left N^-1 to F
        a = a >= q ? a - q : a;
        dot29_mac(d, a, c.F[j]);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) dot29_mac(d, y[kk], c.E[kk][j]);
        u64 v = dot29_reduce_q(d, c.qm[j]);
        if (rs) {
            const u64 r = rs[(size_t)j * n + ridx];
            v = add_mod(v, neg ? neg_mod(r, q) : r, q);
        }
        return v;
    };
    u64 y[K];
    const u64 *acc, *rs;
    int ridx;
    bool neg;
    setup(item, y, acc, rs, ridx, neg);
    if (pair < 0 && L <= 4) {
        // small L: every load of the coefficient is issued before any product
        // (the launches are latency-bound: long-scoreboard stalls dominate)
        u64 av[L], bv[L], rv[L];
#pragma unroll
        for (int j = 0; j < L; ++j) {
            av[j] = acc[(size_t)j * n + k];
            av[j] = av[j] >= c.qm[j].q ? av[j] - c.qm[j].q : av[j];
            bv[j] = base ? base[(size_t)j * n + k] : 0;
            if (ex) bv[j] = add_mod(bv[j], ex[(size_t)j * n + k], c.qm[j].q);
            rv[j] = rs ? rs[(size_t)j * n + ridx] : 0;
        }
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const u64 q = c.qm[j].q;
            Dot29 d;
            dot29_mac(d, av[j], c.F[j]);
#pragma unroll
            for (int kk = 0; kk < K; ++kk) dot29_mac(d, y[kk], c.E[kk][j]);
            u64 v = dot29_reduce_q(d, c.qm[j]);
            if (rs) v = add_mod(v, neg ? neg_mod(rv[j], q) : rv[j], q);
            v = add_mod(v, bv[j], q);
            out[(size_t)j * n + k] = v;
            if (yo) yo[(size_t)j * n + k] = shoup_q(v, c.dhi[j], c.dhi_sh[j], q);
        }
    } else if (pair < 0) {
#pragma unroll 2
        for (int j = 0; j < L; ++j) {
            const u64 q = c.qm[j].q;
            u64 v = term(j, y, acc, rs, ridx, neg);
            if (base) v = add_mod(v, base[(size_t)j * n + k], q);
            if (ex) v = add_mod(v, ex[(size_t)j * n + k], q);
            out[(size_t)j * n + k] = v;
            if (yo) yo[(size_t)j * n + k] = shoup_q(v, c.dhi[j], c.dhi_sh[j], q);
        }
    } else {  // merged rotation of item `pair`, half of the limbs
        u64 y2[K];
        const u64 *acc2, *rs2;
        int ridx2;
        bool neg2;
        setup(pair, y2, acc2, rs2, ridx2, neg2);
        const int jlo = pv <= -3 ? L / 2 : 0, jhi = pv <= -3 ? L : L / 2;
#pragma unroll 1
        for (int j = jlo; j < jhi; ++j) {
            const u64 q = c.qm[j].q;
            u64 v = add_mod(term(j, y, acc, rs, ridx, neg), term(j, y2, acc2, rs2, ridx2, neg2), q);
            if (base) v = add_mod(v, base[(size_t)j * n + k], q);
            if (ex) v = add_mod(v, ex[(size_t)j * n + k], q);
            out[(size_t)j * n + k] = v;
            if (yo) yo[(size_t)j * n + k] = shoup_q(v, c.dhi[j], c.dhi_sh[j], q);
        }
    }
}

// lazy: ACC is the inverse NTT without its final x N^-1 (NttJob::lazy_out);
// N^-1 rides in (P/p_k)^-1 (the y_k) and in P^-1 (the acc_j term)
template <int L, int K>
static ModDownK<L, K> make_moddown_k(const RnsParams& P, bool lazy = false) {
    const DevConsts& h = P.host;
    ModDownK<L, K> c{};
    c.n = P.n;
    for (int kk = 0; kk < K; ++kk) {
        c.pk[kk] = h.mod[L + kk].q;
        c.phat_inv[kk] = lazy ? host_mulmod(h.phat_inv[kk], h.ninv[L + kk], c.pk[kk]) : h.phat_inv[kk];
        c.phat_inv_sh[kk] = lazy ? shoup_factor(c.phat_inv[kk], c.pk[kk]) : h.phat_inv_sh[kk];
    }
    for (int j = 0; j < L; ++j) {
        c.qm[j] = h.mod[j];
        c.dhi[j] = h.dig_hat_inv[j];
        c.dhi_sh[j] = h.dig_hat_inv_sh[j];
        const u64 q = h.mod[j].q;
        c.F[j] = split29(lazy ? host_mulmod(h.Pinv_q[j], h.ninv[j], q) : h.Pinv_q[j]);
        for (int kk = 0; kk < K; ++kk)
            c.E[kk][j] = split29((q - host_mulmod(h.phat_q[kk][j], h.Pinv_q[j], q)) % q);
    }
    return c;
}

// The key switch's inverse column phase fused with ModDown (E4) for the
// fixed shapes: one CTA = one (item, polynomial, LN-column tile).  The L+K
// limb tiles of ACC (block phase already inverted by K2) are loaded once,
// inverse-transformed in shared memory (lazy: N^-1 rides in the ModDown
// constants, make_moddown_k(P, true)), and ModDown + base + extra + the
// rotated c0 of the source run on the tile; the accumulators cross HBM once
// (written by K2, read here) instead of three times, and one launch goes.
// PAIR (level 0): the CTAs of a D_1 item also transform their O_1 partner's
// tiles and add both ModDowns (same sums as k_ks_moddown_k's split pair);
// the partner's CTAs exit.  Same words as k_ntt_cols + k_ks_moddown_k.
template <int LOGN, int L, int K, int LN, int RADIX = 3>
__global__ void __launch_bounds__(Ntt2<LOGN>::TC, 256 / Ntt2<LOGN>::TC * (RADIX == 3 ? 3 : 4)) k_ks_cols_moddown(
    const __grid_constant__ ModDownK<L, K> c, const DevConsts* __restrict__ dc, const u64* __restrict__ ACC,
    const u64* const* BASE, const u64* const* RSRC, const u32* ginv, u64* const* OUT, const u64* const* EXTRA,
    const int* PAIR, u64* const* YOUT, const u64* const* XACC) {
    using G = Ntt2<LOGN>;
    constexpr int LK = L + K, T = G::TC, CTAS = G::R2 / LN, SEG = LN / 2;
    constexpr int VL = LK * LN;                 // lines: (limb, column)
    constexpr int TILE = LN * G::R1, PER = TILE / T;  // elements per thread and limb
    constexpr int TWS = 2 * G::R1 + 2;          // per-limb twiddle stride (16 B pad: limbs on distinct banks)
    static_assert(PER >= 1 && TILE % T == 0 && T % VL == 0, "tile smaller than the CTA");
    extern __shared__ u64 smem[];
    u64* tiles = smem;              // [R1][VL], line = limb * LN + column
    u64* tws = smem + LK * TILE;    // [LK][TWS] (w, w_shoup) pairs
    const int n = c.n;
    const int tileid = blockIdx.x % CTAS;
    const int rest = blockIdx.x / CTAS;
    const int p = rest & 1;
    const int item = rest >> 1;
    const int pv = PAIR ? PAIR[item] : -1;
    if (pv <= -3) return;  // an O_1 partner: evaluated by its D_1's CTAs
    const int col0 = tileid * LN;
    for (int j = 0; j < LK; ++j)
        for (int i = threadIdx.x; i < G::R1; i += T) cp_async16(tws + (size_t)j * TWS + 2 * i, dc->tw[j].inv + 2 * i);
    auto addr = [](int l, int pos) { return pos * VL + l; };
    auto at = [](int j, int e) { return (e / LN) * VL + j * LN + (e % LN); };  // element e of limb j's tile
    // every thread keeps one line (tid % VL) in every pass: its modulus and
    // twiddle row are per-thread constants
    const int myl = threadIdx.x % VL;
    const u64 myq = dc->mod[myl / LN].q;
    const u64* mytw = tws + (size_t)(myl / LN) * TWS;
    // inverse column phase of item `it`'s LK tiles of polynomial p, in smem:
    // all limbs in the same passes (radix-8, 16 lines)
    auto transform = [&](int it) {
        const u64* acc = ACC + ((size_t)it * 2 + p) * LK * n;
#pragma unroll
        for (int j = 0; j < LK; ++j) {
#pragma unroll
            for (int r = 0; r < G::R1 * SEG / T; ++r) {
                const int i = threadIdx.x + T * r, cc = i / SEG, h = i % SEG;
                cp_async16(tiles + (size_t)cc * VL + j * LN + 2 * h, acc + (size_t)j * n + (size_t)cc * G::R2 + col0 + 2 * h);
            }
        }
        cp_async_wait_all();
        __syncthreads();
        const u64* xa = XACC ? XACC[it] : nullptr;  // an odd step's accumulators, same shared ModDown
        if (xa) {
            xa += (size_t)p * LK * n;
#pragma unroll
            for (int r = 0; r < LK * TILE / T; ++r) {
                const int i = threadIdx.x + T * r, cc = i / VL, l = i % VL, j = l / LN;
                const u64 q2 = 2 * dc->mod[j].q;
                u64& t = tiles[(size_t)cc * VL + l];
                const u64 s = t + xa[(size_t)j * n + (size_t)cc * G::R2 + col0 + (l % LN)];
                t = s >= q2 ? s - q2 : s;
            }
            __syncthreads();
        }
        auto twf = [&](int sl, int, int blk) {
            const int k = (1 << sl) + blk;
            return *reinterpret_cast<const ulonglong2*>(mytw + 2 * k);
        };
        line_ntt_v<G::A, 0, true, RADIX, VL>(tiles, SpecQ{myq}, addr, twf, whole_cta());
    };
    // ModDown of element e of the transformed tiles of item `it` (+ its rotated c0)
    auto moddown = [&](int it, int e, u64 out[L]) {
        const int k = (e / LN) * G::R2 + col0 + (e % LN);
        u64 y[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk)
            y[kk] = shoup_q(tiles[at(L + kk, e)], c.phat_inv[kk], c.phat_inv_sh[kk], c.pk[kk]);
        const u64* rs = (RSRC && p == 0) ? RSRC[it] : nullptr;
        bool neg = false;
        const int ridx = rs ? automorph_src(ginv ? ginv[it] : 0u, k, n, neg) : k;
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const u64 q = c.qm[j].q;
            u64 a = tiles[at(j, e)];
            a = a >= q ? a - q : a;
            Dot29 d;
            dot29_mac(d, a, c.F[j]);
#pragma unroll
            for (int kk = 0; kk < K; ++kk) dot29_mac(d, y[kk], c.E[kk][j]);
            u64 v = dot29_reduce_q(d, c.qm[j]);
            if (rs) {
                const u64 r = rs[(size_t)j * n + ridx];
                v = add_mod(v, neg ? neg_mod(r, q) : r, q);
            }
            out[j] = v;
        }
    };
    transform(item);
    u64 v[PER][L];
#pragma unroll
    for (int r = 0; r < PER; ++r) moddown(item, threadIdx.x + T * r, v[r]);
    if (pv >= 0) {  // D_1 of a merged pair: add the rotation of its O_1 partner
        __syncthreads();
        transform(pv);
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            u64 w[L];
            moddown(pv, threadIdx.x + T * r, w);
#pragma unroll
            for (int j = 0; j < L; ++j) v[r][j] = add_mod(v[r][j], w[j], c.qm[j].q);
        }
    }
    u64* out = OUT[item] + (size_t)p * L * n;
    u64* yo = (p == 1 && YOUT) ? YOUT[item] : nullptr;
    const u64* base = BASE ? BASE[item] : nullptr;  // per-item entries may be null (hoisted odd steps)
    if (base) base += (size_t)p * L * n;
    const u64* ex = EXTRA ? EXTRA[item] : nullptr;
    if (ex) ex += (size_t)p * L * n;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int e = threadIdx.x + T * r;
        const size_t k = (size_t)(e / LN) * G::R2 + col0 + (e % LN);
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const u64 q = c.qm[j].q;
            u64 x = v[r][j];
            if (base) x = add_mod(x, base[(size_t)j * n + k], q);
            if (ex) x = add_mod(x, ex[(size_t)j * n + k], q);
            out[(size_t)j * n + k] = x;
            if (yo) yo[(size_t)j * n + k] = shoup_q(x, c.dhi[j], c.dhi_sh[j], q);
        }
    }
}

template <int LOGN, int L, int K, int LN>
static bool cols_moddown_ln(const DevConsts* dc, const RnsParams& P, const u64* ACC, const u64* const* BASE,
                            const u64* const* RSRC, const u32* ginv, u64* const* OUT, int items, cudaStream_t st,
                            const u64* const* EXTRA, const int* PAIR, u64* const* YOUT, const u64* const* XACC);

template <int LOGN, int L, int K>
static bool cols_moddown_t(const DevConsts* dc, const RnsParams& P, const u64* ACC, const u64* const* BASE,
                           const u64* const* RSRC, const u32* ginv, u64* const* OUT, int items, cudaStream_t st,
                           const u64* const* EXTRA, const int* PAIR, u64* const* YOUT, const u64* const* XACC) {
    using G = Ntt2<LOGN>;
    static const int ln = [] {
        const char* e = std::getenv("CSSC_COLS_MODDOWN_LN");
        return e ? std::atoi(e) : 4;
    }();
    // 4-column tiles (radix-4 passes, 40 KB smem, 3 CTAs per SM) measured faster
    // than 8 (80 KB, 2 CTAs per SM): C5 6.08 vs 6.19 ms
    if (ln == 8)
        return cols_moddown_ln<LOGN, L, K, 8>(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, XACC);
    return cols_moddown_ln<LOGN, L, K, 4>(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, XACC);
}

template <int LOGN, int L, int K, int LN>
static bool cols_moddown_ln(const DevConsts* dc, const RnsParams& P, const u64* ACC, const u64* const* BASE,
                            const u64* const* RSRC, const u32* ginv, u64* const* OUT, int items, cudaStream_t st,
                            const u64* const* EXTRA, const int* PAIR, u64* const* YOUT, const u64* const* XACC) {
    using G = Ntt2<LOGN>;
    if constexpr (G::R2 < 16 || G::R1 * LN < G::TC) {
        return false;
    } else {
        constexpr int smem = ((L + K) * LN * G::R1 + (L + K) * (2 * G::R1 + 2)) * 8;
        const unsigned grid = (unsigned)items * 2 * (G::R2 / LN);
        static const int radix = [] {
            const char* e = std::getenv("CSSC_CMD_RADIX");  // radix-4 passes (64 regs, 4 CTAs/SM) measured 0.2 % faster at C5
            return e ? std::atoi(e) : 2;
        }();
        if (radix == 2) {
            smem_optin_k(k_ks_cols_moddown<LOGN, L, K, LN, 2>, smem);
            k_ks_cols_moddown<LOGN, L, K, LN, 2><<<grid, G::TC, smem, st>>>(make_moddown_k<L, K>(P, true), dc, ACC,
                                                                            BASE, RSRC, ginv, OUT, EXTRA, PAIR, YOUT,
                                                                            XACC);
        } else {
            smem_optin_k(k_ks_cols_moddown<LOGN, L, K, LN>, smem);
            k_ks_cols_moddown<LOGN, L, K, LN><<<grid, G::TC, smem, st>>>(make_moddown_k<L, K>(P, true), dc, ACC, BASE,
                                                                         RSRC, ginv, OUT, EXTRA, PAIR, YOUT, XACC);
        }
        CSSC_CHECK_LAUNCH();
        return true;
    }
}

// The fused kernel gives each CTA a whole (item, polynomial) column tile of
// all L+K limbs: launches of fewer than one wave of such CTAs (a lone
// rotation, C1/C2's small levels) keep the two-kernel path, whose separate
// launches spread the same work over more CTAs.
bool ks_cols_moddown_applies(const RnsParams& P, int items) {
    static const bool off = std::getenv("CSSC_NO_COLS_MODDOWN") != nullptr;
    const auto& cf = P.cfg;
    if (off || cf.L != 2 || cf.K != 2 || cf.alpha != 2 || (cf.logn != 13 && cf.logn != 14)) return false;
    const long ctas = (long)items * 2 * (64 / 4);  // R2 / LN: R2 = 64 at 2^13 and 2^14, LN = 4
    return ctas >= 3L * 148;
}

bool launch_ks_cols_moddown(const DevConsts* dc, const RnsParams& P, const u64* ACC, const u64* const* BASE,
                            const u64* const* RSRC, const u32* ginv, u64* const* OUT, int items, cudaStream_t st,
                            const u64* const* EXTRA, const int* PAIR, u64* const* YOUT, const u64* const* XACC) {
    if (!items || !ks_cols_moddown_applies(P, items)) return false;
    const auto& cf = P.cfg;
    {
        switch (cf.logn) {
            case 13:
                return cols_moddown_t<13, 2, 2>(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, XACC);
            case 14:
                return cols_moddown_t<14, 2, 2>(dc, P, ACC, BASE, RSRC, ginv, OUT, items, st, EXTRA, PAIR, YOUT, XACC);
            default: return false;
        }
    }
    return false;
}

void launch_ks_moddown(const DevConsts* dc, const RnsParams& P, const u64* ACC,
                       const u64* const* BASE, const u64* const* RSRC, const u32* ginv,
                       u64* const* OUT, int items, cudaStream_t st, const u64* const* EXTRA, const int* PAIR,
                       u64* const* YOUT, bool lazy_in) {
    if (!items) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        dim3 g = ew_grid(P.n, items);
        g.z = 2;
        constexpr int LT = decltype(l_)::value, KT = decltype(k_)::value;
        if constexpr (LT > 0)
            k_ks_moddown_k<LT, KT><<<g, EW_THREADS, 0, st>>>(make_moddown_k<LT, KT>(P, lazy_in), ACC, BASE, RSRC,
                                                            ginv, OUT, EXTRA, PAIR, YOUT);
        else if (lazy_in)
            throw std::invalid_argument("unscaled inverse-NTT input needs a fixed RNS shape");
        else if (YOUT)
            throw std::invalid_argument("hoisted ModUp factors need a fixed RNS shape");
        else
            k_ks_moddown<SHAPE_ARGS><<<g, EW_THREADS, 0, st>>>(dc, ACC, BASE, RSRC, ginv, OUT, EXTRA, PAIR);
    });
    CSSC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// masks and plaintext products
// ---------------------------------------------------------------------------
template <int LT, int KT, int AT>
__global__ void k_mask_accum(const DevConsts* __restrict__ dc, const u64* __restrict__ MT,
                             const int* slice_off, const int* slice_items, const int* item_mask,
                             const u64* __restrict__ MASKS, u64* __restrict__ RES) {
    const int n = dc->n, L = LT ? LT : dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = blockIdx.y;
    const int b = slice_off[s], e = slice_off[s + 1];
    const size_t CT = (size_t)2 * L * n;
    u64 acc[2 * MAXL];
#pragma unroll
    for (int x = 0; x < 2 * L; ++x) acc[x] = 0;
    for (int x = b; x < e; ++x) {
        const int it = slice_items[x];
        const u64* mt = MT + (size_t)it * CT + k;
        const u64* mk = MASKS + (size_t)item_mask[it] * L * n + k;
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const Modulus md = dc->mod[j];
            const u64 m = mk[(size_t)j * n];
            acc[j] = add_mod(acc[j], mul_mod(mt[(size_t)j * n], m, md), md.q);
            acc[L + j] = add_mod(acc[L + j], mul_mod(mt[(size_t)(L + j) * n], m, md), md.q);
        }
    }
#pragma unroll
    for (int x = 0; x < 2 * L; ++x) RES[(size_t)s * CT + (size_t)x * n + k] = acc[x];
}

void launch_mask_accum(const DevConsts* dc, const RnsParams& P, const u64* MT,
                       const int* slice_off, const int* slice_items, const int* item_mask,
                       const u64* MASKS, u64* RES, int slices, cudaStream_t st) {
    if (!slices) return;
    dispatch_shape(P, [&](auto l_, auto k_, auto a_) {
        k_mask_accum<SHAPE_ARGS><<<ew_grid(P.n, slices), EW_THREADS, 0, st>>>(dc, MT, slice_off, slice_items,
                                                                              item_mask, MASKS, RES);
    });
    CSSC_CHECK_LAUNCH();
}

// X[item][poly][L][N] *= PT[item][L][N]
__global__ void k_pointwise_plain(const DevConsts* __restrict__ dc, u64* X, const u64* PT,
                                  int polys) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    for (int p = 0; p < polys; ++p)
        for (int j = 0; j < L; ++j) {
            const size_t o = (((size_t)item * polys + p) * L + j) * n + k;
            X[o] = mul_mod(X[o], PT[((size_t)item * L + j) * n + k], dc->mod[j]);
        }
}

void launch_pointwise_plain(const DevConsts* dc, const RnsParams& P, u64* X, const u64* PT,
                            int items, int polys, cudaStream_t st) {
    if (!items) return;
    k_pointwise_plain<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, X, PT, polys);
    CSSC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// encoding, encryption, decryption
// ---------------------------------------------------------------------------
__global__ void k_encode_scatter(const DevConsts* __restrict__ dc, const int64_t* vals,
                                 const u64* offs, u64* M, size_t mstride) {
    const int S = dc->n / 2;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64 b = offs[item];
    if (j >= S || (u64)j >= offs[item + 1] - b) return;
    const int64_t t = (int64_t)dc->t;
    int64_t v = vals[b + j] % t;
    if (v < 0) v += t;
    M[(size_t)item * mstride + dc->pos0[j]] = (u64)v;
}

void launch_encode_scatter(const DevConsts* dc, const RnsParams& P, const int64_t* vals,
                           const u64* offs, u64* M, int items, cudaStream_t st, size_t mstride) {
    if (!items) return;
    if (!mstride) mstride = (size_t)P.n;
    cudaMemset2DAsync(M, mstride * 8, 0, (size_t)P.n * 8, (size_t)items, st);
    k_encode_scatter<<<dim3((unsigned)(P.S / EW_THREADS + 1), (unsigned)items), EW_THREADS, 0, st>>>(
        dc, vals, offs, M, mstride);
    CSSC_CHECK_LAUNCH();
}

// Client A + Client B fused: row record {nz_begin, len, pos, slice}; entry j of
// the row sits in aligned column j (csr_to_cssc, sparse.cpp:79-117), which
// chunk cols[col_base + j] = {chunk, k, h} holds at flat slot k h + pos
// (generate_chunks, chunk.cpp:10-52); the vector chunk takes v[col] at the
// same slot (reorg_vector, reorg.cpp).  Padding stays 0 (memset).
// One thread per row entry (load-balanced for power-law rows: a hub row of
// thousands of entries no longer serialises on a few lanes): entry e belongs
// to row record r with rpre[r] <= e < rpre[r + 1] (binary search over the
// exclusive prefix of the row lengths), at aligned column j = e - rpre[r].
template <class CIT, class VAT, class VT>
__global__ void k_pack_cssc(const DevConsts* __restrict__ dc, const CIT* __restrict__ CI,
                            const VAT* __restrict__ VA, const VT* __restrict__ V,
                            const int4* __restrict__ rows, const int* __restrict__ rpre, int n_rows,
                            const int2* __restrict__ slices, const int4* __restrict__ cols, int n_chunks,
                            u64* __restrict__ M, size_t mstride) {
    __shared__ int range[2];
    const int e0 = blockIdx.x * blockDim.x;
    const int e = e0 + threadIdx.x;
    const int total = __ldg(rpre + n_rows);
    auto row_of = [&](int x, int lo, int hi) {  // last r in [lo, hi] with rpre[r] <= x
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(rpre + mid) <= x) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    // the CTA's first and last entries bound every thread's search; both are
    // located cooperatively (each round: every thread samples one row prefix,
    // __syncthreads_count narrows [lo, hi] by the CTA width), so two rounds
    // of loads replace a ~log2(rows)-deep dependent chain
    if (e0 >= total) return;  // uniform per CTA
    const int x0 = e0, x1 = min(e0 + (int)blockDim.x, total) - 1;
    int lo0 = 0, hi0 = n_rows - 1, lo1 = 0, hi1 = n_rows - 1;
    const int nt = blockDim.x;
    for (int round = 0; round < 2 && (hi0 > lo0 || hi1 > lo1); ++round) {
        // sample r_t = lo + ceil(t * span / nt): the last r with rpre[r] <= x lies
        // in [r_(c-1), r_c - 1], c = #samples <= x (rpre is non-decreasing)
        const int s0 = hi0 - lo0 + 1, s1 = hi1 - lo1 + 1;
        const int r0 = lo0 + (int)(((long)threadIdx.x * s0 + nt - 1) / nt);
        const int r1 = lo1 + (int)(((long)threadIdx.x * s1 + nt - 1) / nt);
        const bool p0 = r0 <= hi0 && __ldg(rpre + r0) <= x0;
        const bool p1 = r1 <= hi1 && __ldg(rpre + r1) <= x1;
        const int c0 = __syncthreads_count(p0), c1 = __syncthreads_count(p1);
        auto narrow = [&](int c, int& lo, int& hi, int span) {
            const int a = lo + (int)(((long)(c - 1) * span + nt - 1) / nt);      // sample c-1 (c >= 1: rpre[lo] <= x)
            const int b = c < nt ? lo + (int)(((long)c * span + nt - 1) / nt) - 1 : hi;
            lo = a;
            hi = min(b, hi);
        };
        narrow(c0, lo0, hi0, s0);
        narrow(c1, lo1, hi1, s1);
    }
    if (threadIdx.x < 2) range[threadIdx.x] = threadIdx.x ? row_of(x1, lo1, hi1) : row_of(x0, lo0, hi0);
    __syncthreads();
    if (e >= total) return;
    const int lo = row_of(e, range[0], range[1]);
    const int4 rec = rows[lo];
    const int j = e - __ldg(rpre + lo);
    const int2 sl = slices[rec.w];
    const int64_t t = (int64_t)dc->t;
    const int4 c = __ldg(cols + sl.x + j);
    if (c.x < 0) return;  // a chunk another rank evaluates (sharded jobs)
    const u32 pos = dc->pos0[c.y * c.z + rec.z];
    int64_t a = (int64_t)VA[rec.x + j] % t;
    int64_t b = (int64_t)V[(int64_t)sl.y + (int64_t)CI[rec.x + j]] % t;
    M[(size_t)c.x * mstride + pos] = (u64)(a < 0 ? a + t : a);
    M[(size_t)(n_chunks + c.x) * mstride + pos] = (u64)(b < 0 ? b + t : b);
}

template <class CIT, class VAT, class VT>
static void pack_t(const DevConsts* dc, const void* CI, const void* VA, const void* V, const int4* rows,
                   const int* rpre, int n_rows, long entries, const int2* slices, const int4* cols, int n_chunks,
                   u64* M, size_t mstride, cudaStream_t st) {
    k_pack_cssc<CIT, VAT, VT><<<(unsigned)((entries + 127) / 128), 128, 0, st>>>(
        dc, static_cast<const CIT*>(CI), static_cast<const VAT*>(VA), static_cast<const VT*>(V), rows, rpre, n_rows,
        slices, cols, n_chunks, M, mstride);
}

template <class CIT>
static void pack_ci(int va_w, int v_w, const DevConsts* dc, const void* CI, const void* VA, const void* V,
                    const int4* rows, const int* rpre, int n_rows, long entries, const int2* slices, const int4* cols,
                    int n_chunks, u64* M, size_t mstride, cudaStream_t st) {
    if (va_w == 1 && v_w == 1)
        pack_t<CIT, int8_t, int8_t>(dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride, st);
    else if (va_w == 1)
        pack_t<CIT, int8_t, int64_t>(dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride, st);
    else if (v_w == 1)
        pack_t<CIT, int64_t, int8_t>(dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride, st);
    else
        pack_t<CIT, int64_t, int64_t>(dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride,
                                      st);
}

void launch_pack_cssc(const DevConsts* dc, const RnsParams& P, const void* CI, const void* VA, const void* V,
                      int ci_w, int va_w, int v_w, const int4* rows, const int* rpre, int n_rows, long entries,
                      const int2* slices, const int4* cols, int n_chunks, u64* M, size_t mstride, cudaStream_t st) {
    if (!n_chunks) return;
    cudaMemset2DAsync(M, mstride * 8, 0, (size_t)P.n * 8, (size_t)2 * n_chunks, st);
    if (n_rows && entries > 0) {
        if (ci_w == 2)
            pack_ci<uint16_t>(va_w, v_w, dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride,
                              st);
        else if (ci_w == 4)
            pack_ci<uint32_t>(va_w, v_w, dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride,
                              st);
        else
            pack_ci<uint64_t>(va_w, v_w, dc, CI, VA, V, rows, rpre, n_rows, entries, slices, cols, n_chunks, M, mstride,
                              st);
    }
    CSSC_CHECK_LAUNCH();
}

// PT[item][L][N] = centred lift of M[item][N] (mod t) to each q_j (coef form)
__global__ void k_plain_lift(const DevConsts* __restrict__ dc, const u64* M, u64* PT) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64 t = dc->t, m = M[(size_t)item * n + k];
    for (int j = 0; j < L; ++j) {
        const u64 q = dc->mod[j].q;
        PT[((size_t)item * L + j) * n + k] = m <= t / 2 ? m : q - (t - m);
    }
}

void launch_plain_lift(const DevConsts* dc, const RnsParams& P, const u64* M, u64* PT, int items,
                       cudaStream_t st) {
    if (!items) return;
    k_plain_lift<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, M, PT);
    CSSC_CHECK_LAUNCH();
}

// U[item][L][N]: one ChaCha block per thread (8 coefficients of u, the block
// counter = k / 8 as everywhere), all in registers -- no shuffles, no idle
// lanes; each thread writes its 8 words per limb as four 16-byte stores
__global__ void __launch_bounds__(128) k_enc_sample_u(const DevConsts* __restrict__ dc, SeedKey seed,
                                                      const u64* streams, u64* U) {
    const int n = dc->n, L = dc->L;
    const int item = blockIdx.y;
    const u64 id = streams[item];
    const int b = blockIdx.x * 128 + threadIdx.x;  // ChaCha block = coefficients 8b .. 8b+7
    if (8 * b >= n) return;
    u32 blk[16];
    chacha20_block(seed, (u32)b, DOM_ENC_U, (u32)id, (u32)(id >> 32), blk);
    int64_t u[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) u[w] = ternary_of(word64(blk, w));
    for (int j = 0; j < L; ++j) {
        const u64 q = dc->mod[j].q;
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(U + ((size_t)item * L + j) * n + 8 * (size_t)b);
#pragma unroll
        for (int w = 0; w < 4; ++w) dst[w] = make_ulonglong2(lift_signed(u[2 * w], q), lift_signed(u[2 * w + 1], q));
    }
}

void launch_enc_sample_u(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams,
                         u64* U, int items, cudaStream_t st) {
    if (!items) return;
    k_enc_sample_u<<<dim3((unsigned)((P.n / 8 + 127) / 128), (unsigned)items), 128, 0, st>>>(dc, seed, streams, U);
    CSSC_CHECK_LAUNCH();
}

// C[item][2][L][N] = PK[p] (.) U  (NTT domain)
__global__ void k_enc_pk(const DevConsts* __restrict__ dc, const u64* PK, const u64* U, u64* C) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    for (int j = 0; j < L; ++j) {
        const Modulus md = dc->mod[j];
        const u64 u = U[((size_t)item * L + j) * n + k];
        for (int p = 0; p < 2; ++p)
            C[((size_t)item * (2 * L + 1) + (size_t)p * L + j) * n + k] =
                mul_mod(__ldg(PK + ((size_t)p * L + j) * n + k), u, md);
    }
}

void launch_enc_pk(const DevConsts* dc, const RnsParams& P, const u64* PK, const u64* U, u64* C,
                   int items, cudaStream_t st) {
    if (!items) return;
    k_enc_pk<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, PK, U, C);
    CSSC_CHECK_LAUNCH();
}

// OUT = C + (e0 + Delta m, e1): a 128-thread CTA draws the 16 + 16 ChaCha
// blocks of its 128 coefficients (4 lanes per block), then one thread per
// coefficient finishes every limb with coalesced loads and stores
// E (int8 [item][2][N], drawn ahead by k_enc_sample_e): read the e draws
// instead of running ChaCha again (same words)
template <bool FROM_E>
__global__ void __launch_bounds__(128) k_enc_finish(const DevConsts* __restrict__ dc, SeedKey seed,
                                                    const u64* streams, const u64* C, size_t cstride,
                                                    const u64* MSG, size_t mstride, u64* const* OUT,
                                                    const int8_t* __restrict__ E) {
    const int n = dc->n, L = dc->L;
    const int item = blockIdx.y;
    const int kk = threadIdx.x, k = blockIdx.x * 128 + kk;
    int64_t e0, e1;
    if constexpr (FROM_E) {
        e0 = E[((size_t)item * 2) * n + k];
        e1 = E[((size_t)item * 2 + 1) * n + k];
    } else {
        __shared__ u32 blk[32][16];
        const u64 id = streams[item];
        const int g = threadIdx.x >> 2;
        chacha20_block_x4(seed, (u32)(blockIdx.x * 16 + (g & 15)), g < 16 ? DOM_ENC_E0 : DOM_ENC_E1, (u32)id,
                          (u32)(id >> 32), blk[g]);
        __syncthreads();
        e0 = cbd_of(word64(blk[kk >> 3], kk & 7));
        e1 = cbd_of(word64(blk[16 + (kk >> 3)], kk & 7));
    }
    const size_t cm = (size_t)item * cstride + k;
    const u64 m = MSG[(size_t)item * mstride + k];
    u64* out = OUT[item];
    for (int j = 0; j < L; ++j) {
        const u64 q = dc->mod[j].q;
        const size_t o0 = cm + (size_t)j * n;
        const size_t o1 = cm + (size_t)(L + j) * n;
        u64 c0 = add_mod(C[o0], lift_signed(e0, q), q);
        c0 = add_mod(c0, shoup(m, dc->delta[j], dc->delta_sh[j], q), q);
        const u64 c1 = add_mod(C[o1], lift_signed(e1, q), q);
        out[(size_t)j * n + k] = c0;
        out[((size_t)L + j) * n + k] = c1;
    }
}

// the e draws of k_enc_finish / k_mul_extend_enc, ahead of time: one ChaCha
// block per thread (8 coefficients, block counter = k / 8), in registers, one
// 8-byte store of the 8 int8 draws
__global__ void __launch_bounds__(128) k_enc_sample_e(SeedKey seed, const u64* streams, int8_t* E, int n) {
    const int item = blockIdx.y, poly = blockIdx.z;
    const u64 id = streams[item];
    const int b = blockIdx.x * 128 + threadIdx.x;
    if (8 * b >= n) return;
    u32 blk[16];
    chacha20_block(seed, (u32)b, poly ? DOM_ENC_E1 : DOM_ENC_E0, (u32)id, (u32)(id >> 32), blk);
    u64 packed = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) packed |= (u64)(uint8_t)(int8_t)cbd_of(word64(blk, w)) << (8 * w);
    *reinterpret_cast<u64*>(E + ((size_t)item * 2 + poly) * n + 8 * (size_t)b) = packed;
}

void launch_enc_sample_e(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams, int8_t* E,
                         int items, cudaStream_t st) {
    (void)dc;
    if (!items) return;
    k_enc_sample_e<<<dim3((unsigned)((P.n / 8 + 127) / 128), (unsigned)items, 2), 128, 0, st>>>(seed, streams, E,
                                                                                                 P.n);
    CSSC_CHECK_LAUNCH();
}

void launch_enc_finish(const DevConsts* dc, const RnsParams& P, SeedKey seed, const u64* streams,
                       const u64* CM, u64* const* OUT, int items, cudaStream_t st, const u64* MSG, size_t cstride,
                       size_t mstride, const int8_t* E) {
    if (!items) return;
    if (!cstride) cstride = (size_t)(2 * P.cfg.L + 1) * P.n;
    if (!MSG) {
        MSG = CM + (size_t)2 * P.cfg.L * P.n;
        mstride = cstride;
    }
    const dim3 g((unsigned)(P.n / 128), (unsigned)items);
    if (E)
        k_enc_finish<true><<<g, 128, 0, st>>>(dc, seed, streams, CM, cstride, MSG, mstride, OUT, E);
    else
        k_enc_finish<false><<<g, 128, 0, st>>>(dc, seed, streams, CM, cstride, MSG, mstride, OUT, nullptr);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_mul_s(const DevConsts* __restrict__ dc, u64* X, const u64* S_NTT) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    for (int j = 0; j < L; ++j) {
        const size_t o = ((size_t)item * L + j) * n + k;
        X[o] = mul_mod(X[o], S_NTT[(size_t)j * n + k], dc->mod[j]);
    }
}

void launch_mul_s(const DevConsts* dc, const RnsParams& P, u64* X, const u64* S_NTT, int items,
                  cudaStream_t st) {
    if (!items) return;
    k_mul_s<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, X, S_NTT);
    CSSC_CHECK_LAUNCH();
}

// E5: m = round(t (c0 + c1 s) / Q) mod t; maxdev = max |fraction| (2^-64 units)
__global__ void k_dec_scale(const DevConsts* __restrict__ dc, const u64* const* CT,
                            const u64* X, u64* M, unsigned long long* maxdev) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64* c0 = CT[item];
    u64 shi = 0, slo = 0;
    for (int i = 0; i < L; ++i) {
        const u64 q = dc->mod[i].q;
        const u64 x = add_mod(c0[(size_t)i * n + k], X[((size_t)item * L + i) * n + k], q);
        const u64 xi = shoup(x, dc->QhatInv[i], dc->QhatInv_sh[i], q);
        add128(shi, slo, umulhi(xi, dc->T1[i]), xi * dc->T1[i]);
        add128(shi, slo, 0, umulhi(xi, dc->T0[i]));
    }
    const u64 r = shi + (slo >> 63);
    M[(size_t)item * n + k] = r % dc->t;
    const int64_t d = (int64_t)slo;
    unsigned long long ad = d < 0 ? (unsigned long long)0 - (unsigned long long)d : (unsigned long long)d;
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, ad, off);
        ad = o > ad ? o : ad;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(maxdev + item, ad);
}

void launch_dec_scale(const DevConsts* dc, const RnsParams& P, const u64* const* CT,
                      const u64* X, u64* M, unsigned long long* maxdev, int items,
                      cudaStream_t st) {
    if (!items) return;
    cudaMemsetAsync(maxdev, 0, sizeof(unsigned long long) * items, st);
    k_dec_scale<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, CT, X, M, maxdev);
    CSSC_CHECK_LAUNCH();
}

// Decryption's t/Q scaling fused into the column phase of the forward NTT
// mod t (the decode): one CTA per (slice, column tile) reads the L residues of
// d = c0 + c1 s (coefficient form, D[slice][L][N]) at each of its tile's
// coefficients, computes m = round(t d / Q) mod t (E5, as k_dec_scale) and the
// largest rounding distance, then runs the column phase mod t and stores the
// tile like k_ntt_cols; k_ntt_blocks finishes the transform.
template <int LOGN, int LN>
__global__ void __launch_bounds__(Ntt2<LOGN>::TC) k_dec_cols(const DevConsts* __restrict__ dc, const u64* __restrict__ D,
                                                             u64* __restrict__ M, unsigned long long* maxdev) {
    using G = Ntt2<LOGN>;
    constexpr int T = G::TC;
    constexpr int CTAS = G::R2 / LN;
    constexpr int SEG = LN / 2;
    extern __shared__ u64 smem[];
    u64* tile = smem;
    u64* tws = smem + LN * G::R1;
    const int tileid = blockIdx.x % CTAS;
    const int item = blockIdx.x / CTAS;
    const int L = dc->L;
    const int tp = dc->np - 1;
    const u64 t = dc->t;
    const int col0 = tileid * LN;
    const u64* tw = dc->tw[tp].fwd;
    for (int i = threadIdx.x; i < G::R1; i += T) cp_async16(tws + 2 * i, tw + 2 * i);
    const u64* d = D + (size_t)item * L * G::N;
    unsigned long long ad_max = 0;
    for (int e = threadIdx.x; e < G::R1 * LN; e += T) {
        const int c = e / LN, jl = e % LN;
        const int k = c * G::R2 + col0 + jl;
        u64 shi = 0, slo = 0;
        for (int i = 0; i < L; ++i) {
            const u64 q = dc->mod[i].q;
            const u64 xi = shoup(__ldg(d + (size_t)i * G::N + k), dc->QhatInv[i], dc->QhatInv_sh[i], q);
            add128(shi, slo, umulhi(xi, dc->T1[i]), xi * dc->T1[i]);
            add128(shi, slo, 0, umulhi(xi, dc->T0[i]));
        }
        tile[c * LN + jl] = (shi + (slo >> 63)) % t;
        const int64_t dv = (int64_t)slo;
        const unsigned long long ad = dv < 0 ? (unsigned long long)0 - (unsigned long long)dv : (unsigned long long)dv;
        ad_max = ad > ad_max ? ad : ad_max;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, ad_max, off);
        ad_max = o > ad_max ? o : ad_max;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(maxdev + item, ad_max);
    cp_async_wait_all();
    __syncthreads();
    auto addr = [](int l, int pos) { return pos * LN + l; };
    auto twf = [&](int sl, int, int blk) {
        const int kk = (1 << sl) + blk;
        return make_ulonglong2(tws[2 * kk], tws[2 * kk + 1]);
    };
    line_ntt_v<G::A, 0, false, 3, LN>(tile, ConstQ{dc->mod[tp].q}, addr, twf, whole_cta());
    u64* dst = M + (size_t)item * G::N;
    for (int i = threadIdx.x; i < G::R1 * SEG; i += T) {
        const int c = i / SEG, h = i % SEG;
        *reinterpret_cast<ulonglong2*>(dst + (size_t)c * G::R2 + col0 + 2 * h) =
            make_ulonglong2(tile[c * LN + 2 * h], tile[c * LN + 2 * h + 1]);
    }
}

template <int LOGN>
static void dec_ntt_t(const DevConsts* dc, const RnsParams& P, u64* D, u64* M, u64* slots,
                      unsigned long long* maxdev, int items, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int L = P.cfg.L;
    NttJob jd;
    jd.src = D;
    jd.dst = D;
    jd.limbs = L;
    for (int i = 0; i < L; ++i) jd.pidx[i] = (signed char)i;
    launch_ntt_phase(dc, LOGN, true, true, jd, items, st);  // inverse column phase of d
    cudaMemsetAsync(maxdev, 0, sizeof(unsigned long long) * items, st);
    // 2-column tiles unless 8-column tiles already give one CTA per SM: the
    // per-coefficient scaling dominates, and a single result has only R2
    // columns
    smem_optin_k(k_dec_cols<LOGN, 8>, (8 * G::R1 + 2 * G::R1) * 8);
    smem_optin_k(k_dec_cols<LOGN, 2>, (2 * G::R1 + 2 * G::R1) * 8);
    if ((long)items * (G::R2 / 8) >= 148)
        k_dec_cols<LOGN, 8><<<items * (G::R2 / 8), G::TC, (8 * G::R1 + 2 * G::R1) * 8, st>>>(dc, D, M, maxdev);
    else
        k_dec_cols<LOGN, 2><<<items * (G::R2 / 2), G::TC, (2 * G::R1 + 2 * G::R1) * 8, st>>>(dc, D, M, maxdev);
    CSSC_CHECK_LAUNCH();
    NttJob jm;
    jm.src = M;
    jm.dst = M;
    jm.limbs = 1;
    jm.pidx[0] = (signed char)P.t_index();
    launch_ntt_phase(dc, LOGN, false, false, jm, items, st);  // forward block phase mod t
    if (slots) launch_decode_gather(dc, P, M, slots, items, st);
}

// D (d = c0 + c1 s after the inverse block phase) -> slots, see k_dec_cols
void launch_decrypt_ntt(const DevConsts* dc, const RnsParams& P, u64* D, u64* M, u64* slots,
                        unsigned long long* maxdev, int items, cudaStream_t st) {
    if (!items) return;
    switch (P.cfg.logn) {
        case 10: dec_ntt_t<10>(dc, P, D, M, slots, maxdev, items, st); break;
        case 11: dec_ntt_t<11>(dc, P, D, M, slots, maxdev, items, st); break;
        case 12: dec_ntt_t<12>(dc, P, D, M, slots, maxdev, items, st); break;
        case 13: dec_ntt_t<13>(dc, P, D, M, slots, maxdev, items, st); break;
        case 14: dec_ntt_t<14>(dc, P, D, M, slots, maxdev, items, st); break;
        case 15: dec_ntt_t<15>(dc, P, D, M, slots, maxdev, items, st); break;
        default: throw std::invalid_argument("decrypt: unsupported logn");
    }
}

__global__ void k_decode_gather(const DevConsts* __restrict__ dc, const u64* M, u64* slots) {
    const int S = dc->n / 2;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    if (j >= S) return;
    slots[(size_t)item * S + j] = M[(size_t)item * dc->n + dc->pos0[j]];
}

// pipeline download: result r's first rows[r] slots as u32 at out + off[r]
__global__ void k_decode_rows(const DevConsts* __restrict__ dc, const u64* M, u32* out, const int* rows,
                              const int* off) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    if (j >= rows[item]) return;
    out[off[item] + j] = (u32)M[(size_t)item * dc->n + dc->pos0[j]];
}

void launch_decode_rows(const DevConsts* dc, const RnsParams& P, const u64* M, u32* out, const int* rows,
                        const int* off, int max_rows, int items, cudaStream_t st) {
    if (!items || max_rows <= 0) return;
    k_decode_rows<<<dim3((unsigned)((max_rows + EW_THREADS - 1) / EW_THREADS), (unsigned)items), EW_THREADS, 0,
                    st>>>(dc, M, out, rows, off);
    CSSC_CHECK_LAUNCH();
}

void launch_decode_gather(const DevConsts* dc, const RnsParams& P, const u64* M, u64* slots,
                          int items, cudaStream_t st) {
    if (!items) return;
    k_decode_gather<<<dim3((unsigned)(P.S / EW_THREADS + 1), (unsigned)items), EW_THREADS, 0, st>>>(
        dc, M, slots);
    CSSC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// key generation helpers
// ---------------------------------------------------------------------------
__global__ void k_sample_small(int n, SeedKey seed, u32 n0, u64 id, int kind, int64_t* out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n / 8) return;
    u32 blk[16];
    chacha20_block(seed, (u32)b, n0, (u32)id, (u32)(id >> 32), blk);
    for (int w = 0; w < 8; ++w) {
        const u64 x = word64(blk, w);
        out[8 * b + w] = kind == 0 ? ternary_of(x) : cbd_of(x);
    }
}

void launch_sample_small(int logn, SeedKey seed, u32 dom, u64 id, int kind, int64_t* out,
                         cudaStream_t st) {
    const int n = 1 << logn;
    k_sample_small<<<(n / 8 + 63) / 64, 64, 0, st>>>(n, seed, dom, id, kind, out);
    CSSC_CHECK_LAUNCH();
}

// uniform residues for limbs [limb0, limb0+limbs): coefficient k uses words 2k, 2k+1
__global__ void k_sample_uniform(const DevConsts* __restrict__ dc, SeedKey seed, u32 dom, int digit,
                                 u64 id, int limb0, u64* out) {
    const int n = dc->n;
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = limb0 + blockIdx.y;
    if (b >= n / 4) return;
    const Modulus md = dc->mod[l];
    u32 blk[16];
    chacha20_block(seed, (u32)b, dom | ((u32)l << 8) | ((u32)digit << 16), (u32)id,
                   (u32)(id >> 32), blk);
    for (int w = 0; w < 4; ++w) {
        const u64 hi = word64(blk, 2 * w), lo = word64(blk, 2 * w + 1);
        const u64 h = reduce128(0, hi, md.q, md.mu1, md.mu0);
        out[(size_t)blockIdx.y * n + 4 * b + w] = reduce128(h, lo, md.q, md.mu1, md.mu0);
    }
}

void launch_sample_uniform(const DevConsts* dc, int logn, SeedKey seed, u32 dom, int digit, u64 id,
                           int limbs, int limb0, u64* out, cudaStream_t st) {
    const int n = 1 << logn;
    k_sample_uniform<<<dim3((unsigned)((n / 4 + 63) / 64), (unsigned)limbs), 64, 0, st>>>(
        dc, seed, dom, digit, id, limb0, out);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_lift_small(const DevConsts* __restrict__ dc, const int64_t* s, int limb0,
                             u64* out) {
    const int n = dc->n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int l = blockIdx.y;
    out[(size_t)l * n + k] = lift_signed(s[k], dc->mod[limb0 + l].q);
}

void launch_lift_small(const DevConsts* dc, int logn, const int64_t* s, int limbs, int limb0,
                       u64* out, cudaStream_t st) {
    k_lift_small<<<ew_grid(1 << logn, limbs), EW_THREADS, 0, st>>>(dc, s, limb0, out);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_automorph_small(int n, u32 ginv, const int64_t* in, int64_t* out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    bool neg;
    const int idx = automorph_src(ginv, k, n, neg);
    out[k] = neg ? -in[idx] : in[idx];
}

void launch_automorph_small(int logn, u32 g, const int64_t* in, int64_t* out, cudaStream_t st) {
    const int n = 1 << logn;
    // inverse of g in (Z/2N)^*: g^(N-1)
    const u64 two_n = 2 * (u64)n;
    u64 ginv = 1, b = g;
    for (u64 e = (u64)n - 1; e; e >>= 1) {
        if (e & 1) ginv = ginv * b % two_n;
        b = b * b % two_n;
    }
    k_automorph_small<<<(n + 127) / 128, 128, 0, st>>>(n, (u32)ginv, in, out);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_key_combine(const DevConsts* __restrict__ dc, const u64* A, const u64* E,
                              const u64* S, const u64* SP, int dlo, int dhi, u64* out) {
    const int n = dc->n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const Modulus md = dc->mod[j];
    const size_t o = (size_t)j * n + k;
    u64 v = add_mod(mul_mod(A[o], S[o], md), E[o], md.q);
    v = neg_mod(v, md.q);
    if (SP && j >= dlo && j < dhi)
        v = add_mod(v, mul_mod(dc->P_q[j], SP[o], md), md.q);
    out[o] = v;
}

// floor(w 2^64 / q) by restoring division (key generation only)
__global__ void k_shoup_companions(const DevConsts* __restrict__ dc, const u64* W, u64* WS, int LK, int n,
                                   size_t count) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const u64 q = dc->mod[(int)((i / n) % LK)].q;
    u64 r = W[i], quo = 0;  // r < q < 2^62: r << 1 never overflows
    for (int b = 0; b < 64; ++b) {
        r <<= 1;
        quo <<= 1;
        if (r >= q) {
            r -= q;
            quo |= 1;
        }
    }
    WS[i] = quo;
}

void launch_shoup_companions(const DevConsts* dc, const u64* W, u64* WS, int LK, int n, int polys,
                             cudaStream_t st) {
    const size_t count = (size_t)polys * LK * n;
    k_shoup_companions<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(dc, W, WS, LK, n, count);
    CSSC_CHECK_LAUNCH();
}

void launch_key_combine(const DevConsts* dc, int logn, int limbs, const u64* A, const u64* E,
                        const u64* S, const u64* SP, int digit_lo, int digit_hi, u64* out,
                        cudaStream_t st) {
    k_key_combine<<<ew_grid(1 << logn, limbs), EW_THREADS, 0, st>>>(dc, A, E, S, SP, digit_lo,
                                                                    digit_hi, out);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_square(const DevConsts* __restrict__ dc, const u64* S, u64* out) {
    const int n = dc->n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const size_t o = (size_t)j * n + k;
    out[o] = mul_mod(S[o], S[o], dc->mod[j]);
}

void launch_square(const DevConsts* dc, int logn, int limbs, const u64* S, u64* out,
                   cudaStream_t st) {
    k_square<<<ew_grid(1 << logn, limbs), EW_THREADS, 0, st>>>(dc, S, out);
    CSSC_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// generic ciphertext ops
// ---------------------------------------------------------------------------
__global__ void k_add(const DevConsts* __restrict__ dc, const u64* const* A, const u64* const* B,
                      u64* const* OUT) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    for (int p = 0; p < 2; ++p)
        for (int j = 0; j < L; ++j) {
            const size_t o = ((size_t)p * L + j) * n + k;
            OUT[item][o] = add_mod(A[item][o], B[item][o], dc->mod[j].q);
        }
}

void launch_add(const DevConsts* dc, const RnsParams& P, const u64* const* A,
                const u64* const* B, u64* const* OUT, int items, cudaStream_t st) {
    if (!items) return;
    k_add<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, A, B, OUT);
    CSSC_CHECK_LAUNCH();
}

// ACC[item] (2 (L+K) limbs) += XACC[item] (nullable entries): the key-switch
// accumulators of an odd step summed into its doubling step's before the one
// shared INTT + ModDown; lazy-safe (inputs < 2q, output < 2q)
__global__ void k_acc_add(const DevConsts* __restrict__ dc, u64* ACC, const u64* const* XACC, int LK) {
    const int n = dc->n;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    const u64* x = XACC[item];
    if (!x) return;
    u64* a = ACC + (size_t)item * 2 * LK * n;
    for (int j = 0; j < 2 * LK; ++j) {
        const u64 q2 = 2 * dc->mod[j % LK].q;
        const size_t o = (size_t)j * n + k;
        const u64 s = a[o] + x[o];
        a[o] = s >= q2 ? s - q2 : s;
    }
}

void launch_acc_add(const DevConsts* dc, const RnsParams& P, u64* ACC, const u64* const* XACC, int items,
                    cudaStream_t st) {
    if (!items || !XACC) return;
    k_acc_add<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, ACC, XACC, P.cfg.L + P.cfg.K);
    CSSC_CHECK_LAUNCH();
}

// OUT[item] = (phi_g(SRC[item].c0), untouched c1): the c0 term of a rotation
// whose key switch is folded into another's ModDown
__global__ void k_automorph_c0(const DevConsts* __restrict__ dc, const u64* const* SRC, const u32* ginv,
                               u64* const* OUT) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    bool neg;
    const int idx = automorph_src(ginv[item], k, n, neg);
    for (int j = 0; j < L; ++j) {
        const u64 v = SRC[item][(size_t)j * n + idx];
        OUT[item][(size_t)j * n + k] = neg ? neg_mod(v, dc->mod[j].q) : v;
    }
}

void launch_automorph_c0(const DevConsts* dc, const RnsParams& P, const u64* const* SRC, const u32* ginv,
                         u64* const* OUT, int items, cudaStream_t st) {
    if (!items) return;
    k_automorph_c0<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, SRC, ginv, OUT);
    CSSC_CHECK_LAUNCH();
}

// OUT[item].c0 (=|+=) sum_t phi_t(SRC[item][t].c0), t < 3 (GI[item][t] = 0: no
// term): the c0 terms of the rotations a stage folds into one ModDown beyond
// the one its ModDown gathers itself (DESIGN 2.9)
__global__ void k_automorph_sum(const DevConsts* __restrict__ dc, u64* const* OUT, const u64* const* SRC,
                                const u32* GI, int accumulate) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int item = blockIdx.y;
    u64* out = OUT[item];
    int idx[3];
    bool neg[3];
#pragma unroll
    for (int t = 0; t < 3; ++t) idx[t] = GI[item * 3 + t] ? automorph_src(GI[item * 3 + t], k, n, neg[t]) : -1;
    for (int j = 0; j < L; ++j) {
        const u64 q = dc->mod[j].q;
        u64 v = accumulate ? out[(size_t)j * n + k] : 0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (idx[t] < 0) continue;
            const u64 x = SRC[item * 3 + t][(size_t)j * n + idx[t]];
            v = add_mod(v, neg[t] ? neg_mod(x, q) : x, q);
        }
        out[(size_t)j * n + k] = v;
    }
}

void launch_automorph_sum(const DevConsts* dc, const RnsParams& P, u64* const* OUT, const u64* const* SRC,
                          const u32* GI, bool accumulate, int items, cudaStream_t st) {
    if (!items) return;
    k_automorph_sum<<<ew_grid(P.n, items), EW_THREADS, 0, st>>>(dc, OUT, SRC, GI, accumulate ? 1 : 0);
    CSSC_CHECK_LAUNCH();
}

__global__ void k_fold_mod(const DevConsts* __restrict__ dc, u64* W) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y % L;  // limb of row blockIdx.y = (result, poly, limb)
    u64* w = W + (size_t)blockIdx.y * n + k;
    *w = reduce64(*w, dc->mod[j]);
}

void launch_fold_mod(const DevConsts* dc, const RnsParams& P, u64* W, int results, cudaStream_t st) {
    if (!results) return;
    k_fold_mod<<<dim3((unsigned)(P.n / EW_THREADS), (unsigned)(results * 2 * P.cfg.L)), EW_THREADS, 0, st>>>(dc, W);
    CSSC_CHECK_LAUNCH();
}

// OUT = sum of `count` ciphertexts (the diagonal method's accumulation):
// one thread per (coefficient, limb); lazy sums of < 31 canonical terms,
// reduced by the 32-bit quotient estimate
__global__ void k_sum_items(const DevConsts* __restrict__ dc, const u64* const* A, int count, u64* OUT) {
    const int n = dc->n, L = dc->L;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;  // limb of [c0 | c1]
    const Modulus md = dc->mod[x % L];
    const size_t o = (size_t)x * n + k;
    u64 acc = 0;
    int lazy = 0;
    for (int i = 0; i < count; ++i) {
        acc += A[i][o];
        if (++lazy == 30) {
            acc = reduce_small_quot(acc, md);
            lazy = 1;
        }
    }
    OUT[o] = reduce_small_quot(acc, md);
}

void launch_sum_items(const DevConsts* dc, const RnsParams& P, const u64* const* A, int count, u64* OUT,
                      cudaStream_t st) {
    k_sum_items<<<dim3((unsigned)(P.n / EW_THREADS), (unsigned)(2 * P.cfg.L)), EW_THREADS, 0, st>>>(dc, A, count,
                                                                                                 OUT);
    CSSC_CHECK_LAUNCH();
}


}  // namespace cssc

namespace cssc {

// ---------------------------------------------------------------------------
// roofline probe: the radix-16 forward butterfly network of line_pass
// (correction-free lazy Shoup, as the forward NTT runs it), fed from
// registers only (no memory traffic), to measure the integer peak the NTT can
// approach.  Each iteration = 4 stages x 8 butterflies.  Values wrap; only the
// instruction stream matters.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bfly_peak(u64 q, u64 w0, u64 w0sh, int iters, u64* sink) {
    u64 v[16];
    u64 w = w0, wsh = w0sh;
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = (threadIdx.x * 16 + c + blockIdx.x) % q;
    const u64 two_q = 2 * q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int h = 1 << (3 - u);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                if (c & h) continue;
                const u64 x = v[c];
                const u64 y = shoup_lazy_q(v[c + h], w, wsh, q);
                v[c] = x + y;
                v[c + h] = x - y + two_q;
            }
        }
        w += 1;  // keep the twiddle live per iteration (as per-stage table loads would)
    }
    u64 s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s ^= v[c];
    if (s == 0x1234567) sink[0] = s;
}

double probe_butterfly_peak(const DevConsts* dc_host_copy_q, u64 q, u64 w, u64 wsh, cudaStream_t st) {
    (void)dc_host_copy_q;
    auto ok = [](cudaError_t e, const char* what) {
        if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
    };
    u64* sink = nullptr;
    ok(cudaMalloc(&sink, 8), "cudaMalloc");
    int dev = 0, sms = 148;
    ok(cudaGetDevice(&dev), "device");
    ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    const int blocks = sms * 8, threads = 256, iters = 2048;
    cudaEvent_t a = nullptr, b = nullptr;
    ok(cudaEventCreate(&a), "event");
    ok(cudaEventCreate(&b), "event");
    k_bfly_peak<<<blocks, threads, 0, st>>>(q, w, wsh, 64, sink);  // warm
    CSSC_CHECK_LAUNCH();
    ok(cudaEventRecord(a, st), "record");
    k_bfly_peak<<<blocks, threads, 0, st>>>(q, w, wsh, iters, sink);
    ok(cudaEventRecord(b, st), "record");
    ok(cudaEventSynchronize(b), "probe");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    CSSC_CHECK_LAUNCH();
    const double bfly = (double)blocks * threads * iters * 32.0;
    return bfly / (ms * 1e-3);
}

}  // namespace cssc
