// mul_fused.cu -- the ct x ct multiply and the masked accumulation fused
// around the NTT block phase.
//
//   k_mul_blocks_tensor : for one limb j of Q u B and one tile of 16 blocks of
//                         one item: the NTT block phase of the four extended
//                         inputs (a0 a1 b0 b1), the tensor product
//                           z0 = a0 b0,  z1 = a0 b1 + a1 b0,  z2 = a1 b1,
//                         and the INTT block phase of z0 .. z2.
// It replaces the forward block phase, k_mul_tensor and the inverse block
// phase (three launches and two round trips of seven polynomials through
// HBM).  The column phases before and after stay standard NTT launches.  The
// arithmetic is the same as the separate kernels (modular products of the same
// residues), so the words are identical.
#include <stdexcept>
#include <string>

#include "bfv_kernels.cuh"
#include "ntt.cuh"

namespace cssc {

template <int LOGN>
constexpr int mulb_threads() { return LOGN >= 15 ? 256 : 128; }

// k_mul_blocks_tensor runs its four forward and three inverse tile transforms
// on two 128-thread groups with named barriers (tiles g, g+2): a serial chain
// of 2 + 2 transforms instead of 7, at the occupancy of a 256-thread CTA
// (four groups measured no faster: the register file then halves the CTAs).
constexpr int kMulGroups = 2, kGroupThreads = 128;

template <int LOGN, int LT, int KT, int LN = 16>
__global__ void __launch_bounds__(kMulGroups * kGroupThreads) k_mul_blocks_tensor(const DevConsts* __restrict__ dc,
                                                                                  const u64* __restrict__ T,
                                                                                  u64* __restrict__ Z, int M) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = LN * PITCH;  // LN blocks per tile (8 at 2^15: half the smem, more CTAs per SM)
    constexpr int NT = kMulGroups * kGroupThreads;
    constexpr int PER = LN * G::R2 / NT;
    constexpr int CTAS = G::R1 / LN;
    constexpr int MAXR = LN >= 16 ? 4 : 3;  // radix-8 passes keep all threads of a group busy on 8 lines
    static_assert(PER >= 1, "tile smaller than the CTA");
    u64* tile = smem;            // 4 tiles: a0 a1 b0 b1, then z0 z1 z2 in the first three
    u64* tws = smem + 4 * TW;
    const int L = LT ? LT : dc->L, K = KT ? KT : dc->K;  // M: 2L over Q u R, 2L + 1 over Q u B
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j = bid % M;
    const int item = bid / M;
    const int prime = j < L ? j : K + j;  // B primes follow P in the prime table
    const Modulus md = dc->mod[prime];
    const u64 q = md.q;
    const int blk0 = tileid * LN;
    const size_t base = (size_t)blk0 * G::R2;
    const size_t PM = (size_t)M * G::N;
    const int grp = threadIdx.x / kGroupThreads;
    const ThreadGroup tg = cta_slice(grp, kMulGroups);
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl, int l, int blk) { return block_tw<LOGN, LN>(tws, sl, l, blk); };
    const u64* src = T + (size_t)item * 4 * PM + (size_t)j * G::N + base;
    load_block_twiddles<LOGN, LN>(tws, dc->tw[prime].fwd, blk0);
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int x = threadIdx.x + NT * r;
            cp_async8(tile + p * TW + saddr(x), src + p * PM + x);
        }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 1
    for (int p = grp; p < 4; p += kMulGroups)
        line_ntt_v<G::B, 0, false, MAXR, LN>(tile + p * TW, SpecQ{q}, addr, twf, tg);
    __syncthreads();
    // tensor: all four inputs canonicalised (cheap 32-bit quotient estimate),
    // so z1 = a0 b1 + a1 b0 < 2 q^2 < 2^117 is one 128-bit sum under a single
    // Barrett reduction (range < 2^(k+63)) instead of two reductions and an add
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int s0 = saddr(threadIdx.x + NT * r);
        const u64 a0 = reduce_small_quot_q(tile[s0], md), a1 = reduce_small_quot_q(tile[TW + s0], md);
        const u64 b0 = reduce_small_quot_q(tile[2 * TW + s0], md), b1 = reduce_small_quot_q(tile[3 * TW + s0], md);
        // products as 29-bit Karatsuba column sums (three IMAD.WIDE.U32 each),
        // one Barrett reduction per output: the canonical words of mul_mod
        Dot29 d0, d1, d2;
        dot29_mac_var(d0, a0, b0);
        dot29_mac_var(d1, a0, b1);
        dot29_mac_var(d1, a1, b0);
        dot29_mac_var(d2, a1, b1);
        tile[s0] = dot29_reduce_q(d0, md);
        tile[TW + s0] = dot29_reduce_q(d1, md);
        tile[2 * TW + s0] = dot29_reduce_q(d2, md);
    }
    __syncthreads();
    load_block_twiddles<LOGN, LN>(tws, dc->tw[prime].inv, blk0);
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 1
    for (int p = grp; p < 3; p += kMulGroups)
        line_ntt_v<G::B, 0, true, MAXR, LN>(tile + p * TW, SpecQ{q}, addr, twf, tg);
    __syncthreads();
    u64* dst = Z + (size_t)item * 3 * PM + (size_t)j * G::N + base;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int x = threadIdx.x + NT * r;
            dst[p * PM + x] = tile[p * TW + saddr(x)];
        }
}

// Masked inter-chunk accumulation around the block phase: for one slice s,
// one limb j2 of [c0 | c1] (prime j2 mod L) and one tile of 16 blocks: for each
// chunk of the slice, the NTT block phase of its folded ciphertext (after the
// forward column phase, MT), times the chunk's mask tile (NTT form), summed
// (inter_chunk_sum, aggregate.cpp:55-74); then the INTT block phase of the sum,
// written to the slice's result ciphertext for the inverse column phase.
// Replaces the forward block phase, k_mask_accum and the inverse block phase.
template <int LOGN, int LN = 16>
__global__ void __launch_bounds__(2 * kGroupThreads) k_mask_blocks(const DevConsts* __restrict__ dc,
                                                                   const u64* __restrict__ MT,
                                                                   const int* __restrict__ slice_off,
                                                                   const int* __restrict__ slice_items,
                                                                   const int* __restrict__ item_mask,
                                                                   const u64* __restrict__ MASKS,
                                                                   u64* const* OUT) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = LN * PITCH;
    constexpr int NG = 2;  // groups: chunks x = b + g, b + g + 2, ... each into its own partial sum
    constexpr int NT = NG * kGroupThreads;
    constexpr int PERG = LN * G::R2 / kGroupThreads;  // elements per thread within a group
    constexpr int PER = LN * G::R2 / NT;
    constexpr int CTAS = G::R1 / LN;
    static_assert(PER >= 1, "tile smaller than the CTA");
    u64* work = smem;             // NG work tiles
    u64* acc = smem + NG * TW;    // NG partial sums
    u64* tws = smem + 2 * NG * TW;
    const int L = dc->L;
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j2 = bid % (2 * L);
    const int sl = bid / (2 * L);
    const int j = j2 % L;
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const int blk0 = tileid * LN;
    const size_t base = (size_t)blk0 * G::R2;
    const int grp = threadIdx.x / kGroupThreads;
    const ThreadGroup tg = cta_slice(grp, NG);
    u64* wk = work + grp * TW;
    u64* ac = acc + grp * TW;
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl_, int l, int blk) { return block_tw<LOGN, LN>(tws, sl_, l, blk); };
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].fwd, blk0);
    cp_async_wait_all();
    __syncthreads();
    const int b = slice_off[sl], e = slice_off[sl + 1];
    bool any = false;
#pragma unroll 1
    for (int x = b + grp; x < e; x += NG) {
        const int it = slice_items[x];
        const u64* src = MT + ((size_t)it * 2 * L + j2) * G::N + base;
#pragma unroll
        for (int r = 0; r < PERG; ++r) {
            const int y = tg.tid + kGroupThreads * r;
            cp_async8(wk + saddr(y), src + y);
        }
        cp_async_wait_all();
        tg.sync();
        line_ntt_v<G::B, 0, false, (LN >= 16 ? 4 : 2), LN>(wk, SpecQ{q}, addr, twf, tg);
        const u64* mk = MASKS + ((size_t)item_mask[it] * L + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PERG; ++r) {
            const int y = tg.tid + kGroupThreads * r, s0 = saddr(y);
            const u64 p = mul_mod_q(wk[s0], __ldg(mk + y), md);  // lazy (< 31q) x canonical mask
            ac[s0] = any ? add_mod(ac[s0], p, q) : p;
        }
        any = true;
        tg.sync();  // work tile reloaded next round
    }
    if (!any)
#pragma unroll
        for (int r = 0; r < PERG; ++r) ac[saddr(tg.tid + kGroupThreads * r)] = 0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int s0 = saddr(threadIdx.x + NT * r);
        acc[s0] = add_mod(acc[s0], acc[TW + s0], q);
    }
    __syncthreads();
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].inv, blk0);
    cp_async_wait_all();
    __syncthreads();
    line_ntt_v<G::B, 0, true, 2, LN>(acc, SpecQ{q}, addr, twf, whole_cta());  // radix-4: more threads busy
    u64* dst = OUT[sl] + (size_t)j2 * G::N + base;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int y = threadIdx.x + NT * r;
        dst[y] = acc[saddr(y)];
    }
}

// The pipeline's decrypting variant of k_mask_blocks: for one slice, one
// prime j < L and one tile, groups 0-1 sum the c0 limb and groups 2-3 the c1
// limb of the slice's chunks (block phase x mask; even / odd chunks), then d = c0 + c1 s (s in NTT form,
// the key holder's decryption product, done where c1 already is in the NTT
// domain) goes through the inverse block phase into D[slice][j].  The
// inverse column phase of D and the t/Q scaling follow (k_dec_cols).  The
// slice's result ciphertext is never materialised: the pipeline returns only
// its decryption, and d mod q_j is the same residue c0 + INTT(NTT(c1) s)
// gives, so the slots are unchanged.
template <int LOGN, int LN = 16>
__global__ void __launch_bounds__(4 * kGroupThreads) k_mask_dec_blocks(const DevConsts* __restrict__ dc,
                                                                       const u64* __restrict__ MT,
                                                                       const int* __restrict__ slice_off,
                                                                       const int* __restrict__ slice_items,
                                                                       const int* __restrict__ item_mask,
                                                                       const u64* __restrict__ MASKS,
                                                                       const u64* __restrict__ S_NTT,
                                                                       u64* __restrict__ D) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = LN * PITCH;
    constexpr int NG = 4;  // groups 0, 1: c0 (even / odd chunks), groups 2, 3: c1
    constexpr int NT = NG * kGroupThreads;
    constexpr int PERG = LN * G::R2 / kGroupThreads;
    constexpr int PER = LN * G::R2 / NT;
    constexpr int CTAS = G::R1 / LN;
    u64* work = smem;
    u64* acc = smem + NG * TW;
    u64* tws = smem + 2 * NG * TW;
    const int L = dc->L;
    int bid = blockIdx.x;
    const int tileid = bid % CTAS;
    bid /= CTAS;
    const int j = bid % L;
    const int sl = bid / L;
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const int blk0 = tileid * LN;
    const size_t base = (size_t)blk0 * G::R2;
    const int grp = threadIdx.x / kGroupThreads;
    const ThreadGroup tg = cta_slice(grp, NG);
    const int j2 = (grp >> 1) * L + j;
    u64* wk = work + grp * TW;
    u64* ac = acc + grp * TW;
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl_, int l, int blk) { return block_tw<LOGN, LN>(tws, sl_, l, blk); };
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].fwd, blk0);
    cp_async_wait_all();
    __syncthreads();
    const int b = slice_off[sl], e = slice_off[sl + 1];
    bool any = false;
#pragma unroll 1
    for (int x = b + (grp & 1); x < e; x += 2) {
        const int it = slice_items[x];
        const u64* src = MT + ((size_t)it * 2 * L + j2) * G::N + base;
#pragma unroll
        for (int r = 0; r < PERG; ++r) {
            const int y = tg.tid + kGroupThreads * r;
            cp_async8(wk + saddr(y), src + y);
        }
        cp_async_wait_all();
        tg.sync();
        line_ntt_v<G::B, 0, false, (LN >= 16 ? 4 : 2), LN>(wk, SpecQ{q}, addr, twf, tg);
        const u64* mk = MASKS + ((size_t)item_mask[it] * L + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PERG; ++r) {
            const int y = tg.tid + kGroupThreads * r, s0 = saddr(y);
            const u64 p = mul_mod_q(wk[s0], __ldg(mk + y), md);
            ac[s0] = any ? add_mod(ac[s0], p, q) : p;
        }
        any = true;
        tg.sync();
    }
    if (!any)
#pragma unroll
        for (int r = 0; r < PERG; ++r) ac[saddr(tg.tid + kGroupThreads * r)] = 0;
    __syncthreads();
    const u64* sk = S_NTT + (size_t)j * G::N + base;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int y = threadIdx.x + NT * r, s0 = saddr(y);
        const u64 c0 = add_mod(acc[s0], acc[TW + s0], q), c1 = add_mod(acc[2 * TW + s0], acc[3 * TW + s0], q);
        acc[s0] = add_mod(c0, mul_mod_q(c1, __ldg(sk + y), md), q);
    }
    __syncthreads();
    load_block_twiddles<LOGN, LN>(tws, dc->tw[j].inv, blk0);
    cp_async_wait_all();
    __syncthreads();
    line_ntt_v<G::B, 0, true, 2, LN>(acc, SpecQ{q}, addr, twf, whole_cta());  // radix-4: more threads busy
    u64* dst = D + ((size_t)sl * L + j) * G::N + base;
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int y = threadIdx.x + NT * r;
        dst[y] = acc[saddr(y)];
    }
}

template <int LOGN>
static void maskdec_t(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                      const int* slice_items, const int* item_mask, const u64* MASKS, const u64* S_NTT, u64* D,
                      int slices, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int smem = (8 * G::LINES * G::PITCH + 2 * G::TWB) * 8;
    const int smemh = (8 * 8 * G::PITCH + 2 * btw_entries<LOGN, 8>()) * 8;
    smem_optin_k(k_mask_dec_blocks<LOGN>, smem);
    smem_optin_k(k_mask_dec_blocks<LOGN, 8>, smemh);
    if (blocks_use_ln8((long)slices * P.cfg.L * G::CTAS_B) && 8 * G::R2 >= 4 * kGroupThreads)  // small: 8-block tiles
        k_mask_dec_blocks<LOGN, 8><<<slices * P.cfg.L * (G::R1 / 8), 4 * kGroupThreads, smemh, st>>>(
            dc, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D);
    else
        k_mask_dec_blocks<LOGN><<<slices * P.cfg.L * G::CTAS_B, 4 * kGroupThreads, smem, st>>>(
            dc, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("mask-decrypt launch: ") + cudaGetErrorString(e));
}

void launch_mask_dec_blocks(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                            const int* slice_items, const int* item_mask, const u64* MASKS, const u64* S_NTT,
                            u64* D, int slices, cudaStream_t st) {
    if (!slices) return;
    switch (P.cfg.logn) {
        case 10: maskdec_t<10>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        case 11: maskdec_t<11>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        case 12: maskdec_t<12>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        case 13: maskdec_t<13>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        case 14: maskdec_t<14>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        case 15: maskdec_t<15>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, S_NTT, D, slices, st); break;
        default: throw std::invalid_argument("mask-decrypt: unsupported logn");
    }
}

template <int LOGN>
static void maskb_t(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                    const int* slice_items, const int* item_mask, const u64* MASKS, u64* const* OUT, int slices,
                    cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int smem = (4 * G::LINES * G::PITCH + 2 * G::TWB) * 8;
    const int smemh = (4 * 8 * G::PITCH + 2 * btw_entries<LOGN, 8>()) * 8;
    smem_optin_k(k_mask_blocks<LOGN>, smem);
    smem_optin_k(k_mask_blocks<LOGN, 8>, smemh);
    if (blocks_use_ln8((long)slices * 2 * P.cfg.L * G::CTAS_B) && 8 * G::R2 >= 2 * kGroupThreads)  // small: 8-block tiles
        k_mask_blocks<LOGN, 8><<<slices * 2 * P.cfg.L * (G::R1 / 8), 2 * kGroupThreads, smemh, st>>>(
            dc, MT, slice_off, slice_items, item_mask, MASKS, OUT);
    else
        k_mask_blocks<LOGN><<<slices * 2 * P.cfg.L * G::CTAS_B, 2 * kGroupThreads, smem, st>>>(
            dc, MT, slice_off, slice_items, item_mask, MASKS, OUT);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("mask blocks launch: ") + cudaGetErrorString(e));
}

void launch_mask_blocks(const DevConsts* dc, const RnsParams& P, const u64* MT, const int* slice_off,
                        const int* slice_items, const int* item_mask, const u64* MASKS, u64* const* OUT,
                        int slices, cudaStream_t st) {
    if (!slices) return;
    switch (P.cfg.logn) {
        case 10: maskb_t<10>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        case 11: maskb_t<11>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        case 12: maskb_t<12>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        case 13: maskb_t<13>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        case 14: maskb_t<14>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        case 15: maskb_t<15>(dc, P, MT, slice_off, slice_items, item_mask, MASKS, OUT, slices, st); break;
        default: throw std::invalid_argument("mask: unsupported logn");
    }
}

// Client-side polynomial product around the block phase (encryption: u x pk,
// decryption: c1 x s): for one limb j < L and one tile of one item, the block
// phase of IN (after the forward column phase), times each of the NMUL
// NTT-form multipliers, and the inverse block phase of each product, written
// to OUT limb p*L + j.  CTAs with j == L (only when XTRA is set) run the
// inverse block phase of limb `xlimb` of XTRA in place with prime `xprime`:
// the encoded message riding in the encryption's inverse NTT.
template <int LOGN, int NMUL>
__global__ void __launch_bounds__(mulb_threads<LOGN>()) k_blocks_mul_inv(const DevConsts* __restrict__ dc,
                                                                         const u64* __restrict__ IN,
                                                                         const u64* __restrict__ MUL,
                                                                         u64* __restrict__ OUT, size_t out_stride,
                                                                         u64* __restrict__ XTRA, int xlimb,
                                                                         int xprime, const u64* __restrict__ MULSH) {
    using G = Ntt2<LOGN>;
    extern __shared__ u64 smem[];
    constexpr int PITCH = G::PITCH;
    constexpr int TW = G::LINES * PITCH;
    constexpr int NT = mulb_threads<LOGN>();
    constexpr int PER = G::LINES * G::R2 / NT;
    u64* tile = smem;  // input, then NMUL products
    u64* tws = smem + (NMUL + 1) * TW;
    const int L = dc->L, J = XTRA ? L + 1 : L;
    int bid = blockIdx.x;
    const int tileid = bid % G::CTAS_B;
    bid /= G::CTAS_B;
    const int j = bid % J;
    const int item = bid / J;
    const int blk0 = tileid * G::LINES;
    const size_t base = (size_t)blk0 * G::R2;
    auto saddr = [](int x) { return (x >> G::B) * PITCH + (x & (G::R2 - 1)); };
    auto addr = [](int l, int pos) { return l * PITCH + pos; };
    auto twf = [&](int sl, int l, int blk) { return block_tw<LOGN>(tws, sl, l, blk); };
    if (j == L) {  // the extra limb: inverse block phase only, in place
        const Modulus mx = dc->mod[xprime];
        u64* x = XTRA + (size_t)item * out_stride + (size_t)xlimb * G::N + base;
        load_block_twiddles<LOGN>(tws, dc->tw[xprime].inv, blk0);
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int y = threadIdx.x + NT * r;
            cp_async8(tile + saddr(y), x + y);
        }
        cp_async_wait_all();
        __syncthreads();
        line_ntt<G::B, 0, true>(tile, mx.q, addr, twf);
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int y = threadIdx.x + NT * r;
            x[y] = tile[saddr(y)];
        }
        return;
    }
    const Modulus md = dc->mod[j];
    const u64 q = md.q;
    const u64* in = IN + ((size_t)item * L + j) * G::N + base;
    load_block_twiddles<LOGN>(tws, dc->tw[j].fwd, blk0);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int y = threadIdx.x + NT * r;
        cp_async8(tile + saddr(y), in + y);
    }
    cp_async_wait_all();
    __syncthreads();
    line_ntt_q<G::B, 0, false>(tile, q, addr, twf);
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        const int y = threadIdx.x + NT * r, s0 = saddr(y);
        const u64 w = tile[s0];  // lazy (< 31q) x canonical multiplier
#pragma unroll
        for (int p = 0; p < NMUL; ++p) {
            const size_t o = ((size_t)p * L + j) * G::N + base + y;
            // fixed multipliers (pk, s) with stored Shoup companions: no Barrett reduction
            tile[(p + 1) * TW + s0] = MULSH ? shoup_q(w, __ldg(MUL + o), __ldg(MULSH + o), q) : mul_mod_q(w, __ldg(MUL + o), md);
        }
    }
    __syncthreads();
    load_block_twiddles<LOGN>(tws, dc->tw[j].inv, blk0);
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 1
    for (int p = 0; p < NMUL; ++p) line_ntt_q<G::B, 0, true>(tile + (p + 1) * TW, q, addr, twf);
#pragma unroll
    for (int p = 0; p < NMUL; ++p) {
        u64* dst = OUT + (size_t)item * out_stride + ((size_t)p * L + j) * G::N + base;
#pragma unroll
        for (int r = 0; r < PER; ++r) {
            const int y = threadIdx.x + NT * r;
            dst[y] = tile[(p + 1) * TW + saddr(y)];
        }
    }
}

template <int LOGN, int NMUL>
static void bmi_t(const DevConsts* dc, const RnsParams& P, const u64* IN, const u64* MUL, u64* OUT,
                  size_t out_stride, u64* XTRA, int xlimb, int xprime, int items, cudaStream_t st, const u64* MULSH) {
    using G = Ntt2<LOGN>;
    const int smem = ((NMUL + 1) * G::LINES * G::PITCH + 2 * G::TWB) * 8;
    smem_optin_k(k_blocks_mul_inv<LOGN, NMUL>, smem);
    const int J = P.cfg.L + (XTRA ? 1 : 0);
    k_blocks_mul_inv<LOGN, NMUL><<<items * J * G::CTAS_B, mulb_threads<LOGN>(), smem, st>>>(
        dc, IN, MUL, OUT, out_stride, XTRA, xlimb, xprime, MULSH);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("blocks-mul launch: ") + cudaGetErrorString(e));
}

template <int LOGN>
static void bmi_logn(const DevConsts* dc, const RnsParams& P, const u64* IN, const u64* MUL, int nmul, u64* OUT,
                     size_t out_stride, u64* XTRA, int xlimb, int xprime, int items, cudaStream_t st,
                     const u64* MULSH) {
    if (nmul == 1)
        bmi_t<LOGN, 1>(dc, P, IN, MUL, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH);
    else if (nmul == 2)
        bmi_t<LOGN, 2>(dc, P, IN, MUL, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH);
    else
        throw std::invalid_argument("blocks-mul: 1 or 2 multipliers");
}

void launch_blocks_mul_inv(const DevConsts* dc, const RnsParams& P, const u64* IN, const u64* MUL, int nmul,
                           u64* OUT, size_t out_stride, u64* XTRA, int xlimb, int xprime, int items,
                           cudaStream_t st, const u64* MULSH) {
    if (!items) return;
    switch (P.cfg.logn) {
        case 10: bmi_logn<10>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        case 11: bmi_logn<11>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        case 12: bmi_logn<12>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        case 13: bmi_logn<13>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        case 14: bmi_logn<14>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        case 15: bmi_logn<15>(dc, P, IN, MUL, nmul, OUT, out_stride, XTRA, xlimb, xprime, items, st, MULSH); break;
        default: throw std::invalid_argument("blocks-mul: unsupported logn");
    }
}

template <int LOGN, int LT, int KT>
static void mulb_t(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items, cudaStream_t st) {
    using G = Ntt2<LOGN>;
    const int M = P.mul_limbs();
    // 2^15 (B = 7): 16-block tiles need 100 KB of smem (2 CTAs per SM); 8-block
    // tiles halve it (CSSC_MULB_LN=16 keeps 16)
    static const int ln_env = [] {
        const char* e = std::getenv("CSSC_MULB_LN");
        return e ? std::atoi(e) : 0;
    }();
    if (LOGN >= 15 && ln_env != 16) {
        constexpr int LN = 8;
        const int smem = (4 * LN * G::PITCH + 2 * btw_entries<LOGN, LN>()) * 8;
        smem_optin_k(k_mul_blocks_tensor<LOGN, LT, KT, LN>, smem);
        k_mul_blocks_tensor<LOGN, LT, KT, LN><<<items * M * (G::R1 / LN), kMulGroups * kGroupThreads, smem, st>>>(
            dc, T, Z, M);
    } else {
        const int smem = (4 * G::LINES * G::PITCH + 2 * G::TWB) * 8;
        smem_optin_k(k_mul_blocks_tensor<LOGN, LT, KT>, smem);
        k_mul_blocks_tensor<LOGN, LT, KT><<<items * M * G::CTAS_B, kMulGroups * kGroupThreads, smem, st>>>(dc, T, Z,
                                                                                                          M);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("mul blocks launch: ") + cudaGetErrorString(e));
}

template <int LOGN>
static void mulb_logn(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items, cudaStream_t st) {
    const auto& c = P.cfg;
    if (c.L == 2 && c.K == 2)
        mulb_t<LOGN, 2, 2>(dc, P, T, Z, items, st);
    else if (c.L == 4 && c.K == 4)
        mulb_t<LOGN, 4, 4>(dc, P, T, Z, items, st);
    else
        mulb_t<LOGN, 0, 0>(dc, P, T, Z, items, st);
}

void launch_mul_blocks_tensor(const DevConsts* dc, const RnsParams& P, const u64* T, u64* Z, int items,
                              cudaStream_t st) {
    if (!items) return;
    switch (P.cfg.logn) {
        case 10: mulb_logn<10>(dc, P, T, Z, items, st); break;
        case 11: mulb_logn<11>(dc, P, T, Z, items, st); break;
        case 12: mulb_logn<12>(dc, P, T, Z, items, st); break;
        case 13: mulb_logn<13>(dc, P, T, Z, items, st); break;
        case 14: mulb_logn<14>(dc, P, T, Z, items, st); break;
        case 15: mulb_logn<15>(dc, P, T, Z, items, st); break;
        default: throw std::invalid_argument("multiply: unsupported logn");
    }
}

}  // namespace cssc
