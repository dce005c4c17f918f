// bfly_bench.cu -- register-resident butterfly throughput of the Shoup
// variants considered for the NTT (radix-16 network, as k_bfly_peak).
//   fwd_exact : current forward butterfly (full 64-bit high product, y < 2q)
//   fwd_approx: quotient from three 32-bit partial products (y < 4q) plus one
//               conditional subtraction of 4q on x (values stay < 8q)
//   inv_exact : current inverse butterfly (sum csub 2q, lazy Shoup of x - y + 2q)
//   inv_approx: the same with the approximate quotient (values stay < 4q)
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bfly tools/bfly_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

using u64 = unsigned long long;
using u32 = unsigned int;

__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) { return a * w - __umul64hi(a, wsh) * q; }
// floor(a wsh / 2^64) - e, e in {0, 1, 2}: the low x low product is dropped and
// the two cross products contribute only their high halves
__device__ __forceinline__ u64 shoup_lazy4(u64 a, u64 w, u64 wsh, u64 q) {
    const u32 ah = (u32)(a >> 32), al = (u32)a, sh = (u32)(wsh >> 32), sl = (u32)wsh;
    const u64 mid = (u64)__umulhi(ah, sl) + __umulhi(al, sh);
    const u64 qh = (u64)ah * sh + mid;
    return a * w - qh * q;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_bfly(u64 q, u64 w0, u64 w0sh, int iters, u64* sink) {
    u64 v[16];
    u64 w = w0, wsh = w0sh;
#pragma unroll
    for (int c = 0; c < 16; ++c) v[c] = (threadIdx.x * 16 + c + blockIdx.x) % q;
    const u64 two_q = 2 * q, four_q = 4 * q;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int h = 1 << (3 - u);
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                if (c & h) continue;
                if (MODE == 0) {
                    const u64 x = v[c];
                    const u64 y = shoup_lazy(v[c + h], w, wsh, q);
                    v[c] = x + y;
                    v[c + h] = x - y + two_q;
                } else if (MODE == 1) {
                    u64 x = v[c];
                    x = x >= four_q ? x - four_q : x;
                    const u64 y = shoup_lazy4(v[c + h], w, wsh, q);
                    v[c] = x + y;
                    v[c + h] = x - y + four_q;
                } else if (MODE == 2) {
                    const u64 x = v[c], y = v[c + h];
                    u64 s = x + y;
                    v[c] = s >= two_q ? s - two_q : s;
                    v[c + h] = shoup_lazy(x - y + two_q, w, wsh, q);
                } else {
                    const u64 x = v[c], y = v[c + h];
                    u64 s = x + y;
                    v[c] = s >= four_q ? s - four_q : s;
                    v[c + h] = shoup_lazy4(x - y + four_q, w, wsh, q);
                }
            }
        }
        w += 1;
    }
    u64 s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s ^= v[c];
    if (s == 0x1234567) sink[0] = s;
}

template <int MODE>
double run(u64 q, u64 w, u64 wsh, u64* sink) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 2048;
    k_bfly<MODE><<<blocks, threads>>>(q, w, wsh, 64, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(a);
        k_bfly<MODE><<<blocks, threads>>>(q, w, wsh, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double bfly = (double)blocks * threads * iters * 32;
    return bfly / (best * 1e-3) / 1e9;
}

// exhaustive-ish host check of the approximate quotient's range on random inputs
static u64 rng = 88172645463325252ull;
static u64 next() {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    return rng;
}

int main() {
    const u64 q = 288230376151711717ull;  // < 2^58 (not necessarily prime: only the range matters)
    const u64 w = 123456789012345678ull % q;
    const u64 wsh = (u64)(((unsigned __int128)w << 64) / q);
    int bad = 0;
    for (int i = 0; i < 1000000; ++i) {
        const u64 a = next(), ww = next() % q;
        const u64 s = (u64)(((unsigned __int128)ww << 64) / q);
        const u32 ah = (u32)(a >> 32), al = (u32)a, sh = (u32)(s >> 32), sl = (u32)s;
        const u64 mid = (u64)(((u64)ah * sl) >> 32) + (((u64)al * sh) >> 32);
        const u64 qh = (u64)ah * sh + mid;
        const u64 r = a * ww - qh * q;
        const unsigned __int128 exact = (unsigned __int128)a * ww % q;
        if (r >= 4 * q || r % q != (u64)exact) ++bad;
    }
    printf("host check: %d bad of 1e6\n", bad);
    u64* sink;
    cudaMalloc(&sink, 8);
    printf("fwd_exact  %.1f Gbfly/s\n", run<0>(q, w, wsh, sink));
    printf("fwd_approx %.1f Gbfly/s\n", run<1>(q, w, wsh, sink));
    printf("inv_exact  %.1f Gbfly/s\n", run<2>(q, w, wsh, sink));
    printf("inv_approx %.1f Gbfly/s\n", run<3>(q, w, wsh, sink));
    return 0;
}
