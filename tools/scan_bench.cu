// Microbenchmark (not product): streaming the 16 B/slot SoA at N = 16M on one B200.
//   copy-read : plain vectorized read + xor reduce (the achievable read bandwidth)
//   tile-loop : the admission scan's tile loop structure (512 thr, 4 slots/thread, depth D,
//               per-tile __syncthreads_or) with thresholds that accept nothing
//   tma-loop  : same classification, SoA tiles staged by cp.async.bulk + mbarrier ring
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scan_bench scan_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copy_read(const ulonglong2* lt, const uint4* ag, const uint4* rf, long long n4, unsigned long long* out) {
    unsigned long long acc = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        ulonglong2 a = __ldcs(lt + 2 * i), b = __ldcs(lt + 2 * i + 1);
        uint4 c = __ldcs(ag + i), d = __ldcs(rf + i);
        acc ^= a.x ^ a.y ^ b.x ^ b.y ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
    if (acc == 0x1234567) out[0] = acc;
}

template <int D>
__global__ void __launch_bounds__(512, 1) tile_loop(const unsigned long long* lt, const unsigned int* ag, const unsigned int* rf,
                                                    long long cap, unsigned long long thr, unsigned long long* out) {
    const int T = blockDim.x, tid = threadIdx.x;
    const long long TV = T * 4;
    long long per = (cap + gridDim.x - 1) / gridDim.x;
    per = (per + 3) / 4 * 4;
    const long long lo = blockIdx.x * per, hi = min(cap, lo + per);
    __shared__ int cnt;
    if (tid == 0) cnt = 0;
    __syncthreads();
    struct Q { ulonglong2 a, b; uint4 c, d; } q[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
        long long i = lo + d * TV + tid * 4;
        if (i + 4 <= hi) { q[d].a = __ldcs((const ulonglong2*)(lt + i)); q[d].b = __ldcs((const ulonglong2*)(lt + i + 2)); q[d].c = __ldcs((const uint4*)(ag + i)); q[d].d = __ldcs((const uint4*)(rf + i)); }
    }
    for (long long base = lo; base < hi; base += D * TV) {
#pragma unroll
        for (int d = 0; d < D; ++d) {
            long long tb = base + d * TV;
            if (tb >= hi) break;
            int acc = 0;
            unsigned long long x[4] = {q[d].a.x, q[d].a.y, q[d].b.x, q[d].b.y};
            unsigned int r[4] = {q[d].d.x, q[d].d.y, q[d].d.z, q[d].d.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += (x[k] <= thr) + (r[k] == 0 && x[k] <= thr);
            if (acc) atomicAdd(&cnt, acc);
            long long i = tb + D * TV + tid * 4;
            if (i + 4 <= hi) { q[d].a = __ldcs((const ulonglong2*)(lt + i)); q[d].b = __ldcs((const ulonglong2*)(lt + i + 2)); q[d].c = __ldcs((const uint4*)(ag + i)); q[d].d = __ldcs((const uint4*)(rf + i)); }
            __syncthreads_or(acc);
        }
    }
    if (tid == 0 && cnt) out[0] = cnt;
}

__device__ __forceinline__ void mbar_init(unsigned long long* m, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(m)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned phase) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n"
                 :: "r"((unsigned)__cvta_generic_to_shared(m)), "r"(phase) : "memory");
}

template <int S>
__global__ void __launch_bounds__(512, 1) tma_loop(const unsigned long long* lt, const unsigned int* ag, const unsigned int* rf,
                                                   long long cap, unsigned long long thr, unsigned long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int T = blockDim.x, tid = threadIdx.x;
    const int TV = T * 4;
    long long per = (cap + gridDim.x - 1) / gridDim.x;
    per = (per + 3) / 4 * 4;
    const long long lo = blockIdx.x * per, hi = min(cap, lo + per);
    unsigned long long* s_lt = (unsigned long long*)sm;
    unsigned int* s_ag = (unsigned int*)(sm + (size_t)S * TV * 8);
    unsigned int* s_rf = (unsigned int*)(sm + (size_t)S * TV * 12);
    __shared__ __align__(8) unsigned long long mb[S];
    __shared__ int cnt;
    const int ntiles = (int)((hi - lo + TV - 1) / TV);
    if (tid == 0) {
        cnt = 0;
        for (int s = 0; s < S; ++s) mbar_init(&mb[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](int t) {
        const int s = t % S;
        const long long b = lo + (long long)t * TV;
        const unsigned nsl = (unsigned)min((long long)TV, hi - b);
        mbar_expect_tx(&mb[s], nsl * 16);
        bulk_g2s(s_lt + (size_t)s * TV, lt + b, nsl * 8, &mb[s]);
        bulk_g2s(s_ag + (size_t)s * TV, ag + b, nsl * 4, &mb[s]);
        bulk_g2s(s_rf + (size_t)s * TV, rf + b, nsl * 4, &mb[s]);
    };
    if (tid == 0) for (int t = 0; t < S && t < ntiles; ++t) issue(t);
    for (int t = 0; t < ntiles; ++t) {
        const int s = t % S;
        mbar_wait(&mb[s], (t / S) & 1);
        const long long b = lo + (long long)t * TV;
        int acc = 0;
        if (b + tid * 4 < hi) {
            ulonglong2 a = *(const ulonglong2*)(s_lt + (size_t)s * TV + tid * 4);
            ulonglong2 c = *(const ulonglong2*)(s_lt + (size_t)s * TV + tid * 4 + 2);
            uint4 r = *(const uint4*)(s_rf + (size_t)s * TV + tid * 4);
            unsigned long long x[4] = {a.x, a.y, c.x, c.y};
            unsigned int rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += (x[k] <= thr) + (rr[k] == 0 && x[k] <= thr);
        }
        if (acc) atomicAdd(&cnt, acc);
        __syncthreads_or(acc);
        if (tid == 0 && t + S < ntiles) issue(t + S);
    }
    if (tid == 0 && cnt) out[0] = cnt;
}

int main() {
    const long long N = 64ll << 20;  // 1 GiB of SoA: far beyond the 126 MB L2
    unsigned long long* lt; unsigned int *ag, *rf; unsigned long long* out;
    CK(cudaMalloc(&lt, N * 8)); CK(cudaMalloc(&ag, N * 4)); CK(cudaMalloc(&rf, N * 4)); CK(cudaMalloc(&out, 8));
    {   // random contents (no compressible / constant pages)
        unsigned long long* h = (unsigned long long*)malloc(N * 8);
        unsigned long long x = 88172645463325252ull;
        for (long long i = 0; i < N; ++i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = x; }
        CK(cudaMemcpy(lt, h, N * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ag, h, N * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(rf, (char*)h + N * 4, N * 4, cudaMemcpyHostToDevice));
        free(h);
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto timeit = [&](const char* name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        cudaEventRecord(a);
        const int it = 20;
        for (int i = 0; i < it; ++i) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double us = ms * 1000 / it;
        printf("%-22s %8.1f us  %7.0f GB/s\n", name, us, N * 16.0 / (us * 1e-6) / 1e9);
    };
    timeit("copy-read grid=4xSM", [&] { copy_read<<<sms * 4, 512>>>((const ulonglong2*)lt, (const uint4*)ag, (const uint4*)rf, N / 4, out); });
    timeit("copy-read grid=1xSM", [&] { copy_read<<<sms, 512>>>((const ulonglong2*)lt, (const uint4*)ag, (const uint4*)rf, N / 4, out); });
    timeit("tile-loop D=2", [&] { tile_loop<2><<<sms, 512>>>(lt, ag, rf, N, 0, out); });
    timeit("tile-loop D=3", [&] { tile_loop<3><<<sms, 512>>>(lt, ag, rf, N, 0, out); });
    timeit("tile-loop D=4", [&] { tile_loop<4><<<sms, 512>>>(lt, ag, rf, N, 0, out); });
    {
        size_t sm3 = 3 * 2048 * 16, sm4 = 4 * 2048 * 16, sm6 = 6 * 2048 * 16;
        cudaFuncSetAttribute(tma_loop<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm3);
        cudaFuncSetAttribute(tma_loop<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm4);
        cudaFuncSetAttribute(tma_loop<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm6);
        timeit("tma-loop S=3", [&] { tma_loop<3><<<sms, 512, sm3>>>(lt, ag, rf, N, 0, out); });
        timeit("tma-loop S=4", [&] { tma_loop<4><<<sms, 512, sm4>>>(lt, ag, rf, N, 0, out); });
        timeit("tma-loop S=6", [&] { tma_loop<6><<<sms, 512, sm6>>>(lt, ag, rf, N, 0, out); });
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
}
