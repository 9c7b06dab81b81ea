// Latency microbenchmarks for the admission kernel's serial phases (one CTA of 544 threads):
// %globaltimer read, clock64 read, __syncthreads, dependent L2 load, global store + fence.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned long long* out, unsigned long long* buf, int iters) {
    __shared__ unsigned long long s[1];
    unsigned long long t0, t1, x = 0;
    // 1. globaltimer reads (dependent through the sum)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        x += g;
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / iters;
    // 2. syncthreads
    t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = (t1 - t0) / iters;
    // 3. dependent L2 loads (pointer chase over a small ring in L2)
    unsigned long long p = threadIdx.x == 0 ? buf[0] : 0;
    t0 = clock64();
    if (threadIdx.x == 0)
        for (int i = 0; i < iters; ++i) p = __ldcg(buf + (p & 1023));
    t1 = clock64();
    if (threadIdx.x == 0) out[2] = (t1 - t0) / iters;
    // 4. syncthreads_or
    t0 = clock64();
    int acc = 0;
    for (int i = 0; i < iters; ++i) acc += __syncthreads_or(threadIdx.x == (unsigned)i);
    t1 = clock64();
    if (threadIdx.x == 0) out[3] = (t1 - t0) / iters;
    // 5. threadfence after a store
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) {
            buf[2048 + i] = i;
            __threadfence();
        }
    }
    t1 = clock64();
    if (threadIdx.x == 0) out[4] = (t1 - t0) / iters;
    // 6. atomicAdd round trip (returned value used)
    unsigned long long q = 0;
    t0 = clock64();
    if (threadIdx.x == 0)
        for (int i = 0; i < iters; ++i) q += atomicAdd(buf + 4096 + (q & 7), 1ull);
    t1 = clock64();
    if (threadIdx.x == 0) out[5] = (t1 - t0) / iters;
    if (threadIdx.x == 0) out[6] = x + p + acc + q + s[0];
}

int main() {
    unsigned long long *out, *buf;
    cudaMalloc(&out, 64 * 8);
    cudaMalloc(&buf, 8192 * 8);
    unsigned long long h[8192];
    for (int i = 0; i < 8192; ++i) h[i] = (i * 7 + 13) & 1023;
    cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) k<<<1, 544>>>(out, buf, 200);
    cudaDeviceSynchronize();
    unsigned long long r[8];
    cudaMemcpy(r, out, 64, cudaMemcpyDeviceToHost);
    printf("cycles: globaltimer %llu, syncthreads(544) %llu, L2 dep load %llu, syncthreads_or %llu, store+fence %llu, atomic rt %llu\n",
           r[0], r[1], r[2], r[3], r[4], r[5]);
    // launch overhead: empty cooperative-size kernel, 148 x 544, 220 KB smem
    return 0;
}
