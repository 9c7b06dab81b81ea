// Next-use index of the Belady baseline, built on the device from the materialized requests:
// BeladyPolicy::BeladyPolicy (baselines.cpp:34-46, paths relative to /root/reference/proj)
// keeps per key its sorted request ids and the chain position of its first occurrence. Here the
// request blocks are sorted by key (stable, so request order is kept within a key); the run of a
// key is its CSR row of request ids, and its first element gives the depth.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "cs_launch.h"

namespace csb {

namespace {

__global__ void bel_req_of_flat(const long long* blk_off, long long n_req, unsigned int* req_of) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n_req; r += (long long)gridDim.x * blockDim.x)
        for (long long f = blk_off[r]; f < blk_off[r + 1]; ++f) req_of[f] = (unsigned int)r;
}

__global__ void bel_iota(unsigned int* v, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = (unsigned int)i;
}

__global__ void bel_heads(const unsigned long long* k, long long n, unsigned int* head) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        head[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

// kid = inclusive scan of the heads - 1
__global__ void bel_fill(const unsigned int* head, const unsigned int* kid1, const unsigned int* flat,
                         const unsigned int* req_of, const long long* blk_off, long long n, unsigned int* ref,
                         long long* ref_off, int* depth, unsigned int* kid_of) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned int kid = kid1[i] - 1u;
        const unsigned int f = flat[i];
        const unsigned int r = req_of[f];
        ref[i] = r;
        kid_of[f] = kid;
        if (head[i]) {
            ref_off[kid] = i;
            depth[kid] = (int)((long long)f - blk_off[r]);  // depth_.emplace: the first occurrence
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ref_off[kid1[n - 1]] = n;
}

void ckb(cudaError_t e) {
    if (e != cudaSuccess) throw e;
}

}  // namespace

long long build_belady_index(const unsigned long long* keys, long long n_flat, const long long* blk_off, long long n_req,
                             unsigned int* ref, long long* ref_off, int* depth, unsigned int* kid_of, cudaStream_t s) {
    if (n_flat <= 0) return 0;
    if (n_flat >= (1ll << 31)) return -1;  // cub sizes and 32-bit request / key ids
    unsigned long long* k_out = nullptr;
    unsigned int *v_in = nullptr, *v_out = nullptr, *head = nullptr, *kid1 = nullptr, *req_of = nullptr;
    void* tmp = nullptr;
    long long n_kids = -1;
    try {
        ckb(cudaMalloc(&k_out, 8 * n_flat));
        ckb(cudaMalloc(&v_in, 4 * n_flat));
        ckb(cudaMalloc(&v_out, 4 * n_flat));
        ckb(cudaMalloc(&head, 4 * n_flat));
        ckb(cudaMalloc(&kid1, 4 * n_flat));
        ckb(cudaMalloc(&req_of, 4 * n_flat));
        const int n = (int)n_flat;
        size_t b1 = 0, b2 = 0;
        ckb(cub::DeviceRadixSort::SortPairs(nullptr, b1, keys, k_out, v_in, v_out, n, 0, 64, s));
        ckb(cub::DeviceScan::InclusiveSum(nullptr, b2, head, kid1, n, s));
        ckb(cudaMalloc(&tmp, b1 > b2 ? b1 : b2));
        const int g = 592, t = 256;
        bel_req_of_flat<<<g, t, 0, s>>>(blk_off, n_req, req_of);
        bel_iota<<<g, t, 0, s>>>(v_in, n_flat);
        ckb(cudaGetLastError());
        ckb(cub::DeviceRadixSort::SortPairs(tmp, b1, keys, k_out, v_in, v_out, n, 0, 64, s));  // stable
        bel_heads<<<g, t, 0, s>>>(k_out, n_flat, head);
        ckb(cub::DeviceScan::InclusiveSum(tmp, b2, head, kid1, n, s));
        bel_fill<<<g, t, 0, s>>>(head, kid1, v_out, req_of, blk_off, n_flat, ref, ref_off, depth, kid_of);
        ckb(cudaGetLastError());
        unsigned int last = 0;
        ckb(cudaMemcpyAsync(&last, kid1 + n_flat - 1, 4, cudaMemcpyDeviceToHost, s));
        ckb(cudaStreamSynchronize(s));
        n_kids = last;
    } catch (cudaError_t) {
        n_kids = -1;
    }
    for (void* q : {(void*)k_out, (void*)v_in, (void*)v_out, (void*)head, (void*)kid1, (void*)req_of, tmp})
        if (q) cudaFree(q);
    return n_kids;
}

}  // namespace csb
