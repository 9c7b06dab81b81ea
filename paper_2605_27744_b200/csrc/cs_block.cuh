// Block-level building blocks shared by the admission kernel: reductions and an exact
// MSB-first radix select over distinct 64-bit keys (last_touch ticks are unique per resident
// block, so a k-th smallest value identifies exactly k elements).
#pragma once

#include "cs_device.cuh"

namespace csb {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

struct RedSmem {
    long long v[32];
    unsigned long long u[32];
    unsigned long long w[32];
};

__device__ __forceinline__ long long block_sum(long long x, RedSmem& R) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if (lane_id() == 0) R.v[warp_id()] = x;
    __syncthreads();
    if (warp_id() == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        long long y = lane_id() < nw ? R.v[lane_id()] : 0;
        for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        if (lane_id() == 0) R.v[0] = y;
    }
    __syncthreads();
    const long long r = R.v[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ long long block_min(long long x, RedSmem& R) {
    for (int o = 16; o; o >>= 1) x = min(x, __shfl_xor_sync(0xffffffffu, x, o));
    __syncthreads();
    if (lane_id() == 0) R.v[warp_id()] = x;
    __syncthreads();
    if (warp_id() == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        long long y = lane_id() < nw ? R.v[lane_id()] : 0x7fffffffffffffffll;
        for (int o = 16; o; o >>= 1) y = min(y, __shfl_xor_sync(0xffffffffu, y, o));
        if (lane_id() == 0) R.v[0] = y;
    }
    __syncthreads();
    const long long r = R.v[0];
    __syncthreads();
    return r;
}

// Number of v[0, m) below x. v lives in shared memory, 16-byte aligned: 128-bit loads, four
// independent counters and an unrolled body keep many loads in flight (a plain loop is bound by
// the shared-memory latency at one CTA per SM).
__device__ __forceinline__ int count_below(const unsigned long long* v, int m, unsigned long long x) {
    int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
    int k = 0;
#pragma unroll 4
    for (; k + 4 <= m; k += 4) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(v + k);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(v + k + 2);
        r0 += a.x < x;
        r1 += a.y < x;
        r2 += b.x < x;
        r3 += b.y < x;
    }
    for (; k < m; ++k) r0 += v[k] < x;
    return r0 + r1 + r2 + r3;
}

struct SelectSmem {
    unsigned int hist[256];
    unsigned long long acc_or, acc_and;
    unsigned long long prefix;
    unsigned long long hmax;  // finalize_list: largest candidate written for the list
    int k;
    int tmp;
};

// k-th smallest (1 <= k <= count) of the values v[j] (j < m) whose tag[j] == want (tag may
// be null = all). v may live in shared or global memory. All threads of the block call it.
// The digits above the highest bit in which the selected values differ are skipped.
__device__ inline unsigned long long block_kth(const unsigned long long* v, const unsigned char* tag,
                                               unsigned char want, int m, int k, SelectSmem& S) {
    if (threadIdx.x == 0) {
        S.acc_or = 0ull;
        S.acc_and = ~0ull;
    }
    __syncthreads();
    unsigned long long o = 0ull, a = ~0ull;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        if (tag && tag[j] != want) continue;
        const unsigned long long x = v[j];
        o |= x;
        a &= x;
    }
    for (int s = 16; s; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if (lane_id() == 0) {
        atomicOr(&S.acc_or, o);
        atomicAnd(&S.acc_and, a);
    }
    __syncthreads();
    const unsigned long long diff = S.acc_or ^ S.acc_and;
    const unsigned long long same = S.acc_and;
    if (diff == 0ull) {  // a single distinct value
        __syncthreads();
        return same;
    }
    const int hb = 63 - __clzll((long long)diff);
    int shift = (hb / 8) * 8;
    unsigned long long hmask = (shift + 8 >= 64) ? 0ull : ~((1ull << (shift + 8)) - 1ull);
    unsigned long long prefix = same & hmask;
    int kk = k;
    for (;;) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) S.hist[b] = 0u;
        __syncthreads();
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            if (tag && tag[j] != want) continue;
            const unsigned long long x = v[j];
            if ((x & hmask) == prefix) atomicAdd(&S.hist[(x >> shift) & 255ull], 1u);
        }
        __syncthreads();
        if (warp_id() == 0) {
            unsigned int c[8];
            unsigned int s = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = S.hist[lane_id() * 8 + q];
                s += c[q];
            }
            unsigned int inc = s;
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned int t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane_id() >= d) inc += t;
            }
            const unsigned int exc = inc - s;
            if (exc < (unsigned)kk && (unsigned)kk <= inc) {
                unsigned int cum = exc;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (cum + c[q] >= (unsigned)kk) {
                        S.prefix = prefix | ((unsigned long long)(lane_id() * 8 + q) << shift);
                        S.k = kk - (int)cum;
                        break;
                    }
                    cum += c[q];
                }
            }
        }
        __syncthreads();
        prefix = S.prefix;
        kk = S.k;
        hmask |= (255ull << shift);
        if (shift == 0) break;
        shift -= 8;
    }
    __syncthreads();
    return prefix;
}

// Barrier of a warp group of `n` threads (a multiple of 32) on named barrier `id` (1..15).
__device__ __forceinline__ void group_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// block_kth for a warp group (threads gt = 0..gn-1 of the group, named barrier bar), so two
// groups of one CTA select from two lists at once. v in shared memory; all values distinct.
__device__ inline unsigned long long group_kth(const unsigned long long* v, int m, int k, SelectSmem& S, int gt,
                                               int gn, int bar) {
    if (gt == 0) {
        S.acc_or = 0ull;
        S.acc_and = ~0ull;
    }
    group_sync(bar, gn);
    unsigned long long o = 0ull, a = ~0ull;
    for (int j = gt; j < m; j += gn) {
        const unsigned long long x = v[j];
        o |= x;
        a &= x;
    }
    for (int s = 16; s; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if ((gt & 31) == 0) {
        atomicOr(&S.acc_or, o);
        atomicAnd(&S.acc_and, a);
    }
    group_sync(bar, gn);
    const unsigned long long diff = S.acc_or ^ S.acc_and;
    const unsigned long long same = S.acc_and;
    if (diff == 0ull) {
        group_sync(bar, gn);
        return same;
    }
    const int hb = 63 - __clzll((long long)diff);
    int shift = (hb / 8) * 8;
    unsigned long long hmask = (shift + 8 >= 64) ? 0ull : ~((1ull << (shift + 8)) - 1ull);
    unsigned long long prefix = same & hmask;
    int kk = k;
    for (;;) {
        for (int b = gt; b < 256; b += gn) S.hist[b] = 0u;
        group_sync(bar, gn);
        for (int j = gt; j < m; j += gn) {
            const unsigned long long x = v[j];
            if ((x & hmask) == prefix) atomicAdd(&S.hist[(x >> shift) & 255ull], 1u);
        }
        group_sync(bar, gn);
        if (gt < 32) {
            const int ln = gt;
            unsigned int c[8];
            unsigned int sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c[q] = S.hist[ln * 8 + q];
                sum += c[q];
            }
            unsigned int inc = sum;
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned int t = __shfl_up_sync(0xffffffffu, inc, d);
                if (ln >= d) inc += t;
            }
            const unsigned int exc = inc - sum;
            if (exc < (unsigned)kk && (unsigned)kk <= inc) {
                unsigned int cum = exc;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (cum + c[q] >= (unsigned)kk) {
                        S.prefix = prefix | ((unsigned long long)(ln * 8 + q) << shift);
                        S.k = kk - (int)cum;
                        break;
                    }
                    cum += c[q];
                }
            }
        }
        group_sync(bar, gn);
        prefix = S.prefix;
        kk = S.k;
        hmask |= (255ull << shift);
        if (shift == 0) break;
        shift -= 8;
    }
    group_sync(bar, gn);
    return prefix;
}

}  // namespace csb
