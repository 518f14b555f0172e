// kernel_lb.cuh -- lower bound on the hindsight optimum for simultaneous arrivals.
//
// For an instance whose requests all arrive at the same round a0, the k requests that
// finish first occupy vol_i = s_i o_i + o_i (o_i + 1) / 2 slot-rounds each inside
// rounds a0+1 .. c_(k), with capacity M per round (the volume argument of P:319), so
//   c_(k) - a0 >= ceil(V_k / M),   V_k = sum of the k smallest volumes,
// and also c_(k) - a0 >= o_(k), the k-th smallest output length.  Hence
//   OPT = sum_k (c_(k) - a0) >= LB = sum_k max(ceil(V_k / M), o_(k)).
// One CTA per instance: bitonic sorts of the volumes and of the output lengths in shared
// memory, a block scan of the sorted volumes, a block reduction of the terms.
#pragma once
#include "params.cuh"

namespace kv {

__device__ __forceinline__ void block_bitonic_sort(long long *v, int NPi)
{
    for (int k = 2; k <= NPi; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < (NPi >> 1); i += blockDim.x) {
                const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                const int hi = lo + j;
                const bool up = (lo & k) == 0;
                const long long x = v[lo], y = v[hi];
                if ((x > y) == up) { v[lo] = y; v[hi] = x; }
            }
            __syncthreads();
        }
}

// lb[k] = LB_sorted of instance k, or -1 if its requests do not all arrive together or it
// has more than max_n requests; 0 for an empty instance.  blockDim.x = 512, dynamic shared
// memory = 2 * next_pow2(max_n) * 8 bytes + 64 bytes.
__global__ void __launch_bounds__(512) k_lb_sorted(long long n_inst, const long long *offset, const int4 *req,
                                                    const int *mem, int max_n, long long *lb)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int NPmax = next_pow2(max(max_n, 2));
    long long *vol = reinterpret_cast<long long *>(smem_raw);
    long long *os = vol + NPmax;
    __shared__ long long warp_part[16];
    __shared__ int flag;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (long long inst = blockIdx.x; inst < n_inst; inst += gridDim.x) {
        const long long off = offset[inst];
        const int n = (int)(offset[inst + 1] - off);
        const long long M = mem[inst];
        if (threadIdx.x == 0) flag = 0;
        __syncthreads();
        if (n > max_n || M < 1) {
            if (threadIdx.x == 0) lb[inst] = -1;
            __syncthreads();
            continue;
        }
        if (n == 0) {
            if (threadIdx.x == 0) lb[inst] = 0;
            __syncthreads();
            continue;
        }
        const int NPi = next_pow2(max(n, 2));
        const int a0 = req[off].x;
        for (int i = threadIdx.x; i < NPi; i += blockDim.x) {
            long long v = 0x7fffffffffffffffll, o = 0x7fffffffffffffffll;
            if (i < n) {
                const int4 r = req[off + i];
                if (r.x != a0) atomicOr(&flag, 1);
                o = r.z;
                v = (long long)r.y * r.z + (long long)r.z * (r.z + 1) / 2;
            }
            vol[i] = v;
            os[i] = o;
        }
        __syncthreads();
        if (flag) {
            if (threadIdx.x == 0) lb[inst] = -1;
            __syncthreads();
            continue;
        }
        block_bitonic_sort(vol, NPi);
        block_bitonic_sort(os, NPi);
        // inclusive scan of vol[0..n) in chunks of blockDim.x, then the terms
        long long carry = 0, acc = 0;
        for (int base = 0; base < n; base += blockDim.x) {
            const int i = base + threadIdx.x;
            long long x = i < n ? vol[i] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const long long y = __shfl_up_sync(KV_FULL, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) warp_part[wid] = x;
            __syncthreads();
            long long wp = 0;
            for (int w = 0; w < wid; ++w) wp += warp_part[w];
            long long chunk_total = 0;
            for (int w = 0; w < nwarps; ++w) chunk_total += warp_part[w];
            const long long Vk = carry + wp + x;                  // sum of the i+1 smallest volumes
            if (i < n) {
                const long long c1 = (Vk + M - 1) / M;
                acc += c1 > os[i] ? c1 : os[i];
            }
            carry += chunk_total;
            __syncthreads();
        }
        acc = warp_sum_i64(acc);
        if (lane == 0) warp_part[wid] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            long long tot = 0;
            for (int w = 0; w < nwarps; ++w) tot += warp_part[w];
            lb[inst] = tot;
        }
        __syncthreads();
    }
}

}  // namespace kv
