// kernel_gen.cuh -- NEXT-3: on-device generation of Arrival-Model-2 instances on the
// lambda x M sweep grid of configuration C5, from an integer counter-based specification
// (workloads.am2_counter is the host reference; include/kvsched.h states the spec).
//
//   instance g = instance_id0 + k; cell = g mod (n_lambda n_m); lambda index = cell / n_m;
//   M = m_values[cell % n_m];  u(stream, j) = Philox4x32-10(counter (lo g, hi g, stream, j),
//   key (lo seed, hi seed));  mulhi(u, r) = (u r) >> 32
//   T = T_lo + mulhi(u(0,0).x, T_hi - T_lo + 1)
//   arrivals at round r (1..T): smallest c with u(1, r).x < cdf[lambda][c]  (Poisson by inversion)
//   request i (arrival order): w = u(2, i); s = s_lo + mulhi(w.x, s_hi - s_lo + 1);
//                              o = 1 + mulhi(w.y, M - s); o~ = o.
#pragma once
#include "params.cuh"

namespace kv {

struct GenAm2 {
    long long n_inst, id0;
    unsigned long long seed;
    int n_lambda, n_m;
    const unsigned long long *cdf;   // [n_lambda][32]
    const int *m_values;             // [n_m]
    int T_lo, T_hi, s_lo, s_hi;
};

__device__ __forceinline__ uint4 gen_u(unsigned long long g, unsigned long long seed, unsigned stream, unsigned j)
{
    return philox4x32_10(make_uint4((uint32_t)g, (uint32_t)(g >> 32), stream, j),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

__device__ __forceinline__ int gen_count(const GenAm2 &G, unsigned long long g, int li, int r)
{
    const unsigned long long u = gen_u(g, G.seed, 1u, (unsigned)r).x;
    const unsigned long long *c = G.cdf + (size_t)li * 32;
    int k = 0;
    while (k < 31 && u >= c[k]) ++k;
    return k;
}

// sizes into off[k+1] (off[0] = 0); a scan turns them into offsets
__global__ void k_gen_am2_count(const GenAm2 G, long long *off)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < G.n_inst;
         k += (long long)gridDim.x * blockDim.x) {
        const unsigned long long g = (unsigned long long)(G.id0 + k);
        const int cell = (int)(g % (unsigned long long)(G.n_lambda * G.n_m));
        const int li = cell / G.n_m;
        const int T = G.T_lo + (int)__umulhi(gen_u(g, G.seed, 0u, 0u).x, (unsigned)(G.T_hi - G.T_lo + 1));
        long long n = 0;
        for (int r = 1; r <= T; ++r) n += gen_count(G, g, li, r);
        off[k + 1] = n;
        if (k == 0) off[0] = 0;
    }
}

// in-place inclusive scan of x[1..n] (x[0] = 0): per-block scans, block-sum scan, fix-up
constexpr int kScanBlock = 1024;

__device__ __forceinline__ long long block_incl_scan(long long v, long long *tmp)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(KV_FULL, v, d);
        if (lane >= d) v += y;
    }
    if (lane == 31) tmp[wid] = v;
    __syncthreads();
    if (wid == 0) {
        long long w = lane < (int)(blockDim.x >> 5) ? tmp[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long y = __shfl_up_sync(KV_FULL, w, d);
            if (lane >= d) w += y;
        }
        tmp[lane] = w;
    }
    __syncthreads();
    const long long r = v + (wid > 0 ? tmp[wid - 1] : 0);
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanBlock) k_scan_blocks(long long *x, long long n, long long *bsum)
{
    __shared__ long long tmp[32];
    const long long i = 1 + blockIdx.x * (long long)kScanBlock + threadIdx.x;
    const long long v = i <= n ? x[i] : 0;
    const long long s = block_incl_scan(v, tmp);
    if (i <= n) x[i] = s;
    if (threadIdx.x == kScanBlock - 1) bsum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kScanBlock) k_scan_sums(long long *bsum, long long nb)
{
    __shared__ long long tmp[32];
    __shared__ long long last;
    long long carry = 0;
    for (long long base = 0; base < nb; base += kScanBlock) {
        const long long i = base + threadIdx.x;
        const long long v = i < nb ? bsum[i] : 0;
        const long long s = block_incl_scan(v, tmp) + carry;
        if (i < nb) bsum[i] = s;
        if (threadIdx.x == kScanBlock - 1) last = s;
        __syncthreads();
        carry = last;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanBlock) k_scan_fix(long long *x, long long n, const long long *bsum)
{
    if (blockIdx.x == 0) return;
    const long long i = 1 + blockIdx.x * (long long)kScanBlock + threadIdx.x;
    if (i <= n) x[i] += bsum[blockIdx.x - 1];
}

// one warp per instance: arrival rounds from the per-round counts, then the request rows
__global__ void __launch_bounds__(128) k_gen_am2_fill(const GenAm2 G, const long long *off, int4 *req, int *mem)
{
    __shared__ int cum[4][1025];                        // per warp: cumulative counts by round
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    int *cw = cum[wid];
    for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + wid; k < G.n_inst; k += warps) {
        const unsigned long long g = (unsigned long long)(G.id0 + k);
        const int cell = (int)(g % (unsigned long long)(G.n_lambda * G.n_m));
        const int li = cell / G.n_m;
        const int M = G.m_values[cell % G.n_m];
        const int T = G.T_lo + (int)__umulhi(gen_u(g, G.seed, 0u, 0u).x, (unsigned)(G.T_hi - G.T_lo + 1));
        int carry = 0;
        for (int r0 = 1; r0 <= T; r0 += 32) {           // inclusive prefix of counts over rounds
            const int r = r0 + lane;
            int c = r <= T ? gen_count(G, g, li, r) : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(KV_FULL, c, d);
                if (lane >= d) c += y;
            }
            if (r <= T) cw[r] = carry + c;
            carry += __shfl_sync(KV_FULL, c, 31);
        }
        __syncwarp();
        const long long o0 = off[k];
        const int n = (int)(off[k + 1] - o0);
        for (int i = lane; i < n; i += 32) {
            int lo = 1, hi = T;                          // smallest r with cum[r] > i
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (cw[mid] > i) hi = mid; else lo = mid + 1;
            }
            const uint4 w = gen_u(g, G.seed, 2u, (unsigned)i);
            const int s = G.s_lo + (int)__umulhi(w.x, (unsigned)(G.s_hi - G.s_lo + 1));
            const int o = 1 + (int)__umulhi(w.y, (unsigned)max(M - s, 0));
            req[o0 + i] = make_int4(lo, s, o, o);
        }
        if (lane == 0) mem[k] = M;
        __syncwarp();
    }
}

}  // namespace kv
