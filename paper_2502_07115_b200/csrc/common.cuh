// common.cuh -- warp-level building blocks shared by the simulation kernels (sm_100a).
//
// Nothing here is shared with oracle/ (the CPU checker); the Philox block below is an
// independent implementation of Salmon et al., SC'11 (checked against the published
// known-answer vectors through sched_philox4x32_10 in tests/test_gpu_parity.py).
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

#define KV_FULL 0xffffffffu
#define KV_INF 0x7fffffff
// alpha-beta: at most this many clearing passes per overflow, then LIVELOCK (DESIGN Q29)
#define KV_BETA_MAX_PASSES 65536
// lane kernel scope: arrivals at most 2^29, so a run ends before the default round cap
#define KV_LANE_MAX_A (1 << 29)

namespace kv {

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), all four output words.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// alpha-beta eviction draw (DESIGN Q14): counter (t, pass, idx, 0), key = halves of
// seed ^ gid * 0x9E3779B97F4A7C15, output word 0.
__device__ __forceinline__ uint32_t evict_draw(uint64_t seed, uint64_t gid, int t, int pass, int idx)
{
    const uint64_t K = seed ^ (gid * 0x9E3779B97F4A7C15ull);
    return philox4x32_10(make_uint4((uint32_t)t, (uint32_t)pass, (uint32_t)idx, 0u),
                         make_uint2((uint32_t)K, (uint32_t)(K >> 32))).x;
}

// ---------------------------------------------------------------------------------------
// warp reductions
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ long long warp_sum_i64(long long v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(KV_FULL, v, o);
    return v;
}

__device__ __forceinline__ int warp_max_i32(int v) { return __reduce_max_sync(KV_FULL, v); }
__device__ __forceinline__ int warp_min_i32(int v) { return __reduce_min_sync(KV_FULL, v); }

// ---------------------------------------------------------------------------------------
// Waiting queue R as a two-level bitmap over ranks (rank = position in the policy's key
// order).  bm[w] holds ranks 32w..32w+31; bit (w & 31) of sm[w >> 5] says bm[w] != 0.
// Up to 32 summary words -> 32768 ranks.  The head (smallest waiting rank) is one ballot
// over the summary, one shuffle and one shared load.
// ---------------------------------------------------------------------------------------
struct WarpQueue {
    uint32_t *bm;
    uint32_t *sm;
    int ns;              // summary words in use (<= 32)
};

// insert rank r (may be called by several lanes at once)
__device__ __forceinline__ void q_insert(const WarpQueue &q, int r)
{
    atomicOr(&q.bm[r >> 5], 1u << (r & 31));
    atomicOr(&q.sm[r >> 10], 1u << ((r >> 5) & 31));
}

// smallest rank in the queue, KV_INF if empty (warp-uniform; call with all lanes)
__device__ __forceinline__ int q_first(const WarpQueue &q)
{
    const int lane = lane_id();
    const uint32_t sw = lane < q.ns ? q.sm[lane] : 0u;
    const uint32_t b = __ballot_sync(KV_FULL, sw != 0u);
    if (b == 0u) return KV_INF;
    const int l0 = __ffs(b) - 1;
    const uint32_t w0 = __shfl_sync(KV_FULL, sw, l0);
    const int wi = (l0 << 5) + __ffs(w0) - 1;
    const uint32_t word = q.bm[wi];
    return (wi << 5) + __ffs(word) - 1;
}

// remove the head h (the smallest rank) and return the new head (warp-uniform)
__device__ __forceinline__ int q_pop_head(const WarpQueue &q, int h)
{
    const uint32_t word = q.bm[h >> 5] & ~(1u << (h & 31));
    __syncwarp();
    if (lane_id() == 0) {
        q.bm[h >> 5] = word;
        if (word == 0u) q.sm[h >> 10] &= ~(1u << ((h >> 5) & 31));
    }
    __syncwarp();
    if (word != 0u) return (h & ~31) + __ffs(word) - 1;   // remaining bits are all > h
    return q_first(q);
}

// remove an arbitrary rank r (lane 0 only; caller syncs)
__device__ __forceinline__ void q_erase_lane0(const WarpQueue &q, int r)
{
    const uint32_t word = q.bm[r >> 5] & ~(1u << (r & 31));
    q.bm[r >> 5] = word;
    if (word == 0u) q.sm[r >> 10] &= ~(1u << ((r >> 5) & 31));
}

__host__ __device__ __forceinline__ int next_pow2(int x)
{
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// instance-level counters every kernel writes in its epilogue
struct InstResult {
    long long tel, rounds, decision_rounds, evictions;
    int makespan, peak, status;
};

}  // namespace kv
