// kernel_mcring.cuh -- MC-SF (Algorithm 1) and MC-Benchmark (Algorithm 2,
// P:1076-1103) for large budgets (C3, C4: M = 16492): one warp per instance.
//
// Two launches per batch:
//
//   k_mc_prep<POL>   one CTA per instance.  Validates the rows (DESIGN Q8), computes the
//                    round cap (Q23), ranks the requests ((o~, idx) for MC-SF, P:175 / Q5;
//                    idx for MC-Benchmark) with a bitonic sort in shared memory and
//                    writes two 8-byte streams: rq8[rank] = {s | w << 16, idx} (the head's
//                    entry) and arr8[idx] = {a, rank} (the arrival stream).  Invalid /
//                    unsupported instances get their status here; MC-SF instances with
//                    o~ > o are listed for k_prot (alpha = 0, DESIGN Q10) with the entries
//                    it reads.
//   k_mc_ring<POL>   the round loop.  Per warp in shared memory:
//                      * the projected-memory profile of the window [t+1, t+L] (Eq. 5 LHS of
//                        the in-flight set) as 16-bit slots -- valid because every
//                        admission certified Prof <= M <= 32767 on its window -- so one
//                        32-bit word holds two rounds and the warp covers 64 rounds per
//                        pass with 16x2 SIMD adds/maxima (VIADD2 / VIMNMX.U16x2);
//                      * the waiting queue as a rank bitmap (common.cuh);
//                      * the arrival stream staged by cp.async.bulk (global -> shared, one
//                        mbarrier per 32-entry chunk, four chunks in flight), so arrival
//                        intake and the "does an arrival sort before the head" look-ahead
//                        read shared memory, not HBM/L2.
//                    A candidate (s, w) fits at round t iff max_{1<=u<=w} Prof(t+u) + u <=
//                    M - s (Eq. 5; one SIMD max pass).  When it does not, the first round
//                    at which it fits while the profile only advances (Alg. 1 breaks at the
//                    head, so nothing else changes meanwhile) is found for the next 31
//                    rounds: position u blocks the offsets D in [max(u-w,0), min(u-1,
//                    Prof+u-(M-s)-1)]; positions 32..w only through their maximum (their
//                    interval starts at 0), so only positions 1..31 and w+1..w+31 need the
//                    per-position interval -- one lane each.  Requests whose window exceeds
//                    the ring (w + 31 > L) take a per-position path that also reads the
//                    long list (kernel_ring.cuh).
#pragma once
#include <cub/block/block_radix_sort.cuh>
#include "kernel_ring.cuh"

namespace kv {

#define KV_PREP_WARP_N 1024                  // k_mc_prep_w takes instances up to this size
#ifndef KV_PREP_RADIX
#define KV_PREP_RADIX 1                      // k_mc_prep: CUB block radix sort for 2048 <= NP <= 16384
#endif
#ifndef KV_PREP_CTA_LO
#define KV_PREP_CTA_LO 128                   // instances of KV_PREP_CTA_LO < n <= 1024: k_mc_prep<POL, 256>
#endif                                       // (KV_PREP_CTA_LO >= 1024: all on k_mc_prep_w)
#define KV_STAGE_CH 32                       // arrival entries per staged chunk
#define KV_STAGE_SLOTS 4                     // chunks resident / in flight per warp
#define KV_STAGE_ENTRIES (KV_STAGE_CH + 2)   // one extra on each side for 16-byte alignment

// ---------------------------------------------------------------------------------------
// bulk copy + mbarrier (PTX)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// one thread: arm `bar` for `bytes` and start the global -> shared bulk copy that completes it
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0u;
}

// The arrival stream of one instance, staged chunk by chunk.  Chunk c (entries 32c..32c+31)
// lives in slot c & 3; the global copy starts at the even entry at or below off + 32c so
// that source and size are 16-byte multiples (34 entries = 272 bytes).  Warp-uniform state:
// chunks [c0, iss) issued, [c0, rdy) landed (waited); `phase` bit b = parity of slot b's
// next completion, `pend` bit b = a copy on slot b not yet waited (possibly of an earlier
// instance: it is waited before the slot is reused, keeping the parities consistent).
struct Stage {
    int2 *buf;          // [KV_STAGE_SLOTS][KV_STAGE_ENTRIES]
    uint64_t *bar;      // [KV_STAGE_SLOTS]
    const int2 *src;    // arr8 + off (this instance's entries)
    int shift;          // (off & 1): position of entry 32c in its slot
    int nch;            // chunks of this instance
    int c0, iss, rdy;
    uint32_t phase, pend;
};

__device__ __forceinline__ void stage_wait_slot(Stage &S, int b)
{
    while (!mbar_try_wait(&S.bar[b], (S.phase >> b) & 1u)) {
    }
    S.phase ^= 1u << b;
    S.pend &= ~(1u << b);
}

__device__ __forceinline__ void stage_issue(Stage &S)
{
    const int hi = min(S.c0 + KV_STAGE_SLOTS, S.nch);
    while (S.iss < hi) {
        const int c = S.iss, b = c & (KV_STAGE_SLOTS - 1);
        if ((S.pend >> b) & 1u) stage_wait_slot(S, b);
        __syncwarp();
        if (lane_id() == 0)
            bulk_g2s(S.buf + b * KV_STAGE_ENTRIES, S.src + (KV_STAGE_CH * c - S.shift),
                     KV_STAGE_ENTRIES * (uint32_t)sizeof(int2), &S.bar[b]);
        S.pend |= 1u << b;
        ++S.iss;
    }
}

// make chunks c_lo..c_hi readable (c_hi - c_lo <= 1); chunks below c_lo are released
__device__ __forceinline__ void stage_need(Stage &S, int c_lo, int c_hi)
{
    if (c_lo > S.c0) {
        S.c0 = c_lo;
        if (S.rdy < S.c0) S.rdy = S.c0;
        stage_issue(S);
    }
    while (S.rdy <= c_hi) {
        if (S.rdy >= S.iss) stage_issue(S);
        stage_wait_slot(S, S.rdy & (KV_STAGE_SLOTS - 1));
        ++S.rdy;
    }
}

__device__ __forceinline__ void stage_begin(Stage &S, const int2 *arr8, long long off, int n)
{
    S.src = arr8 + off;
    S.shift = (int)(off & 1);
    S.nch = (n + KV_STAGE_CH - 1) / KV_STAGE_CH;
    S.c0 = S.iss = S.rdy = 0;
    stage_issue(S);
}

// entry k (lane-divergent): shared memory if its chunk has landed, else global
__device__ __forceinline__ int2 stage_get(const Stage &S, int k)
{
    const int c = k / KV_STAGE_CH;
    if (c >= S.c0 && c < S.rdy)
        return S.buf[(c & (KV_STAGE_SLOTS - 1)) * KV_STAGE_ENTRIES + S.shift + (k - KV_STAGE_CH * c)];
    return S.src[k];
}

// ---------------------------------------------------------------------------------------
// 16-bit profile ring: slot r & (L-1) = absolute round r; word j = rounds 2j, 2j+1 (mod L)
// ---------------------------------------------------------------------------------------
struct R16 {
    uint16_t *p;
    uint2 *q;           // quads: rounds 4j .. 4j+3 (mod L)
    int L, mask, qmask;
};

// in-window halfword masks of a quad: rounds t+u0 .. t+u0+3 against positions [1, e]
__device__ __forceinline__ uint32_t half_in(int u, int e) { return (u >= 1 && u <= e) ? 0xffffu : 0u; }

// The first-fit horizon: a blocked head is resolved for offsets D in [0, KV_FF_D]; position
// u blocks D in [max(u-w, 0), min(u-1, Prof(t+u)+u-(M-s)-1, KV_FF_D)], so every position
// u >= KV_FF_D + 1 inside the window (u <= w) blocks a prefix [0, ...] and only the maximum
// of Prof(t+u)+u over them matters.  With four rounds per quad, the quads whose first
// position is <= KV_FF_D + 1 ("head" quads, positions 1..A, A <= KV_FF_D + 4 = 31) are kept
// apart from the rest, so the head positions are the only ones needing one lane each.
#define KV_FF_D 27

// max over u in [1, w] of Prof(t+u) + u: ma over the head quads (positions <= A), mb over
// the rest; 0 if empty.  Four rounds per lane (one 8-byte shared load, two 16x2 adds, 128
// rounds per warp pass); returns A, the last position of the head quads.
__device__ __forceinline__ int r16_window_max(const R16 &R, int t, int w, int &ma, int &mb)
{
    const int lane = lane_id();
    uint32_t acc_a = 0u, acc_b = 0u;
    const int Q0 = (t + 1) >> 2, Q1 = (t + w) >> 2;
    // warp-uniform masks of the first quad (rounds <= t) and the last quad (rounds > t+w)
    const unsigned long long fm = ~0ull << (16 * ((t + 1) & 3));
    const unsigned long long em = ~0ull >> (16 * (3 - ((t + w) & 3)));
    for (int q = Q0 + lane; q <= Q1; q += 32) {
        const uint2 v = R.q[q & R.qmask];
        const int u0 = 4 * q - t;                       // -2..1 on the first quad
        uint32_t z0 = __vadd2(v.x, ((uint32_t)u0 & 0xffffu) | ((uint32_t)(u0 + 1) << 16));
        uint32_t z1 = __vadd2(v.y, ((uint32_t)(u0 + 2) & 0xffffu) | ((uint32_t)(u0 + 3) << 16));
        if (q == Q0) { z0 &= (uint32_t)fm; z1 &= (uint32_t)(fm >> 32); }
        if (q == Q1) { z0 &= (uint32_t)em; z1 &= (uint32_t)(em >> 32); }
        const uint32_t z = __vmaxu2(z0, z1);
        if (u0 <= KV_FF_D + 1) acc_a = __vmaxu2(acc_a, z);
        else acc_b = __vmaxu2(acc_b, z);
    }
    ma = (int)__reduce_max_sync(KV_FULL, max(acc_a & 0xffffu, acc_a >> 16));
    mb = (int)__reduce_max_sync(KV_FULL, max(acc_b & 0xffffu, acc_b >> 16));
    const int qa = (t + KV_FF_D + 1) >> 2;              // quad holding position KV_FF_D + 1
    return 4 * qa - t + 3;
}

// First offset D in [1, KV_FF_D] at which (s, w) fits while the profile only advances,
// KV_FF_D + 1 if none; the caller knows D = 0 fails.  mb = max Prof(t+u)+u over the window
// positions A+1..w (A from r16_window_max, KV_FF_D + 1 <= A <= KV_FF_D + 4).  Needs
// w + KV_FF_D <= L.
__device__ __forceinline__ int r16_first_fit(const R16 &R, int t, int w, int room, int A, int mb)
{
    const int lane = lane_id();
    uint32_t cov = 0u;
    const uint32_t all = 0xffffffffu >> (31 - KV_FF_D);
    const int gb = mb - room - 1;                          // positions A+1..w block [0, gb]
    if (gb >= 0) cov = gb >= KV_FF_D ? all : (0xffffffffu >> (31 - gb));
    if (lane < A) {
        const int ua = lane + 1;                           // head positions 1..A
        const int v = R.p[(t + ua) & R.mask];
        const int lo = max(ua - w, 0), hi = min(min(ua - 1, v + ua - room - 1), KV_FF_D);
        if (hi >= lo) cov |= (0xffffffffu >> (31 - hi)) & (0xffffffffu << lo);
    }
    const int uc = max(A, w) + 1 + lane;                   // positions max(A, w)+1 .. w+KV_FF_D
    if (uc <= w + KV_FF_D) {
        const int v = R.p[(t + uc) & R.mask];
        const int lo = uc - w, hi = min(v + uc - room - 1, KV_FF_D);
        if (hi >= lo) cov |= (0xffffffffu >> (31 - hi)) & (0xffffffffu << lo);
    }
    cov = __reduce_or_sync(KV_FULL, cov);
    return cov == all ? KV_FF_D + 1 : __ffs(~cov) - 1;
}

__device__ __forceinline__ int r16_at(const R16 &R, const LongList &G, int t, int u)
{
    const int far = G.used ? long_prof(G, t + u) : 0;
    return u <= R.L ? (int)R.p[(t + u) & R.mask] : far;
}

// Per-position path for windows past the ring (w + 31 > L): the Eq. 5 test at D = 0 and,
// when multi, the first fit over D in [0, 31] (kernel_ring.cuh's ring_first_fit on R16).
__device__ __forceinline__ int r16_fit_slow(const R16 &R, const LongList &G, int t, int s, int w, int M, bool multi)
{
    const int lane = lane_id();
    const int room = M - s;
    const int span = multi ? w + 31 : w;
    uint32_t cov = 0u;
    for (int base = 1; base <= span; base += 32) {
        const int u = base + lane;
        const int v = r16_at(R, G, t, u);
        if (u <= span) {
            const int lo = max(u - w, 0);
            const int hi = min(min(u - 1, v + u - room - 1), 31);
            if (hi >= lo) cov |= (0xffffffffu >> (31 - hi)) & (0xffffffffu << lo);
        }
    }
    cov = __reduce_or_sync(KV_FULL, cov);
    if (!multi) return cov & 1u ? 1 : 0;
    return cov == KV_FULL ? 32 : __ffs(~cov) - 1;
}

// Prof(t+u) += s + u for u in [1, min(w, L)] (four rounds per lane: one 8-byte load/store;
// a halfword never carries: the sum is <= M, certified by the Eq. 5 test)
__device__ __forceinline__ void r16_ramp(const R16 &R, int t, int w, int s)
{
    const int e = min(w, R.L);
    const int Q0 = (t + 1) >> 2, Q1 = (t + e) >> 2;
    const unsigned long long fm = ~0ull << (16 * ((t + 1) & 3));
    const unsigned long long em = ~0ull >> (16 * (3 - ((t + e) & 3)));
    for (int q = Q0 + lane_id(); q <= Q1; q += 32) {
        const int u0 = 4 * q - t;
        const int b = s + u0;
        uint32_t a0 = ((uint32_t)b & 0xffffu) | ((uint32_t)(b + 1) << 16);
        uint32_t a1 = ((uint32_t)(b + 2) & 0xffffu) | ((uint32_t)(b + 3) << 16);
        if (q == Q0) { a0 &= (uint32_t)fm; a1 &= (uint32_t)(fm >> 32); }
        if (q == Q1) { a0 &= (uint32_t)em; a1 &= (uint32_t)(em >> 32); }
        uint2 v = R.q[q & R.qmask];
        v.x += a0;
        v.y += a1;
        R.q[q & R.qmask] = v;
    }
}

// ring_jump (kernel_ring.cuh) on the 16-bit ring: window start t -> tn, returns max Prof(r)
// over r in [t+1, E]; slots leaving the window are re-initialised from the long list.
__device__ __forceinline__ int r16_jump(const R16 &R, LongList &G, int t, int E, int tn)
{
    const int lane = lane_id();
    if (tn == t + 1 && E == tn && !G.used) {            // the common single-round advance
        const int slot = tn & R.mask;
        const int v = R.p[slot];
        __syncwarp();
        if (lane == 0) R.p[slot] = 0;
        __syncwarp();
        return v;
    }
    const int L = R.L, mask = R.mask;
    int v = 0;
    const int dn = max(min(E - t, L), 0);
    for (int base = 1; base <= dn; base += 32) {
        const int tau = base + lane;
        if (tau <= dn) v = max(v, (int)R.p[(t + tau) & mask]);
    }
    if (G.used && E - t > L) {
        const bool own = ((G.used >> lane) & 1u) && G.e > t + L && G.e <= E;
        v = max(v, long_prof(G, own ? G.e : E));
    }
    __syncwarp();
    if (tn - t <= L) {
        for (int base = 1; base <= tn - t; base += 32) {
            const int tau = base + lane;
            const int far = G.used ? long_prof(G, t + tau + L) : 0;
            if (tau <= tn - t) R.p[(t + tau) & mask] = (uint16_t)far;
        }
    } else {
        for (int j0 = 0; j0 < L; j0 += 32) {
            const int j = j0 + lane;
            const int r = tn + 1 + ((j - (tn + 1)) & mask);
            const int far = G.used ? long_prof(G, r) : 0;
            R.p[j] = (uint16_t)far;
        }
    }
    if (G.used) G.used &= ~__ballot_sync(KV_FULL, ((G.used >> lane) & 1u) && G.e <= tn + L);
    __syncwarp();
    return warp_max_i32(v);
}

__host__ __device__ inline int mcring_warp_bytes(int L, int NP)
{
    const int b = KV_STAGE_SLOTS * 8 + KV_STAGE_SLOTS * KV_STAGE_ENTRIES * 8 + L * 2 + (NP / 32) * 4 + 32 * 4;
    return (b + 15) & ~15;
}

// Work estimate of an instance for longest-first claiming (rounds ~ the larger of the
// arrival span and the volume the budget must carry; plus one admission per request)
__device__ __forceinline__ uint32_t work_estimate(int a0, int alast, long long vol, int M, int n)
{
    const long long r = max((long long)alast - a0, vol / max(M, 1)) + n;
    return (uint32_t)min(r + 1, 0xffffffffll);
}

// The MC-SF keys (o~ << 15 | idx) of one instance sorted in place in shared memory by a CUB
// block radix sort on the o~ bits only (stable, so ties stay in idx order, P:175 / Q5):
// ceil(bits / 4) passes instead of the bitonic network's log2(NP) (log2(NP) + 1) / 2 stages
// with a block barrier each.  Blocked arrangement: thread t holds keys t IT .. t IT + IT - 1.
template <int BLOCK, int IT>
using PrepSort = cub::BlockRadixSort<uint32_t, BLOCK, IT>;
constexpr size_t kPrepSortBytes = sizeof(typename PrepSort<1024, 16>::TempStorage);      // 1024 threads
constexpr size_t kPrepSortBytes256 = sizeof(typename PrepSort<256, 4>::TempStorage);     // 256 threads

template <int BLOCK, int IT>
__device__ __forceinline__ void prep_radix_sort(uint32_t *keys, int n, int max_len, void *tmp)
{
    const int tid = threadIdx.x;
    uint32_t k[IT];
#pragma unroll
    for (int j = 0; j < IT; ++j) {
        const int i = tid * IT + j;
        k[j] = i < n ? keys[i] : 0xffffffffu;        // padding sorts last (stable: after ties)
    }
    __syncthreads();
    const int eb = min(32, 15 + (32 - __clz(max(max_len, 1))));
    PrepSort<BLOCK, IT>(*reinterpret_cast<typename PrepSort<BLOCK, IT>::TempStorage *>(tmp)).Sort(k, 15, eb);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IT; ++j) keys[tid * IT + j] = k[j];
    __syncthreads();
}

// ---------------------------------------------------------------------------------------
// k_mc_prep: validation, round cap, ranks, the rq8 / arr8 streams (one CTA per instance)
// ---------------------------------------------------------------------------------------
// BLOCK = 1024 takes the instances with more than 1024 requests; BLOCK = 256 those with
// n_lo < n <= 1024 (a CTA radix sort instead of k_mc_prep_w's warp bitonic network).
template <int POL, int BLOCK = 1024>
__global__ void __launch_bounds__(BLOCK) k_mc_prep(const KParams P, uint4 *rq_early, int *arank_early, int n_lo = 0)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(smem_raw);
    __shared__ int s_flags;                 // bit 0 invalid, bit 1 unsupported, bit 2 o~ != o
    __shared__ unsigned long long s_sumo, s_vol;
    const int tid = threadIdx.x, lane = tid & 31;
    const int *reqi = reinterpret_cast<const int *>(P.req);
    for (long long inst = blockIdx.x; inst < P.n_inst; inst += gridDim.x) {
        const long long off = P.offset[inst] - P.row_base;
        const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
        // another prep's instance (instances above the caller's size hint are k_mc_prep_w's:
        // the launches are sized from the hint)
        if ((BLOCK == 1024 ? n <= KV_PREP_WARP_N : (n <= n_lo || n > KV_PREP_WARP_N)) || n > P.max_requests) continue;
        const int M = P.mem[inst];
        if (tid == 0) {
            s_flags = (n > P.max_requests || M > P.max_mem || off + n > P.scratch_rows) ? 2 : 0;
            s_sumo = 0ull;
            s_vol = 0ull;
        }
        __syncthreads();
        int fl = 0;
        long long so = 0, vol = 0;
        if (!(s_flags & 2)) {
            for (int k = tid; k < n; k += blockDim.x) {
                const int4 r = P.req[off + k];
                bool bad = r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1;
                if (k > 0) bad |= reqi[(off + k - 1) * 4] > r.x;
                if (POL == POL_MCSF) {
                    bad |= (long long)r.y + r.w > M || r.w < r.z;
                    if (r.w != r.z) fl |= 4;
                } else {
                    bad |= (long long)r.y + r.z > M;
                }
                if (r.z > P.max_len || (POL == POL_MCSF && r.w > P.max_len)) fl |= 2;
                if (bad) fl |= 1;
                so += r.z;
                vol += (long long)r.y * r.z + (long long)r.z * (r.z + 1) / 2;
                if (POL == POL_MCSF) keys[k] = ((uint32_t)min(max(r.w, 0), 0x1ffff) << 15) | (uint32_t)k;
            }
        }
        fl = __reduce_or_sync(KV_FULL, fl);
        so = warp_sum_i64(so);
        vol = warp_sum_i64(vol);
        if (lane == 0) {
            if (fl) atomicOr(&s_flags, fl);
            if (so) atomicAdd(&s_sumo, (unsigned long long)so);
            if (vol) atomicAdd(&s_vol, (unsigned long long)vol);
        }
        __syncthreads();
        const int flags = s_flags;
        const long long sumo = (long long)s_sumo;
        int capv = -1;
        if (flags & 3) {                                    // INVALID / UNSUPPORTED
            for (int k = tid; k < n; k += blockDim.x) {
                if (P.completion) P.completion[off + k] = -1;
                if (P.start) P.start[off + k] = -1;
            }
            if (tid < 32) write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, (flags & 2) ? ST_UNSUPPORTED : ST_INVALID});
        } else if (n == 0) {
            if (tid < 32) write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, ST_OK});
        } else if (POL == POL_MCSF && (flags & 4) && !P.early_list) {
            for (int k = tid; k < n; k += blockDim.x) {
                if (P.completion) P.completion[off + k] = -1;
                if (P.start) P.start[off + k] = -1;
            }
            if (tid < 32) write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, ST_UNSUPPORTED});
        } else {
            const int NPr = next_pow2(n);
            if (POL == POL_MCSF && KV_PREP_RADIX && BLOCK == 1024 && NPr >= 2048 && NPr <= 16384) {   // block radix sort
                void *tmp = smem_raw + (size_t)P.NP * 4;
                if (NPr == 2048) prep_radix_sort<BLOCK, 2>(keys, n, P.max_len, tmp);
                else if (NPr == 4096) prep_radix_sort<BLOCK, 4>(keys, n, P.max_len, tmp);
                else if (NPr == 8192) prep_radix_sort<BLOCK, 8>(keys, n, P.max_len, tmp);
                else prep_radix_sort<BLOCK, 16>(keys, n, P.max_len, tmp);
            } else if (POL == POL_MCSF && BLOCK == 256 && NPr >= 256 && NPr <= 1024) {
                void *tmp = smem_raw + (size_t)P.NP * 4;
                if (NPr == 256) prep_radix_sort<256, 1>(keys, n, P.max_len, tmp);
                else if (NPr == 512) prep_radix_sort<256, 2>(keys, n, P.max_len, tmp);
                else prep_radix_sort<256, 4>(keys, n, P.max_len, tmp);
            } else if (POL == POL_MCSF) {                   // bitonic sort of (o~, idx) keys
                const int NPi = next_pow2(n);
                for (int k = n + tid; k < NPi; k += blockDim.x) keys[k] = 0xffffffffu;
                __syncthreads();
                for (int k = 2; k <= NPi; k <<= 1) {
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        for (int i = tid; i < (NPi >> 1); i += blockDim.x) {
                            const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                            const int hi = lo + j;
                            const bool up = (lo & k) == 0;
                            const uint32_t x = keys[lo], y = keys[hi];
                            if ((x > y) == up) { keys[lo] = y; keys[hi] = x; }
                        }
                        __syncthreads();
                    }
                }
            }
            if (POL == POL_MCSF && (flags & 4)) {
                // o~ > o somewhere: protected MC-SF with alpha = 0 (k_prot) reads {s, o~, o, idx}
                // per rank and the rank of each idx
                for (int r = tid; r < n; r += blockDim.x) {
                    const int idx = (int)(keys[r] & 0x7fffu);
                    const int4 q = P.req[off + idx];
                    rq_early[off + r] = make_uint4((uint32_t)q.y, (uint32_t)q.w, (uint32_t)q.z, (uint32_t)idx);
                    arank_early[off + idx] = r;
                }
                if (tid == 0) P.early_list[atomicAdd(P.early_count, 1ull)] = inst;
            } else {
                for (int r = tid; r < n; r += blockDim.x) {
                    const int idx = POL == POL_MCSF ? (int)(keys[r] & 0x7fffu) : r;
                    const int4 q = P.req[off + idx];
                    const int w = POL == POL_MCSF ? q.w : q.z;      // MC-SF: o~ = o here
                    P.rq8[off + r] = make_uint2((uint32_t)q.y | ((uint32_t)w << 16), (uint32_t)idx);
                    P.arr8[off + idx] = make_int2(q.x, r);
                }
                const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(reqi[(off + n - 1) * 4], sumo);
                capv = (int)min(cap64, 0x7ffffffell);
            }
        }
        if (tid == 0) {
            P.capv[inst] = capv;
            if (P.estv) P.estv[inst] = capv < 0 ? 0u : work_estimate(reqi[off * 4], reqi[(off + n - 1) * 4],
                                                                     (long long)s_vol, M, n);
        }
        __syncthreads();
    }
}

// k_mc_prep_w: the same for instances of at most KV_PREP_WARP_N requests, one warp each
// (keys in 4 KB of shared memory per warp, the bitonic stages separated by __syncwarp
// instead of block barriers); k_mc_prep then takes only the larger instances.
template <int POL>
__global__ void __launch_bounds__(256) k_mc_prep_w(const KParams P, uint4 *rq_early, int *arank_early,
                                                   int n_hi = KV_PREP_WARP_N)
{
    __shared__ __align__(16) uint32_t keys_all[8][KV_PREP_WARP_N];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t *keys = keys_all[warp];
    const int *reqi = reinterpret_cast<const int *>(P.req);
    const long long nwarps = (long long)gridDim.x * 8;
    for (long long inst = (long long)blockIdx.x * 8 + warp; inst < P.n_inst; inst += nwarps) {
        const long long off = P.offset[inst] - P.row_base;
        const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
        if (n > n_hi && n <= P.max_requests) continue;     // k_mc_prep (hint violators: here)
        const int M = P.mem[inst];
        int fl = (n > P.max_requests || M > P.max_mem || off + n > P.scratch_rows) ? 2 : 0;
        long long so = 0, vol = 0;
        if (!fl) {
            int carry = 0;                                 // a of row k0 - 1
            for (int k0 = 0; k0 < n; k0 += 32) {
                const int k = k0 + lane;
                const int4 r = k < n ? P.req[off + k] : make_int4(0x7fffffff, 1, 1, 1);
                int prev = __shfl_up_sync(KV_FULL, r.x, 1);
                if (lane == 0) prev = carry;
                carry = __shfl_sync(KV_FULL, r.x, 31);
                if (k < n) {
                    bool bad = r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1 || (k > 0 && prev > r.x);
                    if (POL == POL_MCSF) {
                        bad |= (long long)r.y + r.w > M || r.w < r.z;
                        if (r.w != r.z) fl |= 4;
                    } else {
                        bad |= (long long)r.y + r.z > M;
                    }
                    if (r.z > P.max_len || (POL == POL_MCSF && r.w > P.max_len)) fl |= 2;
                    if (bad) fl |= 1;
                    so += r.z;
                    vol += (long long)r.y * r.z + (long long)r.z * (r.z + 1) / 2;
                    if (POL == POL_MCSF) keys[k] = ((uint32_t)min(max(r.w, 0), 0x1ffff) << 15) | (uint32_t)k;
                }
            }
        }
        fl = __reduce_or_sync(KV_FULL, fl);
        so = warp_sum_i64(so);
        vol = warp_sum_i64(vol);
        int capv = -1;
        if (fl & 3) {
            for (int k = lane; k < n; k += 32) {
                if (P.completion) P.completion[off + k] = -1;
                if (P.start) P.start[off + k] = -1;
            }
            write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, (fl & 2) ? ST_UNSUPPORTED : ST_INVALID});
        } else if (n == 0) {
            write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, ST_OK});
        } else if (POL == POL_MCSF && (fl & 4) && !P.early_list) {
            for (int k = lane; k < n; k += 32) {
                if (P.completion) P.completion[off + k] = -1;
                if (P.start) P.start[off + k] = -1;
            }
            write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, ST_UNSUPPORTED});
        } else {
            // (a CUB warp merge sort in place of the bitonic network measured the same on C4,
            // 0.82 ms: the sort is not what bounds this kernel)
            if (POL == POL_MCSF) {
                const int NPi = next_pow2(max(n, 2));
                for (int k = n + lane; k < NPi; k += 32) keys[k] = 0xffffffffu;
                __syncwarp();
                for (int k = 2; k <= NPi; k <<= 1) {
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        for (int i = lane; i < (NPi >> 1); i += 32) {
                            const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                            const int hi = lo + j;
                            const bool up = (lo & k) == 0;
                            const uint32_t x = keys[lo], y = keys[hi];
                            if ((x > y) == up) { keys[lo] = y; keys[hi] = x; }
                        }
                        __syncwarp();
                    }
                }
            }
            if (POL == POL_MCSF && (fl & 4)) {
                for (int r = lane; r < n; r += 32) {
                    const int idx = (int)(keys[r] & 0x7fffu);
                    const int4 q = P.req[off + idx];
                    rq_early[off + r] = make_uint4((uint32_t)q.y, (uint32_t)q.w, (uint32_t)q.z, (uint32_t)idx);
                    arank_early[off + idx] = r;
                }
                if (lane == 0) P.early_list[atomicAdd(P.early_count, 1ull)] = inst;
            } else {
                for (int r = lane; r < n; r += 32) {
                    const int idx = POL == POL_MCSF ? (int)(keys[r] & 0x7fffu) : r;
                    const int4 q = P.req[off + idx];
                    const int w = POL == POL_MCSF ? q.w : q.z;
                    P.rq8[off + r] = make_uint2((uint32_t)q.y | ((uint32_t)w << 16), (uint32_t)idx);
                    P.arr8[off + idx] = make_int2(q.x, r);
                }
                const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(reqi[(off + n - 1) * 4], so);
                capv = (int)min(cap64, 0x7ffffffell);
            }
        }
        if (lane == 0) {
            P.capv[inst] = capv;
            if (P.estv) P.estv[inst] = capv < 0 ? 0u : work_estimate(reqi[off * 4], reqi[(off + n - 1) * 4], vol, M, n);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// k_mc_ring: the round loop
// ---------------------------------------------------------------------------------------
// QREG (instances of at most 1024 requests): the waiting queue is one bitmap word per lane in
// a register (lane l: ranks 32l .. 32l+31) instead of the two-level shared-memory bitmap;
// arrivals stage their bits through smq (shared atomics) and each lane folds its word in.
template <int POL, bool QREG>
__device__ void mcring_instance(const KParams &P, long long inst, const R16 &R, uint32_t *bm, uint32_t *smq,
                                Stage &A)
{
    const int lane = lane_id();
    const int cap = P.capv[inst];
    if (cap < 0) return;                                   // handled by k_mc_prep / k_prot
    const long long off = P.offset[inst] - P.row_base;
    const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
    const int M = P.mem[inst];
    const int L = R.L;
    const uint2 *rq8 = P.rq8 + off;

    const int NPi = next_pow2(max(n, 32));
    const int nw = NPi >> 5;
    for (int i = lane; i < (L >> 2); i += 32) R.q[i] = make_uint2(0u, 0u);
    for (int w = lane; w < nw; w += 32) bm[w] = 0u;
    smq[lane] = 0u;
    __syncwarp();
    WarpQueue Q{bm, smq, (nw + 31) >> 5};
    uint32_t qw = 0u, qhw = 0u;                            // QREG: this lane's word, the head's word
    stage_begin(A, P.arr8, off, n);
    const bool multi = !(P.flags & 1);

    long long suma = 0;
    int2 e0;
    stage_need(A, 0, 0);
    e0 = stage_get(A, 0);
    int t = e0.x;
    int next = 0, a_next = t;
    int h = KV_INF;
    uint2 he = make_uint2(0u, 0u);                         // head entry {s | w << 16, idx}
    bool hstale = false, head_fits = false;
    long long sumc = 0;
    int rounds = 0, drounds = 0, maxc = -1, peak = 0, status = ST_OK;
    LongList G;
    G.p = G.s = G.e = G.idx = 0;
    G.used = 0u;

    for (;;) {
        if (h == KV_INF) {
            if (a_next == KV_INF) {                        // drain
                const int E = min(maxc, cap + 1);
                if (E > t) peak = max(peak, r16_jump(R, G, t, E, t));
                if (maxc > t) rounds += maxc - t;
                if (maxc >= cap + 1) status = ST_LIVELOCK;
                break;
            }
            const int tn = a_next;
            if (tn > t) {                                  // skip rounds t..tn-1
                const int E = min(tn, cap + 1);
                peak = max(peak, r16_jump(R, G, t, E, tn));
                rounds += max(0, min(tn, maxc) - t);
                if (tn > cap) { status = ST_LIVELOCK; break; }
                t = tn;
            }
        }
        if (t > cap) { status = ST_LIVELOCK; break; }

        // arrivals from the staged stream
        while (a_next <= t) {
            stage_need(A, next / KV_STAGE_CH, min(next + 31, n - 1) / KV_STAGE_CH);
            const int k = next + lane;
            const int2 e = k < n ? stage_get(A, k) : make_int2(KV_INF, KV_INF);
            const bool take = e.x <= t;
            const int cnt = __popc(__ballot_sync(KV_FULL, take));
            int rk = KV_INF;
            if (take) {
                rk = e.y;
                if (QREG) atomicOr(&smq[rk >> 5], 1u << (rk & 31));
                else q_insert(Q, rk);
                suma += e.x;
            }
            const int mn = warp_min_i32(rk);
            if (mn < h) { h = mn; hstale = true; head_fits = false; }
            if (QREG) {                                    // fold the staged bits in
                __syncwarp();
                qw |= smq[lane];
                smq[lane] = 0u;
                __syncwarp();
                qhw = __shfl_sync(KV_FULL, qw, (h >> 5) & 31);
            }
            next += cnt;
            a_next = cnt < 32 ? __shfl_sync(KV_FULL, e.x, cnt & 31) : (next < n ? t : KV_INF);
        }
        __syncwarp();

        // decision round t with R non-empty (Alg. 1 / Alg. 2)
        if (hstale) { he = rq8[h]; hstale = false; }
        int jump = 1;
        bool blocked_through = false;
        for (;;) {
            const int s = (int)(he.x & 0xffffu), w = (int)(he.x >> 16), idx = (int)he.y;
            if (!head_fits) {
                int d;
                if (w + KV_FF_D + 4 <= L) {
                    int ma, mb;
                    const int A = r16_window_max(R, t, w, ma, mb);
                    const int room = M - s;
                    d = max(ma, mb) <= room ? 0 : (multi ? r16_first_fit(R, t, w, room, A, mb) : 1);
                    if (d == KV_FF_D + 1) d = 32;          // blocked throughout: jump KV_FF_D + 1
                } else {
                    d = r16_fit_slow(R, G, t, s, w, M, multi);
                }
                if (d > 0) {                               // Eq. 5 violated
                    blocked_through = d == 32;
                    jump = blocked_through ? (w + KV_FF_D + 4 <= L ? KV_FF_D + 1 : 32) : d;
                    break;
                }
            }
            head_fits = false;
            // the next head leaves the queue first so that its entry loads while the ramp is
            // written (a RETRY restarts the instance, so the order is free; MC-Benchmark too).
            // Fusing the ramp with the next head's window pass measured slower (C4 7.47 ->
            // 8.0 ms: the pass must wait for that entry's load)
            int hn;
            if (QREG) {
                const uint32_t bit = 1u << (h & 31);
                if (lane == (h >> 5)) qw &= ~bit;
                qhw &= ~bit;
                if (qhw) {
                    hn = (h & ~31) + __ffs(qhw) - 1;       // the rest of the head's word is > h
                } else {
                    const uint32_t b = __ballot_sync(KV_FULL, qw != 0u);
                    const int l0 = b ? __ffs(b) - 1 : 0;
                    qhw = __shfl_sync(KV_FULL, qw, l0);
                    hn = b ? (l0 << 5) + __ffs(qhw) - 1 : KV_INF;
                }
            } else {
                hn = q_pop_head(Q, h);
            }
            uint2 hen = he;
            if (hn != KV_INF) hen = rq8[hn];
            r16_ramp(R, t, w, s);
            if (w > L && !long_add(G, t, s, t + w, idx)) { status = ST_RETRY; break; }
            const int c = t + w;                           // o = w on this path
            if (lane == 0) {
                if (P.completion) P.completion[off + idx] = c;
                if (P.start) P.start[off + idx] = t;
            }
            sumc += c;
            maxc = max(maxc, c);
            __syncwarp();
            h = hn;
            if (h == KV_INF) break;
            he = hen;
        }
        if (status == ST_RETRY) break;
        if (jump > 1) {
            int T = t + min(jump, cap + 1 - t);
            if (POL == POL_MCSF) {
                // an arrival before T ends the jump only if it sorts before the head
                for (int k = next; a_next < T && k < n; k += 32) {
                    const int kk = k + lane;
                    const int2 e = kk < n ? stage_get(A, kk) : make_int2(KV_INF, KV_INF);
                    const bool before = e.x < T;
                    const uint32_t m = __ballot_sync(KV_FULL, before && e.y < h);
                    if (m) { T = __shfl_sync(KV_FULL, e.x, __ffs(m) - 1); break; }
                    if (!__all_sync(KV_FULL, before)) break;
                }
            }
            head_fits = !blocked_through && T == t + jump;
            jump = T - t;
        }
        drounds += jump;
        rounds += jump;
        peak = max(peak, r16_jump(R, G, t, t + jump, t + jump));
        t += jump;
    }

    if (status == ST_RETRY) {               // rerun by the full-ring launch
        if (lane == 0) P.retry_list[atomicAdd(P.retry_count, 1ull)] = inst;
        return;
    }
    if (status != ST_OK) {
        for (int k = next + lane; k < n; k += 32) {          // not yet arrived (idx = k)
            if (P.completion) P.completion[off + k] = -1;
            if (P.start) P.start[off + k] = -1;
        }
        for (int w = lane; w < nw; w += 32) {
            uint32_t bits = QREG ? qw : bm[w];
            while (bits) {
                const int r = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                const int idx = (int)rq8[r].y;
                if (P.completion) P.completion[off + idx] = -1;
                if (P.start) P.start[off + idx] = -1;
            }
        }
    }
    InstResult res;
    res.tel = sumc - warp_sum_i64(suma);                   // suma: per lane (arrivals it took)
    res.rounds = rounds;
    res.decision_rounds = drounds;
    res.evictions = 0;
    res.makespan = maxc;
    res.peak = peak;
    res.status = status;
    write_result(P, inst, res);
}

#ifndef KV_MCRING_MINB
#define KV_MCRING_MINB 8        // blocks of 4 warps per SM the register budget must allow
#endif
template <int POL, bool QREG = false>
__global__ void __launch_bounds__(128, KV_MCRING_MINB) k_mc_ring(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + (size_t)warp * P.warp_bytes;
    Stage A;
    A.bar = reinterpret_cast<uint64_t *>(base);
    A.buf = reinterpret_cast<int2 *>(base + KV_STAGE_SLOTS * 8);
    unsigned char *rp = base + KV_STAGE_SLOTS * 8 + KV_STAGE_SLOTS * KV_STAGE_ENTRIES * 8;
    R16 R;
    R.p = reinterpret_cast<uint16_t *>(rp);
    R.q = reinterpret_cast<uint2 *>(rp);
    R.L = P.L;
    R.mask = P.L - 1;
    R.qmask = (P.L >> 2) - 1;
    uint32_t *bm = reinterpret_cast<uint32_t *>(rp + P.L * 2);
    uint32_t *smq = bm + P.NP / 32;
    if (lane == 0)
        for (int b = 0; b < KV_STAGE_SLOTS; ++b) mbar_init(&A.bar[b], 1u);
    mbar_fence_init();
    __syncwarp();
    A.phase = 0u;
    A.pend = 0u;

    const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
    long long w = 0;
    if (lane == 0) w = atomicAdd(P.counter, 1ull);
    w = __shfl_sync(KV_FULL, w, 0);
    while (w < n_work) {
        long long nxt = 0;
        if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
        mcring_instance<POL, QREG>(P, P.work_list ? P.work_list[w] : w, R, bm, smq, A);
        w = __shfl_sync(KV_FULL, nxt, 0);
        __syncwarp();
    }
    // no copy may still be writing this warp's shared memory when the block exits
    for (int b = 0; b < KV_STAGE_SLOTS; ++b)
        if ((A.pend >> b) & 1u) stage_wait_slot(A, b);
}

}  // namespace kv
