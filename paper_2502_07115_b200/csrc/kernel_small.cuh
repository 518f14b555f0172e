// kernel_small.cuh -- fused MC-SF / MC-Benchmark simulator for budgets M <= 64.
//
// One warp simulates one instance at a time on a persistent grid.  Everything the round
// loop touches lives on chip:
//   * projected memory profile Prof(t+tau), tau = 1..64, in registers: lane l holds
//     tau = l+1 (P0) and tau = l+33 (P1).  Prof is the left-hand side of Eq. 5
//     for the in-flight set S, so a candidate (s, w) is admissible at round t iff
//         Prof(t+tau) + s + tau <= M  for every tau in [1, w].
//     With o~ >= o the profile beyond a candidate's own window is already feasible (every
//     earlier admission certified its window), so these are exactly the t' in
//     [t+1, t_max(U + {i})] of Eq. 5.  Admission adds the ramp s + tau (Eq. 3);
//     advancing the clock is a shuffle.
//   * the waiting queue R^(t): a bitmap over ranks, one 32-bit word per lane for up to
//     1024 ranks (else a two-level bitmap in shared memory); rank = position in (o~, idx)
//     order for MC-SF (Alg. 1 "ascending order of predicted output length") or idx
//     for MC-Benchmark (arrival order).  MC-SF ranks come from a stable warp
//     counting sort on o~ (<= 63), once per instance.
//   * packed per-request words {o~:6 | idx:14 | s:6 | o:6} by rank, arrivals a by idx,
//     and start rounds p by idx; completions and starts are written to HBM once, coalesced,
//     when the instance ends, and TEL = sum (p + o - a) is reduced in that pass.
// The admission loop walks the queue head in rank order and stops at the first failure
// (Alg. 1 "Break the for loop"): the longest feasible prefix of Eq. 6.
//
// Exact fast paths (DESIGN "Exact fast paths"):
//   * rounds with an empty queue are not iterated: the clock jumps to the next arrival and
//     the skipped rounds' occupancy is read off the profile;
//   * a queue head that fails Eq. 5 keeps failing -- and, by the break rule, blocks every
//     other request -- until the profile has drained enough, a request that sorts before it
//     arrives, or (o~ > o) a request completes early.  first_fit_offset() evaluates Eq. 5
//     for the head at all of the next 64 rounds in one warp pass, and the loop advances
//     straight to the first round at which something can change.  Every skipped round is a
//     decision round whose outcome ("admit nothing") was evaluated, so decision_rounds,
//     peak memory and all outputs equal the one-round-at-a-time loop's
//     (SCHED_FLAG_PER_ROUND runs that loop instead).
// With o~ > o (early completion) a request leaves S before its projected window
// ends; its unused tail is removed from the profile at completion (Eq. 5 sums over the
// requests still in progress).
#pragma once
#include "params.cuh"

#ifndef KV_SMALL_MIN_BLOCKS
#define KV_SMALL_MIN_BLOCKS 9
#endif

namespace kv {

struct SmallSmem {
    uint32_t *keys;      // [NP] packed words by rank (MC-Benchmark: rank = idx)
    uint32_t *kidx;      // [NP] packed words by idx (MC-SF, before ranking)
    int *arr;            // [NP] a by idx
    int *pst;            // [NP] start round p by idx, -1 = not started
    uint16_t *arank;     // [NP] rank of idx (MC-SF)
    uint32_t *bm;        // [NP/32] shared-memory queue words (NP > 1024)
    uint32_t *sm;        // [32] queue summary (NP > 1024) / insert staging (NP <= 1024)
    int *hist;           // [64] o~ histogram / running bucket offsets (MC-SF)
};

__host__ __device__ inline int small_warp_bytes(int NP)
{
    int b = NP * 18 + (NP / 32) * 4 + 32 * 4 + 64 * 4;
    return (b + 15) & ~15;
}

// ---------------------------------------------------------------------------------------
// waiting queue, register version: lane l holds bitmap word l (ranks 32l .. 32l+31)
// ---------------------------------------------------------------------------------------
struct RegQueue {
    uint32_t word;
    uint32_t hw;         // warp-uniform copy of the word holding the head (after first())
    uint32_t *stage;     // [32] shared staging words for inserts

    __device__ __forceinline__ void init(uint32_t *st, uint32_t *, int)
    {
        stage = st;
        word = 0u;
        stage[lane_id()] = 0u;
        __syncwarp();
    }
    __device__ __forceinline__ void insert(bool take, int r)
    {
        if (take) atomicOr(&stage[r >> 5], 1u << (r & 31));
    }
    __device__ __forceinline__ void flush()
    {
        __syncwarp();
        word |= stage[lane_id()];
        stage[lane_id()] = 0u;
        __syncwarp();
    }
    // re-read the head's word after inserts (the head is the smallest rank, h != KV_INF)
    __device__ __forceinline__ void refresh(int h) { hw = __shfl_sync(KV_FULL, word, h >> 5); }
    __device__ __forceinline__ int first()
    {
        const uint32_t b = __ballot_sync(KV_FULL, word != 0u);
        if (b == 0u) return KV_INF;
        const int l0 = __ffs(b) - 1;
        hw = __shfl_sync(KV_FULL, word, l0);
        return (l0 << 5) + __ffs(hw) - 1;
    }
    // remove the head h (the smallest rank); the next head is usually in the same word
    __device__ __forceinline__ int pop(int h)
    {
        const uint32_t bit = 1u << (h & 31);
        if (lane_id() == (h >> 5)) word &= ~bit;
        hw &= ~bit;
        if (hw != 0u) return (h & ~31) + __ffs(hw) - 1;
        return first();
    }
};

// waiting queue, shared-memory version (two-level bitmap, up to 32768 ranks)
struct SmemQueue {
    WarpQueue q;

    __device__ __forceinline__ void init(uint32_t *sm, uint32_t *bm, int nw)
    {
        for (int w = lane_id(); w < nw; w += 32) bm[w] = 0u;
        sm[lane_id()] = 0u;
        __syncwarp();
        q = WarpQueue{bm, sm, (nw + 31) >> 5};
    }
    __device__ __forceinline__ void insert(bool take, int r)
    {
        if (take) q_insert(q, r);
    }
    __device__ __forceinline__ void flush() { __syncwarp(); }
    __device__ __forceinline__ void refresh(int) {}
    __device__ __forceinline__ int first() { return q_first(q); }
    __device__ __forceinline__ int pop(int h) { return q_pop_head(q, h); }
};

// ---------------------------------------------------------------------------------------
// register profile helpers
// ---------------------------------------------------------------------------------------
// shift the register profile so that tau' = tau - d (d >= 1)
__device__ __forceinline__ void prof_shift(int &P0, int &P1, int d)
{
    const int lane = lane_id();
    if (d > 64) d = 64;
    const int j0 = lane + d, j1 = lane + 32 + d;
    const int a0 = __shfl_sync(KV_FULL, P0, j0 & 31);
    const int b0 = __shfl_sync(KV_FULL, P1, j0 & 31);
    const int b1 = __shfl_sync(KV_FULL, P1, j1 & 31);
    P0 = j0 < 32 ? a0 : (j0 < 64 ? b0 : 0);
    P1 = j1 < 64 ? b1 : 0;
}

__device__ __forceinline__ void prof_shift1(int &P0, int &P1)
{
    const int lane = lane_id();
    const int p10 = __shfl_sync(KV_FULL, P1, 0);
    const int n0 = __shfl_down_sync(KV_FULL, P0, 1);
    const int n1 = __shfl_down_sync(KV_FULL, P1, 1);
    P0 = lane == 31 ? p10 : n0;
    P1 = lane == 31 ? 0 : n1;
}

// this lane's share of max Prof(t+tau) over tau in [1, d] (the warp maximum is taken once,
// when the instance ends)
__device__ __forceinline__ int prof_max_lane(int P0, int P1, int d)
{
    const int lane = lane_id();
    const int v = (lane + 1 <= d) ? P0 : 0;
    return max(v, (lane + 33 <= d) ? P1 : 0);
}

// First round offset D >= 0 at which a head candidate (s, w) satisfies Eq. 5 while the
// profile only advances (no admission, arrival or early completion in between).  Profile
// position u = D + tau (tau in [1, w]) rules out the offsets D in [u-w, u-1] for which
// Prof(u) + s + (u - D) > M, i.e. D <= Prof(u) + u - (M-s) - 1: an interval.  The union
// of the intervals of the 64 positions the warp holds is an OR-reduction of bit masks,
// and the answer is its first zero bit.  Offsets 0..31 are resolved first (one 32-bit
// reduction); 32..63 only when all of those are blocked.  Prof is zero beyond tau = 63
// (o~ <= 63), so the head fits by D = 64 at the latest.
// bits [lo, hi] of a 32-bit word, relative to `base`, clipped to [0, 31]: 2^(hi+1) - 2^lo
// with clamped funnel shifts (2^32 -> 0); empty when hi < lo
__device__ __forceinline__ unsigned pow2c(int k) { return __funnelshift_lc(0u, 1u, (unsigned)k); }

__device__ __forceinline__ unsigned interval_bits(int lo, int hi, int base)
{
    lo = max(lo - base, 0);
    const int e = min(max(hi + 1 - base, lo), 32);
    return pow2c(e) - pow2c(lo);
}

__device__ __forceinline__ int first_fit_offset(int P0, int P1, int s, int w, int M)
{
    const int lane = lane_id();
    const int room = M - s;
    const int u0 = lane + 1, u1 = lane + 33;
    const int lo0 = u0 - w, hi0 = min(u0 - 1, P0 + u0 - room - 1);
    const int lo1 = u1 - w, hi1 = min(u1 - 1, P1 + u1 - room - 1);
    const unsigned c0 = __reduce_or_sync(KV_FULL, interval_bits(lo0, hi0, 0) | interval_bits(lo1, hi1, 0));
    if (c0 != 0xffffffffu) return __ffs(~c0) - 1;
    const unsigned c1 = __reduce_or_sync(KV_FULL, interval_bits(lo0, hi0, 32) | interval_bits(lo1, hi1, 32));
    return c1 != 0xffffffffu ? 32 + __ffs(~c1) - 1 : 64;
}

// ---------------------------------------------------------------------------------------
// The round loop and the outputs of one instance; SLOW = some request has o~ > o (early
// completions, MC-SF only), specialised so the o~ = o hot path carries none of it.
template <int POL, bool MULTI, class Queue, bool SLOW>
__device__ __forceinline__ void small_run(const KParams &P, long long inst, const SmallSmem &S, long long off,
                                          int n, int M, long long suma, long long sumo)
{
    const int lane = lane_id();
    InstResult res{0, 0, 0, 0, 0, 0, ST_OK};
    constexpr bool slow = SLOW;
    Queue Q;
    Q.init(S.sm, S.bm, (next_pow2(max(n, 32)) + 31) >> 5);

    const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(S.arr[n - 1], sumo);
    const int cap = (int)min(cap64, 0x7ffffffell);

    // ---- round loop --------------------------------------------------------------------
    int t = S.arr[0];
    int next = 0, a_next = S.arr[0];
    int h = KV_INF;                  // queue head (rank), KV_INF = R empty
    uint32_t hkey = 0u;
    bool hstale = false;
    bool head_fits = false;          // the head's first-fit round was computed and reached
    int P0 = 0, P1 = 0;              // Prof(t+lane+1), Prof(t+lane+33)
    int rounds = 0, drounds = 0;     // rounds: non-idle rounds that were not decision rounds
    int maxc = -1, peak = 0, status = ST_OK;   // peak: per-lane partial maximum
    // early-completion records (slow mode): one lane per in-flight request with o~ > o
    int rc = KV_INF, rs = 0, rp = 0, rw = 0;

    for (;;) {
        if (h == KV_INF) {
            if (!slow) {
                if (a_next == KV_INF) {                       // drain: S only, no arrivals
                    const int E = min(maxc, cap + 1);
                    if (E > t) peak = max(peak, prof_max_lane(P0, P1, min(E - t, 64)));
                    if (maxc > t) rounds += maxc - t;
                    if (maxc >= cap + 1) status = ST_LIVELOCK;
                    break;
                }
                const int tn = a_next;
                if (tn > t) {                                 // skip rounds t..tn-1
                    const int E = min(tn, cap + 1);
                    if (E > t) peak = max(peak, prof_max_lane(P0, P1, min(E - t, 64)));
                    rounds += max(0, min(tn, maxc) - t);
                    if (tn > cap) { status = ST_LIVELOCK; break; }
                    prof_shift(P0, P1, tn - t);
                    t = tn;
                }
            } else if (maxc < t) {                            // S empty: idle jump
                if (a_next == KV_INF) break;
                t = max(t, a_next);
            }
        }
        if (t > cap) { status = ST_LIVELOCK; break; }

        // arrivals a_i <= t join R^(t)
        if (a_next <= t) {
            do {
                const int k = next + lane;
                const int ak = k < n ? S.arr[k] : KV_INF;
                const bool take = ak <= t;
                const int cnt = __popc(__ballot_sync(KV_FULL, take));
                const int rk = take ? ((POL == POL_MCSF) ? (int)S.arank[k] : k) : KV_INF;
                Q.insert(take, rk);
                const int mn = warp_min_i32(rk);
                if (mn < h) { h = mn; hstale = true; head_fits = false; }
                next += cnt;
                a_next = cnt < 32 ? __shfl_sync(KV_FULL, ak, cnt & 31) : (next < n ? S.arr[next] : KV_INF);
            } while (a_next <= t);
            Q.flush();
            Q.refresh(h);
        }

        // early completions (o~ > o): drop the unused projected tail (slow mode only)
        if (slow) {
            uint32_t m = __ballot_sync(KV_FULL, rc == t);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int s_ = __shfl_sync(KV_FULL, rs, l), p_ = __shfl_sync(KV_FULL, rp, l);
                const int e_ = __shfl_sync(KV_FULL, rw, l) + p_ - t;     // tau in [1, e_]
                if (lane + 1 <= e_) P0 -= s_ + t + lane + 1 - p_;
                if (lane + 33 <= e_) P1 -= s_ + t + lane + 33 - p_;
                if (lane == l) rc = KV_INF;
            }
            if (h == KV_INF) {                 // R empty, S non-empty: one plain round
                if (maxc > t) ++rounds;
                if (lane == 0) peak = max(peak, P0);
                prof_shift1(P0, P1);
                ++t;
                continue;
            }
        }

        // decision round t with R non-empty (Alg. 1 / Alg. 2): candidates in rank order,
        // break at the first failure.
        if (hstale) { hkey = S.keys[h]; hstale = false; }
        int jump = 1;
        for (;;) {
            const int w = (POL == POL_MCSF) ? (int)(hkey >> 26) : (int)(hkey & 63u);
            const int s = (int)((hkey >> 6) & 63u), o = (int)(hkey & 63u);
            if (MULTI) {
                if (!head_fits) {
                    const int d = first_fit_offset(P0, P1, s, w, M);
                    if (d > 0) { jump = d; break; }                      // Eq. 5 violated now
                }
                head_fits = false;
            } else {
                const int tau0 = lane + 1, tau1 = lane + 33;
                const bool v = (tau0 <= w && P0 + s + tau0 > M) || (tau1 <= w && P1 + s + tau1 > M);
                if (__any_sync(KV_FULL, v)) break;                      // Eq. 5 violated
            }
            if (lane + 1 <= w) P0 += s + lane + 1;                       // ramp s + tau (Eq. 3)
            if (lane + 33 <= w) P1 += s + lane + 33;
            if (lane == 0) S.pst[(hkey >> 12) & 0x3fffu] = t;            // p_i = t
            maxc = max(maxc, t + o);                                     // c_i = p_i + o_i
            if (SLOW && w > o) {                                          // early completion
                const uint32_t fr = __ballot_sync(KV_FULL, rc == KV_INF);
                if (lane == __ffs(fr) - 1) { rc = t + o; rs = s; rp = t; rw = w; }
            }
            h = Q.pop(h);
            if (h == KV_INF) break;
            hkey = S.keys[h];
        }
        if (MULTI && jump > 1) {
            int T = t + min(jump, cap + 1 - t);
            if (slow) T = min(T, warp_min_i32(rc));
            // an arrival before T ends the jump only if it becomes the new head, i.e. its
            // key (o~, idx) precedes the blocked head's; in arrival order (MC-Benchmark) a
            // newcomer never does.  Other arrivals join R at the landing round (no decision
            // is taken in between, so when exactly they join does not matter).
            if (POL == POL_MCSF) {
                for (int k = next; a_next < T && k < n; k += 32) {
                    const int kk = k + lane;
                    const int ak = kk < n ? S.arr[kk] : KV_INF;
                    const bool before = ak < T;
                    const uint32_t m = __ballot_sync(KV_FULL, before && (int)S.arank[min(kk, n - 1)] < h);
                    if (m) { T = __shfl_sync(KV_FULL, ak, __ffs(m) - 1); break; }
                    if (!__all_sync(KV_FULL, before)) break;
                }
            }
            head_fits = T == t + jump;        // landing where the unchanged head fits
            jump = T - t;
        }
        // rounds t .. t+jump-1: decision rounds (R non-empty), batch memory Prof(t+1..t+jump)
        drounds += jump;
        if (jump == 1) {
            if (lane == 0) peak = max(peak, P0);                          // Mem(t+1)
            prof_shift1(P0, P1);
        } else {
            peak = max(peak, prof_max_lane(P0, P1, jump));
            prof_shift(P0, P1, jump);
        }
        t += jump;
    }

    // ---- outputs: coalesced completion / start, TEL ------------------------------
    __syncwarp();
    long long sumc = 0;
    for (int k = lane; k < n; k += 32) {
        const int p = S.pst[k];
        const uint32_t key = (POL == POL_MCSF) ? S.kidx[k] : S.keys[k];
        const int c = p < 0 ? -1 : p + (int)(key & 63u);
        sumc += c;
        if (P.completion) P.completion[off + k] = c;
        if (P.start) P.start[off + k] = p;
        if (P.lat16) {
            const long long d = (long long)c - S.arr[k];
            P.lat16[off + k] = (c < 0 || d < 0 || d > 65534) ? (uint16_t)0xffffu : (uint16_t)d;
        }
    }
    sumc = warp_sum_i64(sumc);
    res.tel = sumc - suma;
    res.rounds = rounds + drounds;
    res.decision_rounds = drounds;
    res.makespan = maxc;
    res.peak = warp_max_i32(peak);
    res.status = status;
    write_result(P, inst, res);
}

template <int POL, bool MULTI, class Queue>
__device__ void small_instance(const KParams &P, long long inst, const SmallSmem &S)
{
    const int lane = lane_id();
    const long long off = P.offset[inst] - P.row_base;      // row of request 0
    const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
    const int M = P.mem[inst];
    InstResult res{0, 0, 0, 0, 0, 0, ST_OK};

    if (n > P.max_requests || M > P.max_mem) {
        res.status = ST_UNSUPPORTED;
        fill_unscheduled(P, off, n);
        write_result(P, inst, res);
        return;
    }

    // ---- stage + validate (one coalesced 16-byte load per request) ------------------
    stream_wait(P, inst);
    bool bad = false, slow = false;
    long long suma = 0, sumo = 0;
    int carry = 0;                                       // P16 rows: a of the previous chunk
    for (int k0 = 0; k0 < n; k0 += 32) {
        const int k = k0 + lane;
        const int4 r = P.req16 ? load_row_p16(P, off, k, n, carry)
                               : (k < n ? load_row(P, off + k) : make_int4(0, 1, 1, 1));   // {a, s, o, o~}
        if (k >= n) continue;
        bad |= r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1;
        if (POL == POL_MCSF) {
            bad |= r.y + r.w > M || r.w < r.z;            // DESIGN Q8; o~ >= o
            slow |= r.w != r.z;
        } else {
            bad |= r.y + r.z > M;
        }
        suma += r.x;
        sumo += r.z;
        S.arr[k] = r.x;
        S.pst[k] = -1;
        const uint32_t w = (POL == POL_MCSF) ? (uint32_t)r.w : 0u;
        const uint32_t key = (w << 26) | ((uint32_t)k << 12) | (((uint32_t)r.y & 63u) << 6) | ((uint32_t)r.z & 63u);
        if (POL == POL_MCSF) S.kidx[k] = key; else S.keys[k] = key;
    }
    __syncwarp();
    for (int k = lane + 1; k < n; k += 32) bad |= S.arr[k] < S.arr[k - 1];
    bad = __any_sync(KV_FULL, bad);
    slow = __any_sync(KV_FULL, slow);
    suma = warp_sum_i64(suma);
    sumo = warp_sum_i64(sumo);
    if (bad) {
        res.status = ST_INVALID;
        fill_unscheduled(P, off, n);
        write_result(P, inst, res);
        return;
    }
    if (n == 0) {
        write_result(P, inst, res);
        return;
    }

    // ---- MC-SF: ranks in (o~, idx) order by a stable counting sort on o~ <= 63 -----------
    //   rank_i = #{j : o~_j < o~_i} + #{j < i : o~_j = o~_i}
    if (POL == POL_MCSF) {
        S.hist[lane] = 0;
        S.hist[lane + 32] = 0;
        __syncwarp();
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const int v = k < n ? (int)(S.kidx[k] >> 26) : 64 + lane;
            const unsigned peers = __match_any_sync(KV_FULL, v);
            if (k < n && __ffs(peers) - 1 == lane) S.hist[v] += __popc(peers);
            __syncwarp();
        }
        const int h0 = S.hist[2 * lane], h1 = S.hist[2 * lane + 1];
        int x = h0 + h1;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(KV_FULL, x, d);
            if (lane >= d) x += y;
        }
        __syncwarp();
        S.hist[2 * lane] = x - h0 - h1;
        S.hist[2 * lane + 1] = x - h1;
        __syncwarp();
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            const uint32_t key = k < n ? S.kidx[k] : 0u;
            const int v = k < n ? (int)(key >> 26) : 64 + lane;
            const unsigned peers = __match_any_sync(KV_FULL, v);
            if (k < n) {
                const int r = S.hist[v] + __popc(peers & ((1u << lane) - 1u));
                S.keys[r] = key;
                S.arank[k] = (uint16_t)r;
            }
            __syncwarp();
            if (k < n && __ffs(peers) - 1 == lane) S.hist[v] += __popc(peers);
            __syncwarp();
        }
    }
    if (POL == POL_MCSF && slow) small_run<POL, MULTI, Queue, true>(P, inst, S, off, n, M, suma, sumo);
    else small_run<POL, MULTI, Queue, false>(P, inst, S, off, n, M, suma, sumo);
}

template <int POL, bool MULTI, bool QREG>
__global__ void __launch_bounds__(128, KV_SMALL_MIN_BLOCKS) k_mc_small(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + (size_t)warp * P.warp_bytes;
    const int NP = P.NP;
    SmallSmem S;
    S.keys = reinterpret_cast<uint32_t *>(base);
    S.kidx = reinterpret_cast<uint32_t *>(base + NP * 4);
    S.arr = reinterpret_cast<int *>(base + NP * 8);
    S.pst = reinterpret_cast<int *>(base + NP * 12);
    S.arank = reinterpret_cast<uint16_t *>(base + NP * 16);
    S.bm = reinterpret_cast<uint32_t *>(base + NP * 18);
    S.sm = reinterpret_cast<uint32_t *>(base + NP * 18 + (NP / 32) * 4);
    S.hist = reinterpret_cast<int *>(base + NP * 18 + (NP / 32) * 4 + 128);

    // work item w is instance w, or work_list[w] for the instances k_mc_lane handed over
    const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
    long long w = 0;
    if (lane == 0) w = atomicAdd(P.counter, 1ull);
    w = __shfl_sync(KV_FULL, w, 0);
    while (w < n_work) {
        long long nxt = 0;     // claim the next instance now; the latency hides behind this one
        if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
        const long long inst = P.work_list ? P.work_list[w] : w;
        if (QREG) small_instance<POL, MULTI, RegQueue>(P, inst, S);
        else small_instance<POL, MULTI, SmemQueue>(P, inst, S);
        w = __shfl_sync(KV_FULL, nxt, 0);
        __syncwarp();
    }
}

}  // namespace kv
