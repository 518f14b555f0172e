// kernel_small.cuh -- fused MC-SF / MC-Benchmark simulator for budgets M <= 64.
//
// One warp simulates one instance at a time on a persistent grid.  Everything the round
// loop touches lives on chip:
//   * projected memory profile Prof(t+tau), tau = 1..64, in registers: lane l holds
//     tau = l+1 (P0) and tau = l+33 (P1).  Prof is the left-hand side of Eq. 5
//     for the in-flight set S, so a candidate (s, w) is admissible at round t iff
//         Prof(t+tau) + s + tau <= M  for every tau in [1, w]
//     -- one vote over the warp.  With o~ >= o the profile beyond a candidate's own window
//     is already feasible (every earlier admission certified its window), so these are
//     exactly the t' in [t+1, t_max(U + {i})] of Eq. 5.  Admission adds the ramp s + tau
//     (Eq. 3); advancing the clock is a one-lane shuffle.
//   * the waiting queue R^(t): a two-level bitmap over ranks in shared memory; rank =
//     position in (o~, idx) order for MC-SF (Alg. 1 line "ascending order of predicted
//     output length") or idx for MC-Benchmark (arrival order).  The ranks
//     come from a warp bitonic sort of packed keys, done once per instance.
//   * packed per-request words {o~:6 | idx:14 | s:6 | o:6} by rank, arrivals a by idx.
// The admission loop walks the queue head in rank order and stops at the first failure
// (Alg. 1 "Break the for loop"): the longest feasible prefix of Eq. 6.
//
// Rounds with an empty queue are not iterated: nothing can be admitted in them, so the
// clock jumps to the next arrival and the skipped rounds' occupancy is read off the
// profile (DESIGN "Exact fast paths").  With o~ > o (early completion) a request
// leaves S before its projected window ends; those instances run the plain per-round
// loop with the unused tail removed from the profile at completion (Eq. 5 sums over the
// requests still in progress).
#pragma once
#include "params.cuh"

namespace kv {

struct SmallSmem {
    uint32_t *keys;      // [NP] packed words by rank
    int *arr;            // [NP] a by idx
    uint16_t *arank;     // [NP] rank of idx (MC-SF)
    uint32_t *bm;        // [NP/32]
    uint32_t *sm;        // [32]
};

__host__ __device__ inline int small_warp_bytes(int NP)
{
    int b = NP * 4 + NP * 4 + NP * 2 + (NP / 32) * 4 + 32 * 4;
    return (b + 15) & ~15;
}

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

// max of Prof(t+tau) over tau in [1, d]
__device__ __forceinline__ int prof_max(int P0, int P1, int d)
{
    const int lane = lane_id();
    int v = (lane + 1 <= d) ? P0 : 0;
    v = max(v, (lane + 33 <= d) ? P1 : 0);
    return warp_max_i32(v);
}

// Bit D (0 <= D < 64) of the result is set iff a head candidate (s, w) would violate
// Eq. 5 at round t+D while the profile only advances (no admission, arrival or early
// completion in between).  Position u = t+D+tau of the profile rules out the offsets
// D in [u-w, u-1] with Prof(u) + s + (u - D) > M, i.e. D <= Prof(u) + u - (M-s) - 1; the
// union over the 64 positions held by the warp is two OR-reductions.  Prof is zero
// beyond tau = 63 (o~ <= 63), so the head always fits by D = 64.
__device__ __forceinline__ unsigned long long blocked_rounds(int P0, int P1, int s, int w, int M)
{
    const int lane = lane_id();
    const int room = M - s;
    unsigned long long m = 0ull;
    {
        const int u = lane + 1;
        const int lo = max(0, u - w), hi = min(u - 1, P0 + u - room - 1);
        if (hi >= lo) m |= (~0ull >> (63 - hi)) & (~0ull << lo);
    }
    {
        const int u = lane + 33;
        const int lo = max(0, u - w), hi = min(u - 1, P1 + u - room - 1);
        if (hi >= lo) m |= (~0ull >> (63 - hi)) & (~0ull << lo);
    }
    const unsigned lo32 = __reduce_or_sync(KV_FULL, (unsigned)m);
    const unsigned hi32 = __reduce_or_sync(KV_FULL, (unsigned)(m >> 32));
    return ((unsigned long long)hi32 << 32) | lo32;
}

template <int POL, bool MULTI>
__device__ void small_instance(const KParams &P, long long inst, const SmallSmem &S)
{
    const int lane = lane_id();
    const long long off = P.offset[inst];
    const int n = (int)(P.offset[inst + 1] - off);
    const int M = P.mem[inst];
    InstResult res{0, 0, 0, 0, 0, 0, ST_OK};

    if (n > P.max_requests || M > P.max_mem) {
        res.status = ST_UNSUPPORTED;
        fill_unscheduled(P, off, n);
        write_result(P, inst, res);
        return;
    }

    // ---- stage + validate (one coalesced 16-byte load per request) ------------------
    const int NPi = next_pow2(max(n, 32));
    bool bad = false, slow = false;
    long long suma = 0, sumo = 0;
    for (int k = lane; k < NPi; k += 32) {
        uint32_t key = 0xffffffffu;
        if (k < n) {
            const int4 r = P.req[off + k];               // {a, s, o, o~}
            bad |= r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1;
            if (POL == POL_MCSF) {
                bad |= r.y + r.w > M || r.w < r.z;        // DESIGN Q8; o~ >= o
                slow |= r.w != r.z;
            } else {
                bad |= r.y + r.z > M;
            }
            suma += r.x;
            sumo += r.z;
            S.arr[k] = r.x;
            const uint32_t w = (POL == POL_MCSF) ? (uint32_t)r.w : 0u;
            key = (w << 26) | ((uint32_t)k << 12) | (((uint32_t)r.y & 63u) << 6) | ((uint32_t)r.z & 63u);
        }
        S.keys[k] = key;
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

    // ---- MC-SF: sort packed keys by (o~, idx) -> ranks (warp bitonic, once) ----------
    if (POL == POL_MCSF) {
        for (int k = 2; k <= NPi; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < (NPi >> 1); i += 32) {
                    const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                    const int hi = lo + j;
                    const bool up = (lo & k) == 0;
                    const uint32_t x = S.keys[lo], y = S.keys[hi];
                    if ((x > y) == up) { S.keys[lo] = y; S.keys[hi] = x; }
                }
                __syncwarp();
            }
        }
        for (int r = lane; r < n; r += 32) S.arank[(S.keys[r] >> 12) & 0x3fffu] = (uint16_t)r;
    }
    const int nw = (NPi + 31) >> 5;
    for (int w = lane; w < nw; w += 32) S.bm[w] = 0u;
    S.sm[lane] = 0u;
    __syncwarp();
    WarpQueue Q{S.bm, S.sm, (nw + 31) >> 5};

    const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(S.arr[n - 1], sumo);
    const int cap = (int)min(cap64, 0x7ffffffell);

    // ---- round loop --------------------------------------------------------------------
    int t = S.arr[0];
    int next = 0, a_next = S.arr[0];
    int h = KV_INF;                  // queue head (rank), KV_INF = R empty
    uint32_t hkey = 0u;
    bool hstale = false;
    int P0 = 0, P1 = 0;              // Prof(t+lane+1), Prof(t+lane+33)
    long long sumc = 0;
    int rounds = 0, drounds = 0;
    int maxc = -1, peak = 0, status = ST_OK;
    // early-completion records (slow mode): one lane per in-flight request with o~ > o
    int rc = KV_INF, rs = 0, rp = 0, rw = 0;

    for (;;) {
        if (h == KV_INF) {
            if (!slow) {
                if (a_next == KV_INF) {                       // drain: S only, no arrivals
                    const int E = min(maxc, cap + 1);
                    if (E > t) peak = max(peak, prof_max(P0, P1, min(E - t, 64)));
                    if (maxc > t) rounds += maxc - t;
                    if (maxc >= cap + 1) status = ST_LIVELOCK;
                    break;
                }
                const int tn = a_next;
                if (tn > t) {                                 // skip rounds t..tn-1
                    const int E = min(tn, cap + 1);
                    if (E > t) peak = max(peak, prof_max(P0, P1, min(E - t, 64)));
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
        while (a_next <= t) {
            const int k = next + lane;
            const int ak = k < n ? S.arr[k] : KV_INF;
            const bool take = ak <= t;
            const int cnt = __popc(__ballot_sync(KV_FULL, take));
            int rk = KV_INF;
            if (take) {
                rk = (POL == POL_MCSF) ? (int)S.arank[k] : k;
                q_insert(Q, rk);
            }
            const int mn = warp_min_i32(rk);
            if (mn < h) { h = mn; hstale = true; }
            next += cnt;
            a_next = cnt < 32 ? __shfl_sync(KV_FULL, ak, cnt & 31) : (next < n ? S.arr[next] : KV_INF);
        }
        __syncwarp();

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
                peak = max(peak, __shfl_sync(KV_FULL, P0, 0));
                prof_shift1(P0, P1);
                ++t;
                continue;
            }
        }

        // decision round t with R non-empty (Alg. 1 / Alg. 2): candidates in rank order,
        // break at the first failure.  The failing head keeps failing -- and nothing else
        // is admitted -- until it fits, a request arrives or (o~ > o) a request completes
        // early; the coverage test finds the first of those rounds in one pass.
        if (hstale) { hkey = S.keys[h]; hstale = false; }
        int jump = 1;
        for (;;) {
            const int w = (POL == POL_MCSF) ? (int)(hkey >> 26) : (int)(hkey & 63u);
            const int s = (int)((hkey >> 6) & 63u), o = (int)(hkey & 63u);
            if (MULTI) {
                const unsigned long long cov = blocked_rounds(P0, P1, s, w, M);
                if (cov & 1ull) {                                        // Eq. 5 violated now
                    jump = (~cov == 0ull) ? 64 : __ffsll((long long)~cov) - 1;
                    break;
                }
            } else {
                const int tau0 = lane + 1, tau1 = lane + 33;
                const bool v = (tau0 <= w && P0 + s + tau0 > M) || (tau1 <= w && P1 + s + tau1 > M);
                if (__any_sync(KV_FULL, v)) break;                      // Eq. 5 violated
            }
            if (lane + 1 <= w) P0 += s + lane + 1;                       // ramp s + tau (Eq. 3)
            if (lane + 33 <= w) P1 += s + lane + 33;
            const int idx = (int)((hkey >> 12) & 0x3fffu);
            const int c = t + o;                                         // c_i = p_i + o_i
            if (lane == 0) {
                if (P.completion) P.completion[off + idx] = c;
                if (P.start) P.start[off + idx] = t;
            }
            sumc += c;
            maxc = max(maxc, c);
            if (POL == POL_MCSF && w > o) {                               // early completion
                const uint32_t fr = __ballot_sync(KV_FULL, rc == KV_INF);
                if (lane == __ffs(fr) - 1) { rc = c; rs = s; rp = t; rw = w; }
            }
            h = q_pop_head(Q, h);
            if (h == KV_INF) break;
            hkey = S.keys[h];
        }
        if (MULTI && jump > 1) {
            jump = min(jump, a_next - t);                 // a new request may become the head
            jump = min(jump, cap + 1 - t);
            if (slow) jump = min(jump, warp_min_i32(rc) - t);
        }
        // rounds t .. t+jump-1: decision rounds (R non-empty), batch memory Prof(t+1..t+jump)
        drounds += jump;
        rounds += jump;
        if (jump == 1) {
            peak = max(peak, __shfl_sync(KV_FULL, P0, 0));               // Mem(t+1)
            prof_shift1(P0, P1);
        } else {
            peak = max(peak, prof_max(P0, P1, jump));
            prof_shift(P0, P1, jump);
        }
        t += jump;
    }

    if (status != ST_OK) {
        // requests never started (still waiting, or not yet arrived) report -1
        for (int k = next + lane; k < n; k += 32) {
            if (P.completion) P.completion[off + k] = -1;
            if (P.start) P.start[off + k] = -1;
        }
        for (int w = lane; w < nw; w += 32) {
            uint32_t bits = S.bm[w];
            while (bits) {
                const int r = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                const int idx = (POL == POL_MCSF) ? (int)((S.keys[r] >> 12) & 0x3fffu) : r;
                if (P.completion) P.completion[off + idx] = -1;
                if (P.start) P.start[off + idx] = -1;
            }
        }
    }
    res.tel = sumc - suma;
    res.rounds = rounds;
    res.decision_rounds = drounds;
    res.makespan = maxc;
    res.peak = peak;
    res.status = status;
    write_result(P, inst, res);
}

template <int POL, bool MULTI>
__global__ void __launch_bounds__(128) k_mc_small(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + (size_t)warp * P.warp_bytes;
    const int NP = P.NP;
    SmallSmem S;
    S.keys = reinterpret_cast<uint32_t *>(base);
    S.arr = reinterpret_cast<int *>(base + NP * 4);
    S.arank = reinterpret_cast<uint16_t *>(base + NP * 8);
    S.bm = reinterpret_cast<uint32_t *>(base + NP * 10);
    S.sm = reinterpret_cast<uint32_t *>(base + NP * 10 + (NP / 32) * 4);

    long long inst = 0;
    if (lane == 0) inst = atomicAdd(reinterpret_cast<unsigned long long *>(P.counter), 1ull);
    inst = __shfl_sync(KV_FULL, inst, 0);
    while (inst < P.n_inst) {
        long long nxt = 0;     // claim the next instance now; the latency hides behind this one
        if (lane == 0) nxt = atomicAdd(reinterpret_cast<unsigned long long *>(P.counter), 1ull);
        small_instance<POL, MULTI>(P, inst, S);
        inst = __shfl_sync(KV_FULL, nxt, 0);
        __syncwarp();
    }
}

}  // namespace kv
