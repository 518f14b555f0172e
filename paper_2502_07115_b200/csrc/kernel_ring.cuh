// kernel_ring.cuh -- per-instance warp simulator for any budget M (all four policies).
//
// Same round structure as kernel_small.cuh, but the memory profile lives in a ring of L
// int32 slots in shared memory holding the exact profile of the window [t+1, t+L] (slot
// r & (L-1) = absolute round r), so a candidate's Eq. 5 test and its admission are
// ceil(w/32) warp-wide passes over its own window.  L is at most KV_RING_SHORT (2048) so
// that ~20 warps fit an SM; the rare requests whose ramp reaches past the window ("long",
// w > L) are kept one per lane in a LongList: slots entering the window are initialised from
// it and positions beyond the window are computed from it.  An instance that ever has more
// than 32 long requests in flight is handed to a second launch with a ring covering every
// request (status RETRY, internal).  Per-request data stay in HBM/L2 and are fetched when a
// request reaches the head of the queue.
//
//   MC-SF / MC-Benchmark : ring = projected memory of S (Eq. 5 LHS), as in the small kernel.
//                           A blocked head is resolved over the next 32 rounds per pass
//                           (ring_first_fit), arrivals end the jump only if they sort before
//                           the head.
//   alpha / alpha-beta    : ring = actual memory (Eq. 3, true o).  Admission is FCFS with
//                           threshold B = floor((1-alpha)M) on the next-round occupancy
//                           (DESIGN Q12); when Mem(t+1) > M the active set is cleared
//                            or thinned by independent Philox draws (DESIGN Q14).
//                           Rounds in which nothing can happen (head over threshold, no
//                           overflow, no arrival into an empty queue) are found 32 at a time
//                           by one ballot over the ring.  The in-flight set is a bitmap over
//                           idx (plus start rounds in global scratch) walked only on overflow.
#pragma once
#include "params.cuh"

namespace kv {

struct RingSmem {
    int *prof;        // [L]
    uint32_t *bm;     // [NP/32] waiting queue
    uint32_t *sm;     // [32]
    uint32_t *infl;   // [NP/32] in-flight set (alpha policies)
};

__host__ __device__ inline int ring_warp_bytes(int L, int NP, int policy)
{
    int b = L * 4 + (NP / 32) * 4 + 32 * 4;
    if (policy >= POL_ALPHA) b += (NP / 32) * 4;
    return (b + 15) & ~15;
}

// Prof(t+tau) += sign * (base + tau) for tau in [1, e]
__device__ __forceinline__ void ring_ramp(int *prof, int mask, int t, int e, int base, int sign)
{
    for (int tau = lane_id() + 1; tau <= e; tau += 32) prof[(t + tau) & mask] += sign * (base + tau);
}

// In-flight requests whose ramp reaches past the ring window: one per lane.  Active at
// absolute rounds (p, e], holding s + r - p at round r (Eq. 3).  `used` is warp-uniform.
struct LongList {
    int p, s, e, idx;
    uint32_t used;
};

// sum over long requests active at absolute round r of (s + r - p); r may differ per lane,
// all lanes must call
__device__ __forceinline__ int long_prof(const LongList &G, int r)
{
    int v = 0;
    uint32_t m = G.used;
    while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const int p = __shfl_sync(KV_FULL, G.p, l), s = __shfl_sync(KV_FULL, G.s, l);
        const int e = __shfl_sync(KV_FULL, G.e, l);
        if (p < r && r <= e) v += s + r - p;
    }
    return v;
}

__device__ __forceinline__ bool long_add(LongList &G, int p, int s, int e, int idx)
{
    if (G.used == KV_FULL) return false;
    const int l = __ffs(~G.used) - 1;
    if (lane_id() == l) { G.p = p; G.s = s; G.e = e; G.idx = idx; }
    G.used |= 1u << l;
    return true;
}

__device__ __forceinline__ void long_remove_idx(LongList &G, int idx)
{
    G.used &= ~__ballot_sync(KV_FULL, ((G.used >> lane_id()) & 1u) && G.idx == idx);
}

// Profile at window position u (absolute round t+u): ring inside the window, long list beyond.
__device__ __forceinline__ int prof_at(const int *prof, int mask, int L, const LongList &G, int t, int u)
{
    const int far = G.used ? long_prof(G, t + u) : 0;
    return u <= L ? prof[(t + u) & mask] : far;
}

// Advance the window start from t to tn (> t) and return max Prof(r) over r in [t+1, E]
// (E <= tn; the occupancy of the batches of rounds t..E-1).  Slots leaving the window are
// re-initialised for the rounds entering it, from the long list.
__device__ __forceinline__ int ring_jump(int *prof, int mask, int L, LongList &G, int t, int E, int tn)
{
    const int lane = lane_id();
    int v = 0;
    const int dn = max(min(E - t, L), 0);
    for (int base = 1; base <= dn; base += 32) {
        const int tau = base + lane;
        if (tau <= dn) v = max(v, prof[(t + tau) & mask]);
    }
    if (G.used && E - t > L) {
        // rounds beyond the old window: only long requests; maximum at an end point or at E
        const bool own = ((G.used >> lane) & 1u) && G.e > t + L && G.e <= E;
        v = max(v, long_prof(G, own ? G.e : E));
    }
    __syncwarp();
    if (tn - t <= L) {
        for (int base = 1; base <= tn - t; base += 32) {
            const int tau = base + lane;
            const int far = G.used ? long_prof(G, t + tau + L) : 0;
            if (tau <= tn - t) prof[(t + tau) & mask] = far;
        }
    } else {
        for (int j0 = 0; j0 < L; j0 += 32) {                     // whole window rewritten
            const int j = j0 + lane;
            const int r = tn + 1 + ((j - (tn + 1)) & mask);       // round of slot j in [tn+1, tn+L]
            const int far = G.used ? long_prof(G, r) : 0;
            prof[j] = far;
        }
    }
    G.used &= ~__ballot_sync(KV_FULL, ((G.used >> lane) & 1u) && G.e <= tn + L);   // now inside
    __syncwarp();
    return warp_max_i32(v);
}

// Admit a ramp s + tau, tau in [1, w], started at t: the window part into the ring, the
// rest via the long list.  false = long list full.
__device__ __forceinline__ bool ring_admit(int *prof, int mask, int L, LongList &G, int t, int w, int s, int idx)
{
    ring_ramp(prof, mask, t, min(w, L), s, +1);
    if (w > L) return long_add(G, t, s, t + w, idx);
    return true;
}

// First offset D in [0, 31] at which the head (s, w) satisfies Eq. 5 while the profile only
// advances; 32 if it is blocked at all of them.  Position u = D + tau rules out the offsets
// D in [u-w, u-1] with Prof(u) + s + u - D > M (see first_fit_offset in kernel_small.cuh);
// positions beyond w + 31 cannot reach D <= 31.
__device__ __forceinline__ int ring_first_fit(const int *prof, int mask, int L, const LongList &G, int t,
                                              int s, int w, int M)
{
    const int lane = lane_id();
    const int room = M - s;
    unsigned cov = 0u;
    for (int base = 1; base <= w + 31; base += 32) {
        const int u = base + lane;
        const int D = prof_at(prof, mask, L, G, t, u);
        const int lo = max(u - w, 0);
        const int hi = min(min(u - 1, D + u - room - 1), 31);
        if (hi >= lo) cov |= (0xffffffffu >> (31 - hi)) & (0xffffffffu << lo);
    }
    cov = __reduce_or_sync(KV_FULL, cov);
    return cov == 0xffffffffu ? 32 : __ffs(~cov) - 1;
}

template <int POL>
__device__ void ring_instance(const KParams &P, long long inst, const RingSmem &S)
{
    constexpr bool MC = POL == POL_MCSF || POL == POL_MCBENCH;
    const int lane = lane_id();
    const long long off = P.offset[inst] - P.row_base;      // row of request 0
    const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
    const int M = P.mem[inst];
    const int L = P.L, mask = L - 1;
    const int *reqi = reinterpret_cast<const int *>(P.req);
    InstResult res{0, 0, 0, 0, 0, 0, ST_OK};

    // ---- validate (coalesced pass) ------------------------------------------------------
    bool bad = false, unsup = n > P.max_requests || M > P.max_mem || off + n > P.scratch_rows, early = false;
    long long suma = 0, sumo = 0;
    if (!unsup) {
        for (int k = lane; k < n; k += 32) {
            const int4 r = P.req[off + k];
            bad |= r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1;
            if (k > 0) bad |= reqi[(off + k - 1) * 4] > r.x;
            if (POL == POL_MCSF) {
                bad |= (long long)r.y + r.w > M || r.w < r.z;
                early |= r.w != r.z;                 // early completion (o~ > o): k_prot
            } else {
                bad |= (long long)r.y + r.z > M;
            }
            unsup |= r.z > P.max_len || (POL == POL_MCSF && r.w > P.max_len);
            suma += r.x;
            sumo += r.z;
        }
    }
    bad = __any_sync(KV_FULL, bad);
    unsup = __any_sync(KV_FULL, unsup);
    if (POL == POL_MCSF && __any_sync(KV_FULL, early) && !bad && !unsup) {
        // MC-SF with o~ > o equals protected MC-SF with alpha = 0 (no realised overflow can
        // occur when o <= o~): listed for the k_prot launch that follows, else UNSUPPORTED
        if (P.early_list) {
            if (lane == 0) P.early_list[atomicAdd(P.early_count, 1ull)] = inst;
            return;
        }
        unsup = true;
    }
    suma = warp_sum_i64(suma);
    sumo = warp_sum_i64(sumo);
    if (unsup || bad) {
        res.status = unsup ? ST_UNSUPPORTED : ST_INVALID;
        fill_unscheduled(P, off, n);
        write_result(P, inst, res);
        return;
    }
    if (n == 0) { write_result(P, inst, res); return; }

    const int NPi = next_pow2(max(n, 32));
    const int nw = NPi >> 5;
    for (int i = lane; i < L; i += 32) S.prof[i] = 0;
    for (int w = lane; w < nw; w += 32) {
        S.bm[w] = 0u;
        if (!MC) S.infl[w] = 0u;
    }
    S.sm[lane] = 0u;
    __syncwarp();
    WarpQueue Q{S.bm, S.sm, (nw + 31) >> 5};

    const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(reqi[(off + n - 1) * 4], sumo);
    const int cap = (int)min(cap64, 0x7ffffffell);
    const long long B = MC ? 0 : ((long long)(P.alpha_den - P.alpha_num) * M) / P.alpha_den;
    const unsigned long long gid = P.id0 + (unsigned long long)inst;
    const bool multi = !(P.flags & 1);

    int t = reqi[off * 4];
    int next = 0, a_next = t;
    int h = KV_INF;
    uint4 he = make_uint4(0, 0, 0, 0);   // head entry {s, w, o, idx}
    bool hstale = false, head_fits = false;
    long long sumc = 0, evictions = 0;
    int rounds = 0, drounds = 0;
    int maxc = -1, peak = 0, status = ST_OK;
    int mem_prev = 0;                    // alpha: Mem(t) of the previous round
    // alpha-greedy cycle detection (DESIGN Q24): admissions since the last clear-all and the
    // arrival pointer then; a clear-all that evicts everything admitted since the previous
    // one (nothing completed), with no arrival in between and none left to come, repeats
    // that cycle for ever.
    int adm_since_clear = 0, next_at_clear = -1;
    LongList G;
    G.p = G.s = G.e = G.idx = 0;
    G.used = 0u;

    auto fetch = [&](int r) -> uint4 {
        if (POL == POL_MCSF) return P.rq[off + r];
        const int4 q = P.req[off + r];
        return make_uint4((uint32_t)q.y, (uint32_t)q.z, (uint32_t)q.z, (uint32_t)r);
    };

    for (;;) {
        if (h == KV_INF) {
            if (MC) {
                if (a_next == KV_INF) {                        // drain
                    const int E = min(maxc, cap + 1);
                    if (E > t) peak = max(peak, ring_jump(S.prof, mask, L, G, t, E, t));
                    if (maxc > t) rounds += maxc - t;
                    if (maxc >= cap + 1) status = ST_LIVELOCK;
                    break;
                }
                const int tn = a_next;
                if (tn > t) {                                  // skip rounds t..tn-1
                    const int E = min(tn, cap + 1);
                    peak = max(peak, ring_jump(S.prof, mask, L, G, t, E, tn));
                    rounds += max(0, min(tn, maxc) - t);
                    if (tn > cap) { status = ST_LIVELOCK; break; }
                    t = tn;
                }
            } else if (mem_prev == 0) {                        // R and S empty: idle jump
                if (a_next == KV_INF) break;
                t = max(t, a_next);
            }
        }
        if (t > cap) { status = ST_LIVELOCK; break; }

        // arrivals
        while (a_next <= t) {
            const int k = next + lane;
            const int ak = k < n ? reqi[(off + k) * 4] : KV_INF;
            const bool take = ak <= t;
            const int cnt = __popc(__ballot_sync(KV_FULL, take));
            int rk = KV_INF;
            if (take) {
                rk = (POL == POL_MCSF) ? P.arank[off + k] : k;
                q_insert(Q, rk);
            }
            const int mn = warp_min_i32(rk);
            if (mn < h) { h = mn; hstale = true; head_fits = false; }
            next += cnt;
            a_next = cnt < 32 ? __shfl_sync(KV_FULL, ak, cnt & 31) : (next < n ? reqi[(off + next) * 4] : KV_INF);
        }
        __syncwarp();

        const bool had_R = h != KV_INF;
        if (MC) {
            // decision round t with R non-empty (Alg. 1 / Alg. 2)
            if (hstale) { he = fetch(h); hstale = false; }
            int jump = 1;
            bool blocked_through = false;                 // head blocked at all 32 offsets
            for (;;) {
                const int s = (int)he.x, w = (int)he.y, o = (int)he.z, idx = (int)he.w;
                if (!head_fits) {
                    int d;
                    if (multi) {
                        d = ring_first_fit(S.prof, mask, L, G, t, s, w, M);
                    } else {
                        bool bad_ = false;
                        for (int base = 1; base <= w; base += 32) {
                            const int tau = base + lane;
                            const int v = prof_at(S.prof, mask, L, G, t, tau);
                            bad_ |= tau <= w && v + s + tau > M;
                        }
                        d = __any_sync(KV_FULL, bad_) ? 1 : 0;
                    }
                    if (d > 0) { jump = d; blocked_through = d == 32; break; }   // Eq. 5 violated
                }
                head_fits = false;
                // MC-SF: the next head leaves the queue first so that its entry (rank-ordered
                // scratch) loads while the ramp is written; a RETRY restarts the instance, so
                // the order is free (measured on C4: MC-SF 1.6 % faster, MC-Benchmark 3 %
                // slower, so it keeps pop-after-admit)
                int hn = KV_INF;
                uint4 hen = he;
                if (POL == POL_MCSF) {
                    hn = q_pop_head(Q, h);
                    if (hn != KV_INF) hen = fetch(hn);
                }
                if (!ring_admit(S.prof, mask, L, G, t, w, s, idx)) { status = ST_RETRY; break; }
                const int c = t + o;
                if (lane == 0) {
                    if (P.completion) P.completion[off + idx] = c;
                    if (P.start) P.start[off + idx] = t;
                }
                sumc += c;
                maxc = max(maxc, c);
                __syncwarp();
                if (POL != POL_MCSF) {
                    hn = q_pop_head(Q, h);
                    if (hn != KV_INF) hen = fetch(hn);
                }
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
                        const int ak = kk < n ? reqi[(off + kk) * 4] : KV_INF;
                        const bool before = ak < T;
                        const uint32_t m = __ballot_sync(KV_FULL, before && P.arank[off + min(kk, n - 1)] < h);
                        if (m) { T = __shfl_sync(KV_FULL, ak, __ffs(m) - 1); break; }
                        if (!__all_sync(KV_FULL, before)) break;
                    }
                }
                head_fits = !blocked_through && T == t + jump;
                jump = T - t;
            }
            drounds += jump;
            rounds += jump;
            peak = max(peak, ring_jump(S.prof, mask, L, G, t, t + jump, t + jump));
            t += jump;
            continue;
        }

        // ---- alpha / alpha-beta ----------------------------------------------------------
        const int occ = S.prof[(t + 1) & mask];           // Mem(t+1) of S
        const bool idle_before = occ == 0;
        long long Lnext = occ;
        int admitted = 0;
        if (had_R) {
            ++drounds;
            if (hstale) { he = fetch(h); hstale = false; }
            for (;;) {
                const int s = (int)he.x, o = (int)he.z, idx = (int)he.w;
                if (Lnext + s + 1 > B) break;                   // (1-alpha)M threshold
                Lnext += s + 1;
                if (!ring_admit(S.prof, mask, L, G, t, o, s, idx)) { status = ST_RETRY; break; }
                const int c = t + o;
                if (lane == 0) {
                    if (P.completion) P.completion[off + idx] = c;
                    if (P.start) P.start[off + idx] = t;
                    P.pstart[off + idx] = t;                            // start scratch
                    S.infl[idx >> 5] |= 1u << (idx & 31);
                }
                sumc += c;
                ++admitted;
                ++adm_since_clear;
                __syncwarp();
                h = q_pop_head(Q, h);
                if (h == KV_INF) break;
                he = fetch(h);
            }
        }
        if (status == ST_RETRY) break;
        __syncwarp();
        int mem = S.prof[(t + 1) & mask];
        bool cycle = false;
        if (mem > M) {
            // overflow of the batch of round t (DESIGN Q13): clear or thin
            const int *pst = P.pstart;
            const long long ev_before = evictions;
            int pass = 0;
            for (;; ++pass) {
                if (pass == KV_BETA_MAX_PASSES) { status = ST_LIVELOCK; break; }   // DESIGN Q29
                int left = 0;
                for (int wb = 0; wb < nw; wb += 32) {
                    const int wi = wb + lane;
                    uint32_t bits = wi < nw ? S.infl[wi] : 0u;
                    uint32_t keep = bits;
                    while (__any_sync(KV_FULL, bits != 0u)) {
                        int j = -1, pj = 0, sj = 0, oj = 0;
                        bool ev = false, act = false;
                        if (bits) {
                            j = (wi << 5) + __ffs(bits) - 1;
                            bits &= bits - 1;
                            pj = pst[off + j];
                            sj = reqi[(off + j) * 4 + 1];
                            oj = reqi[(off + j) * 4 + 2];
                            act = pj + oj > t;
                            if (!act) keep &= ~(1u << (j & 31));   // completed earlier
                            else {
                                ev = (POL == POL_ALPHA) ||
                                     (unsigned long long)evict_draw(P.seed, gid, t, pass, j) < P.beta_thresh;
                                if (ev) keep &= ~(1u << (j & 31));
                            }
                        }
                        left += __popc(__ballot_sync(KV_FULL, act && !ev));
                        uint32_t evm = __ballot_sync(KV_FULL, ev);
                        if (evm) {
                            evictions += __popc(evm);
                            sumc -= warp_sum_i64(ev ? (long long)(pj + oj) : 0ll);
                            const int mn = warp_min_i32(ev ? j : KV_INF);
                            if (mn < h) { h = mn; hstale = true; }
                            if (ev) {
                                q_insert(Q, j);
                                if (P.completion) P.completion[off + j] = -1;
                                if (P.start) P.start[off + j] = -1;
                            }
                            if (POL == POL_ALPHA_BETA) {
                                while (evm) {                       // remove its ramp
                                    const int l = __ffs(evm) - 1;
                                    evm &= evm - 1;
                                    const int s_ = __shfl_sync(KV_FULL, sj, l);
                                    const int p_ = __shfl_sync(KV_FULL, pj, l);
                                    const int o_ = __shfl_sync(KV_FULL, oj, l);
                                    const int j_ = __shfl_sync(KV_FULL, j, l);
                                    __syncwarp();
                                    ring_ramp(S.prof, mask, t, min(p_ + o_ - t, L), s_ + t - p_, -1);
                                    long_remove_idx(G, j_);
                                }
                            }
                        }
                    }
                    if (wi < nw) S.infl[wi] = keep;
                }
                __syncwarp();
                if (POL == POL_ALPHA) {
                    for (int i = lane; i < L; i += 32) S.prof[i] = 0;
                    __syncwarp();
                    G.used = 0u;
                    mem = 0;
                    cycle = next == n && next_at_clear == next && evictions - ev_before == adm_since_clear;
                    next_at_clear = next;
                    adm_since_clear = 0;
                    break;
                }
                mem = S.prof[(t + 1) & mask];
                if (mem <= M || left == 0) break;
            }
        }
        if (cycle || status == ST_LIVELOCK) { status = ST_LIVELOCK; break; }
        if (idle_before && admitted == 0 && h != KV_INF) { status = ST_LIVELOCK; break; }
        if (had_R || !idle_before) ++rounds;
        __syncwarp();
        const int mnow = ring_jump(S.prof, mask, L, G, t, t + 1, t + 1);   // Mem(t+1) of the batch
        peak = max(peak, mnow);
        mem_prev = mnow;
        ++t;

        // Rounds r = t, t+1, ... in which nothing can happen: no overflow (Mem(r+1) <= M),
        // S non-empty, and either the FCFS head stays over the threshold (a newcomer never
        // precedes it) or, with R empty, nothing arrives.  Found 32 at a time by a ballot
        // over the ring; their counters are accumulated without iterating them.
        if (multi && mem_prev > 0) {
            const int sh = h != KV_INF ? (hstale ? (int)fetch(h).x : (int)he.x) : 0;
            for (;;) {
                const int r = t + lane;
                const int v = S.prof[(r + 1) & mask];
                const bool quiet = r <= cap && v > 0 && v <= M &&
                                   (h != KV_INF ? (long long)v + sh + 1 > B : r < a_next);
                const uint32_t qm = __ballot_sync(KV_FULL, quiet);
                const int k = qm == KV_FULL ? 32 : __ffs(~qm) - 1;   // quiet rounds t..t+k-1
                if (k == 0) break;
                mem_prev = __shfl_sync(KV_FULL, v, k - 1);
                peak = max(peak, ring_jump(S.prof, mask, L, G, t, t + k, t + k));
                rounds += k;
                if (h != KV_INF) drounds += k;
                t += k;
                if (k < 32) break;
            }
        }
    }

    if (status == ST_RETRY) {               // rerun by the full-ring launch (kvsched.cu)
        if (lane == 0) P.retry_list[atomicAdd(P.retry_count, 1ull)] = inst;
        return;
    }
    if (status != ST_OK) {
        for (int k = next + lane; k < n; k += 32) {
            if (P.completion) P.completion[off + k] = -1;
            if (P.start) P.start[off + k] = -1;
        }
        for (int w = lane; w < nw; w += 32) {
            uint32_t bits = S.bm[w];
            while (bits) {
                const int r = (w << 5) + __ffs(bits) - 1;
                bits &= bits - 1;
                const int idx = (POL == POL_MCSF) ? (int)P.rq[off + r].w : r;
                if (P.completion) P.completion[off + idx] = -1;
                if (P.start) P.start[off + idx] = -1;
            }
        }
    }
    if (!MC) {
        // makespan of the final schedule
        int mx = -1;
        if (status == ST_OK)
            for (int k = lane; k < n; k += 32) mx = max(mx, P.pstart[off + k] + reqi[(off + k) * 4 + 2]);
        maxc = warp_max_i32(mx);
    }
    res.tel = sumc - suma;
    res.rounds = rounds;
    res.decision_rounds = drounds;
    res.evictions = evictions;
    res.makespan = maxc;
    res.peak = peak;
    res.status = status;
    write_result(P, inst, res);
}

template <int POL>
__global__ void __launch_bounds__(128) k_ring(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + (size_t)warp * P.warp_bytes;
    RingSmem S;
    S.prof = reinterpret_cast<int *>(base);
    S.bm = reinterpret_cast<uint32_t *>(base + P.L * 4);
    S.sm = reinterpret_cast<uint32_t *>(base + P.L * 4 + (P.NP / 32) * 4);
    S.infl = reinterpret_cast<uint32_t *>(base + P.L * 4 + (P.NP / 32) * 4 + 128);

    // work item w is instance w, or work_list[w] for the full-ring rerun of RETRY instances
    const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
    long long w = 0;
    if (lane == 0) w = atomicAdd(P.counter, 1ull);
    w = __shfl_sync(KV_FULL, w, 0);
    while (w < n_work) {
        long long nxt = 0;
        if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
        ring_instance<POL>(P, P.work_list ? P.work_list[w] : w, S);
        w = __shfl_sync(KV_FULL, nxt, 0);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// MC-SF rank prepass for the ring kernel: one CTA per instance sorts (o~, idx) keys in
// shared memory (bitonic) and writes per-rank entries {s, o~, o, idx} and rank[idx].
// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_rank_sort(const KParams P, uint4 *rq, int *arank)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(smem_raw);
    for (long long inst = blockIdx.x; inst < P.n_inst; inst += gridDim.x) {
        const long long off = P.offset[inst] - P.row_base;
        const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
        if (n <= 0 || n > P.max_requests || off + n > P.scratch_rows) continue;
        const int NPi = next_pow2(n);
        for (int k = threadIdx.x; k < NPi; k += blockDim.x) {
            uint32_t key = 0xffffffffu;
            if (k < n) {
                const uint32_t w = (uint32_t)min(max(P.req[off + k].w, 0), 0x1ffff);
                key = (w << 15) | (uint32_t)k;
            }
            keys[k] = key;
        }
        __syncthreads();
        for (int k = 2; k <= NPi; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < (NPi >> 1); i += blockDim.x) {
                    const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1));
                    const int hi = lo + j;
                    const bool up = (lo & k) == 0;
                    const uint32_t x = keys[lo], y = keys[hi];
                    if ((x > y) == up) { keys[lo] = y; keys[hi] = x; }
                }
                __syncthreads();
            }
        }
        for (int r = threadIdx.x; r < n; r += blockDim.x) {
            const int idx = (int)(keys[r] & 0x7fffu);
            const int4 q = P.req[off + idx];
            rq[off + r] = make_uint4((uint32_t)q.y, (uint32_t)q.w, (uint32_t)q.z, (uint32_t)idx);
            arank[off + idx] = r;
        }
        __syncthreads();
    }
}

}  // namespace kv
