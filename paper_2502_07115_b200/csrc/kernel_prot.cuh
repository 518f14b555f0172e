// kernel_prot.cuh -- MC-SF under prediction error with a protection margin.
//
// The scheduler sees noisy predictions o~ (o~ ~ U((1-eps)o, (1+eps)o), integer-
// rounded on the host), runs Algorithm 1 "as if the effective budget were (1-alpha)M"
// (P:526), and "an overflow triggers a clearing event, where all active requests are
// evicted and re-queued".  One warp per instance; two shared-memory rings over the
// window [t+1, t+L] (plus long-request lists beyond it, see kernel_ring.cuh):
//   Pp  the projection of Eq. 5: o~-ramps of the requests in S^(t) (an underestimated
//       request drops out of it once its predicted window ends, the indicator of P:141);
//   Pa  the realised occupancy of Eq. 3 with the true o (overflow detection, peak).
// A request that completes before its predicted end (o < o~) leaves S at c = p + o; the
// unused tail of its projection is removed then.  Such requests are chained per completion
// round (bucket head per ring slot in shared memory, links in global scratch).
// Rounds are processed one at a time, except idle rounds and runs of quiet rounds (blocked
// head, no overflow, no early completion), which are jumped up to 32 at a time.
#pragma once
#include "kernel_ring.cuh"

namespace kv {

struct ProtSmem {
    int *pp;          // [L] projection ring
    int *pa;          // [L] realised-occupancy ring
    int *rel;         // [L] early-completion chain heads by completion slot (-1 = empty)
    uint32_t *bm;     // [NP/32] waiting queue
    uint32_t *sm;     // [32]
    uint32_t *infl;   // [NP/32] in-flight set
};

__host__ __device__ inline int prot_warp_bytes(int L, int NP)
{
    int b = 3 * L * 4 + 2 * (NP / 32) * 4 + 32 * 4;
    return (b + 15) & ~15;
}

__device__ void prot_instance(const KParams &P, long long inst, const ProtSmem &S)
{
    const int lane = lane_id();
    const long long off = P.offset[inst] - P.row_base;      // row of request 0
    const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
    const int M = P.mem[inst];
    const int L = P.L, mask = L - 1;
    const int *reqi = reinterpret_cast<const int *>(P.req);
    InstResult res{0, 0, 0, 0, 0, 0, ST_OK};

    // DESIGN Q26b: a cleared request's prediction is raised to the tokens it is known to need
    // and the instance is re-ranked (keys sorted in the ring area, which a clearing resets)
    const bool raise = P.policy == POL_MCSF_PROT_RAISE;
    bool bad = false, unsup = n > P.max_requests || M > P.max_mem || off + n > P.scratch_rows ||
                              (raise && next_pow2(max(n, 2)) > 3 * L);
    long long suma = 0, sumo = 0;
    if (!unsup) {
        for (int k = lane; k < n; k += 32) {
            const int4 r = P.req[off + k];
            bad |= r.x < 0 || r.y < 1 || r.z < 1 || r.w < 1;
            if (k > 0) bad |= reqi[(off + k - 1) * 4] > r.x;
            bad |= (long long)r.y + r.z > M;                    // physically feasible
            unsup |= r.z > P.max_len || r.w > P.max_len;
            suma += r.x;
            sumo += r.z;
        }
    }
    bad = __any_sync(KV_FULL, bad);
    unsup = __any_sync(KV_FULL, unsup);
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
    for (int i = lane; i < L; i += 32) { S.pp[i] = 0; S.pa[i] = 0; S.rel[i] = -1; }
    for (int w = lane; w < nw; w += 32) { S.bm[w] = 0u; S.infl[w] = 0u; }
    S.sm[lane] = 0u;
    WarpQueue Q{S.bm, S.sm, (nw + 31) >> 5};
    uint4 *rqw = const_cast<uint4 *>(P.rq) + off;           // Q26b rewrites the ranks
    int *arw = const_cast<int *>(P.arank) + off;
    if (raise)
        for (int k = lane; k < n; k += 32) P.pstart[off + k] = -1;   // -1 = not in S, not completed
    __syncwarp();

    const long long cap64 = P.round_cap > 0 ? P.round_cap : default_cap(reqi[(off + n - 1) * 4], sumo);
    const int cap = (int)min(cap64, 0x7ffffffell);
    const int B = (int)(((long long)(P.alpha_den - P.alpha_num) * M) / P.alpha_den);   // (1-alpha)M
    const bool multi = !(P.flags & 1);                  // SCHED_FLAG_PER_ROUND: no jumps
    int *relnext = P.relnext + off;                     // chain links by idx
    int *pst = P.pstart + off;                          // start rounds by idx

    int t = reqi[off * 4];
    int next = 0, a_next = t;
    int h = KV_INF;
    uint4 he = make_uint4(0, 0, 0, 0);
    bool hstale = false;
    long long sumc = 0, evictions = 0;
    int rounds = 0, drounds = 0, peak = 0, status = ST_OK, mem_prev = 0;
    int adm_since_clear = 0, next_at_clear = -1;     // cycle rule (DESIGN Q24)
    LongList Gp, Ga;
    Gp.p = Gp.s = Gp.e = Gp.idx = 0;
    Gp.used = 0u;
    Ga = Gp;

    for (;;) {
        if (h == KV_INF && mem_prev == 0) {               // R and S empty: idle jump
            if (a_next == KV_INF) break;
            t = max(t, a_next);                           // rings and long lists are empty
        }
        if (t > cap) { status = ST_LIVELOCK; break; }

        while (a_next <= t) {                             // arrivals
            const int k = next + lane;
            const int ak = k < n ? reqi[(off + k) * 4] : KV_INF;
            const bool take = ak <= t;
            const int cnt = __popc(__ballot_sync(KV_FULL, take));
            int rk = KV_INF;
            if (take) {
                rk = P.arank[off + k];
                q_insert(Q, rk);
            }
            const int mn = warp_min_i32(rk);
            if (mn < h) { h = mn; hstale = true; }
            next += cnt;
            a_next = cnt < 32 ? __shfl_sync(KV_FULL, ak, cnt & 31) : (next < n ? reqi[(off + next) * 4] : KV_INF);
        }
        __syncwarp();

        // completions before the predicted end (o < o~): the request leaves S^(t), so its
        // projection beyond t drops out of Eq. 5
        {
            int prev = -1, cur = S.rel[t & mask];
            while (cur >= 0) {
                const int nxt = relnext[cur];
                const int p_ = pst[cur];
                const int o_ = reqi[(off + cur) * 4 + 2];
                if (p_ + o_ == t) {
                    const int s_ = reqi[(off + cur) * 4 + 1], w_ = reqi[(off + cur) * 4 + 3];
                    ring_ramp(S.pp, mask, t, min(p_ + w_ - t, L), s_ + t - p_, -1);
                    if (p_ + w_ > t + L) long_remove_idx(Gp, cur);
                    __syncwarp();
                    if (lane == 0) { if (prev < 0) S.rel[t & mask] = nxt; else relnext[prev] = nxt; }
                } else {
                    prev = cur;                            // a later completion on the same slot
                }
                __syncwarp();
                cur = nxt;
            }
        }
        __syncwarp();

        const bool had_R = h != KV_INF;
        const bool idle_before = S.pa[(t + 1) & mask] == 0;
        int admitted = 0;
        if (had_R) {
            ++drounds;
            if (hstale) { he = P.rq[off + h]; hstale = false; }
            for (;;) {                                     // Alg. 1 on budget (1-alpha)M
                const int s = (int)he.x, w = (int)he.y, o = (int)he.z, idx = (int)he.w;
                bool viol = false;
                for (int base = 1; base <= w; base += 32) {
                    const int tau = base + lane;
                    const int v = prof_at(S.pp, mask, L, Gp, t, tau);
                    viol |= tau <= w && v + s + tau > B;
                }
                if (__any_sync(KV_FULL, viol)) break;
                // the next head leaves the queue first so that its entry loads while the two
                // ramps are written (a RETRY restarts the instance, so the order is free)
                const int hn = q_pop_head(Q, h);
                uint4 hen = he;
                if (hn != KV_INF) hen = P.rq[off + hn];
                if (!ring_admit(S.pp, mask, L, Gp, t, w, s, idx) || !ring_admit(S.pa, mask, L, Ga, t, o, s, idx)) {
                    status = ST_RETRY;
                    break;
                }
                const int c = t + o;
                if (lane == 0) {
                    if (P.completion) P.completion[off + idx] = c;
                    if (P.start) P.start[off + idx] = t;
                    pst[idx] = t;
                    S.infl[idx >> 5] |= 1u << (idx & 31);
                    if (w > o) { relnext[idx] = S.rel[c & mask]; S.rel[c & mask] = idx; }
                }
                sumc += c;
                ++admitted;
                ++adm_since_clear;
                __syncwarp();
                h = hn;
                if (h == KV_INF) break;
                he = hen;
            }
            if (status == ST_RETRY) break;
        }
        __syncwarp();

        // realised overflow: clear every active request
        bool cycle = false;
        if (S.pa[(t + 1) & mask] > M) {
            long long ev = 0;
            for (int wb = 0; wb < nw; wb += 32) {
                const int wi = wb + lane;
                uint32_t bits = wi < nw ? S.infl[wi] : 0u;
                while (__any_sync(KV_FULL, bits != 0u)) {
                    int j = -1;
                    bool act = false;
                    if (bits) {
                        j = (wi << 5) + __ffs(bits) - 1;
                        bits &= bits - 1;
                        act = pst[j] + reqi[(off + j) * 4 + 2] > t;
                    }
                    const uint32_t am = __ballot_sync(KV_FULL, act);
                    if (am) {
                        ev += __popc(am);
                        sumc -= warp_sum_i64(act ? (long long)(pst[j] + reqi[(off + j) * 4 + 2]) : 0ll);
                        if (act) {
                            const int rj = arw[j];
                            if (raise) {
                                // ran rounds p..t-1, unfinished (c > t): o >= t - p + 1 (Q26b)
                                const int need = t - pst[j] + 1;
                                if ((int)rqw[rj].y < need) rqw[rj].y = (uint32_t)need;
                                pst[j] = -1;
                            }
                            q_insert(Q, rj);
                            if (P.completion) P.completion[off + j] = -1;
                            if (P.start) P.start[off + j] = -1;
                        }
                    }
                }
                if (wi < nw) S.infl[wi] = 0u;
            }
            __syncwarp();
            if (raise) {
                // re-rank by (o~, idx) with the raised predictions: keys in the ring area
                __threadfence_block();
                __syncwarp();
                uint32_t *keys = reinterpret_cast<uint32_t *>(S.pp);   // pp, pa, rel: 3L words
                const int NPk = next_pow2(max(n, 2));
                for (int k = lane; k < NPk; k += 32)
                    keys[k] = k < n ? (((uint32_t)min((int)rqw[arw[k]].y, 0x1ffff) << 15) | (uint32_t)k) : 0xffffffffu;
                __syncwarp();
                for (int kk = 2; kk <= NPk; kk <<= 1) {
                    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                        for (int i = lane; i < (NPk >> 1); i += 32) {
                            const int lo = ((i & ~(jj - 1)) << 1) | (i & (jj - 1));
                            const int hi = lo + jj;
                            const bool up = (lo & kk) == 0;
                            const uint32_t x = keys[lo], y = keys[hi];
                            if ((x > y) == up) { keys[lo] = y; keys[hi] = x; }
                        }
                        __syncwarp();
                    }
                }
                for (int r = lane; r < n; r += 32) {
                    const int idx = (int)(keys[r] & 0x7fffu);
                    const int4 q = P.req[off + idx];
                    rqw[r] = make_uint4((uint32_t)q.y, keys[r] >> 15, (uint32_t)q.z, (uint32_t)idx);
                    arw[idx] = r;
                }
                __threadfence_block();
                __syncwarp();
                // the waiting queue: every arrived request not in S and not completed
                for (int w = lane; w < nw; w += 32) S.bm[w] = 0u;
                S.sm[lane] = 0u;
                __syncwarp();
                for (int k = lane; k < next; k += 32)
                    if (pst[k] < 0) q_insert(Q, arw[k]);
                __syncwarp();
            }
            // the head is a rank: recompute it over the re-queued set
            h = q_first(Q);
            hstale = h != KV_INF;
            for (int i = lane; i < L; i += 32) { S.pp[i] = 0; S.pa[i] = 0; S.rel[i] = -1; }
            Gp.used = 0u;
            Ga.used = 0u;
            __syncwarp();
            evictions += ev;
            cycle = !raise && next == n && next_at_clear == next && ev == adm_since_clear;
            next_at_clear = next;
            adm_since_clear = 0;
        }
        if (cycle) { status = ST_LIVELOCK; break; }
        if (idle_before && admitted == 0 && h != KV_INF) {
            // S empty and the head does not fit an empty worker (s + o~ > (1-alpha)M): stuck
            // for ever unless a request still to arrive sorts before it (DESIGN Q25)
            bool rescue = false;
            for (int k = next; k < n && !rescue; k += 32) {
                const int kk = k + lane;
                rescue = __any_sync(KV_FULL, kk < n && P.arank[off + kk] < h);
            }
            if (!rescue) { status = ST_LIVELOCK; break; }
        }
        if (had_R || !idle_before) ++rounds;
        const int mnow = ring_jump(S.pa, mask, L, Ga, t, t + 1, t + 1);   // Mem(t+1)
        ring_jump(S.pp, mask, L, Gp, t, t, t + 1);
        peak = max(peak, mnow);
        mem_prev = mnow;
        ++t;

        // Rounds r = t, t+1, ... in which nothing can happen, found 32 at a time: S non-empty
        // and no overflow (0 < Mem(r+1) <= M), no early completion chained on r, no arrival
        // that sorts before the head (any arrival if R is empty), and the head violates
        // Eq. 5 on (1-alpha)M at r (ring_first_fit: the projection only advances meanwhile).
        while (multi && mem_prev > 0) {
            int d = 32;
            if (h != KV_INF) {
                if (hstale) { he = P.rq[off + h]; hstale = false; }
                d = ring_first_fit(S.pp, mask, L, Gp, t, (int)he.x, (int)he.y, B);
            }
            if (d == 0) break;
            int Ta = a_next;
            if (h != KV_INF) {
                Ta = KV_INF;
                for (int k = next; k < n; k += 32) {
                    const int kk = k + lane;
                    const int ak = kk < n ? reqi[(off + kk) * 4] : KV_INF;
                    const bool before = ak < t + 32;
                    const uint32_t m = __ballot_sync(KV_FULL, before && P.arank[off + min(kk, n - 1)] < h);
                    if (m) { Ta = __shfl_sync(KV_FULL, ak, __ffs(m) - 1); break; }
                    if (!__all_sync(KV_FULL, before)) break;
                }
            }
            const int r = t + lane;
            const int v = S.pa[(r + 1) & mask];
            const bool quiet = lane < d && r <= cap && r < Ta && v > 0 && v <= M && S.rel[r & mask] < 0;
            const uint32_t qm = __ballot_sync(KV_FULL, quiet);
            const int k = qm == KV_FULL ? 32 : __ffs(~qm) - 1;          // quiet rounds t..t+k-1
            if (k == 0) break;
            mem_prev = __shfl_sync(KV_FULL, v, k - 1);
            peak = max(peak, ring_jump(S.pa, mask, L, Ga, t, t + k, t + k));
            ring_jump(S.pp, mask, L, Gp, t, t, t + k);
            rounds += k;
            if (h != KV_INF) drounds += k;
            t += k;
            if (k < 32) break;
        }
    }

    if (status == ST_RETRY && raise) {
        // the re-ranks have rewritten this instance's entries, so it cannot restart on the
        // full ring: UNSUPPORTED (documented in kvsched.h)
        fill_unscheduled(P, off, n);
        write_result(P, inst, InstResult{0, 0, 0, 0, 0, 0, ST_UNSUPPORTED});
        return;
    }
    if (status == ST_RETRY) {
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
                const int idx = (int)P.rq[off + r].w;
                if (P.completion) P.completion[off + idx] = -1;
                if (P.start) P.start[off + idx] = -1;
            }
        }
    }
    int mx = -1;
    if (status == ST_OK)
        for (int k = lane; k < n; k += 32) mx = max(mx, pst[k] + reqi[(off + k) * 4 + 2]);
    res.tel = sumc - suma;
    res.rounds = rounds;
    res.decision_rounds = drounds;
    res.evictions = evictions;
    res.makespan = warp_max_i32(mx);
    res.peak = peak;
    res.status = status;
    write_result(P, inst, res);
}

__global__ void __launch_bounds__(128) k_prot(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *base = smem_raw + (size_t)warp * P.warp_bytes;
    ProtSmem S;
    S.pp = reinterpret_cast<int *>(base);
    S.pa = S.pp + P.L;
    S.rel = S.pa + P.L;
    S.bm = reinterpret_cast<uint32_t *>(S.rel + P.L);
    S.infl = S.bm + P.NP / 32;
    S.sm = S.infl + P.NP / 32;

    const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
    long long w = 0;
    if (lane == 0) w = atomicAdd(P.counter, 1ull);
    w = __shfl_sync(KV_FULL, w, 0);
    while (w < n_work) {
        long long nxt = 0;
        if (lane == 0) nxt = atomicAdd(P.counter, 1ull);
        prot_instance(P, P.work_list ? P.work_list[w] : w, S);
        w = __shfl_sync(KV_FULL, nxt, 0);
        __syncwarp();
    }
}

}  // namespace kv
