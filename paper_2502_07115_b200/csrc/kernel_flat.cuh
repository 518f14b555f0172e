// kernel_flat.cuh -- MC-SF / MC-Benchmark, one LANE per instance, for instances whose
// requests all arrive in the same round (Arrival Model 1; configuration C2) and
// that are too large for k_mc_lane's shared-memory columns.
//
// With every request present from the first round, the waiting queue R^(t) is always a
// suffix of the policy's order -- (o~, idx) for MC-SF, idx for MC-Benchmark
// -- because Algorithm 1 admits the longest feasible prefix and nothing
// ever joins.  So the queue is one integer (the next rank h), and the per-request keys are
// read from global memory one at a time, in rank order, one admission ahead; no per-request
// shared memory is needed and any n (up to the build's limit) fits.  Everything else is
// k_mc_lane's: the byte-SWAR register profile, the exact first-fit fixpoint (first_fit),
// one jump + the admission at its landing round per loop iteration, the peak fold.
//
// Staging (warp-cooperative, per claimed instance): the rows are read once, coalesced;
// the instance is checked (all a equal, s >= 1, 1 <= o < 4 NW, o~ = o for MC-SF, s + o <=
// M, M <= 64, the caller's hints) and, for MC-SF, ranked by a stable counting sort on o~
// (<= 63, __match_any_sync per 32 rows); the packed keys {w:6 | s:6 | idx:15} are written in
// rank order to global scratch.  Instances that fail the checks go to k_mc_small.
#pragma once
#include "kernel_lane.cuh"

namespace kv {

template <int NW>
struct FlatInst {
    uint32_t P[NW];
    uint32_t key, key2;          // keys of ranks h and h+1 (s, w, idx): loaded two ahead
    long long inst, off, sumc, suma;
    int t, n, M, h, maxc, peak, dr, nr;
    bool active, dec;
};

// Claim and stage the next instance of the work list (warp-uniform): validate its rows,
// rank them (MC-SF: stable counting sort on o~) and write the packed keys in policy order.
// Instances outside the kernel's scope are appended to retry_list (k_mc_small runs them).
// false when the list is exhausted.
template <int POL, int NW>
__device__ __forceinline__ bool flat_stage(const KParams &P, uint32_t *keys, int *hist, long long &inst_out,
                                           long long &off_out, int &n_out, int &M_out, int &a0_out)
{
    const int lane = lane_id();
    const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
    for (;;) {
        long long w = 0;
        if (lane == 0) w = (long long)atomicAdd(P.counter, 1ull);
        w = __shfl_sync(KV_FULL, w, 0);
        if (w >= n_work) return false;
        const long long inst = P.work_list ? P.work_list[w] : w;
        const long long off = P.offset[inst] - P.row_base;
        const int n = (int)(P.offset[inst + 1] - P.offset[inst]);
        const int M = P.mem[inst];
        bool ok = n >= 1 && n <= 32767 && M <= 64 && n <= P.max_requests && M <= P.max_mem &&
                  off + n <= P.scratch_rows;
        int a0 = 0;
        if (ok) {
            // one pass: validate and (MC-SF) histogram o~; rows loaded four chunks at a time
            a0 = P.req[off].x;
            // a run ends by a0 + sum o < a0 + 64 n: keep it below the default round cap 2^30
            ok = (long long)a0 + 64ll * n < (1ll << 30);
        }
        if (ok) {
            if (POL == POL_MCSF) {
                hist[lane] = 0;
                hist[lane + 32] = 0;
                __syncwarp();
            }
            bool bad = false;
            for (int k0 = 0; k0 < n; k0 += 128) {
                int4 r[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int k = k0 + 32 * c + lane;
                    r[c] = k < n ? P.req[off + k] : make_int4(a0, 1, 1, 1);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int k = k0 + 32 * c + lane;
                    if (k < n) {
                        bad |= r[c].x != a0 || r[c].x < 0 || r[c].y < 1 || r[c].z < 1 || r[c].w < 1 ||
                               r[c].y + r[c].z > M || r[c].z >= 4 * NW;
                        if (POL == POL_MCSF) bad |= r[c].w != r[c].z;
                    }
                    if (POL == POL_MCSF && k0 + 32 * c < n) {
                        const int v = k < n ? min(max(r[c].z, 0), 63) : 64 + lane;
                        const unsigned peers = __match_any_sync(KV_FULL, v);
                        if (k < n && __ffs(peers) - 1 == lane) hist[v] += __popc(peers);
                        __syncwarp();
                    }
                }
            }
            ok = !__any_sync(KV_FULL, bad);
        }
        if (!ok) {                                              // k_mc_small runs it
            if (lane == 0) {
                const unsigned long long slot = atomicAdd(P.retry_count, 1ull);
                P.retry_list[slot] = inst;
            }
            continue;
        }
        // keys in policy order: stable counting sort on o~ (MC-SF), idx order (MC-Benchmark)
        if (POL == POL_MCSF) {
            const int h0 = hist[2 * lane], h1 = hist[2 * lane + 1];
            int x = h0 + h1;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(KV_FULL, x, d);
                if (lane >= d) x += y;
            }
            __syncwarp();
            hist[2 * lane] = x - h0 - h1;
            hist[2 * lane + 1] = x - h1;
            __syncwarp();
            for (int k0 = 0; k0 < n; k0 += 128) {
                int4 r[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int k = k0 + 32 * c + lane;
                    r[c] = k < n ? P.req[off + k] : make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (k0 + 32 * c >= n) break;
                    const int k = k0 + 32 * c + lane;
                    const int v = k < n ? r[c].z : 64 + lane;
                    const unsigned peers = __match_any_sync(KV_FULL, v);
                    if (k < n) {
                        const int rk = hist[v] + __popc(peers & ((1u << lane) - 1u));
                        keys[off + rk] = (uint32_t)r[c].z | ((uint32_t)r[c].y << 6) | ((uint32_t)k << 12);
                    }
                    __syncwarp();
                    if (k < n && __ffs(peers) - 1 == lane) hist[v] += __popc(peers);
                    __syncwarp();
                }
            }
        } else {
            for (int k = lane; k < n; k += 32) {
                const int4 r = P.req[off + k];
                keys[off + k] = (uint32_t)r.z | ((uint32_t)r.y << 6) | ((uint32_t)k << 12);
            }
        }
        __threadfence_block();
        __syncwarp();
        inst_out = inst;
        off_out = off;
        n_out = n;
        M_out = M;
        a0_out = a0;
        return true;
    }
}

// Stage the next instance of the work list into lane tl (warp-uniform).  false when the
// list is exhausted.
template <int POL, int NW>
__device__ __forceinline__ bool flat_refill(const KParams &P, uint32_t *keys, int *hist, FlatInst<NW> &L, int tl)
{
    long long inst, off;
    int n, M, a0;
    if (!flat_stage<POL, NW>(P, keys, hist, inst, off, n, M, a0)) return false;
    {
        const int lane = lane_id();
        const uint32_t first = keys[off];
        const uint32_t second = n > 1 ? keys[off + 1] : 0u;
        if (lane == tl) {
#pragma unroll
            for (int i = 0; i < NW; ++i) L.P[i] = 0u;
            L.key = first;
            L.key2 = second;
            L.inst = inst;
            L.off = off;
            L.sumc = 0;
            L.suma = (long long)a0 * n;
            L.t = a0;
            L.n = n;
            L.M = M;
            L.h = 0;
            L.maxc = -1;
            L.peak = 0;
            L.dr = L.nr = 0;
            L.active = true;
            L.dec = false;
        }
        return true;
    }
}

// first_fit with a short dependency chain, for the latency-bound flat kernel (few lanes in
// flight): the prefix maximum is taken inside each word first (independent across words),
// then only the word maxima are chained (one max per word) and folded back in.
template <int NW>
__device__ __forceinline__ int first_fit_ll(const uint32_t (&P)[NW], int L, int w, unsigned char *fcol,
                                            uint32_t &pk16)
{
    const uint32_t b64 = 0x00400040u;
    const uint32_t kL = (uint32_t)(64 - L) * 0x00010001u;
    uint32_t pe_l[NW], po_l[NW], mw[NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const uint32_t xe = __byte_perm(P[i], 0u, 0x4240);
        const uint32_t xo = __byte_perm(P[i], 0u, 0x4341);
        pk16 = __vimax3_s16x2_relu(pk16, xe, xo);
        const uint32_t te = (uint32_t)(4 * i + 1) | ((uint32_t)(4 * i + 3) << 16);
        const uint32_t to = (uint32_t)(4 * i + 2) | ((uint32_t)(4 * i + 4) << 16);
        const uint32_t ce = add_fma(__viaddmin_s16x2(xe, kL, b64), te);
        const uint32_t co = add_fma(__viaddmin_s16x2(xo, kL, b64), to);
        const uint32_t t1 = __vimax_s16x2_relu(ce, co);                       // (max c1 c2, max c3 c4)
        po_l[i] = __vimax_s16x2_relu(t1, __byte_perm(t1, 0u, 0x1010));       // (l2, l4)
        pe_l[i] = __vimax_s16x2_relu(ce, __byte_perm(po_l[i], 0u, 0x1044));  // (c1, max(c3, l2))
        mw[i] = __byte_perm(po_l[i], 0u, 0x3232);                            // l4, both halves
    }
    uint32_t run = b64, fw[16];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        fw[i] = __byte_perm(__vimax_s16x2_relu(pe_l[i], run), __vimax_s16x2_relu(po_l[i], run), 0x6240);
        run = __vimax_s16x2_relu(run, mw[i]);
    }
#pragma unroll
    for (int i = NW; i < 16; ++i) fw[i] = 0u;
#pragma unroll
    for (int c = 0; c < (NW + 3) / 4; ++c)
        *reinterpret_cast<uint4 *>(fcol + c * 512) = make_uint4(fw[4 * c], fw[4 * c + 1], fw[4 * c + 2], fw[4 * c + 3]);
    int D = 0;
    for (;;) {
        const int x = min(D + w, 4 * NW) - 1;
        const int f = (int)fcol[(x >> 4) * 512 + (x & 15)] - 64;
        if (f <= D) break;
        D = f;
    }
    return D;
}

template <int POL, int NW>
__global__ void __launch_bounds__(128, 4) k_mc_flat(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wbase = smem_raw + (size_t)warp * 2048;
    unsigned char *fcol = wbase + lane * 16;                 // F bytes: [4][32 lanes][16]
    int *hist = reinterpret_cast<int *>(wbase);              // aliases F: staging only
    uint32_t *keys = P.flat_keys;                            // [rows] keys in policy order

    // lanes that take instances: all 32 unless the grid has more warps than 32-lane warps
    // need (small launches spread the instances thinner, see launch_flat)
    uint32_t lanes = KV_FULL;
    {
        const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
        const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
        const long long lpw = (n_work + warps_total - 1) / warps_total;
        if (lpw < 32) lanes = lpw < 1 ? 1u : (1u << lpw) - 1u;
    }

    FlatInst<NW> L;
    L.active = false;
    uint32_t pk16 = 0u;
    bool more = true;
    for (;;) {
        uint32_t idle = __ballot_sync(KV_FULL, !L.active) & lanes;
        while (idle && more) {
            const int tl = __ffs(idle) - 1;
            more = flat_refill<POL, NW>(P, keys, hist, L, tl);
            if (lane == tl) pk16 = 0u;
            idle &= idle - 1;
        }
        if (!__any_sync(KV_FULL, L.active)) break;

        int jump = 0;
        bool admit = false;
        if (L.active) {
            if (L.h == L.n) {                                // every request admitted: drain S
                pk16 = max_bytes16(L.P, pk16);
                if (L.dec) { ++L.dr; L.nr += max(0, L.maxc - L.t - 1); }
                else L.nr += max(0, L.maxc - L.t);
                L.peak = max(L.peak, hmax16(pk16));
                if (P.tel) P.tel[L.inst] = L.sumc - L.suma;
                if (P.rounds) P.rounds[L.inst] = (long long)(L.dr + L.nr);
                if (P.drounds) P.drounds[L.inst] = (long long)L.dr;
                if (P.evictions) P.evictions[L.inst] = 0;
                if (P.makespan) P.makespan[L.inst] = L.maxc;
                if (P.peak) P.peak[L.inst] = L.peak;
                if (P.status) P.status[L.inst] = ST_OK;
                L.active = false;
            } else {
                // Eq. 5 for the head at this round and, if it fails, the first round it holds;
                // the rounds before it are decision rounds that admit nothing (no arrivals)
                const int w = (int)(L.key & 63u), s = (int)((L.key >> 6) & 63u);
                const int D = first_fit_ll(L.P, L.M - s, w, fcol, pk16);
                jump = D;
                L.dr += D;
                admit = true;
            }
        }
#ifndef KV_FLAT_SHIFT_VOTE
#define KV_FLAT_SHIFT_VOTE 0   // latency-bound launch: predicated stages beat the vote (C2 1.35 -> 1.31 ms)
#endif
        shift_bytes<NW, KV_FLAT_SHIFT_VOTE>(L.P, jump);      // all 32 lanes (jump 0 = no-op)
        if (jump > 0) {
            L.t += jump;
            L.dec = false;
        }
        if (admit) {                                         // p = t, c = t + o (Eq. 3)
            const int w = (int)(L.key & 63u), s = (int)((L.key >> 6) & 63u), idx = (int)(L.key >> 12);
            L.dec = true;
            const uint32_t S4 = rep4(s);
            const uint32_t Kw = rep4(127 - w);
#pragma unroll
            for (int i = 0; i < NW; ++i)
                L.P[i] = add_fma(L.P[i], add_fma(S4, tau_word(i)) & ~sign_bytes(Kw + tau_word(i)));
            const int c = L.t + w;
            if (P.start) P.start[L.off + idx] = L.t;
            if (P.completion) P.completion[L.off + idx] = c;
            L.sumc += c;
            L.maxc = max(L.maxc, c);
            // the next head's key was loaded a step ago; load the one after it now, so the
            // global-memory latency hides behind a whole step
            ++L.h;
            L.key = L.key2;
            if (L.h + 1 < L.n) L.key2 = keys[L.off + L.h + 1];
        }
    }
}


// =======================================================================================
// k_mc_flatq -- the same method with one instance per QUAD of lanes (8 per warp).
//
// k_mc_flat gives an instance one lane, so C2's 10^4 instances fill only ~1.7 warps per SM
// and every admission is one lane's dependent chain over the whole 64-byte profile (issue
// 25 %).  Here lane q of a quad holds profile words 4q..4q+3 (bytes tau = 16q+1 .. 16q+16):
//   * Eq. 5 + the exact first fit: c and the prefix maximum F (first_fit) inside each lane's
//     16 positions, then an exclusive max-scan of the lanes' maxima across the quad (two
//     shuffles); F is written to the quad's 64 bytes of shared memory and the fixpoint
//     D <- F(D + w) reads it (all four lanes, broadcast);
//   * the ramp add is local (each lane its own words);
//   * the profile shift by D bytes goes through the quad's 128-byte shared buffer (words
//     16..31 stay zero): store four words, load five, funnel-shift;
//   * the peak fold is local, max-reduced over the quad when the instance ends.
// Staging is flat_stage (warp-cooperative, as in k_mc_flat); all four lanes of a quad run
// the same instance, so quads diverge only between instances, as lanes did.
// =======================================================================================
template <int WPL>
struct FlatQ {
    uint32_t P[WPL];             // this lane's profile words
    uint32_t key, key2;
    const uint32_t *kp;          // keys of this instance, in policy order
    long long inst, off, sumc, suma;
    int t, n, M, h, maxc, dr, nr;
    bool active, dec;
};

// group-local first fit (G lanes, WPL = 16 / G words each).  ql = lane within the group;
// F = the group's 64 bytes.
template <int G>
__device__ __forceinline__ int flatq_first_fit(const uint32_t (&P)[16 / G], int L, int w, int ql, unsigned char *F,
                                               uint32_t &pk16)
{
    constexpr int WPL = 16 / G;
    const uint32_t b64 = 0x00400040u;
    const uint32_t kL = (uint32_t)(64 - L) * 0x00010001u;
    uint32_t pe_l[WPL], po_l[WPL], mw[WPL];
#pragma unroll
    for (int i = 0; i < WPL; ++i) {
        const int g = WPL * ql + i;                             // global word index
        const uint32_t xe = __byte_perm(P[i], 0u, 0x4240);
        const uint32_t xo = __byte_perm(P[i], 0u, 0x4341);
        pk16 = __vimax3_s16x2_relu(pk16, xe, xo);
        const uint32_t te = (uint32_t)(4 * g + 1) | ((uint32_t)(4 * g + 3) << 16);
        const uint32_t to = te + 0x00010001u;
        const uint32_t ce = add_fma(__viaddmin_s16x2(xe, kL, b64), te);
        const uint32_t co = add_fma(__viaddmin_s16x2(xo, kL, b64), to);
        const uint32_t t1 = __vimax_s16x2_relu(ce, co);
        po_l[i] = __vimax_s16x2_relu(t1, __byte_perm(t1, 0u, 0x1010));
        pe_l[i] = __vimax_s16x2_relu(ce, __byte_perm(po_l[i], 0u, 0x1044));
        mw[i] = __byte_perm(po_l[i], 0u, 0x3232);
    }
    // exclusive prefix over the lane's words, then over the group's lanes
    uint32_t ex[WPL];
    uint32_t run = b64;
#pragma unroll
    for (int i = 0; i < WPL; ++i) {
        ex[i] = run;
        run = __vimax_s16x2_relu(run, mw[i]);
    }
    uint32_t inc = run;
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const uint32_t y = __shfl_up_sync(KV_FULL, inc, d, G);
        if (ql >= d) inc = __vimax_s16x2_relu(inc, y);
    }
    uint32_t before = __shfl_up_sync(KV_FULL, inc, 1, G);       // over lanes < ql
    if (ql == 0) before = b64;
    uint32_t fw[WPL];
#pragma unroll
    for (int i = 0; i < WPL; ++i) {
        const uint32_t r = __vimax_s16x2_relu(ex[i], before);
        fw[i] = __byte_perm(__vimax_s16x2_relu(pe_l[i], r), __vimax_s16x2_relu(po_l[i], r), 0x6240);
    }
    if (WPL == 4) *reinterpret_cast<uint4 *>(F + 16 * ql) = make_uint4(fw[0], fw[1 % WPL], fw[2 % WPL], fw[3 % WPL]);
    else if (WPL == 2) *reinterpret_cast<uint2 *>(F + 8 * ql) = make_uint2(fw[0], fw[1 % WPL]);
    else *reinterpret_cast<uint32_t *>(F + 4 * ql) = fw[0];
    __syncwarp();
    int D = 0;
    for (;;) {
        const int x = min(D + w, 64) - 1;
        const int f = (int)F[x] - 64;
        if (f <= D) break;
        D = f;
    }
    return D;
}

// P <- P shifted down by d bytes across the group (d <= 63; d = 0 is the identity); all
// 32 lanes call it (no vote: on C2 nearly every step shifts)
template <int G>
__device__ __forceinline__ void flatq_shift(uint32_t (&P)[16 / G], int d, int ql, uint32_t *pbuf)
{
    constexpr int WPL = 16 / G;
#pragma unroll
    for (int i = 0; i < WPL; ++i) pbuf[WPL * ql + i] = P[i];
    __syncwarp();
    const int w0 = WPL * ql + (d >> 2), sh = (d & 3) * 8;
    uint32_t v[WPL + 1];
#pragma unroll
    for (int i = 0; i <= WPL; ++i) v[i] = pbuf[w0 + i];              // words >= 16 are zero
#pragma unroll
    for (int i = 0; i < WPL; ++i) P[i] = __funnelshift_r(v[i], v[i + 1], sh);
    __syncwarp();
}

// shared memory per warp: F bytes [32/G groups][64] (>= 256 bytes: also the staging
// histogram), shift buffers [32/G][32 words]
template <int G>
__host__ __device__ constexpr int flatq_fbytes() { return (32 / G) * 64 > 256 ? (32 / G) * 64 : 256; }
template <int G>
__host__ __device__ constexpr int flatq_warp_bytes() { return flatq_fbytes<G>() + (32 / G) * 128; }

template <int POL, int G>
__global__ void __launch_bounds__(128) k_mc_flatq(const KParams P)
{
    constexpr int WPL = 16 / G, NG = 32 / G;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = lane / G, ql = lane % G;
    unsigned char *wbase = smem_raw + (size_t)warp * flatq_warp_bytes<G>();
    unsigned char *F = wbase + 64 * q;
    uint32_t *pbuf = reinterpret_cast<uint32_t *>(wbase + flatq_fbytes<G>() + 128 * q);
    int *hist = reinterpret_cast<int *>(wbase);                  // aliases F: staging only
    uint32_t *keys = P.flat_keys;
#pragma unroll
    for (int i = 0; i < WPL; ++i) pbuf[16 + WPL * ql + i] = 0u;    // zero tail of the shift buffer

    // groups that take instances: all unless the grid has more warps than needed
    uint32_t groups_l = KV_FULL;                                 // lanes of the groups in use
    {
        const long long n_work = P.work_list ? (long long)*P.work_count : P.n_inst;
        const long long warps_total = (long long)gridDim.x * (blockDim.x >> 5);
        const long long gpw = (n_work + warps_total - 1) / warps_total;
        if (gpw < NG) groups_l = gpw < 1 ? ((1u << G) - 1u) : (uint32_t)((1ull << (G * gpw)) - 1ull);
    }

    FlatQ<WPL> L;
    L.active = false;
    uint32_t pk16 = 0u;
    bool more = true;
    __syncwarp();
    for (;;) {
        // idle groups: bit G*k set for group k
        uint32_t idle = __ballot_sync(KV_FULL, !L.active && ql == 0) & groups_l;
        while (idle && more) {
            const int tq = (__ffs(idle) - 1) / G;
            long long inst, off;
            int n, M, a0;
            more = flat_stage<POL, 16>(P, keys, hist, inst, off, n, M, a0);
            if (more && q == tq) {
#pragma unroll
                for (int i = 0; i < WPL; ++i) L.P[i] = 0u;
                L.kp = keys + off;
                L.key = L.kp[0];
                L.key2 = n > 1 ? L.kp[1] : 0u;
                L.inst = inst;
                L.off = off;
                L.sumc = 0;
                L.suma = (long long)a0 * n;
                L.t = a0;
                L.n = n;
                L.M = M;
                L.h = 0;
                L.maxc = -1;
                L.dr = L.nr = 0;
                L.active = true;
                L.dec = false;
                pk16 = 0u;
            }
            idle &= idle - 1;
            __syncwarp();
        }
        if (!__any_sync(KV_FULL, L.active)) break;

        // instances whose every request is admitted: drain S, write the results
        const bool drain = L.active && L.h == L.n;
        if (__any_sync(KV_FULL, drain)) {
            uint32_t pk = max_bytes16(L.P, pk16);
#pragma unroll
            for (int d = 1; d < G; d <<= 1) pk = __vimax_s16x2_relu(pk, __shfl_xor_sync(KV_FULL, pk, d));
            if (drain) {
                if (L.dec) { ++L.dr; L.nr += max(0, L.maxc - L.t - 1); }
                else L.nr += max(0, L.maxc - L.t);
                if (ql == 0) {
                    if (P.tel) P.tel[L.inst] = L.sumc - L.suma;
                    if (P.rounds) P.rounds[L.inst] = (long long)(L.dr + L.nr);
                    if (P.drounds) P.drounds[L.inst] = (long long)L.dr;
                    if (P.evictions) P.evictions[L.inst] = 0;
                    if (P.makespan) P.makespan[L.inst] = L.maxc;
                    if (P.peak) P.peak[L.inst] = hmax16(pk);
                    if (P.status) P.status[L.inst] = ST_OK;
                }
                L.active = false;
            }
        }

        // Eq. 5 for the head at this round and, if it fails, the first round it holds
        // (every group computes; only active ones use it)
        const bool go = L.active;
        const int w = (int)(L.key & 63u), s = (int)((L.key >> 6) & 63u);
        const int D = flatq_first_fit<G>(L.P, (go ? L.M : 64) - s, go ? w : 1, ql, F, pk16);
        const int jump = go ? D : 0;
        flatq_shift<G>(L.P, jump, ql, pbuf);
        if (go) {
            L.dr += D;
            if (jump > 0) L.t += jump;
            // admission at the landing round: p = t, c = t + o (Eq. 3)
            const int idx = (int)(L.key >> 12);
            L.dec = true;
            const uint32_t S4 = rep4(s);
            const uint32_t Kw = rep4(127 - w);
#pragma unroll
            for (int i = 0; i < WPL; ++i) {
                const uint32_t tw = tau_word(0) + (uint32_t)(4 * (WPL * ql + i)) * 0x01010101u;
                L.P[i] = add_fma(L.P[i], add_fma(S4, tw) & ~sign_bytes(Kw + tw));
            }
            const int c = L.t + w;
            if (ql == 0) {
                if (P.start) P.start[L.off + idx] = L.t;
                if (P.completion) P.completion[L.off + idx] = c;
            }
            L.sumc += c;
            L.maxc = max(L.maxc, c);
            ++L.h;
            L.key = L.key2;
            if (L.h + 1 < L.n) L.key2 = L.kp[L.h + 1];
        }
        __syncwarp();
    }
}

}  // namespace kv
