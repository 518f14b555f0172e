// kernel_lane.cuh -- MC-SF / MC-Benchmark with ONE LANE PER INSTANCE (the C5 bench path).
//
// k_mc_small spends a warp on one instance: 32 lanes evaluate Eq. 5 at 64 profile
// positions in parallel, but every control step (queue pop, head decode, loop tests) is
// executed by all 32 lanes for that one instance.  For small budgets (M <= 64) the whole
// projected profile fits in 64 bytes, so here each lane runs its own instance and holds
// its profile in NW registers, four rounds per register (SWAR bytes):
//
//   byte tau-1 of P[0..NW-1] = Prof(t + tau)          (Eq. 5 LHS for the in-flight S)
//
// One loop iteration is one event of the lane's instance.  For the queue head (s, w)
// first_fit() returns the first round offset D at which Eq. 5 holds while the profile only
// advances -- D = 0: it fits now -- by an exact prefix-maximum fixpoint (see there).  The
// lane then jumps D rounds (all decision rounds that admit nothing) and admits the
// head at the landing round in the same iteration (ramp s + tau on tau <= w, Eq. 3 P:105,
// four bytes per add); MC-SF stops the jump early at an arrival that might sort before the
// head.  Rounds with an empty queue are skipped to the next arrival.  The 32 lanes of a
// warp run 32 instances in lock step; a lane whose instance ends is refilled by the warp.
//
// Waiting queue R^(t): a 96-bit rank bitmap in three registers (rank = position in
// (o~, idx) order for MC-SF; idx for MC-Benchmark).  Per-request words live
// in shared memory, column `lane` of a [96][32] u32 array (bank = lane: conflict-free):
//   low half  at position = rank : key {w:6 | s:3 | idx:7}
//   high half at position = idx  : {rank:7 | a_(idx+1) - a_idx : 9}
// Instances are claimed 32 per atomic; the warp stages a claimed instance cooperatively
// (coalesced 16-byte row loads prefetched one refill ahead, stable counting sort on o~ for
// the MC-SF ranks) into the idle lane's column.
//
// Scope (checked per instance): 1 <= n <= 96, M <= 64, 1 <= s <= 7, o~ = o for MC-SF,
// s + o <= M, arrivals sorted with gaps <= 511 and a <= 2^29, the caller's size hints, and no
// user round cap (MC rounds never exceed max_a + sum o <= 2^29 + 95 * 511 + 96 * 63 < 2^30,
// so the default cap min(2^30, 16 (max_a + sum o) + 64) is never reached).  Size
// violations are listed before the launch (k_lane_split), row violations -- including
// invalid instances, whose status the general kernel assigns -- by the kernel; k_mc_small
// runs both lists.  Outputs are identical to k_mc_small's (and the oracle's) field by field.
#pragma once
#include "params.cuh"

namespace kv {

#ifndef KV_LANE_NP
#define KV_LANE_NP 96
#endif
// Requests per instance on the lane path.  96 keeps a warp's shared memory at 14 KB (request
// words + first-fit bytes) so that 16 warps fit an SM; on C5 ~1 % of the instances are
// larger and run on k_mc_small.
constexpr int LANE_NP = KV_LANE_NP;
constexpr int LANE_NC = LANE_NP / 32;        // row chunks of 32 per instance
static_assert(LANE_NP <= 96, "the waiting-queue bitmap has three words");
constexpr int LANE_NW = 16;                  // profile words (bytes tau = 1..64)
constexpr int LANE_WARP_BYTES = LANE_NP * 32 * 4 + 2048;   // request words, F bytes (+ hist in refill)

__device__ __forceinline__ uint32_t rep4(int x) { return (uint32_t)x * 0x01010101u; }
__host__ __device__ constexpr uint32_t tau_word(int i)
{
    return (uint32_t)(4 * i + 1) | ((uint32_t)(4 * i + 2) << 8) | ((uint32_t)(4 * i + 3) << 16) |
           ((uint32_t)(4 * i + 4) << 24);
}
// 0xFF in every byte whose bit 7 is set, 0x00 elsewhere (prmt sign replication)
__device__ __forceinline__ uint32_t sign_bytes(uint32_t m)
{
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(m));
    return r;
}

template <int NW>
struct LaneInst {                            // one lane's instance (registers)
    uint32_t P[NW];
    uint32_t q0, q1, q2;                     // waiting queue bitmap over ranks (<= 96)
    long long inst, off, sumc, suma;
    int t, a_next, next, n, M, h, s, w, hidx;
    int maxc, peak, dr, nr;
    bool active, dec, hstale;
};

// Size scope of the lane path (and the caller's size hints, whose violations k_mc_small
// reports): decided from the CSR offsets and budgets alone, before any row is read.
__device__ __forceinline__ bool lane_size_ok(const KParams &P, int n, int M)
{
    return n >= 1 && n <= (P.lane_max_n > 0 ? P.lane_max_n : LANE_NP) && M <= 64 && n <= P.max_requests &&
           M <= P.max_mem;
}

// Lists the instances outside the size scope (retry_list / retry_count of the KParams it is
// given) so that k_mc_small can run them beside k_mc_lane; one thread per instance,
// warp-aggregated appends.
// With `other` set, an out-of-scope instance whose first and last arrivals differ (it can
// never run on k_mc_flat, which takes simultaneous arrivals) goes to `other` / `other_count`
// instead, so the flat kernel does not stage it only to reject it.
__global__ void k_lane_split(const KParams P, long long *other, unsigned long long *other_count)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (long long k0 = blockIdx.x * (long long)blockDim.x; k0 < P.n_inst; k0 += stride) {
        const long long k = k0 + threadIdx.x;
        bool out = false, flat = false;
        if (k < P.n_inst) {
            const long long n = P.offset[k + 1] - P.offset[k];
            out = !lane_size_ok(P, n > 0x7fffffffll ? 0x7fffffff : (int)n, P.mem[k]);
            if (out) {
                const long long off = P.offset[k] - P.row_base;
                flat = !other || (n > 0 && P.req[off].x == P.req[off + n - 1].x);   // (other = null when streaming)
            }
        }
#pragma unroll
        for (int pass = 0; pass < 2; ++pass) {
            const bool mine = out && (pass == 0 ? flat : !flat);
            const unsigned m = __ballot_sync(KV_FULL, mine);
            if (!m) continue;
            unsigned long long *cnt = pass == 0 ? P.retry_count : other_count;
            long long *list = pass == 0 ? P.retry_list : other;
            unsigned long long base = 0;
            if (lane == __ffs(m) - 1) base = atomicAdd(cnt, (unsigned long long)__popc(m));
            base = __shfl_sync(KV_FULL, base, __ffs(m) - 1);
            if (mine) list[base + __popc(m & ((1u << lane) - 1u))] = k;
        }
    }
}

// -------------------------------------------------------------------------------------
// Work feed of one warp.  Instances are claimed 32 at a time (one atomic); lane j holds
// the CSR offset, size and budget of instance base + j.  The request rows of the next
// instance to stage are loaded one refill ahead (lane l holds rows l, l+32, l+64),
// so the global-memory latency overlaps the simulation instead of stalling the warp.
struct LaneFeed {
    long long base;          // first instance of the batch (warp-uniform)
    int cnt, cur;            // batch size, next instance to stage (warp-uniform)
    long long off;           // lane j: first row of instance base + j
    long long id;            // lane j: that instance (work_list[base + j] with a work list)
    int n, M;                // lane j: its size and budget
    int4 r[LANE_NC];         // rows of instance base + cur (prefetched)
    int rdy;                 // streamed host path: chunks <= rdy are known to have landed
};

// R16: the streamed host path's P16 wire rows, decoded here (load_row_p16)
template <bool R16>
__device__ __forceinline__ void feed_prefetch(const KParams &P, LaneFeed &F)
{
    const int lane = lane_id();
    const long long off = __shfl_sync(KV_FULL, F.off, F.cur);
    const int n = __shfl_sync(KV_FULL, F.n, F.cur);
    const int m = n <= LANE_NP ? n : 0;          // out-of-scope sizes are not staged
    if (R16 && P.stream_ready && m > 0) {        // (streamed host path only) chunks land in
                                                 // order: poll a new one only
        const long long id = __shfl_sync(KV_FULL, F.id, F.cur);
        const int ch = (int)((unsigned)id / (unsigned)P.stream_chunk);
        if (ch > F.rdy) {
            stream_wait(P, id);
            F.rdy = ch;
        }
    }
    if (R16) {
        int carry = 0;
#pragma unroll
        for (int c = 0; c < LANE_NC; ++c) {
            const int k = lane + 32 * c;
            const int4 x = m > 32 * c ? load_row_p16(P, off, k, m, carry) : make_int4(0, 0, 0, 0);
            F.r[c] = k < m ? x : make_int4(0x3fffffff, 1, 1, 1);
        }
        return;
    }
#pragma unroll
    for (int c = 0; c < LANE_NC; ++c) {
        const int k = lane + 32 * c;
        F.r[c] = k < m ? P.req[off + k] : make_int4(0x3fffffff, 1, 1, 1);   // (device path: rows resident)
    }
}

// claim the next batch; false when the work counter is exhausted (warp-uniform)
template <bool R16>
__device__ __forceinline__ bool feed_claim(const KParams &P, LaneFeed &F)
{
    const int lane = lane_id();
    long long base = 0;
    if (lane == 0) base = (long long)atomicAdd(P.counter, 32ull);
    base = __shfl_sync(KV_FULL, base, 0);
    if (base >= P.n_inst) return false;
    F.base = base;
    F.cnt = (int)min(32ll, P.n_inst - base);
    F.cur = 0;
    if (lane < F.cnt) {
        const long long k = P.work_list ? P.work_list[base + lane] : base + lane;
        const long long o0 = P.offset[k];
        F.id = k;
        F.off = o0 - P.row_base;
        F.n = (int)(P.offset[k + 1] - o0);
        F.M = P.mem[k];
    } else {
        F.id = 0;
        F.off = 0;
        F.n = 0;
        F.M = 0;
    }
    feed_prefetch<R16>(P, F);
    return true;
}

// Stage instances into the idle lanes of `idle` (warp-uniform).  Returns false once the
// work counter is exhausted.
template <int POL, int NW, bool R16>
__device__ __forceinline__ bool lane_refill(const KParams &P, uint32_t *data, int *hist, LaneInst<NW> &L,
                                            uint32_t idle, LaneFeed &F)
{
    const int lane = lane_id();
    uint16_t *d16 = reinterpret_cast<uint16_t *>(data);
    while (idle) {
        const int tl = __ffs(idle) - 1;
        if (F.cur >= F.cnt && !feed_claim<R16>(P, F)) return false;
        const long long inst = __shfl_sync(KV_FULL, F.id, F.cur);
        const long long off = __shfl_sync(KV_FULL, F.off, F.cur);
        const int n = __shfl_sync(KV_FULL, F.n, F.cur);
        const int M = __shfl_sync(KV_FULL, F.M, F.cur);
        int4 r[LANE_NC];
#pragma unroll
        for (int c = 0; c < LANE_NC; ++c) r[c] = F.r[c];
        if (++F.cur < F.cnt) feed_prefetch<R16>(P, F);
        // in scope, and within the caller's size hints (k_mc_small reports violations)
        // instances outside the size scope were listed by k_lane_split before this launch
        if (!lane_size_ok(P, n, M)) continue;
        bool ok = true;
        int an[LANE_NC];
        long long suma = 0;
        {
            bool bad = false;
#pragma unroll
            for (int c = 0; c < LANE_NC; ++c) {
                const int k = lane + 32 * c;
                int nx = __shfl_down_sync(KV_FULL, r[c].x, 1);
                const int nx0 = __shfl_sync(KV_FULL, r[c < LANE_NC - 1 ? c + 1 : LANE_NC - 1].x, 0);
                if (lane == 31) nx = nx0;
                an[c] = (k + 1 < n) ? nx - r[c].x : 0;           // a_(k+1) - a_k
                if (k < n) {
                    bad |= r[c].x < 0 || r[c].y < 1 || r[c].y > 7 || r[c].z < 1 || r[c].w < 1 ||
                           r[c].y + r[c].z > M ||
                           r[c].z >= 4 * NW ||             // window within the profile words
                           r[c].x > KV_LANE_MAX_A;         // the default round cap stays out of reach
                    if (POL == POL_MCSF) bad |= r[c].w != r[c].z;
                    bad |= an[c] < 0 || an[c] > 511;
                    suma += r[c].x;
                }
            }
            ok = !__any_sync(KV_FULL, bad);
        }
        if (!ok) {
            if (lane == 0) {
                const unsigned long long slot = atomicAdd(P.retry_count, 1ull);
                P.retry_list[slot] = inst;
            }
            continue;
        }
        suma = warp_sum_i64(suma);
        const int a0 = __shfl_sync(KV_FULL, r[0].x, 0);
        // ranks: (o~, idx) order by a stable counting sort on o~ (MC-SF); idx (MC-Benchmark)
        int rank[LANE_NC];
        if (POL == POL_MCSF) {
            hist[lane] = 0;
            hist[lane + 32] = 0;
            __syncwarp();
#pragma unroll
            for (int c = 0; c < LANE_NC; ++c) {
                const int k = lane + 32 * c;
                const int v = k < n ? r[c].z : 64 + lane;
                const unsigned peers = __match_any_sync(KV_FULL, v);
                if (k < n && __ffs(peers) - 1 == lane) hist[v] += __popc(peers);
                __syncwarp();
            }
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
#pragma unroll
            for (int c = 0; c < LANE_NC; ++c) {
                const int k = lane + 32 * c;
                const int v = k < n ? r[c].z : 64 + lane;
                const unsigned peers = __match_any_sync(KV_FULL, v);
                rank[c] = k < n ? hist[v] + __popc(peers & ((1u << lane) - 1u)) : 0;
                __syncwarp();
                if (k < n && __ffs(peers) - 1 == lane) hist[v] += __popc(peers);
                __syncwarp();
            }
        } else {
#pragma unroll
            for (int c = 0; c < LANE_NC; ++c) rank[c] = lane + 32 * c;
        }
#pragma unroll
        for (int c = 0; c < LANE_NC; ++c) {
            const int k = lane + 32 * c;
            if (k < n) {
                const uint32_t key = (uint32_t)r[c].z | ((uint32_t)r[c].y << 6) | ((uint32_t)k << 9);
                d16[(rank[c] * 32 + tl) * 2] = (uint16_t)key;
                d16[(k * 32 + tl) * 2 + 1] = (uint16_t)(rank[c] | (an[c] << 7));
            }
        }
        __syncwarp();
        if (lane == tl) {
#pragma unroll
            for (int i = 0; i < NW; ++i) L.P[i] = 0u;
            L.q0 = L.q1 = L.q2 = 0u;
            L.inst = inst;
            L.off = off;
            L.sumc = 0;
            L.suma = suma;
            L.t = a0;
            L.a_next = a0;
            L.next = 0;
            L.n = n;
            L.M = M;
            L.h = KV_INF;
            L.s = L.w = L.hidx = 0;
            L.maxc = -1;
            L.peak = 0;
            L.dr = L.nr = 0;
            L.active = true;
            L.dec = false;
            L.hstale = false;
        }
        idle &= idle - 1;
    }
    return true;
}

template <int NW, bool R16>
__device__ __forceinline__ void lane_write_result(const KParams &P, const LaneInst<NW> &L)
{
    if (P.tel) P.tel[L.inst] = L.sumc - L.suma;
    if (P.rounds) P.rounds[L.inst] = (long long)(L.dr + L.nr);
    if (P.drounds) P.drounds[L.inst] = (long long)L.dr;
    if (P.evictions) P.evictions[L.inst] = 0;
    if (P.makespan) P.makespan[L.inst] = L.maxc;
    if (P.peak) P.peak[L.inst] = L.peak;
    if (P.status) P.status[L.inst] = ST_OK;
    if (R16 && P.stream_done) stream_count(P, L.inst);
}

// max over the profile bytes, as 16x2 halves (values <= 64)
template <int NW>
__device__ __forceinline__ uint32_t max_bytes16(const uint32_t (&P)[NW], uint32_t acc)
{
#pragma unroll
    for (int i = 0; i < NW; ++i)
        acc = __vimax3_s16x2_relu(acc, __byte_perm(P[i], 0u, 0x4240), __byte_perm(P[i], 0u, 0x4341));
    return acc;
}

// ... of the bytes tau = 1..d only (a superset of whole words; the rest stay in P and are
// folded later), in tiers so that the common short gaps fold one or two words
template <int NW>
__device__ __forceinline__ uint32_t max_bytes16_prefix(const uint32_t (&P)[NW], uint32_t acc, int d)
{
    if (d <= 4)
        return __vimax3_s16x2_relu(acc, __byte_perm(P[0], 0u, 0x4240), __byte_perm(P[0], 0u, 0x4341));
    if (d <= 8) {
        acc = __vimax3_s16x2_relu(acc, __byte_perm(P[0], 0u, 0x4240), __byte_perm(P[0], 0u, 0x4341));
        return __vimax3_s16x2_relu(acc, __byte_perm(P[1], 0u, 0x4240), __byte_perm(P[1], 0u, 0x4341));
    }
    return max_bytes16(P, acc);
}

// P <- P shifted down by d bytes (Prof(t+d+tau) becomes position tau).  Byte 4 NW - 1 is
// always zero (every window ends before it), so d >= 4 NW - 1 clears the profile.  The
// word stages are predicated moves (FMA pipe); with VOTE a stage is skipped by the whole
// warp when no lane needs it (both kernels measured faster without: KV_*_SHIFT_VOTE 0).
template <int NW, bool VOTE = true>
__device__ __forceinline__ void shift_bytes(uint32_t (&P)[NW], int d)
{
    d = min(d, 4 * NW - 1);
    const int q = d >> 2;
#pragma unroll
    for (int b = 8; b >= 1; b >>= 1) {
        if (b >= NW) continue;
        const bool on = (q & b) != 0;
        if (!VOTE || __any_sync(KV_FULL, on)) {
#pragma unroll
            for (int i = 0; i < NW; ++i)
                if (on) P[i] = i + b < NW ? P[i + b] : 0u;
        }
    }
    const int sh = (d & 3) * 8;
#pragma unroll
    for (int i = 0; i < NW - 1; ++i) P[i] = __funnelshift_r(P[i], P[i + 1], sh);
    P[NW - 1] >>= sh;
}

// x + y on the FMA pipe (IMAD), leaving the ALU pipe -- the kernel's binding resource --
// to the SWAR / DPX work
__device__ __forceinline__ uint32_t add_fma(uint32_t x, uint32_t y)
{
    uint32_t r;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return r;
}

// -------------------------------------------------------------------------------------
// First round offset D >= 0 at which the head (s, w) satisfies Eq. 5 while the profile
// only advances (no admission, arrival or early completion in between).  Position u
// (relative to t) blocks exactly the offsets D in [u - w, c_u - 1] with
//     c_u = max(0, min(u, Prof(t+u) + u - (M - s)))
// (for D < u, u lies in the window [D+1, D+w] iff D >= u - w, and fails iff
// Prof(t+u) + s + u - D > M).  So D is feasible iff every u <= D + w has c_u <= D, i.e.
//     feasible(D)  <=>  F(D + w) <= D,       F(x) = max_{u <= x} c_u,
// and D* is the least fixpoint of D <- F(D + w) from D = 0 (F is non-decreasing, so every
// D skipped by that iteration is infeasible).  Positions past 64 hold no projection
// (c_u = u - (M-s) <= D there), so F(x) = F(min(x, 64)).
// c and F are computed four rounds at a time in 16x2 halves (DPX VIADDMNMX / VIMNMX),
// F is packed to bytes in the lane's shared-memory column, and the fixpoint walks it.
// The same pass folds every profile byte into pk16 (peak memory, see k_mc_lane).
template <int NW>
__device__ __forceinline__ int first_fit(const uint32_t (&P)[NW], int L, int w, unsigned char *fcol,
                                         uint32_t &pk16)
{
    // every 16-bit value below carries a bias of 64 so that it stays positive and plain
    // 32-bit adds (FMA pipe) never carry between the halves
    const uint32_t b64 = 0x00400040u;
    const uint32_t kL = (uint32_t)(64 - L) * 0x00010001u;     // 64 - L in both halves (>= 1)
    uint32_t run = b64;                                       // F of the previous word, both halves
    uint32_t fw[16];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const uint32_t xe = __byte_perm(P[i], 0u, 0x4240);    // Prof at tau = 4i+1, 4i+3
        const uint32_t xo = __byte_perm(P[i], 0u, 0x4341);    // Prof at tau = 4i+2, 4i+4
        pk16 = __vimax3_s16x2_relu(pk16, xe, xo);
        const uint32_t te = (uint32_t)(4 * i + 1) | ((uint32_t)(4 * i + 3) << 16);
        const uint32_t to = (uint32_t)(4 * i + 2) | ((uint32_t)(4 * i + 4) << 16);
        // 64 + c' with c' = min(Prof - L, 0) + tau = min(tau, Prof + tau - L) in [-62, 64];
        // c = max(c', 0) comes from starting the running maximum at the bias
        const uint32_t ce = add_fma(__viaddmin_s16x2(xe, kL, b64), te);
        const uint32_t co = add_fma(__viaddmin_s16x2(xo, kL, b64), to);
        // prefix maximum over tau = 4i+1, 4i+2, 4i+3, 4i+4
        const uint32_t t1 = __vimax3_s16x2_relu(ce, co, run);  // lo = F(4i+2), hi = max(run, c3, c4)
        const uint32_t po = __vimax_s16x2_relu(t1, __byte_perm(t1, 0u, 0x1010));   // (F2, F4)
        const uint32_t pe = __vimax_s16x2_relu(ce, __byte_perm(run, po, 0x5410));  // (F1, F3)
        run = __byte_perm(po, 0u, 0x3232);
        fw[i] = __byte_perm(pe, po, 0x6240);                  // bytes 64 + F(4i+1) .. 64 + F(4i+4)
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

__device__ __forceinline__ int hmax16(uint32_t v) { return max((int)(v & 0xffffu), (int)(v >> 16)); }

// -------------------------------------------------------------------------------------
template <int POL, int NW, bool R16 = false>
__global__ void __launch_bounds__(128, 4) k_mc_lane(const KParams P)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char *wbase = smem_raw + (size_t)warp * LANE_WARP_BYTES;
    uint32_t *data = reinterpret_cast<uint32_t *>(wbase);
    unsigned char *fcol = wbase + LANE_NP * 32 * 4 + lane * 16;   // F bytes: [4][32 lanes][16]
    int *hist = reinterpret_cast<int *>(wbase + LANE_NP * 32 * 4);   // aliases F: refill only
    const uint32_t *col = data + lane;           // this lane's column: word k at col[32 k]

    LaneInst<NW> L;
    L.active = false;
    LaneFeed F;
    F.cnt = F.cur = 0;
    F.rdy = -1;
    uint32_t pk16 = 0u;
    bool more = true;
    for (;;) {
        const uint32_t idle = __ballot_sync(KV_FULL, !L.active);
        if (idle && more) {
            more = lane_refill<POL, NW, R16>(P, data, hist, L, idle, F);
            if (idle & (1u << lane)) pk16 = 0u;
        }
        if (!__any_sync(KV_FULL, L.active)) break;

        // One step of this lane's instance.  No lane leaves the iteration early: the
        // profile shift at the end votes across the warp.
        int jump = 0;
        bool admit = false;
        if (L.active) {
            // arrivals a_i <= t join R^(t)
            while (L.a_next <= L.t) {
                const uint32_t d = col[32 * L.next] >> 16;
                const int r = (int)(d & 127u);
                const uint32_t bit = 1u << (r & 31);
                const int wq = r >> 5;
                L.q0 |= wq == 0 ? bit : 0u;
                L.q1 |= wq == 1 ? bit : 0u;
                L.q2 |= wq == 2 ? bit : 0u;
                if (r < L.h) { L.h = r; L.hstale = true; }
                // streamed host path: the consumed half now keeps a_idx mod 2^16 for the
                // latency16 output (a lane instance's latency is < 2^16, see the scope)
                if (R16) reinterpret_cast<uint16_t *>(const_cast<uint32_t *>(col + 32 * L.next))[1] = (uint16_t)L.a_next;
                L.a_next = (++L.next < L.n) ? L.a_next + (int)(d >> 7) : KV_INF;
            }

            if (L.h == KV_INF) {
                // R empty: every projected byte is final (no admission can add to it); the
                // ones about to leave the profile are folded into the peak first
                if (L.next == L.n) {                         // R and arrivals exhausted: drain S
                    pk16 = max_bytes16(L.P, pk16);
                    if (L.dec) { ++L.dr; L.nr += max(0, L.maxc - L.t - 1); }
                    else L.nr += max(0, L.maxc - L.t);
                    L.peak = max(L.peak, hmax16(pk16));
                    lane_write_result<NW, R16>(P, L);
                    L.active = false;
                } else if (L.maxc <= L.t) {                  // S and R empty: idle until a_next
                    L.t = L.a_next;                          // (the profile is all zero)
                } else {
                    // rounds t .. a_next-1: S only (non-idle while t < maxc), no decision
                    const int tn = L.a_next;
                    pk16 = max_bytes16_prefix(L.P, pk16, min(tn, L.maxc) - L.t);
                    if (L.dec) { ++L.dr; L.nr += max(0, min(tn, L.maxc) - L.t - 1); }
                    else L.nr += max(0, min(tn, L.maxc) - L.t);
                    jump = tn - L.t;
                }
            } else {
                if (L.hstale) {
                    const uint32_t key = col[32 * L.h] & 0xffffu;
                    L.w = (int)(key & 63u);
                    L.s = (int)((key >> 6) & 7u);
                    L.hidx = (int)(key >> 9);
                    L.hstale = false;
                }
                // Eq. 5 for the head at this round and, if it fails, the first round it holds
                const int D = first_fit(L.P, L.M - L.s, L.w, fcol, pk16);
                admit = true;
                if (D > 0) {
                    // rounds t .. t+D-1 are decision rounds that admit nothing; the head is
                    // admitted at t+D in this same step.  MC-SF: an arrival at or before t+D
                    // may sort before the head, so stop at it instead (it joins R there and
                    // the next step decides); MC-Benchmark: arrivals queue behind the head.
                    jump = D;
                    if (POL == POL_MCSF && L.a_next - L.t <= D) {
                        jump = L.a_next - L.t;
                        admit = false;
                    }
                    L.dr += jump;
                }
            }
        }
#ifndef KV_LANE_SHIFT_VOTE
#define KV_LANE_SHIFT_VOTE 0   // predicated stages beat the per-stage vote (C5 2.89 -> 2.83 ms)
#endif
        shift_bytes<NW, KV_LANE_SHIFT_VOTE>(L.P, jump);        // all 32 lanes (jump 0 = no-op)
        if (jump > 0) {
            L.t += jump;
            L.dec = false;
        }
        if (admit) {                                           // p = t, c = t + o (Eq. 3)
            L.dec = true;
            const uint32_t S4 = rep4(L.s);
            const uint32_t Kw = rep4(127 - L.w);
#pragma unroll
            for (int i = 0; i < NW; ++i)
                L.P[i] = add_fma(L.P[i], add_fma(S4, tau_word(i)) & ~sign_bytes(Kw + tau_word(i)));
            const int c = L.t + L.w;
            if (P.start) P.start[L.off + L.hidx] = L.t;
            if (P.completion) P.completion[L.off + L.hidx] = c;
            if (R16 && P.lat16) P.lat16[L.off + L.hidx] = (uint16_t)(c - (int)(col[32 * L.hidx] >> 16));
            L.sumc += c;
            L.maxc = max(L.maxc, c);
            const int h = L.h;
            const uint32_t nb = ~(1u << (h & 31));
            const int wq = h >> 5;
            L.q0 &= wq == 0 ? nb : ~0u;
            L.q1 &= wq == 1 ? nb : ~0u;
            L.q2 &= wq == 2 ? nb : ~0u;
            // next head: lowest set rank (independent selects, no branches)
            int nh = L.q2 ? 63 + __ffs(L.q2) : KV_INF;
            nh = L.q1 ? 31 + __ffs(L.q1) : nh;
            L.h = L.q0 ? __ffs(L.q0) - 1 : nh;
            L.hstale = true;
        }
    }
}

}  // namespace kv
