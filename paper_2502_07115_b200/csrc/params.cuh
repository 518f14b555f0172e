// params.cuh -- launch parameters and the per-instance epilogue shared by the kernels.
#pragma once
#include <stdint.h>
#include "common.cuh"

namespace kv {

enum { POL_MCSF = 0, POL_MCBENCH = 1, POL_ALPHA = 2, POL_ALPHA_BETA = 3, POL_MCSF_PROT = 4, POL_MCSF_PROT_RAISE = 5 };
enum { ST_OK = 0, ST_INVALID = 1, ST_LIVELOCK = 2, ST_UNSUPPORTED = 3, ST_RETRY = 4 /* internal */ };

struct KParams {
    // batch
    long long n_inst;
    const long long *offset;
    long long row_base;         // offset[k] - row_base = row of instance k's first request in req
    const int4 *req;            // {a, s, o, o~}
    const int *mem;
    unsigned long long id0;
    // policy
    int policy, alpha_num, alpha_den, flags;
    unsigned long long beta_thresh, seed;
    long long round_cap;
    // capacity (validated hints)
    int max_requests, max_mem, max_len;
    int NP;                     // per-warp rank capacity (pow2 >= max_requests, >= 32)
    int L;                      // ring kernel: profile ring length (pow2 > max_len + 32)
    int warp_bytes;             // dynamic shared memory per warp
    // outputs (any may be null)
    int *completion, *start;
    long long *tel, *rounds, *drounds, *evictions;
    int *makespan, *peak, *status;
    // scratch
    unsigned long long *counter; // persistent-grid work counter (zeroed before launch)
    int *pstart;                // alpha policies: start round of each request (scratch)
    int *relnext;               // protected MC-SF: early-completion chain links (scratch)
    const uint4 *rq;            // MC-SF ring path: per-rank entries {s, o~, o, idx}
    const int *arank;           // MC-SF ring path: rank of request idx
    long long *retry_list;      // ring kernel: instances handed to the full-ring launch
    unsigned long long *retry_count;
    const long long *work_list; // full-ring launch: the instances to (re)run
    const unsigned long long *work_count;
    uint32_t *flat_keys;        // k_mc_flat: [rows] per-request keys in policy order (scratch)
    long long *early_list;      // k_ring<MCSF>: instances with o~ > o, handed to k_prot (alpha = 0)
    unsigned long long *early_count;
    // rows of the per-request scratch above (sized from the max_requests hint); an instance
    // whose rows fall past it (only possible after an instance that broke the caller's
    // hint) is UNSUPPORTED instead of writing out of bounds
    long long scratch_rows;
    // k_mc_prep -> k_mc_ring (kernel_mcring.cuh)
    uint2 *rq8;                 // [rows] per rank: {s | w << 16, idx}
    int2 *arr8;                 // [rows + 64] per idx (arrival order): {a, rank}
    int *capv;                  // [n_inst] round cap, -1 = instance finished by k_mc_prep / k_prot
    uint32_t *estv;             // [n_inst] work estimate (0 = nothing to simulate) or null
    int lane_max_n;             // k_mc_lane takes instances of at most this many requests (0 = LANE_NP)
    // streamed host path (sched_run_instances_host): request rows land chunk by chunk while
    // the kernels run; instance k belongs to chunk k / stream_chunk.  A kernel waits for
    // stream_ready[chunk] before reading an instance's rows (and reads them past L1), and
    // counts the instance in stream_done[chunk] once its outputs are written.
    const int *stream_ready;    // null = not streamed
    unsigned int *stream_done;
    int *stream_err;            // set if a wait gave up (bounded spin)
    long long stream_chunk;
    // streamed host path with SCHED_REQ_P16 rows: the kernels read the 2-byte wire rows and
    // decode them themselves (load_row_p16), so no decode kernel stands between a chunk's
    // copy and its first reader; null otherwise
    const uint16_t *req16;
    // streamed host path: latency16 (c_i - a_i, 65535 = unscheduled) written by the kernels
    // themselves beside / instead of the completion rounds; null otherwise
    uint16_t *lat16;
};

// wait (lane 0 spins, bounded) until the rows of instance `inst` have landed; warp-uniform
__device__ __forceinline__ void stream_wait(const KParams &P, long long inst)
{
    if (!P.stream_ready) return;
    if (lane_id() == 0) {
        const volatile int *f = P.stream_ready + (unsigned)inst / (unsigned)P.stream_chunk;   // (ni < 2^31)
        long long spins = 0;
        while (*f == 0) {
            __nanosleep(200);
            if (++spins > (1ll << 24)) { atomicExch(P.stream_err, 1); break; }   // ~3 s: give up
        }
        __threadfence();
    }
    __syncwarp();
}

// a request row: past L1 when rows are still landing (a cached line could predate them)
__device__ __forceinline__ int4 load_row(const KParams &P, long long r)
{
    return P.stream_ready ? __ldcg(P.req + r) : P.req[r];
}

// Rows k0 + lane (k = that, all 32 lanes call it together) of an instance in SCHED_REQ_P16
// form ({o-1:6 | s-1:3 | gap:7}, a_(-1) = 0, o~ = o; include/kvsched.h): a_k is the prefix
// sum of the gaps, `carry` = a of the row before k0 (0 for the first chunk; updated).  Rows
// k >= n decode as gap 0.  Read past L1: the rows may still be landing.
__device__ __forceinline__ int4 load_row_p16(const KParams &P, long long off, int k, int n, int &carry)
{
    const int lane = lane_id();
    const uint32_t v = k < n ? (uint32_t)__ldcg(reinterpret_cast<const unsigned short *>(P.req16) + off + k) : 0u;
    int a = (int)(v >> 9);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(KV_FULL, a, d);
        if (lane >= d) a += y;
    }
    a += carry;
    carry = __shfl_sync(KV_FULL, a, 31);
    const int o = (int)(v & 63u) + 1;
    return make_int4(a, (int)((v >> 6) & 7u) + 1, o, o);
}

// the instance's outputs are written: count it for its chunk's release
__device__ __forceinline__ void stream_count(const KParams &P, long long inst)
{
    __threadfence();
    atomicAdd(P.stream_done + (unsigned)inst / (unsigned)P.stream_chunk, 1u);   // (ni < 2^31 when streamed)
}

// Lane 0 writes the per-instance outputs.
__device__ __forceinline__ void write_result(const KParams &P, long long inst, const InstResult &r)
{
    if (P.stream_done) {                // every lane's per-request writes before the count
        __threadfence();
        __syncwarp();
    }
    if (lane_id() != 0) return;
    const bool ok = r.status == ST_OK;
    if (P.tel) P.tel[inst] = ok ? r.tel : -1;
    if (P.rounds) P.rounds[inst] = ok ? r.rounds : -1;
    if (P.drounds) P.drounds[inst] = r.decision_rounds;
    if (P.evictions) P.evictions[inst] = r.evictions;
    if (P.makespan) P.makespan[inst] = ok ? r.makespan : -1;
    if (P.peak) P.peak[inst] = r.peak;
    if (P.status) P.status[inst] = r.status;
    if (P.stream_done) stream_count(P, inst);
}

// Every request of an instance rejected before simulation: completion = start = -1.
__device__ __forceinline__ void fill_unscheduled(const KParams &P, long long off, int n)
{
    for (int k = lane_id(); k < n; k += 32) {
        if (P.completion) P.completion[off + k] = -1;
        if (P.start) P.start[off + k] = -1;
        if (P.lat16) P.lat16[off + k] = 0xffffu;
    }
}

__device__ __forceinline__ long long default_cap(long long amax, long long sum_o)
{
    long long cap = 16 * (amax + sum_o) + 64;          // DESIGN Q23
    return cap > (1ll << 30) ? (1ll << 30) : cap;
}

}  // namespace kv
