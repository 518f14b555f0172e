/*
 * kvsched.h -- C ABI of libkvsched.so, the B200 (sm_100a) batched simulator of the online
 * batch scheduler of arXiv 2502.07115 ("Online Scheduling for LLM Inference with KV Cache
 * Constraints") and its baseline policies.
 *
 * Citations "P:<n>" are lines of the paper's LaTeX source.  Where the paper is
 * silent the reading adopted is named "DESIGN Qn" and listed in DESIGN.md.
 *
 * The model.  One worker with KV budget M.  Request i arrives at round a_i with a
 * prompt of s_i tokens and an output of o_i tokens (the scheduler sees a prediction o~_i,
 * P:91).  Started at round p_i it is processed for o_i consecutive unit rounds,
 * holding s_i + k KV slots at round p_i + k for k = 1..o_i (Eq. 3), and completes at
 * c_i = p_i + o_i.  TEL = sum_i (c_i - a_i).
 *
 * Policies.
 *   SCHED_MCSF        Algorithm 1: each round sort the waiting queue by o~
 *                     (ties by arrival position, DESIGN Q5) and admit the longest prefix for
 *                     which Eq. 5 holds at every future round.  o~ > o is allowed
 *                     (the request leaves at p + o, DESIGN Q10); for M > 64 such instances
 *                     run on the protected kernel with alpha = 0, which gives the same
 *                     schedule when o <= o~.
 *   SCHED_MC_BENCH    Algorithm 2: the same test in arrival order, projected
 *                     with the true o.
 *   SCHED_ALPHA       alpha-protection greedy: FCFS admission while the next-
 *                     round occupancy plus s_i+1 stays <= floor((1-alpha)M); when the batch
 *                     of a round needs more than M, every active request is cleared.
 *   SCHED_ALPHA_BETA  alpha-protection beta-clearing: on overflow each active request
 *                     is cleared with probability beta, in whole passes until the batch fits
 *                     (DESIGN Q14); draws are Philox4x32-10 on (t, pass, idx, 0) keyed by
 *                     seed ^ (gid * 0x9E3779B97F4A7C15).
 *   SCHED_MCSF_PROTECTED_RAISE  the same, except that a cleared request re-enters the queue
 *                     with its prediction raised to the tokens it is known to need,
 *                     max(o~, t - p + 1) for a request started at p and cleared at t
 *                     (DESIGN Q26b); instances with more than 3 x 1024 requests, or whose
 *                     rerun needs the full ring, are UNSUPPORTED.
 *   SCHED_MCSF_PROTECTED  MC-SF under prediction error: Algorithm 1 with the
 *                     possibly wrong predictions o~ against the budget floor((1-alpha)M); when
 *                     the realised occupancy of a batch exceeds M every active request is
 *                     cleared and re-queued.
 *
 * Conventions for every entry point.
 *   - Integers only cross the boundary.  All sizes are in KV slots (tokens) and rounds.
 *   - Unless a function says "host", every pointer is a CUDA device pointer on the context's
 *     device, caller-owned; the library never retains or frees caller memory.
 *   - Work is enqueued asynchronously on the context's stream; nothing synchronises the host
 *     unless stated (sched_run_instances synchronises when a size hint is 0, for packed rows
 *     or a latency16 output, and -- on the shared-memory ring path -- when n_instances x
 *     max_requests rows of scratch would exceed 256 MB, to read the true row count).  The
 *     MC policies may also use a library-owned side stream, joined back into the context's
 *     stream before the call's work on it ends.
 *   - Argument errors are detected synchronously, nothing is enqueued, a negative SCHED_E_*
 *     is returned and sched_last_error() describes it.  Per-instance data problems never
 *     fail the call: they set that instance's status (SCHED_INST_*).
 *   - Outputs are a pure function of (inputs, policy, instance_id0): they do not depend on
 *     the grid shape, the number of GPUs or the order instances are processed in.
 */
#ifndef KVSCHED_H
#define KVSCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVSCHED_ABI_VERSION 2

/* return codes */
enum {
    SCHED_OK = 0,
    SCHED_E_ARG = -1,      /* bad argument (null pointer, n < 0, unknown policy, alpha out of
                              [0,1), misaligned req, size limits exceeded)              */
    SCHED_E_CUDA = -2,     /* a CUDA runtime call or kernel launch failed                 */
    SCHED_E_NOMEM = -3,    /* scratch allocation failed                                   */
    SCHED_E_STATE = -4     /* bad context                                                 */
};

/* policies (see above) */
enum { SCHED_MCSF = 0, SCHED_MC_BENCH = 1, SCHED_ALPHA = 2, SCHED_ALPHA_BETA = 3, SCHED_MCSF_PROTECTED = 4,
       SCHED_MCSF_PROTECTED_RAISE = 5 };

/* per-instance status */
enum {
    SCHED_INST_OK = 0,
    SCHED_INST_INVALID = 1,    /* data error: a not sorted, a < 0, s/o/o~ < 1; MC-SF: s+o~ > M
                                  or o~ < o; other policies: s+o > M (DESIGN Q8)          */
    SCHED_INST_LIVELOCK = 2,   /* round cap passed, or alpha head-of-line blocked for ever   */
    SCHED_INST_UNSUPPORTED = 3 /* instance exceeds the caller's size hints / kernel limits
                                  (also: more than 32 requests longer than the ring window
                                  -- 2048 rounds, 1024 for SCHED_MCSF_PROTECTED -- in flight
                                  at once when the full-length ring of the rerun does not
                                  fit shared memory)                                       */
};

/* Limits of this build (sched_run_instances returns SCHED_E_ARG beyond them). */
#define SCHED_MAX_REQUESTS_PER_INSTANCE 32768
#define SCHED_MAX_LEN 32735     /* max over requests of max(o, o~): a 2^15-slot ring covers
                                   a request's window plus the 32-round look-ahead          */

/* sched_policy.flags.  SCHED_FLAG_PER_ROUND makes the MC kernels evaluate Eq. 5 for one
 * round per loop iteration instead of resolving a blocked queue head over up to 64
 * rounds in one warp pass (same results; for A/B measurement).                          */
#define SCHED_FLAG_PER_ROUND 1
/* SCHED_FLAG_WARP_PER_INSTANCE disables the one-lane-per-instance MC kernel (k_mc_lane),
 * which otherwise runs every MC-SF / MC-Benchmark instance within its scope (M <= 64,
 * n <= 96, s <= 7, o~ = o, no round cap) and hands the rest to the one-warp-per-instance
 * kernel (same results; for A/B measurement).                                           */
#define SCHED_FLAG_WARP_PER_INSTANCE 2

typedef struct sched_ctx sched_ctx;   /* opaque: device, stream, scratch, timers */

/* A batch of independent instances in CSR form.                                        */
typedef struct {
    int64_t n_instances;        /* >= 0                                                     */
    const int64_t *req_offset;  /* [n_instances+1]; offset[0] = 0, non-decreasing; the
                                   requests of instance k are rows offset[k]..offset[k+1]-1 */
    const int32_t *req;         /* [n_req][4] rows {a_i, s_i, o_i, o~_i}, 16-byte aligned;
                                   rows of an instance sorted by a (non-decreasing); the row
                                   position inside the instance is the request id idx and
                                   the tie-break of every order (DESIGN Q5).  With req_format
                                   SCHED_REQ_U16X4_DELTA the rows are uint16 {a_i - a_(i-1)
                                   (a_(-1) = 0), s_i, o_i, o~_i}, 8-byte aligned             */
    const int32_t *mem_limit;   /* [n_instances] budget M of each instance           */
    int64_t instance_id0;       /* global id of instance 0 (shards; alpha-beta RNG key gid)  */
    int32_t max_requests;       /* upper bound on requests per instance, or 0 = measure      */
    int32_t max_mem;            /* upper bound on M, or 0 = measure                          */
    int32_t max_len;            /* upper bound on max(o_i, o~_i), or 0 = measure             */
    int32_t req_format;         /* SCHED_REQ_I32X4 (0) or SCHED_REQ_U16X4_DELTA (1): half the
                                   bytes to move; decoded on the device before the run (the
                                   device-pointer call then synchronises once to read the row
                                   count).  Not accepted by sched_latency / sched_lb_sorted.  */
} sched_instances;

enum { SCHED_REQ_I32X4 = 0, SCHED_REQ_U16X4_DELTA = 1, SCHED_REQ_U8X4_DELTA = 2, SCHED_REQ_P16 = 3 };
/* SCHED_REQ_P16: one uint16 per request, bits 0-5 = o_i - 1, bits 6-8 = s_i - 1, bits 9-15 =
 * a_i - a_(i-1) (a_(-1) = 0), and o~_i = o_i (the paper's experiments) -- 2 bytes per
 * request for batches with o <= 64, s <= 8 and arrival gaps <= 127 (the C5 sweep);
 * 2-byte aligned; decoded on the device.                                                 */
/* SCHED_REQ_U8X4_DELTA: rows are uint8 {a_i - a_(i-1) (a_(-1) = 0), s_i, o_i, o~_i}, 4-byte
 * aligned -- a quarter of the int32 bytes for batches whose gaps and sizes fit a byte (the
 * C5 sweep); decoded on the device like SCHED_REQ_U16X4_DELTA.                           */
/* "measure" runs a reduction kernel and synchronises the stream to read the bounds.
 * Instances that exceed a caller-given bound get status SCHED_INST_UNSUPPORTED.            */

typedef struct {
    int32_t policy;             /* SCHED_MCSF .. SCHED_MCSF_PROTECTED_RAISE                  */
    int32_t alpha_num;          /* alpha = alpha_num / alpha_den in [0, 1) (alpha policies and
                                   SCHED_MCSF_PROTECTED);                                   */
    int32_t alpha_den;          /*   budget B = ((den - num) * M) / den (DESIGN Q15)         */
    int32_t flags;              /* SCHED_FLAG_* bits, 0 = defaults                           */
    uint64_t beta_thresh;       /* alpha-beta: evict iff u32 draw < beta_thresh, in [1, 2^32];
                                   round(beta * 2^32); 2^32 = always (beta = 1).  At most
                                   65536 passes per overflow, then LIVELOCK (DESIGN Q29)     */
    uint64_t seed;              /* alpha-beta RNG key                                        */
    int64_t round_cap;          /* > 0: absolute round after which the run is LIVELOCK;
                                   <= 0: min(2^30, 16 (max_a + sum_i o_i) + 64) (DESIGN Q23)  */
} sched_policy;

/* Outputs; every pointer may be NULL (= not requested).                                 */
typedef struct {
    int32_t *completion;        /* [n_req] c_i of the last admission not later evicted, else -1 */
    int32_t *start;             /* [n_req] p_i likewise, else -1                            */
    int64_t *tel;               /* [n_instances] sum_i (c_i - a_i); -1 unless OK      */
    int64_t *rounds;            /* [n_instances] |union_i [a_i, c_i)| (DESIGN Q11); -1 unless OK */
    int64_t *decision_rounds;   /* [n_instances] rounds whose waiting queue was non-empty     */
    int64_t *evictions;         /* [n_instances] requests cleared (alpha policies)           */
    int32_t *makespan;          /* [n_instances] max_i c_i; -1 unless OK                     */
    int32_t *peak_mem;          /* [n_instances] max over processed rounds of the batch's KV
                                   occupancy sum (s_j + t+1 - p_j) (Eq. 3 at t+1)            */
    int32_t *status;            /* [n_instances] SCHED_INST_*                                */
    uint16_t *latency16;        /* [n_req] compact schedule for transfers: c_i - a_i when the
                                   request completed and c_i - a_i <= 65534, else 65535
                                   (completion = a_i + latency16).  Computed on the device
                                   from the completion rounds after the run, or written by
                                   the kernels themselves on the streamed host path (ABI
                                   version 2).                                              */
} sched_outputs;

/* Create a context on `device` that enqueues on `cuda_stream` (a cudaStream_t; NULL = the
 * legacy default stream).  *out receives the context.                                    */
int sched_init(sched_ctx **out, int device, void *cuda_stream);

/* Change the stream later calls enqueue on.                                               */
int sched_set_stream(sched_ctx *ctx, void *cuda_stream);

/* Simulate every instance of `inst` under `pol` (device pointers), on persistent grids.
 * MC policies with M <= 64: one LANE per instance (byte-profile kernel k_mc_lane for n <= 96,
 * k_mc_flatq -- one instance per 8-lane group -- for larger simultaneous-arrival instances),
 * the rest one warp per instance (k_mc_small); MC policies with 64 < M <= 32767: one warp per
 * instance on a 16-bit profile ring (k_mc_prep + k_mc_ring); the alpha policies and larger
 * budgets: the 32-bit ring kernels (k_ring, k_prot) ("Kernels").  Per-instance data errors set that instance's status only.
 * Returns SCHED_E_ARG (nothing enqueued) for bad arguments, including an unknown policy or
 * flag, alpha outside [0, 1), or beta_thresh outside [1, 2^32] for SCHED_ALPHA_BETA.      */
int sched_run_instances(sched_ctx *ctx, const sched_instances *inst, const sched_policy *pol,
                        const sched_outputs *out);

/* Same, with HOST pointers in `inst` and `out` (pinned memory recommended): copies inputs to
 * context-owned device buffers, runs, copies the requested outputs back and synchronises
 * the stream before returning.  The copies overlap the simulation: MC policies with
 * SCHED_REQ_P16 rows (M <= 64) are STREAMED -- one persistent lane launch reads each chunk's
 * wire rows as soon as a stream memory operation flags them landed and the copy-out stream
 * releases chunk k once all its instances are counted; everything else runs as a chunked
 * pipeline (copy-in / kernels / copy-out per chunk on separate streams).  Per-instance int64
 * (resp. int32) outputs laid out field-major at one pitch in host memory are copied with one
 * 2-D copy per chunk.  Uses the driver's stream memory operations (cuStreamWriteValue32 /
 * cuStreamWaitValue32, resolved at run time); without them the chunked pipeline runs.      */
int sched_run_instances_host(sched_ctx *ctx, const sched_instances *inst,
                             const sched_policy *pol, const sched_outputs *out);

/* TEL of every instance from a completion array (device): tel[k] = sum_i (c_i - a_i) over
 * instance k, or -1 if some c_i < 0; *tel_total = sum of the non-negative tel[k].  Either
 * output may be NULL.  Only inst->n_instances, req_offset and req are read.               */
int sched_latency(sched_ctx *ctx, const sched_instances *inst, const int32_t *completion,
                  int64_t *tel, int64_t *tel_total);

/* Lower bound on the hindsight optimum (Eqs. 1-4) of instances whose requests all
 * arrive at the same round: with vol_i = s_i o_i + o_i (o_i+1)/2, V_k the sum of the
 * k smallest volumes and o_(k) the k-th smallest output length, the k-th completion is at
 * least max(ceil(V_k / M), o_(k)) rounds after the arrival (volume argument of P:319), so
 * lb[k] = sum_k max(ceil(V_k / M), o_(k)) <= OPT.  lb[k] = -1 if instance k's arrivals differ
 * or it has more than 8192 requests; 0 if it is empty.  Device pointers; uses
 * inst->max_requests as a hint (0 = measure).                                            */
int sched_lb_sorted(sched_ctx *ctx, const sched_instances *inst, int64_t *lb);

/* Wall clock of a schedule under an affine batch time (SPEC's DurationModel, standing in for
 * the Vidur timing of P:459; DESIGN Q28).  Feasibility stays in rounds; round r (first arrival
 * r0 <= r < makespan) processes tokens(r) = sum_{p_i = r} s_i + #{i : p_i < r < c_i} and lasts
 * c0 + c1 tokens(r); W(r0) = 0.  Per instance k (device pointers; any output may be NULL):
 *   tel_wall[k] = sum_i W(c_i) - W(a_i); makespan_wall[k] = W(max_i c_i)   (-1 if a request
 *   has no schedule, i.e. start or completion < 0);
 *   bins[k][b] = sum of tokens(r) over rounds with floor(W(r) / bin_width) = b < n_bins
 *   (per-bin throughput, Fig. 5);
 *   mem_trace[k][j] = sum_{i: p_i <= r < c_i} (s_i + r + 1 - p_i), r = r0 + j < makespan,
 *   0 beyond (memory over time, Figs. 6 and 9).
 * start / completion are the outputs of sched_run_instances for `inst` (I32X4 rows).      */
typedef struct {
    int64_t c0, c1;             /* batch time c0 + c1 tokens, integer time units (> 0)      */
    int64_t bin_width;          /* throughput bin width in time units (0 = no bins)         */
    int32_t n_bins;             /* bins per instance                                        */
    int32_t trace_len;          /* memory-trace rounds per instance                         */
} sched_clock;

int sched_wallclock(sched_ctx *ctx, const sched_instances *inst, const int32_t *start,
                    const int32_t *completion, const sched_clock *clk, int64_t *tel_wall,
                    int64_t *makespan_wall, int64_t *bins, int32_t *mem_trace);

/* On-device generation of Arrival-Model-2 instances on a lambda x M sweep grid
 * (configuration C5), from an integer counter-based specification; the bytes equal those of
 * the host reference workloads.am2_counter.  Instance k (global id g = instance_id0 + k):
 *   cell = g mod (n_lambda n_m); lambda index = cell / n_m; M = m_values[cell mod n_m];
 *   u(stream, j) = Philox4x32-10(counter (lo32 g, hi32 g, stream, j), key (lo32 seed, hi32 seed));
 *   mulhi(u, r) = (u r) >> 32;
 *   T = T_lo + mulhi(u(0,0)[0], T_hi - T_lo + 1);
 *   arrivals at round r = 1..T: the smallest c with u(1,r)[0] < poisson_cdf[lambda][c];
 *   request i in arrival order: s = s_lo + mulhi(u(2,i)[0], s_hi - s_lo + 1),
 *   o = 1 + mulhi(u(2,i)[1], M - s), o~ = o.
 * poisson_cdf[l][c] = floor(P(Poisson(lambda_l) <= c) 2^32), c = 0..31, the last = 2^32.
 * Requires 0 <= T_lo <= T_hi <= 1024, 1 <= s_lo <= s_hi < every m_value.                */
typedef struct {
    int64_t n_instances;
    int64_t instance_id0;
    uint64_t seed;
    int32_t n_lambda, n_m;
    const uint64_t *poisson_cdf;  /* device [n_lambda][32]                                  */
    const int32_t *m_values;      /* device [n_m]                                           */
    int32_t T_lo, T_hi, s_lo, s_hi;
} sched_gen_am2;

/* req_offset[0..n] (device) <- CSR offsets of the generated batch (count + device scan).   */
int sched_gen_am2_count(sched_ctx *ctx, const sched_gen_am2 *spec, int64_t *req_offset);

/* Fill req [req_offset[n]][4] {a, s, o, o~} and mem_limit [n] (device) for the offsets that
 * sched_gen_am2_count produced.                                                           */
int sched_gen_am2_fill(sched_ctx *ctx, const sched_gen_am2 *spec, const int64_t *req_offset,
                       int32_t *req, int32_t *mem_limit);

/* The counter-based RNG of the alpha-beta policy, exposed for known-answer tests:
 * out[4i..4i+3] = Philox4x32-10(counter ctr[4i..4i+3], key key[2i..2i+1]) (Salmon et al.,
 * SC'11) for i < n.  Device pointers.                                                    */
int sched_philox4x32_10(sched_ctx *ctx, int64_t n, const uint32_t *ctr, const uint32_t *key,
                        uint32_t *out);

/* Kernel accounting of this context since the last reset: number of kernel launches the
 * library made, and the summed device time (ms, CUDA events on the context's stream) of
 * the simulation kernels when timing is enabled.  Host pointers; either may be NULL.     */
int sched_set_timing(sched_ctx *ctx, int enable);
int sched_get_stats(sched_ctx *ctx, int64_t *launches, double *sim_kernel_ms,
                    int64_t *sim_kernel_launches);
int sched_reset_stats(sched_ctx *ctx);

/* Per-kernel split of the same accounting: entry i (0-based, in order of first launch
 * since the last reset) names a simulation kernel (static string) with its summed device
 * time (ms) and launch count.  SCHED_E_ARG when i is out of range (the caller stops
 * there).  Host pointers; any may be NULL.                                               */
int sched_get_kernel_stats(sched_ctx *ctx, int32_t i, const char **name, double *ms,
                           int64_t *launches);

/* Name of the simulation kernel the last sched_run_instances call launched (static string). */
const char *sched_last_kernel(const sched_ctx *ctx);   /* the main one when a call launches several */

/* Release the context's scratch and the context.                                         */
int sched_finalize(sched_ctx *ctx);

/* Text of the last error on this context ("" if none); NULL ctx -> last sched_init error. */
const char *sched_last_error(const sched_ctx *ctx);

/* ABI version compiled into the library (KVSCHED_ABI_VERSION).                          */
int sched_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KVSCHED_H */
