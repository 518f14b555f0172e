// kvsched.cu -- C ABI of libkvsched.so (see include/kvsched.h for the contract).
//
// Host side: argument validation, size bounds, scratch management, kernel selection and
// launch on the context's stream.  All simulation work runs in the kernels of
// kernel_small.cuh / kernel_ring.cuh; there is no CPU path.
#include <cuda.h>            // CUstream / CUdeviceptr types of the stream memory operations only
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>
#include <string.h>

#include <chrono>
#include <utility>
#include <vector>

#include "../../include/kvsched.h"
#include "kernel_clock.cuh"
#include "kernel_gen.cuh"
#include "kernel_lb.cuh"
#include "kernel_prot.cuh"
#include "kernel_ring.cuh"
#include "kernel_mcring.cuh"
#include "kernel_small.cuh"
#include "kernel_lane.cuh"
#include "kernel_flat.cuh"

using namespace kv;

namespace {

constexpr int kBlock = 128;                   // 4 warps, one instance per warp
constexpr int kSmallMaxMem = 64;              // register profile covers tau = 1..64
constexpr int kSmallMaxRequests = 16384;      // 14-bit idx in the packed word
#ifndef KV_RING_SHORT
#define KV_RING_SHORT 2048                    // ring window of the first k_ring launch
#endif
#ifndef KV_PROT_SHORT
#define KV_PROT_SHORT 1024                    // ... and of the first k_prot launch
#endif

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct sched_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    size_t max_smem_optin = 0;
    char err[512] = {0};
    const char *last_kernel = "";
    DevBuf counter, bounds, rq, arank, pstart, relnext, total, retry, scan, dec, h_pk, comp, fkeys;
    DevBuf rq8, arr8, capv, lpt;               // k_mc_prep -> k_mc_ring
    DevBuf h_off, h_req, h_mem, h_out;         // device staging for the host path
    // accounting
    long long launches = 0, sim_launches = 0;
    double sim_ms = 0.0;
    bool timing = false;
    struct Timed {
        cudaEvent_t e0, e1;
        const char *name;
    };
    struct KStat {
        const char *name;
        double ms;
        long long launches;
    };
    std::vector<Timed> pending;
    std::vector<KStat> kstats;
    std::vector<cudaEvent_t> free_events;
    cudaStream_t s_in = nullptr, s_out = nullptr;     // host path copy streams
    cudaStream_t s_side = nullptr;                    // k_mc_small beside k_mc_lane (device path)
    cudaEvent_t ev_split = nullptr, ev_side = nullptr;
    bool side_ok = false;                             // run_impl may use s_side (device path only)
    // streamed host path: rows land chunk by chunk while one persistent lane launch runs
    // (KParams::stream_*); the lane grid leaves `stream_reserve` SMs to the side-stream and
    // latency16 kernels, and the side-stream kernels are capped at `grid_cap` blocks
    bool stream_mode = false;
    bool stream_off = false;                          // retrying a streamed call on the chunked path
    const int *stream_ready = nullptr;
    unsigned int *stream_done = nullptr;
    int *stream_err = nullptr;
    long long stream_chunk = 1;
    int stream_reserve = 0, grid_cap = 0;
    const uint16_t *stream_req16 = nullptr;           // the P16 wire rows the kernels decode
    uint16_t *stream_lat16 = nullptr;                 // latency16 written by the kernels
    std::vector<std::pair<const char *, cudaEvent_t>> *trace = nullptr;   // KVSCHED_STREAM_TRACE marks
    DevBuf sel;                                       // DeviceSelect scratch (streamed path)
    DevBuf sflags;
    int lane_grid_div = 1;                            // host path: lane grid = full occupancy / this
    // host path: extra compute streams, each with its own per-run scratch, so that the
    // kernels of consecutive chunks overlap (one chunk's tail with the next one's start)
    struct RunScratch {
        cudaStream_t stream = nullptr;
        DevBuf counter, bounds, rq, arank, pstart, relnext, retry, comp, fkeys, rq8, arr8, capv, lpt;
    };
    RunScratch extra[7];
    std::vector<cudaEvent_t> chunk_events;
};

static char g_init_err[512];

static int fail(sched_ctx *c, int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c ? c->err : g_init_err, 512, fmt, ap);
    va_end(ap);
    return code;
}

#define CUDA_TRY(ctx, call)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return fail((ctx), SCHED_E_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int grow(sched_ctx *c, DevBuf &b, size_t bytes)
{
    if (bytes <= b.bytes && b.p) return SCHED_OK;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes;
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(c, SCHED_E_NOMEM, "cudaMalloc(%zu) failed", want);
    }
    b.bytes = want;
    return SCHED_OK;
}

cudaEvent_t take_event(sched_ctx *c)
{
    if (!c->free_events.empty()) {
        cudaEvent_t e = c->free_events.back();
        c->free_events.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// ---- bounds: max requests per instance, max M, max(o, o~) -------------------------------
__global__ void k_bounds(long long n_inst, const long long *off, const int4 *req, const int *mem, int *out)
{
    int mn = 0, mm = 0, ml = 0;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n_inst;
         k += (long long)gridDim.x * blockDim.x) {
        const long long lo = off[k], hi = off[k + 1];
        mn = max(mn, (int)min(hi - lo, (long long)KV_INF));
        mm = max(mm, mem[k]);
        for (long long i = lo; i < hi; ++i) ml = max(ml, max(req[i].z, req[i].w));
    }
    mn = __reduce_max_sync(KV_FULL, mn);
    mm = __reduce_max_sync(KV_FULL, mm);
    ml = __reduce_max_sync(KV_FULL, ml);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&out[0], mn);
        atomicMax(&out[1], mm);
        atomicMax(&out[2], ml);
    }
}

// ---- TEL from a completion array: one warp per instance ---------------------------
__global__ void __launch_bounds__(128) k_latency(long long n_inst, const long long *off, const int4 *req,
                                                 const int *comp, long long *tel, unsigned long long *total)
{
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n_inst; k += warps) {
        const long long lo = off[k], hi = off[k + 1];
        long long s = 0;
        bool neg = false;
        for (long long i = lo + lane; i < hi; i += 32) {
            const int c = comp[i];
            neg |= c < 0;
            s += (long long)c - req[i].x;
        }
        neg = __any_sync(KV_FULL, neg);
        s = warp_sum_i64(s);
        if (lane == 0) {
            if (tel) tel[k] = neg ? -1 : s;
            if (total && !neg) atomicAdd(total, (unsigned long long)s);
        }
    }
}

// SCHED_REQ_U16X4_DELTA / SCHED_REQ_U8X4_DELTA -> int32 rows: one warp per instance, a_i =
// prefix sum of the gaps.
// Rows of instance k are input rows offset[k]-row_base.. and output rows likewise.
// the wire rows as {gap, s, o, o~}
__device__ __forceinline__ int4 unpack_row(ushort4 r) { return make_int4(r.x, r.y, r.z, r.w); }
__device__ __forceinline__ int4 unpack_row(uchar4 r) { return make_int4(r.x, r.y, r.z, r.w); }
__device__ __forceinline__ int4 unpack_row(uint16_t v)     // SCHED_REQ_P16: {o-1:6 | s-1:3 | gap:7}
{
    const int o = (v & 63) + 1;
    return make_int4(v >> 9, ((v >> 6) & 7) + 1, o, o);
}

template <typename R>
__global__ void __launch_bounds__(128) k_decode_rows(long long n_inst, const long long *offset, long long row_base,
                                                     const R *in, int4 *out)
{
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); k < n_inst; k += warps) {
        const long long lo = offset[k] - row_base, hi = offset[k + 1] - row_base;
        int carry = 0;
        for (long long b = lo; b < hi; b += 32) {
            const long long i = b + lane;
            const int4 r = i < hi ? unpack_row(in[i]) : make_int4(0, 0, 0, 0);
            int a = r.x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(KV_FULL, a, d);
                if (lane >= d) a += y;
            }
            a += carry;
            if (i < hi) out[i] = make_int4(a, r.y, r.z, r.w);
            carry = __shfl_sync(KV_FULL, a, 31);
        }
    }
}

// decode any packed format into int32 rows on the context's stream
static void launch_decode(sched_ctx *c, int fmt, long long n_inst, const long long *doff, long long row_base,
                          const void *in, int4 *out)
{
    long long blocks = (n_inst + 3) / 4;
    if (blocks > 32LL * c->num_sms) blocks = 32LL * c->num_sms;
    if (blocks < 1) blocks = 1;
    if (fmt == SCHED_REQ_U16X4_DELTA)
        k_decode_rows<ushort4><<<(int)blocks, 128, 0, c->stream>>>(n_inst, doff, row_base, (const ushort4 *)in, out);
    else if (fmt == SCHED_REQ_U8X4_DELTA)
        k_decode_rows<uchar4><<<(int)blocks, 128, 0, c->stream>>>(n_inst, doff, row_base, (const uchar4 *)in, out);
    else
        k_decode_rows<uint16_t><<<(int)blocks, 128, 0, c->stream>>>(n_inst, doff, row_base, (const uint16_t *)in, out);
    c->launches++;
}

// completion rounds -> the compact latency16 output (c_i - a_i, 65535 = none / too large)
__global__ void k_latency16(long long n_rows, const int4 *req, const int *completion, uint16_t *lat)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_rows; i += (long long)gridDim.x * blockDim.x) {
        const int c = completion[i];
        const long long d = (long long)c - req[i].x;
        lat[i] = (c < 0 || d < 0 || d > 65534) ? (uint16_t)65535 : (uint16_t)d;
    }
}

// Instances handed to a full-ring rerun that cannot run: status UNSUPPORTED, no schedule.
__global__ void k_mark_unsupported(const KParams P, const long long *list, const unsigned long long *count)
{
    const long long n = (long long)*count;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (long long w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < n; w += warps) {
        const long long inst = list[w];
        const long long off = P.offset[inst] - P.row_base;
        const int m = (int)(P.offset[inst + 1] - P.offset[inst]);
        fill_unscheduled(P, off, m);
        InstResult res{0, 0, 0, 0, 0, 0, ST_UNSUPPORTED};
        write_result(P, inst, res);
    }
}

__global__ void k_philox(long long n, const uint4 *ctr, const uint2 *key, uint4 *out)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = philox4x32_10(ctr[i], key[i]);
}

// exchange the context's per-run scratch and stream with a host-path compute set
void swap_run_scratch(sched_ctx *c, sched_ctx::RunScratch &r)
{
    std::swap(c->stream, r.stream);
    std::swap(c->counter, r.counter);
    std::swap(c->bounds, r.bounds);
    std::swap(c->rq, r.rq);
    std::swap(c->arank, r.arank);
    std::swap(c->pstart, r.pstart);
    std::swap(c->relnext, r.relnext);
    std::swap(c->retry, r.retry);
    std::swap(c->comp, r.comp);
    std::swap(c->fkeys, r.fkeys);
    std::swap(c->rq8, r.rq8);
    std::swap(c->arr8, r.arr8);
    std::swap(c->capv, r.capv);
    std::swap(c->lpt, r.lpt);
}

template <typename K>
int occupancy_grid(sched_ctx *c, K kernel, int block, int smem, long long work_warps, int *grid)
{
    int per_sm = 0;
    CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
    if (per_sm < 1) return fail(c, SCHED_E_ARG, "kernel does not fit one block per SM (smem %d B)", smem);
    long long blocks = (work_warps + (block / 32) - 1) / (block / 32);
    long long cap = (long long)per_sm * c->num_sms;
    *grid = (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
    return SCHED_OK;
}

// warps per block (1..4) such that the per-warp shared memory fits one block
int warps_per_block(const sched_ctx *c, int warp_bytes)
{
    int w = kBlock / 32;
    while (w > 1 && (size_t)w * warp_bytes > c->max_smem_optin) --w;
    return w;
}

// keys[i] = request count of instance i, ids[i] = i (the lane kernel's largest-first order)
__global__ void k_size_keys(long long n, const long long *offset, uint32_t *keys, long long *ids)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long m = offset[i + 1] - offset[i];
        keys[i] = (uint32_t)(m < 0xffffffffll ? m : 0xffffffffll);
        ids[i] = i;
    }
}

// ids[i] = i, *count = n (the value list and count of the longest-first work list)
__global__ void k_iota(long long n, long long *ids, unsigned long long *count)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        ids[i] = i;
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)n;
}

template <typename K>
int launch_sim(sched_ctx *c, K kernel, const KParams &P, int warp_bytes, const char *name, int max_warps_per_sm = 0)
{
    const int wpb = warps_per_block(c, warp_bytes);
    const int block = 32 * wpb, smem = warp_bytes * wpb;
    if ((size_t)smem > c->max_smem_optin)
        return fail(c, SCHED_E_ARG, "%s needs %d B shared memory per warp", name, warp_bytes);
    CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = 1;
    int rc = occupancy_grid(c, kernel, block, smem, P.n_inst, &grid);
    if (rc) return rc;
    if (max_warps_per_sm < 0) {
        // longest-first claiming with fewer instances than two full waves (C3: 4096 long
        // instances): 16 resident warps per SM, so the longest instances, which start first,
        // run with fewer warps beside them (measured on C3: 29.4 ms vs 34-36 ms at full
        // occupancy, 35 ms at 12, 44 ms at 8; C4, 4x the resident warps, is best full)
        int per_sm = 0;
        CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
        const long long full = (long long)per_sm * wpb * c->num_sms;
        max_warps_per_sm = P.n_inst < 2 * full ? 16 : 0;
    }
    if (max_warps_per_sm > 0) {           // fewer resident warps
        const long long cap = (long long)((max_warps_per_sm + wpb - 1) / wpb) * c->num_sms;
        if (grid > cap) grid = (int)cap;
    }
    if (c->grid_cap > 0 && grid > c->grid_cap) grid = c->grid_cap;    // streamed host path
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        e0 = take_event(c);
        e1 = take_event(c);
        CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    }
    kernel<<<grid, block, smem, c->stream>>>(P);
    CUDA_TRY(c, cudaGetLastError());
    if (c->timing) {
        CUDA_TRY(c, cudaEventRecord(e1, c->stream));
        c->pending.push_back({e0, e1, name});
    }
    c->launches++;
    c->sim_launches++;
    c->last_kernel = name;
    return SCHED_OK;
}

// one-lane-per-instance kernel: 4 warps per block, a persistent grid of full occupancy
template <typename K>
int launch_lane(sched_ctx *c, K kernel, const KParams &P, const char *name)
{
    const int block = 128, smem = 4 * LANE_WARP_BYTES;
    CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = 1;
    int rc = occupancy_grid(c, kernel, block, smem, (P.n_inst + 31) / 32, &grid);
    if (rc) return rc;
    // the host path runs several chunks' lane kernels at once: each gets a share of the SMs,
    // so it has several instances per lane and a short tail
    if (c->lane_grid_div > 1) grid = grid / c->lane_grid_div > c->num_sms ? grid / c->lane_grid_div
                                     : (grid < c->num_sms ? grid : c->num_sms);
    if (c->stream_mode && c->stream_reserve > 0) {   // leave SMs for the streaming helpers
        const int cap = (grid / c->num_sms) * (c->num_sms - c->stream_reserve);
        if (grid > cap && cap > 0) grid = cap;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        e0 = take_event(c);
        e1 = take_event(c);
        CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    }
    kernel<<<grid, block, smem, c->stream>>>(P);
    CUDA_TRY(c, cudaGetLastError());
    if (c->timing) {
        CUDA_TRY(c, cudaEventRecord(e1, c->stream));
        c->pending.push_back({e0, e1, name});
    }
    c->launches++;
    c->sim_launches++;
    c->last_kernel = name;
    return SCHED_OK;
}

// simultaneous-arrival lane kernel: 4 warps per block, 2 KB shared memory per warp
template <typename K>
int launch_flat(sched_ctx *c, K kernel, const KParams &P, const char *name)
{
    // Fewer than 32 x 4 x SMs instances (C2: 10^4 = 313 full warps): one warp per block,
    // and fewer lanes per warp (the kernel derives the count from the grid), so the launch
    // has KV_FLAT_WARPS_PER_SM warps on every SM and each warp's divergent step is the union
    // of fewer lanes' paths.
#ifndef KV_FLAT_WARPS_PER_SM
#define KV_FLAT_WARPS_PER_SM 4
#endif
    long long warps = (P.n_inst + 31) / 32;
    int block = 128;
    if (warps < (long long)KV_FLAT_WARPS_PER_SM * c->num_sms) {
        block = 32;
        warps = std::min<long long>(P.n_inst, (long long)KV_FLAT_WARPS_PER_SM * c->num_sms);
    }
    const int smem = (block / 32) * 2048;
    CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = 1;
    int rc = occupancy_grid(c, kernel, block, smem, warps, &grid);
    if (rc) return rc;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        e0 = take_event(c);
        e1 = take_event(c);
        CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    }
    kernel<<<grid, block, smem, c->stream>>>(P);
    CUDA_TRY(c, cudaGetLastError());
    if (c->timing) {
        CUDA_TRY(c, cudaEventRecord(e1, c->stream));
        c->pending.push_back({e0, e1, name});
    }
    c->launches++;
    c->sim_launches++;
    return SCHED_OK;
}

// k_mc_flatq<POL, G>: one instance per group of G lanes (32/G per warp), 4 warps per block;
// enough warps for one instance per group
template <int G, typename K>
int launch_flatq(sched_ctx *c, K kernel, const KParams &P, const char *name)
{
    const long long warps = (P.n_inst + (32 / G) - 1) / (32 / G);
    const int block = 128, smem = 4 * flatq_warp_bytes<G>();
    CUDA_TRY(c, cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int grid = 1;
    int rc = occupancy_grid(c, kernel, block, smem, warps, &grid);
    if (rc) return rc;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
        e0 = take_event(c);
        e1 = take_event(c);
        CUDA_TRY(c, cudaEventRecord(e0, c->stream));
    }
    kernel<<<grid, block, smem, c->stream>>>(P);
    CUDA_TRY(c, cudaGetLastError());
    if (c->timing) {
        CUDA_TRY(c, cudaEventRecord(e1, c->stream));
        c->pending.push_back({e0, e1, name});
    }
    c->launches++;
    c->sim_launches++;
    return SCHED_OK;
}

int check_common(sched_ctx *c, const sched_instances *inst)
{
    if (!c) return SCHED_E_STATE;
    if (!inst) return fail(c, SCHED_E_ARG, "inst is NULL");
    if (inst->n_instances < 0) return fail(c, SCHED_E_ARG, "n_instances < 0");
    if (inst->req_format != SCHED_REQ_I32X4 && inst->req_format != SCHED_REQ_U16X4_DELTA &&
        inst->req_format != SCHED_REQ_U8X4_DELTA && inst->req_format != SCHED_REQ_P16)
        return fail(c, SCHED_E_ARG, "unknown req_format %d", inst->req_format);
    if (inst->n_instances > 0) {
        if (!inst->req_offset || !inst->mem_limit || !inst->req)
            return fail(c, SCHED_E_ARG, "req_offset, req and mem_limit must be non-NULL");
        if (((uintptr_t)inst->req) & (inst->req_format == SCHED_REQ_I32X4 ? 15u :
                                      inst->req_format == SCHED_REQ_U16X4_DELTA ? 7u :
                                      inst->req_format == SCHED_REQ_U8X4_DELTA ? 3u : 1u))
            return fail(c, SCHED_E_ARG, "req is misaligned for its format");
    }
    if (inst->max_requests < 0 || inst->max_mem < 0 || inst->max_len < 0)
        return fail(c, SCHED_E_ARG, "size hints must be >= 0");
    return SCHED_OK;
}

int check_policy(sched_ctx *c, const sched_policy *pol)
{
    if (!pol) return fail(c, SCHED_E_ARG, "pol is NULL");
    if (pol->policy < SCHED_MCSF || pol->policy > SCHED_MCSF_PROTECTED_RAISE)
        return fail(c, SCHED_E_ARG, "unknown policy %d", pol->policy);
    if (pol->flags & ~(SCHED_FLAG_PER_ROUND | SCHED_FLAG_WARP_PER_INSTANCE))
        return fail(c, SCHED_E_ARG, "unknown flags 0x%x", pol->flags);
    if (pol->policy >= SCHED_ALPHA) {
        if (pol->alpha_den <= 0 || pol->alpha_num < 0 || pol->alpha_num >= pol->alpha_den)
            return fail(c, SCHED_E_ARG, "alpha = %d/%d must lie in [0, 1)", pol->alpha_num, pol->alpha_den);
        if (pol->beta_thresh > (1ull << 32)) return fail(c, SCHED_E_ARG, "beta_thresh must be <= 2^32");
        if (pol->policy == SCHED_ALPHA_BETA && pol->beta_thresh == 0)
            return fail(c, SCHED_E_ARG, "alpha-beta needs beta_thresh >= 1 (beta = 0 never clears)");
    }
    return SCHED_OK;
}

}  // namespace

// =========================================================================================
extern "C" {

int sched_abi_version(void) { return KVSCHED_ABI_VERSION; }

int sched_init(sched_ctx **out, int device, void *cuda_stream)
{
    if (!out) return fail(nullptr, SCHED_E_ARG, "out is NULL");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, SCHED_E_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    }
    if (device < 0 || device >= ndev) return fail(nullptr, SCHED_E_ARG, "device %d out of range", device);
    sched_ctx *c = new sched_ctx();
    c->device = device;
    c->stream = (cudaStream_t)cuda_stream;
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        delete c;
        return fail(nullptr, SCHED_E_CUDA, "cudaGetDeviceProperties failed");
    }
    if (prop.major < 10) {
        delete c;
        return fail(nullptr, SCHED_E_CUDA, "device %d is sm_%d%d; this library is built for sm_100a",
                    device, prop.major, prop.minor);
    }
    c->num_sms = prop.multiProcessorCount;
    c->max_smem_optin = prop.sharedMemPerBlockOptin;
    if (grow(c, c->counter, 64) || grow(c, c->bounds, 64) || grow(c, c->total, 64)) {
        delete c;
        return fail(nullptr, SCHED_E_NOMEM, "scratch allocation failed");
    }
    *out = c;
    return SCHED_OK;
}

int sched_set_stream(sched_ctx *c, void *cuda_stream)
{
    if (!c) return SCHED_E_STATE;
    c->stream = (cudaStream_t)cuda_stream;
    return SCHED_OK;
}

}  // extern "C"

static void trace_mark(sched_ctx *c, const char *what)
{
    if (!c->trace) return;
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    cudaEventRecord(e, c->stream);
    c->trace->push_back({what, e});
}

// Streamed host path: the instances outside the lane kernel's size scope, in instance order
// (a stable selection over the CSR offsets and budgets), on the context's stream.
struct OutOfLane {
    KParams P;
    __device__ bool operator()(long long k) const
    {
        const long long n = P.offset[k + 1] - P.offset[k];
        return !lane_size_ok(P, n > 0x7fffffffll ? 0x7fffffff : (int)n, P.mem[k]);
    }
};

static int select_out_of_lane(sched_ctx *c, const KParams &P, long long *list, unsigned long long *count)
{
    const OutOfLane pred{P};
    cub::CountingInputIterator<long long> ids(0);
    size_t tmp = 0;
    CUDA_TRY(c, cub::DeviceSelect::If(nullptr, tmp, ids, list, count, P.n_inst, pred, c->stream));
    int rc = grow(c, c->sel, tmp + 16);
    if (rc) return rc;
    CUDA_TRY(c, cub::DeviceSelect::If(c->sel.p, tmp, ids, list, count, P.n_inst, pred, c->stream));
    c->launches++;
    return SCHED_OK;
}

// Device-pointer run.  Request rows of instance k start at req_offset[k] - row_base in
// `req` (and in the completion / start outputs): row_base lets the pipelined host path run
// chunks whose rows sit in chunk-local buffers while the offsets stay global.
static int run_impl(sched_ctx *c, const sched_instances *inst, const sched_policy *pol,
                    const sched_outputs *out, long long row_base)
{
    int rc = SCHED_OK;

    int max_req = inst->max_requests, max_mem = inst->max_mem, max_len = inst->max_len;
    if (max_req == 0 || max_mem == 0 || max_len == 0) {
        CUDA_TRY(c, cudaMemsetAsync(c->bounds.p, 0, 16, c->stream));
        long long blocks = (inst->n_instances + 255) / 256;
        if (blocks > 4 * (long long)c->num_sms) blocks = 4 * (long long)c->num_sms;
        k_bounds<<<(int)blocks, 256, 0, c->stream>>>(inst->n_instances, reinterpret_cast<const long long *>(inst->req_offset),
                                                     reinterpret_cast<const int4 *>(inst->req),
                                                     inst->mem_limit, (int *)c->bounds.p);
        CUDA_TRY(c, cudaGetLastError());
        c->launches++;
        int hb[4];
        CUDA_TRY(c, cudaMemcpyAsync(hb, c->bounds.p, 16, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        if (max_req == 0) max_req = hb[0];
        if (max_mem == 0) max_mem = hb[1];
        if (max_len == 0) max_len = hb[2];
    }
    if (max_req > SCHED_MAX_REQUESTS_PER_INSTANCE)
        return fail(c, SCHED_E_ARG, "an instance has %d requests; limit %d", max_req, SCHED_MAX_REQUESTS_PER_INSTANCE);
    if (max_len > SCHED_MAX_LEN) return fail(c, SCHED_E_ARG, "request length %d exceeds limit %d", max_len, SCHED_MAX_LEN);
    if (max_req < 1) max_req = 1;
    if (max_len < 1) max_len = 1;

    KParams P;
    memset(&P, 0, sizeof(P));
    P.n_inst = inst->n_instances;
    P.row_base = row_base;
    P.offset = reinterpret_cast<const long long *>(inst->req_offset);
    P.req = reinterpret_cast<const int4 *>(inst->req);
    P.mem = inst->mem_limit;
    P.id0 = (unsigned long long)inst->instance_id0;
    P.policy = pol->policy;
    P.alpha_num = pol->alpha_num;
    P.alpha_den = pol->alpha_den > 0 ? pol->alpha_den : 1;
    P.flags = pol->flags;
    P.beta_thresh = pol->beta_thresh;
    P.seed = pol->seed;
    P.round_cap = pol->round_cap;
    P.max_requests = max_req;
    P.max_mem = max_mem;
    P.max_len = max_len;
    P.completion = out->completion;
    P.start = out->start;
    P.tel = reinterpret_cast<long long *>(out->tel);
    P.rounds = reinterpret_cast<long long *>(out->rounds);
    P.drounds = reinterpret_cast<long long *>(out->decision_rounds);
    P.evictions = reinterpret_cast<long long *>(out->evictions);
    P.makespan = out->makespan;
    P.peak = out->peak_mem;
    P.status = out->status;
    P.counter = reinterpret_cast<unsigned long long *>(c->counter.p);
    P.scratch_rows = 0x7fffffffffffffffll;            // set below where scratch is sized
    if (c->stream_mode) {
        P.stream_ready = c->stream_ready;
        P.stream_done = c->stream_done;
        P.stream_err = c->stream_err;
        P.stream_chunk = c->stream_chunk;
        P.req16 = c->stream_req16;
        P.lat16 = c->stream_lat16;
    }
    CUDA_TRY(c, cudaMemsetAsync(c->counter.p, 0, 8, c->stream));

    const bool mc = pol->policy == SCHED_MCSF || pol->policy == SCHED_MC_BENCH;
    const int np_small = next_pow2(max_req < 32 ? 32 : max_req);
    if (mc && max_mem <= kSmallMaxMem && max_req <= kSmallMaxRequests &&
        (size_t)small_warp_bytes(np_small) <= c->max_smem_optin) {
        P.NP = np_small;
        P.warp_bytes = small_warp_bytes(P.NP);
        const int smem = P.warp_bytes;
        const bool per_round = pol->flags & SCHED_FLAG_PER_ROUND;
        const bool qreg = P.NP <= 1024;          // waiting queue fits one word per lane
        if (!per_round && !(pol->flags & SCHED_FLAG_WARP_PER_INSTANCE) && pol->round_cap <= 0 &&
            (size_t)LANE_WARP_BYTES * 4 <= c->max_smem_optin) {
            // One lane per instance.  Instances outside its size scope (n > 96, M > 64, hint
            // violations) are listed first by k_lane_split and run by k_mc_small on a side
            // stream: that launch waits for free SM slots, so it fills the lane kernel's tail
            // instead of following it.  Instances the lane kernel rejects on their rows
            // (s > 7, o~ != o, gaps, invalid) are listed by it and run by k_mc_small after.
            const size_t ni = (size_t)inst->n_instances;
            if ((rc = grow(c, c->retry, 128 + 3 * ni * 8))) return rc;
            unsigned long long *cnt = reinterpret_cast<unsigned long long *>(c->retry.p);
            long long *list_b = reinterpret_cast<long long *>((char *)c->retry.p + 128);
            long long *list_a = list_b + ni;
            CUDA_TRY(c, cudaMemsetAsync(c->retry.p, 0, 64, c->stream));
            // KVSCHED_LANE_MAXN (experiments): a lower size limit for the lane kernel, the rest
            // going to the side stream's warp-per-instance kernel
            if (const char *e = getenv("KVSCHED_LANE_MAXN")) P.lane_max_n = atoi(e) > 0 && atoi(e) <= LANE_NP ? atoi(e) : 0;
            {
                KParams S = P;
                S.retry_list = list_a;
                S.retry_count = cnt + 1;
                long long blocks = (inst->n_instances + 255) / 256;
                if (blocks > 8LL * c->num_sms) blocks = 8LL * c->num_sms;
                // out-of-scope instances: simultaneous arrivals to list A (k_mc_flatq), the
                // rest straight to list C (k_mc_small), which the flat kernel's rejects join.
                // (Streamed host path: list A is selected in instance order on the side stream
                // below instead, so the side kernel meets the chunks in the order they land.)
                if (!c->stream_mode) {
                    k_lane_split<<<(int)(blocks > 0 ? blocks : 1), 256, 0, c->stream>>>(S, list_a + ni, cnt + 6);
                    CUDA_TRY(c, cudaGetLastError());
                    c->launches++;
                } else if ((rc = select_out_of_lane(c, P, list_a, cnt + 1))) {   // before the lane launch
                    return rc;                                                   // takes the SMs
                }
            }
            const bool side = c->side_ok;
            if (side) {
                if (!c->s_side) CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking));
                if (!c->ev_split) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_split, cudaEventDisableTiming));
                if (!c->ev_side) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
                CUDA_TRY(c, cudaEventRecord(c->ev_split, c->stream));
            }
            P.retry_count = cnt;
            P.retry_list = list_b;
            // profile words: bytes tau = 1 .. 4 NW with byte 4 NW - 1 never reached by a window
            const int nw = max_len < 16 ? 4 : max_len < 32 ? 8 : max_len < 52 ? 13 : 16;
            const bool sf = pol->policy == SCHED_MCSF;
            // Small batches (at most four lanes' worth of instances per lane slot: the 4- and
            // 8-GPU shards of the strong split) claim the largest instances first -- ids sorted
            // by request count (CUB radix sort) -- so the long instances do not end the launch:
            // 2.5*10^5 instances 0.91 -> 0.81 ms, 1.25*10^5 0.61 -> 0.49 ms.  At 10^6 (one GPU) it
            // gains 3 % (2.86 -> 2.76 ms) but scatters rows and results (2.56 GB of DRAM per
            // launch instead of 1.94), so large batches keep index order; size tiers or
            // 32-instance groups ordered by size measured no gain; the host path's quarter-grid
            // chunks measured slower with it.  KVSCHED_LANE_LPT=0/1 overrides.
            const char *llpt = getenv("KVSCHED_LANE_LPT");
            const bool lane_lpt = llpt && llpt[0] && !c->stream_mode ? llpt[0] == '1'
                                                  : c->lane_grid_div == 1 && !c->stream_mode &&
                                                        ni <= 4ull * 32 * 16 * (size_t)c->num_sms;
            if (lane_lpt && ni > 32 && ni < (1ull << 31)) {
                const size_t ng = ni;
                size_t tmp = 0;
                cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                          (const long long *)nullptr, (long long *)nullptr, (int)ng, 0, 32,
                                                          c->stream);
                const size_t a8 = (ng * 4 + 15) & ~(size_t)15;
                if ((rc = grow(c, c->lpt, 2 * a8 + 2 * ng * 8 + tmp + 256))) return rc;
                char *b = reinterpret_cast<char *>(c->lpt.p);
                uint32_t *keys = reinterpret_cast<uint32_t *>(b), *keys2 = reinterpret_cast<uint32_t *>(b + a8);
                long long *ids = reinterpret_cast<long long *>(b + 2 * a8), *order = ids + ng;
                k_size_keys<<<(int)std::min<long long>((long long)(ng + 255) / 256, 4LL * c->num_sms), 256, 0, c->stream>>>(
                    (long long)ni, P.offset, keys, ids);
                CUDA_TRY(c, cudaGetLastError());
                CUDA_TRY(c, cub::DeviceRadixSort::SortPairsDescending(b + 2 * a8 + 2 * ng * 8, tmp, keys, keys2, ids, order,
                                                                      (int)ng, 0, 32, c->stream));
                c->launches += 2;
                P.work_list = order;
            }
#define KV_LANE(NWV) (P.req16 ? (sf ? launch_lane(c, k_mc_lane<POL_MCSF, NWV, true>, P, "k_mc_lane<MCSF,p16>")      \
                                    : launch_lane(c, k_mc_lane<POL_MCBENCH, NWV, true>, P, "k_mc_lane<MCBENCH,p16>")) \
                         : sf ? launch_lane(c, k_mc_lane<POL_MCSF, NWV>, P, "k_mc_lane<MCSF>")                  \
                              : launch_lane(c, k_mc_lane<POL_MCBENCH, NWV>, P, "k_mc_lane<MCBENCH>"))
            trace_mark(c, "lane0");
            rc = nw == 4 ? KV_LANE(4) : nw == 8 ? KV_LANE(8) : nw == 13 ? KV_LANE(13) : KV_LANE(16);
            trace_mark(c, "lane1");
            P.work_list = nullptr;
#undef KV_LANE
            if (rc) return rc;
            P.retry_list = nullptr;
            P.retry_count = nullptr;
            auto small = [&](const KParams &Q) -> int {
                if (per_round) return SCHED_E_STATE;           // not reached: per-round skips the lane path
                if (pol->policy == SCHED_MCSF)
                    return qreg ? launch_sim(c, k_mc_small<POL_MCSF, true, true>, Q, smem, "k_mc_small<MCSF>")
                                : launch_sim(c, k_mc_small<POL_MCSF, true, false>, Q, smem, "k_mc_small<MCSF,smemq>");
                return qreg ? launch_sim(c, k_mc_small<POL_MCBENCH, true, true>, Q, smem, "k_mc_small<MCBENCH>")
                            : launch_sim(c, k_mc_small<POL_MCBENCH, true, false>, Q, smem, "k_mc_small<MCBENCH,smemq>");
            };
            // list A (size scope): beside the lane kernel on the side stream, or after it.
            // Instances whose requests all arrive together (Arrival Model 1) run one per lane
            // on k_mc_flat; the rest of the list goes on to k_mc_small (list C).
            KParams A = P;
            A.work_list = list_a;
            A.work_count = cnt + 1;
            A.counter = cnt + 2;
            long long *list_c = list_a + ni;
            const size_t key_rows = (size_t)inst->n_instances * (size_t)max_req;   // row bound
            // (streamed host path: no flat kernel -- its staging would read rows still landing)
            const bool flat = !c->stream_mode && key_rows * 4 <= ((size_t)2 << 30) && !grow(c, c->fkeys, key_rows * 4 + 4);
            KParams C = A;                   // list C: k_lane_split's non-simultaneous + flat rejects
            C.work_list = list_c;
            C.work_count = cnt + 6;
            C.counter = cnt + 7;
            auto fallback = [&]() -> int {
                if (!flat) {
                    const int r = small(A);
                    return r ? r : small(C);
                }
                KParams F = A;
                F.flat_keys = reinterpret_cast<uint32_t *>(c->fkeys.p);
                F.scratch_rows = (long long)key_rows;
                F.retry_list = list_c;
                F.retry_count = cnt + 6;
                const int fnw = max_len < 16 ? 4 : max_len < 32 ? 8 : max_len < 52 ? 13 : 16;
                int r;
#define KV_FLAT(NWV) (sf ? launch_flat(c, k_mc_flat<POL_MCSF, NWV>, F, "k_mc_flat<MCSF>")                 \
                         : launch_flat(c, k_mc_flat<POL_MCBENCH, NWV>, F, "k_mc_flat<MCBENCH>"))
                // one instance per quad of lanes (k_mc_flatq); KVSCHED_FLAT_LANE=1 keeps one
                // lane per instance (k_mc_flat, A/B only)
                const char *fl_env = getenv("KVSCHED_FLAT_LANE");
                if (fl_env && fl_env[0] == '1')
                    r = fnw == 4 ? KV_FLAT(4) : fnw == 8 ? KV_FLAT(8) : fnw == 13 ? KV_FLAT(13) : KV_FLAT(16);
                else if (fl_env && fl_env[0] == '4')
                    r = sf ? launch_flatq<4>(c, k_mc_flatq<POL_MCSF, 4>, F, "k_mc_flatq<MCSF>")
                           : launch_flatq<4>(c, k_mc_flatq<POL_MCBENCH, 4>, F, "k_mc_flatq<MCBENCH>");
                else if (fl_env && fl_env[0] == '2')
                    r = sf ? launch_flatq<16>(c, k_mc_flatq<POL_MCSF, 16>, F, "k_mc_flatq<MCSF>")
                           : launch_flatq<16>(c, k_mc_flatq<POL_MCBENCH, 16>, F, "k_mc_flatq<MCBENCH>");
                else
                    r = sf ? launch_flatq<8>(c, k_mc_flatq<POL_MCSF, 8>, F, "k_mc_flatq<MCSF>")
                           : launch_flatq<8>(c, k_mc_flatq<POL_MCBENCH, 8>, F, "k_mc_flatq<MCBENCH>");
#undef KV_FLAT
                if (r) return r;
                return small(C);
            };
            if (side) {
                std::swap(c->stream, c->s_side);
                rc = cudaStreamWaitEvent(c->stream, c->ev_split, 0) == cudaSuccess ? SCHED_OK
                         : fail(c, SCHED_E_CUDA, "cudaStreamWaitEvent failed");
                trace_mark(c, "side0");
                if (!rc) rc = fallback();
                trace_mark(c, "side1");
                if (!rc && cudaEventRecord(c->ev_side, c->stream) != cudaSuccess)
                    rc = fail(c, SCHED_E_CUDA, "cudaEventRecord failed");
                std::swap(c->stream, c->s_side);
            } else {
                rc = fallback();
            }
            if (rc) return rc;
            // list B (rows out of scope; usually empty): a small grid after the lane kernel
            KParams B = P;
            B.work_list = list_b;
            B.work_count = cnt;
            B.counter = cnt + 3;
            B.n_inst = std::min<long long>(P.n_inst, 8LL * c->num_sms);   // grid size only
            rc = small(B);
            if (rc) return rc;
            if (side) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_side, 0));
            c->last_kernel = sf ? "k_mc_lane<MCSF>" : "k_mc_lane<MCBENCH>";   // the main kernel of the call
            return SCHED_OK;
        }
#define KV_SMALL(POLV, MULTIV, QREGV, NAME) launch_sim(c, k_mc_small<POLV, MULTIV, QREGV>, P, smem, NAME)
        if (pol->policy == SCHED_MCSF) {
            if (per_round) return qreg ? KV_SMALL(POL_MCSF, false, true, "k_mc_small<MCSF,per-round>")
                                       : KV_SMALL(POL_MCSF, false, false, "k_mc_small<MCSF,per-round,smemq>");
            return qreg ? KV_SMALL(POL_MCSF, true, true, "k_mc_small<MCSF>")
                        : KV_SMALL(POL_MCSF, true, false, "k_mc_small<MCSF,smemq>");
        }
        if (per_round) return qreg ? KV_SMALL(POL_MCBENCH, false, true, "k_mc_small<MCBENCH,per-round>")
                                   : KV_SMALL(POL_MCBENCH, false, false, "k_mc_small<MCBENCH,per-round,smemq>");
        return qreg ? KV_SMALL(POL_MCBENCH, true, true, "k_mc_small<MCBENCH>")
                    : KV_SMALL(POL_MCBENCH, true, false, "k_mc_small<MCBENCH,smemq>");
#undef KV_SMALL
    }

    // ring kernel.  The first launch uses a window of L_short <= KV_RING_SHORT slots (long
    // requests go through the per-lane long list); instances that overflow the list are
    // rerun by a second launch whose ring covers every request plus the 32-round look-ahead.
    P.NP = next_pow2(max_req < 32 ? 32 : max_req);
    const int L_full = next_pow2(max_len + 33);
    // the protected kernel keeps three per-warp rings: a 1024-slot window doubles its
    // occupancy (measured 1.48x faster on C4 with eps = 0.2 than 2048, 512 is slower)
    int ring_short = pol->policy >= SCHED_MCSF_PROTECTED ? KV_PROT_SHORT : KV_RING_SHORT;   // KVSCHED_RING_WINDOW: experiments only
    if (const char *e = getenv("KVSCHED_RING_WINDOW")) {
        const int v = atoi(e);
        if (v >= 64 && (v & (v - 1)) == 0) ring_short = v;
    }
    int L_short = L_full < ring_short ? L_full : ring_short;
    P.L = L_short;
    const bool prot = pol->policy >= SCHED_MCSF_PROTECTED;
    // MC policies with M <= 32767: the 16-bit profile ring with staged arrivals
    // (kernel_mcring.cuh); KVSCHED_OLD_RING=1 keeps the 32-bit k_ring (A/B only)
    const char *old_ring = getenv("KVSCHED_OLD_RING");
    const bool mcr = mc && max_mem <= 32767 && !(old_ring && old_ring[0] == '1');
    auto wbytes = [&](int L) {
        return mcr ? mcring_warp_bytes(L, P.NP) : prot ? prot_warp_bytes(L, P.NP) : ring_warp_bytes(L, P.NP, pol->policy);
    };
    // MC ring path, batches under two full waves (the launch keeps 16 resident warps per SM,
    // launch_sim): those 16 warps fit a 4096-slot window, so fewer long requests take the
    // per-position path past the ring (C3: 28.9 -> 26.6-27.0 ms; the full-occupancy batches of
    // C4 keep 2048, where a larger window would halve the resident warps)
    if (mcr && !getenv("KVSCHED_RING_WINDOW") && L_full > L_short && KV_RING_SHORT < 4096) {
        int ps2 = 0, ps4 = 0;
        auto kr = k_mc_ring<POL_MCSF, false>;
        const int b2 = 4 * wbytes(L_short), b4 = 4 * wbytes(4096);
        if ((size_t)b4 <= c->max_smem_optin) {
            CUDA_TRY(c, cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, b4));
            CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps2, kr, 128, b2));
            CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps4, kr, 128, b4));
            const long long full = (long long)ps2 * 4 * c->num_sms;
            if ((long long)inst->n_instances < 2 * full && ps4 * 4 >= 16) {
                L_short = L_full < 4096 ? L_full : 4096;
                P.L = L_short;
            }
        }
    }
    P.warp_bytes = wbytes(P.L);
    if ((size_t)P.warp_bytes > c->max_smem_optin)
        return fail(c, SCHED_E_ARG, "ring kernel needs %d B shared memory per warp (L=%d, NP=%d)",
                    P.warp_bytes, P.L, P.NP);
    // retry scratch: counters {ring retry, early, k_prot retry}, then their three lists
    const size_t ni = (size_t)inst->n_instances;
    if ((rc = grow(c, c->retry, 64 + 3 * ni * 8))) return rc;
    unsigned long long *rcnt = reinterpret_cast<unsigned long long *>(c->retry.p);
    P.retry_count = rcnt;
    P.retry_list = reinterpret_cast<long long *>((char *)c->retry.p + 64);
    CUDA_TRY(c, cudaMemsetAsync(c->retry.p, 0, 24, c->stream));
    // MC-SF with early completions (o~ > o) runs on k_prot with alpha = 0 (same schedule:
    // with o <= o~ the realised occupancy never exceeds the projection)
    const bool early = pol->policy == SCHED_MCSF;
    if (early) {
        P.early_list = P.retry_list + ni;
        P.early_count = rcnt + 1;
    }
    // per-request scratch rows: n_instances * max_requests bounds the row count without a
    // device read; for very ragged batches that bound is loose, so read the true count
    size_t slots = (size_t)inst->n_instances * (size_t)max_req;
    if (slots * 20 > ((size_t)256 << 20)) {
        long long last = 0, first = 0;
        CUDA_TRY(c, cudaMemcpyAsync(&last, inst->req_offset + inst->n_instances, 8, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(&first, inst->req_offset, 8, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        const size_t rows = (size_t)(last - first > 0 ? last - first : 1);
        if (rows < slots) slots = rows;
    }
    const char *name = "";
    P.scratch_rows = (long long)slots;
    bool lpt = false;
    uint32_t *lpt_est = nullptr, *lpt_est_sorted = nullptr;
    long long *lpt_ids = nullptr, *lpt_order = nullptr;
    unsigned long long *lpt_count = nullptr;
    void *lpt_tmp = nullptr;
    size_t lpt_tmp_bytes = 0;
    // resident warps per SM of the longest-first launch (KVSCHED_MCRING_WPS: experiments)
    int mcring_wps = -1;                // -1: the rule in launch_sim
    if (const char *e = getenv("KVSCHED_MCRING_WPS")) mcring_wps = atoi(e);
    if (mcr) {
        // k_mc_prep: statuses of invalid / unsupported instances, ranks, the rq8 / arr8
        // streams and round caps; MC-SF instances with o~ > o get k_prot's entries instead
        if ((rc = grow(c, c->rq8, slots * 8)) || (rc = grow(c, c->arr8, (slots + 64) * 8)) ||
            (rc = grow(c, c->capv, ni * 4 + 4)))
            return rc;
        P.rq8 = reinterpret_cast<uint2 *>(c->rq8.p);
        P.arr8 = reinterpret_cast<int2 *>(c->arr8.p);
        P.capv = reinterpret_cast<int *>(c->capv.p);
        // longest-first claiming (KVSCHED_LPT=0 turns it off, A/B only): the prep writes a
        // work estimate per instance, a radix sort orders the ids by it, and the simulation
        // claims from that list; layout est | est_sorted | ids | order | count | cub temp
        const char *lpt_env = getenv("KVSCHED_LPT");
        lpt = ni > 1 && ni < (1ull << 31) && !(lpt_env && lpt_env[0] == '0');
        if (lpt) {
            size_t tmp = 0;
            cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                      (const long long *)nullptr, (long long *)nullptr, (int)ni, 0, 32,
                                                      c->stream);
            const size_t a8 = (ni * 4 + 15) & ~(size_t)15;
            if ((rc = grow(c, c->lpt, 2 * a8 + 2 * ni * 8 + 16 + tmp + 256))) return rc;
            char *b = reinterpret_cast<char *>(c->lpt.p);
            lpt_est = reinterpret_cast<uint32_t *>(b);
            lpt_est_sorted = reinterpret_cast<uint32_t *>(b + a8);
            lpt_ids = reinterpret_cast<long long *>(b + 2 * a8);
            lpt_order = lpt_ids + ni;
            lpt_count = reinterpret_cast<unsigned long long *>(lpt_order + ni);
            lpt_tmp = b + 2 * a8 + 2 * ni * 8 + 16;
            lpt_tmp_bytes = tmp;
            P.estv = lpt_est;
            k_iota<<<(int)std::min<long long>((long long)(ni + 255) / 256, 4LL * c->num_sms), 256, 0, c->stream>>>(
                (long long)ni, lpt_ids, lpt_count);
            CUDA_TRY(c, cudaGetLastError());
            c->launches++;
        }
        if (early) {
            if ((rc = grow(c, c->rq, slots * 16)) || (rc = grow(c, c->arank, slots * 4))) return rc;
            P.rq = reinterpret_cast<const uint4 *>(c->rq.p);
            P.arank = reinterpret_cast<const int *>(c->arank.p);
        }
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (c->timing) {
            e0 = take_event(c);
            e1 = take_event(c);
            CUDA_TRY(c, cudaEventRecord(e0, c->stream));
        }
        uint4 *rq_e = reinterpret_cast<uint4 *>(c->rq.p);
        int *ar_e = reinterpret_cast<int *>(c->arank.p);
        // MC-SF instances of KV_PREP_CTA_LO < n <= KV_PREP_WARP_N requests: one 256-thread CTA
        // each (CUB block radix sort of the keys); smaller ones (and MC-Benchmark, which sorts
        // nothing): one warp each
        const int w_hi = early && KV_PREP_CTA_LO < KV_PREP_WARP_N ? KV_PREP_CTA_LO : KV_PREP_WARP_N;
        {   // instances of <= w_hi requests: one warp each
            auto prep_w = early ? k_mc_prep_w<POL_MCSF> : k_mc_prep_w<POL_MCBENCH>;
            int per_sm = 1;
            CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep_w, 256, 0));
            long long blocks = (long long)(per_sm > 0 ? per_sm : 1) * c->num_sms;
            const long long need = (inst->n_instances + 7) / 8;
            if (blocks > need) blocks = need > 0 ? need : 1;
            prep_w<<<(int)blocks, 256, 0, c->stream>>>(P, rq_e, ar_e, w_hi);
            CUDA_TRY(c, cudaGetLastError());
            c->launches++;
        }
        if (w_hi < KV_PREP_WARP_N && max_req > w_hi) {
            const int ssmem = next_pow2(max_req < 256 ? 256 : std::min(max_req, KV_PREP_WARP_N)) * 4 +
                              (int)kPrepSortBytes256 + 16;
            auto prep = k_mc_prep<POL_MCSF, 256>;
            CUDA_TRY(c, cudaFuncSetAttribute(prep, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem));
            int per_sm = 1;
            CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep, 256, ssmem));
            long long blocks = (long long)(per_sm > 0 ? per_sm : 1) * c->num_sms;
            if (blocks > inst->n_instances) blocks = inst->n_instances > 0 ? inst->n_instances : 1;
            KParams Q = P;
            Q.NP = ssmem > 0 ? next_pow2(max_req < 256 ? 256 : std::min(max_req, KV_PREP_WARP_N)) : P.NP;   // keys region
            prep<<<(int)blocks, 256, ssmem, c->stream>>>(Q, rq_e, ar_e, w_hi);
            CUDA_TRY(c, cudaGetLastError());
            c->launches++;
        }
        if (max_req > KV_PREP_WARP_N) {   // larger instances: one CTA each
            const int ssmem = early ? next_pow2(max_req) * 4 + (int)kPrepSortBytes + 16 : 16;
            auto prep = early ? k_mc_prep<POL_MCSF> : k_mc_prep<POL_MCBENCH>;
            CUDA_TRY(c, cudaFuncSetAttribute(prep, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem));
            int per_sm = 1;
            CUDA_TRY(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, prep, 1024, ssmem));
            long long blocks = (long long)(per_sm > 0 ? per_sm : 1) * c->num_sms;
            if (blocks > inst->n_instances) blocks = inst->n_instances > 0 ? inst->n_instances : 1;
            prep<<<(int)blocks, 1024, ssmem, c->stream>>>(P, rq_e, ar_e, 0);
            CUDA_TRY(c, cudaGetLastError());
            c->launches++;
        }
        if (lpt) {
            CUDA_TRY(c, cub::DeviceRadixSort::SortPairsDescending(lpt_tmp, lpt_tmp_bytes, lpt_est, lpt_est_sorted,
                                                                  lpt_ids, lpt_order, (int)ni, 0, 32, c->stream));
            c->launches++;
        }
        if (c->timing) {
            CUDA_TRY(c, cudaEventRecord(e1, c->stream));
            c->pending.push_back({e0, e1, early ? "k_mc_prep<MCSF>" : "k_mc_prep<MCBENCH>"});
        }
    } else if (pol->policy == SCHED_MCSF || prot) {
        if ((rc = grow(c, c->rq, slots * 16)) || (rc = grow(c, c->arank, slots * 4))) return rc;
        // offsets are relative to the batch: scratch slot = request row (n_req <= slots)
        P.rq = reinterpret_cast<const uint4 *>(c->rq.p);
        P.arank = reinterpret_cast<const int *>(c->arank.p);
        const int ssmem = next_pow2(max_req) * 4;
        CUDA_TRY(c, cudaFuncSetAttribute(k_rank_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, ssmem));
        long long blocks = inst->n_instances < 4LL * c->num_sms ? inst->n_instances : 4LL * c->num_sms;
        k_rank_sort<<<(int)blocks, 1024, ssmem, c->stream>>>(P, reinterpret_cast<uint4 *>(c->rq.p),
                                                             reinterpret_cast<int *>(c->arank.p));
        CUDA_TRY(c, cudaGetLastError());
        c->launches++;
    }
    if (pol->policy >= SCHED_ALPHA || early) {
        if ((rc = grow(c, c->pstart, slots * 4))) return rc;
        P.pstart = reinterpret_cast<int *>(c->pstart.p);
    }
    if (prot || early) {
        if ((rc = grow(c, c->relnext, slots * 4))) return rc;
        P.relnext = reinterpret_cast<int *>(c->relnext.p);
    }
    auto launch_ring = [&](const KParams &Q0) -> int {
        if (mcr) {
            KParams Q = Q0;
            int wps = 0;
            if (lpt && !Q.work_list) {         // first launch: claim longest first
                Q.work_list = lpt_order;
                Q.work_count = lpt_count;
                wps = mcring_wps;
            }
            name = pol->policy == SCHED_MCSF ? "k_mc_ring<MCSF>" : "k_mc_ring<MCBENCH>";
#ifndef KV_MCRING_QREG
#define KV_MCRING_QREG 1
#endif
            if (KV_MCRING_QREG && Q.NP <= 1024)        // the waiting queue in registers
                return pol->policy == SCHED_MCSF ? launch_sim(c, k_mc_ring<POL_MCSF, true>, Q, Q.warp_bytes, name, wps)
                                                 : launch_sim(c, k_mc_ring<POL_MCBENCH, true>, Q, Q.warp_bytes, name, wps);
            return pol->policy == SCHED_MCSF ? launch_sim(c, k_mc_ring<POL_MCSF>, Q, Q.warp_bytes, name, wps)
                                             : launch_sim(c, k_mc_ring<POL_MCBENCH>, Q, Q.warp_bytes, name, wps);
        }
        const KParams &Q = Q0;
        switch (pol->policy) {
        case SCHED_MCSF: name = "k_ring<MCSF>"; return launch_sim(c, k_ring<POL_MCSF>, Q, Q.warp_bytes, name);
        case SCHED_MC_BENCH: name = "k_ring<MCBENCH>"; return launch_sim(c, k_ring<POL_MCBENCH>, Q, Q.warp_bytes, name);
        case SCHED_ALPHA: name = "k_ring<ALPHA>"; return launch_sim(c, k_ring<POL_ALPHA>, Q, Q.warp_bytes, name);
        case SCHED_MCSF_PROTECTED: name = "k_prot<MCSF_PROTECTED>"; return launch_sim(c, k_prot, Q, Q.warp_bytes, name);
        case SCHED_MCSF_PROTECTED_RAISE: name = "k_prot<MCSF_PROTECTED_RAISE>"; return launch_sim(c, k_prot, Q, Q.warp_bytes, name);
        default: name = "k_ring<ALPHA_BETA>"; return launch_sim(c, k_ring<POL_ALPHA_BETA>, Q, Q.warp_bytes, name);
        }
    };
    if ((rc = launch_ring(P))) return rc;
    if (L_short < L_full && (size_t)wbytes(L_full) > c->max_smem_optin) {
        // no room for the full ring: the (rare) instances that overflowed the long list
        // are reported UNSUPPORTED
        k_mark_unsupported<<<64, 128, 0, c->stream>>>(P, P.retry_list, P.retry_count);
        CUDA_TRY(c, cudaGetLastError());
        c->launches++;
    } else if (L_short < L_full) {
        KParams Q = P;
        Q.L = L_full;
        Q.warp_bytes = wbytes(L_full);
        Q.work_list = P.retry_list;
        Q.work_count = P.retry_count;
        Q.retry_list = nullptr;          // the full ring never overflows (no long requests)
        Q.retry_count = nullptr;
        CUDA_TRY(c, cudaMemsetAsync(c->counter.p, 0, 8, c->stream));
        if ((rc = launch_ring(Q))) return rc;
    }
    if (early) {
        // the listed early-completion instances: k_prot (alpha = 0) over the list, with its
        // own long-list overflow rerun at the full ring
        const char *keep = name;
        KParams E = P;
        E.policy = SCHED_MCSF_PROTECTED;
        E.alpha_num = 0;
        E.alpha_den = 1;
        E.early_list = nullptr;
        E.early_count = nullptr;
        E.work_list = P.early_list;
        E.work_count = P.early_count;
        E.retry_list = P.retry_list + 2 * ni;
        E.retry_count = rcnt + 2;
        const int Lp = L_full < KV_PROT_SHORT ? L_full : KV_PROT_SHORT;
        E.L = Lp;
        E.warp_bytes = prot_warp_bytes(Lp, E.NP);
        if ((size_t)E.warp_bytes > c->max_smem_optin)
            return fail(c, SCHED_E_ARG, "k_prot needs %d B shared memory per warp (L=%d, NP=%d)",
                        E.warp_bytes, E.L, E.NP);
        CUDA_TRY(c, cudaMemsetAsync(c->counter.p, 0, 8, c->stream));
        if ((rc = launch_sim(c, k_prot, E, E.warp_bytes, "k_prot<MCSF,early>"))) return rc;
        if (Lp < L_full && (size_t)prot_warp_bytes(L_full, E.NP) > c->max_smem_optin) {
            k_mark_unsupported<<<64, 128, 0, c->stream>>>(E, E.retry_list, E.retry_count);
            CUDA_TRY(c, cudaGetLastError());
            c->launches++;
        } else if (Lp < L_full) {
            KParams Q = E;
            Q.L = L_full;
            Q.warp_bytes = prot_warp_bytes(L_full, E.NP);
            Q.work_list = E.retry_list;
            Q.work_count = E.retry_count;
            Q.retry_list = nullptr;
            Q.retry_count = nullptr;
            CUDA_TRY(c, cudaMemsetAsync(c->counter.p, 0, 8, c->stream));
            if ((rc = launch_sim(c, k_prot, Q, Q.warp_bytes, "k_prot<MCSF,early>"))) return rc;
        }
        c->last_kernel = keep;
    }
    return SCHED_OK;
}

extern "C" {

// latency16 = completion - a on rows [0, n_rows) (device pointers; see kvsched.h)
static int launch_latency16(sched_ctx *c, long long n_rows, const int4 *req, const int *comp, uint16_t *lat)
{
    if (n_rows <= 0) return SCHED_OK;
    long long blocks = (n_rows + 255) / 256;
    if (blocks > 8LL * c->num_sms) blocks = 8LL * c->num_sms;
    k_latency16<<<(int)blocks, 256, 0, c->stream>>>(n_rows, req, comp, lat);
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

// run_impl plus the compact latency16 output (needs the completion rounds: the caller's,
// or context scratch when it did not ask for them)
static int run_outputs(sched_ctx *c, const sched_instances *di, const sched_policy *pol, const sched_outputs *out,
                       long long row_base, long long n_rows)
{
    if (!out->latency16) return run_impl(c, di, pol, out, row_base);
    sched_outputs o = *out;
    int rc;
    if (!o.completion) {
        if ((rc = grow(c, c->comp, (size_t)(n_rows > 0 ? n_rows : 1) * 4))) return rc;
        o.completion = (int32_t *)c->comp.p;
    }
    if ((rc = run_impl(c, di, pol, &o, row_base))) return rc;
    return launch_latency16(c, n_rows, reinterpret_cast<const int4 *>(di->req), o.completion, out->latency16);
}

int sched_run_instances(sched_ctx *c, const sched_instances *inst, const sched_policy *pol,
                        const sched_outputs *out)
{
    int rc = check_common(c, inst);
    if (rc) return rc;
    if ((rc = check_policy(c, pol))) return rc;
    if (!out) return fail(c, SCHED_E_ARG, "out is NULL");
    if (inst->n_instances == 0) return SCHED_OK;
    DeviceGuard g(c->device);
    long long n_req = 0;
    if (inst->req_format != SCHED_REQ_I32X4 || out->latency16) {
        CUDA_TRY(c, cudaMemcpyAsync(&n_req, inst->req_offset + inst->n_instances, 8, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    if (inst->req_format != SCHED_REQ_I32X4) {
        if ((rc = grow(c, c->dec, (size_t)(n_req > 0 ? n_req : 1) * 16))) return rc;
        launch_decode(c, inst->req_format, inst->n_instances, reinterpret_cast<const long long *>(inst->req_offset), 0,
                      inst->req, reinterpret_cast<int4 *>(c->dec.p));
        CUDA_TRY(c, cudaGetLastError());
        c->launches++;
        sched_instances di = *inst;
        di.req = (const int32_t *)c->dec.p;
        di.req_format = SCHED_REQ_I32X4;
        c->side_ok = true;
        rc = run_outputs(c, &di, pol, out, 0, n_req);
        c->side_ok = false;
        return rc;
    }
    c->side_ok = true;
    rc = run_outputs(c, inst, pol, out, 0, n_req);
    c->side_ok = false;
    return rc;
}

// Stream memory operations (driver API, resolved at run time so the library links only the
// runtime): the streamed host path sets its per-chunk flags and holds its copy-out stream
// with them, on the copy engines' front end, without occupying an SM.
typedef CUresult (*pfn_write32_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*pfn_wait32_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static pfn_write32_t g_write32 = nullptr;
static pfn_wait32_t g_wait32 = nullptr;
static double now_ms()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static bool stream_mem_ops(sched_ctx *c)
{
    static int state = 0;                                  // 0 untried, 1 available, 2 not
    if (state == 0) {
        void *w = nullptr, *v = nullptr;
        cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
        const bool ok = cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
                        cudaGetDriverEntryPoint("cuStreamWaitValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
                        q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && w && v;
        if (ok) {
            g_write32 = (pfn_write32_t)w;
            g_wait32 = (pfn_wait32_t)v;
        }
        cudaGetLastError();
        state = ok ? 1 : 2;
    }
    (void)c;
    return state == 1;
}

// Host buffers.  The batch is cut into chunks of whole instances; chunk k's request rows are
// copied in on one stream, simulated on the context's stream, and its outputs copied out on
// a third, so the PCIe transfers of neighbouring chunks overlap the kernels.
int sched_run_instances_host(sched_ctx *c, const sched_instances *inst, const sched_policy *pol,
                             const sched_outputs *out)
{
    int rc = check_common(c, inst);
    if (rc) return rc;
    if ((rc = check_policy(c, pol))) return rc;
    if (!out) return fail(c, SCHED_E_ARG, "out is NULL");
    const long long ni = inst->n_instances;
    if (ni == 0) return SCHED_OK;
    DeviceGuard g(c->device);
    const int64_t *hoff = inst->req_offset;
    const long long n_req = hoff[ni];
    if (n_req < 0 || hoff[0] != 0) return fail(c, SCHED_E_ARG, "req_offset must start at 0 and end >= 0");
    // size hints on the host (the offsets and budgets are host memory here)
    sched_instances hi = *inst;
    if (hi.max_requests == 0 || hi.max_mem == 0 || hi.max_len == 0) {
        long long mr = 0, mm = 0, ml = 0;
        for (long long k = 0; k < ni; ++k) {
            mr = hoff[k + 1] - hoff[k] > mr ? hoff[k + 1] - hoff[k] : mr;
            mm = inst->mem_limit[k] > mm ? inst->mem_limit[k] : mm;
        }
        if (hi.max_len == 0)
            for (long long i = 0; i < n_req; ++i) {
                long long o_, w_;
                if (inst->req_format == SCHED_REQ_U16X4_DELTA) {
                    const uint16_t *r = reinterpret_cast<const uint16_t *>(inst->req) + 4 * i;
                    o_ = r[2];
                    w_ = r[3];
                } else if (inst->req_format == SCHED_REQ_U8X4_DELTA) {
                    const uint8_t *r = reinterpret_cast<const uint8_t *>(inst->req) + 4 * i;
                    o_ = r[2];
                    w_ = r[3];
                } else if (inst->req_format == SCHED_REQ_P16) {
                    o_ = w_ = (reinterpret_cast<const uint16_t *>(inst->req)[i] & 63) + 1;
                } else {
                    const int32_t *r = inst->req + 4 * i;
                    o_ = r[2];
                    w_ = r[3];
                }
                ml = o_ > ml ? o_ : ml;
                ml = w_ > ml ? w_ : ml;
            }
        if (hi.max_requests == 0) hi.max_requests = (int32_t)(mr < 0x7fffffff ? mr : 0x7fffffff);
        if (hi.max_mem == 0) hi.max_mem = (int32_t)mm;
        if (hi.max_len == 0) hi.max_len = (int32_t)(ml < 0x7fffffff ? ml : 0x7fffffff);
        if (hi.max_requests == 0) hi.max_requests = 1;
        if (hi.max_mem == 0) hi.max_mem = 1;
        if (hi.max_len == 0) hi.max_len = 1;
    }
    const bool packed = inst->req_format != SCHED_REQ_I32X4;
    const size_t row_in = inst->req_format == SCHED_REQ_U16X4_DELTA ? 8 : inst->req_format == SCHED_REQ_U8X4_DELTA ? 4
                          : packed ? 2 : 16;                                  // bytes per row on the wire
    const size_t b_off = (size_t)(ni + 1) * 8, b_req = (size_t)n_req * 16, b_mem = (size_t)ni * 4;
    if ((rc = grow(c, c->h_off, b_off)) || (rc = grow(c, c->h_req, b_req)) || (rc = grow(c, c->h_mem, b_mem)))
        return rc;
    if (packed && (rc = grow(c, c->h_pk, (size_t)n_req * 8 + 8))) return rc;
    // device outputs: completion, start [n_req] int32; 4 x int64 + 3 x int32 per instance;
    // latency16 [n_req] uint16
    const size_t o_comp = 0, o_start = o_comp + (size_t)n_req * 4, o_i64 = (o_start + (size_t)n_req * 4 + 15) & ~(size_t)15;
    const size_t o_i32 = o_i64 + (size_t)ni * 8 * 4;
    const size_t o_lat = (o_i32 + (size_t)ni * 4 * 3 + 15) & ~(size_t)15;
    const size_t total = o_lat + (size_t)n_req * 2;
    if ((rc = grow(c, c->h_out, total))) return rc;
    char *ob = (char *)c->h_out.p;
    if (!c->s_in) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
    }
    // compute streams: the context's stream + c->extra (measured on C5: 4 beats 2 and 3 by
    // 4-15 %, 6 is no better); KVSCHED_HOST_STREAMS overrides (experiments)
    int n_streams = 4;
    if (const char *e = getenv("KVSCHED_HOST_STREAMS")) n_streams = atoi(e) >= 1 && atoi(e) <= 8 ? atoi(e) : 4;
    // each chunk's lane kernel gets 1/4 of the SMs (several instances per lane, short tail;
    // the four compute streams keep the GPU full): e2e 5.7 -> 5.0 ms on C5 (2, 6, 8 measured
    // no better); KVSCHED_HOST_GRID_DIV overrides (experiments)
    int grid_div = 4;
    if (const char *e = getenv("KVSCHED_HOST_GRID_DIV")) grid_div = atoi(e) >= 1 ? atoi(e) : 4;
    struct GridDiv {
        sched_ctx *c;
        ~GridDiv() { c->lane_grid_div = 1; }
    } gd{c};
    c->lane_grid_div = grid_div;
    // Streamed pipeline (MC policies on the lane path, SCHED_REQ_P16 rows): the rows are
    // copied in K chunks on s_in, and after each chunk's copy a stream memory operation sets
    // ready[k] (the copy engine's front end writes it: no kernel).  ONE persistent lane launch
    // over the whole batch claims instances in order and waits for an instance's chunk flag
    // before reading its rows, which it decodes itself (k_mc_lane<..., p16>); the size-scope
    // instances run beside it on the side stream (k_mc_small, same flags, same decoding).
    // Every kernel counts an instance in done[chunk] once its outputs are written, and the
    // copy-out stream waits for done[k] >= |chunk k| with a stream wait-value (front end
    // again), then converts chunk k's completions to latency16 and copies it out.  No kernel
    // waits for another kernel's output, so nothing the spinning launches wait on needs an
    // SM; waits are bounded, and a call whose wait gave up is redone on the chunked pipeline.
    // KVSCHED_HOST_STREAM=0 selects the chunked pipeline (A/B).
    {
        const char *se = getenv("KVSCHED_HOST_STREAM");
        const bool lane_path = (pol->policy == SCHED_MCSF || pol->policy == SCHED_MC_BENCH) && hi.max_mem <= kSmallMaxMem &&
                               hi.max_requests <= kSmallMaxRequests && pol->round_cap <= 0 &&
                               !(pol->flags & (SCHED_FLAG_PER_ROUND | SCHED_FLAG_WARP_PER_INSTANCE));
        if (lane_path && inst->req_format == SCHED_REQ_P16 && !(se && se[0] == '0') && !c->stream_off && ni >= 64 &&
            ni < (1ll << 31) &&                                  // 32-bit chunk arithmetic in the kernels
            stream_mem_ops(c)) {
            // K flag chunks (copy-in granularity); the copy-out takes them in groups that grow
            // from one chunk to KVSCHED_HOST_STREAM_GROUP (the first results leave early, the
            // later copies are large)
            long long K = 16;
            if (const char *e = getenv("KVSCHED_HOST_STREAM_CHUNKS")) K = atoll(e) >= 1 ? atoll(e) : K;
            long long gmax = 1;
            if (const char *e = getenv("KVSCHED_HOST_STREAM_GROUP")) gmax = atoll(e) >= 1 ? atoll(e) : gmax;
            if (K > ni) K = ni;
            const long long C = (ni + K - 1) / K;                   // instances per chunk
            K = (ni + C - 1) / C;
            if ((rc = grow(c, c->sflags, (size_t)(2 * K + 2) * 4 + 16))) return rc;
            int *ready = reinterpret_cast<int *>(c->sflags.p);
            unsigned int *done = reinterpret_cast<unsigned int *>(ready + K);
            int *err = reinterpret_cast<int *>(done + K);
            const bool trace = getenv("KVSCHED_STREAM_TRACE") != nullptr;   // event timeline on stderr
            std::vector<std::pair<const char *, cudaEvent_t>> tev;
            auto mark = [&](const char *what, cudaStream_t st) {
                if (!trace) return;
                cudaEvent_t e = nullptr;
                const cudaError_t e1 = cudaEventCreate(&e);
                const cudaError_t e2 = cudaEventRecord(e, st);
                if (e1 != cudaSuccess || e2 != cudaSuccess)
                    fprintf(stderr, "[stream trace] %s: %s / %s\n", what, cudaGetErrorString(e1), cudaGetErrorString(e2));
                tev.push_back({what, e});
            };
            while ((long long)c->chunk_events.size() < 2) c->chunk_events.push_back(take_event(c));
            cudaEvent_t *ev = c->chunk_events.data();
            mark("start", c->stream);
            c->trace = trace ? &tev : nullptr;
            struct TraceOff { sched_ctx *c; ~TraceOff() { c->trace = nullptr; } } trace_off{c};
            // flags and counts cleared before any copy of this call (and after earlier work)
            CUDA_TRY(c, cudaMemsetAsync(c->sflags.p, 0, (size_t)(2 * K + 2) * 4, c->stream));
            CUDA_TRY(c, cudaEventRecord(ev[0], c->stream));
            CUDA_TRY(c, cudaStreamWaitEvent(c->s_in, ev[0], 0));
            CUDA_TRY(c, cudaStreamWaitEvent(c->s_out, ev[0], 0));
            CUDA_TRY(c, cudaMemcpyAsync(c->h_off.p, hoff, b_off, cudaMemcpyHostToDevice, c->s_in));
            CUDA_TRY(c, cudaMemcpyAsync(c->h_mem.p, inst->mem_limit, b_mem, cudaMemcpyHostToDevice, c->s_in));
            CUDA_TRY(c, cudaEventRecord(ev[1], c->s_in));           // offsets and budgets are in
            const long long *doff = (const long long *)c->h_off.p;
            const uint16_t *d16 = reinterpret_cast<const uint16_t *>(c->h_pk.p);
            // copy-in in groups of flag chunks growing from 1 to gmax (one copy, then a flag
            // per chunk): the first rows land early, the later copies are large
            for (long long k = 0, gs = 1; k < K; k += gs, gs = std::min(2 * gs, gmax)) {
                const long long ke = std::min(K, k + gs);
                const long long r0 = hoff[k * C], r1 = hoff[std::min(ni, ke * C)];
                if (r1 > r0)
                    CUDA_TRY(c, cudaMemcpyAsync((char *)c->h_pk.p + r0 * 2, (const char *)inst->req + r0 * 2,
                                                (size_t)(r1 - r0) * 2, cudaMemcpyHostToDevice, c->s_in));
                for (long long j = k; j < ke; ++j)
                    if (g_write32((CUstream)c->s_in, (CUdeviceptr)(ready + j), 1u, 0) != CUDA_SUCCESS)
                        return fail(c, SCHED_E_CUDA, "cuStreamWriteValue32 failed");
                mark("in", c->s_in);
            }
            // the simulation: one launch over everything, gated per chunk
            CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ev[1], 0));
            sched_instances di = hi;
            di.req_format = SCHED_REQ_I32X4;
            di.req_offset = (const int64_t *)doff;
            di.req = nullptr;                                       // the kernels read d16
            di.mem_limit = (const int32_t *)c->h_mem.p;
            sched_outputs dout;
            dout.completion = out->completion ? (int32_t *)(ob + o_comp) : nullptr;
            dout.start = out->start ? (int32_t *)(ob + o_start) : nullptr;
            dout.tel = out->tel ? (int64_t *)(ob + o_i64) : nullptr;
            dout.rounds = out->rounds ? (int64_t *)(ob + o_i64 + ni * 8) : nullptr;
            dout.decision_rounds = out->decision_rounds ? (int64_t *)(ob + o_i64 + ni * 16) : nullptr;
            dout.evictions = out->evictions ? (int64_t *)(ob + o_i64 + ni * 24) : nullptr;
            dout.makespan = out->makespan ? (int32_t *)(ob + o_i32) : nullptr;
            dout.peak_mem = out->peak_mem ? (int32_t *)(ob + o_i32 + ni * 4) : nullptr;
            dout.status = out->status ? (int32_t *)(ob + o_i32 + ni * 8) : nullptr;
            dout.latency16 = nullptr;
            {
                struct StreamGuard {
                    sched_ctx *c;
                    ~StreamGuard()
                    {
                        c->stream_mode = false;
                        c->side_ok = false;
                        c->stream_reserve = 0;
                        c->grid_cap = 0;
                        c->stream_req16 = nullptr;
                        c->stream_lat16 = nullptr;
                    }
                } sg{c};
                c->stream_mode = true;
                c->stream_ready = ready;
                c->stream_done = done;
                c->stream_err = err;
                c->stream_chunk = C;
                c->stream_req16 = d16;
                c->stream_lat16 = out->latency16 ? (uint16_t *)(ob + o_lat) : nullptr;
                c->stream_reserve = 10;              // SMs left to the side-stream kernels (8-12 measured alike)
                c->grid_cap = 96;                    // side-stream fallback kernels (blocks)
                if (const char *e = getenv("KVSCHED_STREAM_RESERVE")) c->stream_reserve = atoi(e);
                if (const char *e = getenv("KVSCHED_STREAM_SIDE_BLOCKS")) c->grid_cap = atoi(e);
                c->side_ok = true;
                c->lane_grid_div = 1;                // one launch over the whole GPU (minus the reserve)
                if ((rc = run_impl(c, &di, pol, &dout, 0))) return rc;
                mark("sim", c->stream);
                if (c->s_side) mark("side", c->s_side);
            }
            // copy-out: chunk k as soon as all its instances are counted
            uint16_t *dlat = (uint16_t *)(ob + o_lat);
            for (long long k = 0, gs = 1; k < K; k += gs, gs = std::min(2 * gs, gmax)) {
                const long long ke = std::min(K, k + gs);
                const long long i0 = k * C, i1 = std::min(ni, ke * C);
                const long long r0 = hoff[i0], r1 = hoff[i1];
                for (long long j = k; j < ke; ++j)
                    if (g_wait32((CUstream)c->s_out, (CUdeviceptr)(done + j), (cuuint32_t)(std::min(ni, (j + 1) * C) - j * C),
                                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                        return fail(c, SCHED_E_CUDA, "cuStreamWaitValue32 failed");
                struct { void *h; const void *d; size_t b; } cp[] = {
                    {out->completion ? out->completion + r0 : nullptr, dout.completion ? dout.completion + r0 : nullptr,
                     (size_t)(r1 - r0) * 4},
                    {out->latency16 ? out->latency16 + r0 : nullptr, dlat + r0, (size_t)(r1 - r0) * 2},
                    {out->start ? out->start + r0 : nullptr, dout.start ? dout.start + r0 : nullptr, (size_t)(r1 - r0) * 4},
                    {out->tel ? out->tel + i0 : nullptr, dout.tel ? dout.tel + i0 : nullptr, (size_t)(i1 - i0) * 8},
                    {out->rounds ? out->rounds + i0 : nullptr, dout.rounds ? dout.rounds + i0 : nullptr, (size_t)(i1 - i0) * 8},
                    {out->decision_rounds ? out->decision_rounds + i0 : nullptr,
                     dout.decision_rounds ? dout.decision_rounds + i0 : nullptr, (size_t)(i1 - i0) * 8},
                    {out->evictions ? out->evictions + i0 : nullptr, dout.evictions ? dout.evictions + i0 : nullptr, (size_t)(i1 - i0) * 8},
                    {out->makespan ? out->makespan + i0 : nullptr, dout.makespan ? dout.makespan + i0 : nullptr, (size_t)(i1 - i0) * 4},
                    {out->peak_mem ? out->peak_mem + i0 : nullptr, dout.peak_mem ? dout.peak_mem + i0 : nullptr, (size_t)(i1 - i0) * 4},
                    {out->status ? out->status + i0 : nullptr, dout.status ? dout.status + i0 : nullptr, (size_t)(i1 - i0) * 4}};
                mark("rel", c->s_out);
                // per-instance fields laid out field-major at one pitch in host memory (the
                // int64 four, the int32 three) go out as one 2-D copy per group: a copy per
                // field and chunk costs more in per-copy overhead than its bytes
                bool grouped[10] = {false};
                for (int g = 0; g < 2; ++g) {
                    const int f0 = g == 0 ? 3 : 7, nf = g == 0 ? 4 : 3;
                    const size_t esz = g == 0 ? 8 : 4;
                    bool ok = true;
                    for (int f = f0; f < f0 + nf; ++f) ok = ok && cp[f].h && cp[f].d && cp[f].b;
                    if (!ok) continue;
                    const ptrdiff_t hp = (char *)cp[f0 + 1].h - (char *)cp[f0].h;
                    for (int f = f0 + 1; f < f0 + nf; ++f)
                        ok = ok && (char *)cp[f].h - (char *)cp[f - 1].h == hp &&
                             (const char *)cp[f].d - (const char *)cp[f - 1].d == (ptrdiff_t)(esz * ni);
                    if (!ok || hp < (ptrdiff_t)cp[f0].b) continue;
                    CUDA_TRY(c, cudaMemcpy2DAsync(cp[f0].h, (size_t)hp, cp[f0].d, esz * ni, cp[f0].b, nf,
                                                  cudaMemcpyDeviceToHost, c->s_out));
                    for (int f = f0; f < f0 + nf; ++f) grouped[f] = true;
                }
                for (int f = 0; f < 10; ++f)
                    if (!grouped[f] && cp[f].h && cp[f].d && cp[f].b)
                        CUDA_TRY(c, cudaMemcpyAsync(cp[f].h, cp[f].d, cp[f].b, cudaMemcpyDeviceToHost, c->s_out));
                mark("out", c->s_out);
            }
            if (trace) {                 // host-side completion times of the marks (poll)
                std::vector<double> when(tev.size(), -1.0);
                const double t0 = now_ms();
                size_t left = tev.size();
                while (left && now_ms() - t0 < 5000.0) {
                    for (size_t i = 0; i < tev.size(); ++i)
                        if (when[i] < 0 && cudaEventQuery(tev[i].second) == cudaSuccess) {
                            when[i] = now_ms() - t0;
                            --left;
                        }
                }
                fprintf(stderr, "[stream trace]");
                for (size_t i = 0; i < tev.size(); ++i) fprintf(stderr, " %s %.3f", tev[i].first, when[i] - when[0]);
                fprintf(stderr, "\n");
                for (auto &e : tev) cudaEventDestroy(e.second);
            }
            // The kernels end on their own (bounded waits); then the copy-out stream can only be
            // held by a count that never completes -- which would be a bug: watch it, and if it
            // does not drain, release every wait and redo the call on the chunked pipeline.
            CUDA_TRY(c, cudaStreamSynchronize(c->s_in));
            CUDA_TRY(c, cudaStreamSynchronize(c->stream));
            if (c->s_side) CUDA_TRY(c, cudaStreamSynchronize(c->s_side));
            bool stuck = false;
            for (int it = 0;; ++it) {
                const cudaError_t q = cudaStreamQuery(c->s_out);
                if (q == cudaSuccess) break;
                if (q != cudaErrorNotReady) CUDA_TRY(c, q);
                if (it > 20000) {                                   // ~2 s after the kernels ended
                    stuck = true;
                    std::vector<unsigned int> big((size_t)K, 0x7fffffffu);
                    CUDA_TRY(c, cudaMemcpy(done, big.data(), (size_t)K * 4, cudaMemcpyHostToDevice));
                    CUDA_TRY(c, cudaStreamSynchronize(c->s_out));
                    break;
                }
                usleep(100);
            }
            int herr = 0;
            CUDA_TRY(c, cudaMemcpy(&herr, err, 4, cudaMemcpyDeviceToHost));
            if (!herr && !stuck) {
                c->last_kernel = pol->policy == SCHED_MCSF ? "k_mc_lane<MCSF,streamed>" : "k_mc_lane<MCBENCH,streamed>";
                return SCHED_OK;
            }
            c->stream_off = true;
            struct Off { sched_ctx *c; ~Off() { c->stream_off = false; } } off_{c};
            return sched_run_instances_host(c, inst, pol, out);
        }
    }
    // the chunked pipeline's extra compute streams (created only here: the streamed path
    // needs its few streams on distinct hardware queues, see above)
    for (auto &r : c->extra) {
        if (!r.stream) CUDA_TRY(c, cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
        if ((rc = grow(c, r.counter, 64)) || (rc = grow(c, r.bounds, 64))) return rc;
    }
    // chunks of ~4 M request rows (64 MB), at most 32 (KVSCHED_HOST_CHUNK_ROWS overrides the
    // chunk size; used by the tests to exercise the pipeline on small batches)
    long long chunk_rows = 4ll << 20;
    if (const char *e = getenv("KVSCHED_HOST_CHUNK_ROWS")) chunk_rows = atoll(e) > 0 ? atoll(e) : chunk_rows;
    long long n_chunks = n_req / chunk_rows;
    if (n_chunks < 1) n_chunks = 1;
    if (n_chunks > 256) n_chunks = 256;
    if (n_chunks > ni) n_chunks = ni;
    while ((long long)c->chunk_events.size() < 2 * n_chunks + 1) c->chunk_events.push_back(take_event(c));
    cudaEvent_t *ev = c->chunk_events.data();
    // the previous work on the context's stream precedes every copy of this call
    CUDA_TRY(c, cudaEventRecord(ev[2 * n_chunks], c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->s_in, ev[2 * n_chunks], 0));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_off.p, hoff, b_off, cudaMemcpyHostToDevice, c->s_in));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_mem.p, inst->mem_limit, b_mem, cudaMemcpyHostToDevice, c->s_in));
    const long long *doff = (const long long *)c->h_off.p;
    for (long long k = 0; k < n_chunks; ++k) {
        const long long i0 = ni * k / n_chunks, i1 = ni * (k + 1) / n_chunks;
        const long long r0 = hoff[i0], r1 = hoff[i1];
        char *dst = packed ? (char *)c->h_pk.p + r0 * row_in : (char *)c->h_req.p + r0 * 16;
        const char *src = (const char *)inst->req + r0 * row_in;
        if (r1 > r0)
            CUDA_TRY(c, cudaMemcpyAsync(dst, src, (size_t)(r1 - r0) * row_in, cudaMemcpyHostToDevice, c->s_in));
        CUDA_TRY(c, cudaEventRecord(ev[2 * k], c->s_in));
        // chunk k computes on stream k mod 3 (with that stream's scratch)
        sched_ctx::RunScratch *rs = (k % n_streams) ? &c->extra[k % n_streams - 1] : nullptr;
        if (rs) swap_run_scratch(c, *rs);
        struct Restore {
            sched_ctx *c;
            sched_ctx::RunScratch *rs;
            ~Restore() { if (rs) swap_run_scratch(c, *rs); }
        } restore{c, rs};
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, ev[2 * k], 0));
        if (packed && i1 > i0) {
            launch_decode(c, inst->req_format, i1 - i0, doff + i0, r0, dst,
                          reinterpret_cast<int4 *>((char *)c->h_req.p + r0 * 16));
            CUDA_TRY(c, cudaGetLastError());
        }
        sched_instances di = hi;
        di.req_format = SCHED_REQ_I32X4;
        di.n_instances = i1 - i0;
        di.req_offset = (const int64_t *)(doff + i0);
        di.req = (const int32_t *)((char *)c->h_req.p + r0 * 16);
        di.mem_limit = (const int32_t *)c->h_mem.p + i0;
        di.instance_id0 = inst->instance_id0 + i0;
        sched_outputs dout;
        dout.completion = out->completion ? (int32_t *)(ob + o_comp) + r0 : nullptr;
        dout.start = out->start ? (int32_t *)(ob + o_start) + r0 : nullptr;
        dout.tel = out->tel ? (int64_t *)(ob + o_i64) + i0 : nullptr;
        dout.rounds = out->rounds ? (int64_t *)(ob + o_i64 + ni * 8) + i0 : nullptr;
        dout.decision_rounds = out->decision_rounds ? (int64_t *)(ob + o_i64 + ni * 16) + i0 : nullptr;
        dout.evictions = out->evictions ? (int64_t *)(ob + o_i64 + ni * 24) + i0 : nullptr;
        dout.makespan = out->makespan ? (int32_t *)(ob + o_i32) + i0 : nullptr;
        dout.peak_mem = out->peak_mem ? (int32_t *)(ob + o_i32 + ni * 4) + i0 : nullptr;
        dout.status = out->status ? (int32_t *)(ob + o_i32 + ni * 8) + i0 : nullptr;
        dout.latency16 = out->latency16 ? (uint16_t *)(ob + o_lat) + r0 : nullptr;
        if (dout.latency16 && !dout.completion) dout.completion = (int32_t *)(ob + o_comp) + r0;   // device scratch
        if (di.n_instances > 0 && (rc = run_outputs(c, &di, pol, &dout, r0, r1 - r0))) return rc;
        CUDA_TRY(c, cudaEventRecord(ev[2 * k + 1], c->stream));
        CUDA_TRY(c, cudaStreamWaitEvent(c->s_out, ev[2 * k + 1], 0));
        struct { void *h; const void *d; size_t b; } cp[] = {
            {out->completion ? out->completion + r0 : nullptr, dout.completion, (size_t)(r1 - r0) * 4},
            {out->latency16 ? out->latency16 + r0 : nullptr, dout.latency16, (size_t)(r1 - r0) * 2},
            {out->start ? out->start + r0 : nullptr, dout.start, (size_t)(r1 - r0) * 4},
            {out->tel ? out->tel + i0 : nullptr, dout.tel, (size_t)(i1 - i0) * 8},
            {out->rounds ? out->rounds + i0 : nullptr, dout.rounds, (size_t)(i1 - i0) * 8},
            {out->decision_rounds ? out->decision_rounds + i0 : nullptr, dout.decision_rounds, (size_t)(i1 - i0) * 8},
            {out->evictions ? out->evictions + i0 : nullptr, dout.evictions, (size_t)(i1 - i0) * 8},
            {out->makespan ? out->makespan + i0 : nullptr, dout.makespan, (size_t)(i1 - i0) * 4},
            {out->peak_mem ? out->peak_mem + i0 : nullptr, dout.peak_mem, (size_t)(i1 - i0) * 4},
            {out->status ? out->status + i0 : nullptr, dout.status, (size_t)(i1 - i0) * 4}};
        for (auto &x : cp)
            if (x.h && x.b) CUDA_TRY(c, cudaMemcpyAsync(x.h, x.d, x.b, cudaMemcpyDeviceToHost, c->s_out));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->s_out));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (auto &r : c->extra) CUDA_TRY(c, cudaStreamSynchronize(r.stream));
    return SCHED_OK;
}

int sched_latency(sched_ctx *c, const sched_instances *inst, const int32_t *completion, int64_t *tel,
                  int64_t *tel_total)
{
    if (!c) return SCHED_E_STATE;
    if (!inst) return fail(c, SCHED_E_ARG, "inst is NULL");
    if (inst->n_instances < 0) return fail(c, SCHED_E_ARG, "n_instances < 0");
    DeviceGuard g(c->device);
    if (tel_total) CUDA_TRY(c, cudaMemsetAsync(tel_total, 0, 8, c->stream));
    if (inst->n_instances == 0) return SCHED_OK;
    if (!inst->req_offset || !inst->req || !completion)
        return fail(c, SCHED_E_ARG, "req_offset, req and completion must be non-NULL");
    if (inst->req_format != SCHED_REQ_I32X4) return fail(c, SCHED_E_ARG, "sched_latency takes SCHED_REQ_I32X4 rows");
    long long blocks = (inst->n_instances + 3) / 4;
    if (blocks > 16LL * c->num_sms) blocks = 16LL * c->num_sms;
    k_latency<<<(int)blocks, 128, 0, c->stream>>>(inst->n_instances,
                                                  reinterpret_cast<const long long *>(inst->req_offset),
                                                  reinterpret_cast<const int4 *>(inst->req), completion,
                                                  reinterpret_cast<long long *>(tel),
                                                  reinterpret_cast<unsigned long long *>(tel_total));
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

int sched_lb_sorted(sched_ctx *c, const sched_instances *inst, int64_t *lb)
{
    int rc = check_common(c, inst);
    if (rc) return rc;
    if (!lb) return fail(c, SCHED_E_ARG, "lb is NULL");
    if (inst->req_format != SCHED_REQ_I32X4) return fail(c, SCHED_E_ARG, "sched_lb_sorted takes SCHED_REQ_I32X4 rows");
    if (inst->n_instances == 0) return SCHED_OK;
    DeviceGuard g(c->device);
    int max_n = inst->max_requests;
    if (max_n == 0) {
        CUDA_TRY(c, cudaMemsetAsync(c->bounds.p, 0, 16, c->stream));
        long long blocks = (inst->n_instances + 255) / 256;
        if (blocks > 4 * (long long)c->num_sms) blocks = 4 * (long long)c->num_sms;
        k_bounds<<<(int)blocks, 256, 0, c->stream>>>(inst->n_instances, reinterpret_cast<const long long *>(inst->req_offset),
                                                     reinterpret_cast<const int4 *>(inst->req), inst->mem_limit,
                                                     (int *)c->bounds.p);
        CUDA_TRY(c, cudaGetLastError());
        c->launches++;
        int hb[4];
        CUDA_TRY(c, cudaMemcpyAsync(hb, c->bounds.p, 16, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        max_n = hb[0];
    }
    if (max_n > 8192) max_n = 8192;                 // larger instances report -1
    if (max_n < 2) max_n = 2;
    const int smem = 2 * next_pow2(max_n) * 8;
    CUDA_TRY(c, cudaFuncSetAttribute(k_lb_sorted, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    long long blocks = inst->n_instances < 8LL * c->num_sms ? inst->n_instances : 8LL * c->num_sms;
    k_lb_sorted<<<(int)blocks, 512, smem, c->stream>>>(inst->n_instances, reinterpret_cast<const long long *>(inst->req_offset),
                                                        reinterpret_cast<const int4 *>(inst->req), inst->mem_limit, max_n,
                                                        reinterpret_cast<long long *>(lb));
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

int sched_wallclock(sched_ctx *c, const sched_instances *inst, const int32_t *start, const int32_t *completion,
                    const sched_clock *clk, int64_t *tel_wall, int64_t *makespan_wall, int64_t *bins, int32_t *mem_trace)
{
    int rc = check_common(c, inst);
    if (rc) return rc;
    if (!clk) return fail(c, SCHED_E_ARG, "clk is NULL");
    if (inst->req_format != SCHED_REQ_I32X4) return fail(c, SCHED_E_ARG, "sched_wallclock takes SCHED_REQ_I32X4 rows");
    if (clk->c0 < 1 || clk->c1 < 0 || clk->bin_width < 0 || clk->n_bins < 0 || clk->trace_len < 0)
        return fail(c, SCHED_E_ARG, "need c0 >= 1, c1 >= 0, bin_width, n_bins, trace_len >= 0");
    if (inst->n_instances == 0) return SCHED_OK;
    if (!start || !completion) return fail(c, SCHED_E_ARG, "start and completion are required");
    DeviceGuard g(c->device);
    ClockParams C{inst->n_instances, reinterpret_cast<const long long *>(inst->req_offset),
                  reinterpret_cast<const int4 *>(inst->req), start, completion, clk->c0, clk->c1, clk->bin_width,
                  clk->n_bins, clk->trace_len, reinterpret_cast<long long *>(tel_wall),
                  reinterpret_cast<long long *>(makespan_wall), bins && clk->n_bins > 0 ? reinterpret_cast<long long *>(bins) : nullptr,
                  mem_trace && clk->trace_len > 0 ? mem_trace : nullptr};
    const int smem = 4 * (int)sizeof(ClockSmem);
    CUDA_TRY(c, cudaFuncSetAttribute(k_wallclock, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    long long blocks = (inst->n_instances + 3) / 4;
    if (blocks > 16LL * c->num_sms) blocks = 16LL * c->num_sms;
    k_wallclock<<<(int)blocks, 128, smem, c->stream>>>(C);
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

static int gen_params(sched_ctx *c, const sched_gen_am2 *sp, GenAm2 *G)
{
    if (!sp) return fail(c, SCHED_E_ARG, "spec is NULL");
    if (sp->n_instances < 0) return fail(c, SCHED_E_ARG, "n_instances < 0");
    if (sp->n_lambda < 1 || sp->n_m < 1 || !sp->poisson_cdf || !sp->m_values)
        return fail(c, SCHED_E_ARG, "need n_lambda, n_m >= 1 and the tables");
    if (sp->T_lo < 0 || sp->T_hi < sp->T_lo || sp->T_hi > 1024)
        return fail(c, SCHED_E_ARG, "need 0 <= T_lo <= T_hi <= 1024");
    if (sp->s_lo < 1 || sp->s_hi < sp->s_lo) return fail(c, SCHED_E_ARG, "need 1 <= s_lo <= s_hi");
    *G = GenAm2{sp->n_instances, sp->instance_id0, sp->seed, sp->n_lambda, sp->n_m,
                reinterpret_cast<const unsigned long long *>(sp->poisson_cdf), sp->m_values,
                sp->T_lo, sp->T_hi, sp->s_lo, sp->s_hi};
    return SCHED_OK;
}

int sched_gen_am2_count(sched_ctx *c, const sched_gen_am2 *spec, int64_t *req_offset)
{
    if (!c) return SCHED_E_STATE;
    GenAm2 G;
    int rc = gen_params(c, spec, &G);
    if (rc) return rc;
    if (!req_offset) return fail(c, SCHED_E_ARG, "req_offset is NULL");
    DeviceGuard g(c->device);
    long long *x = reinterpret_cast<long long *>(req_offset);
    if (G.n_inst == 0) {
        CUDA_TRY(c, cudaMemsetAsync(x, 0, 8, c->stream));
        return SCHED_OK;
    }
    long long blocks = (G.n_inst + 255) / 256;
    if (blocks > 16LL * c->num_sms) blocks = 16LL * c->num_sms;
    k_gen_am2_count<<<(int)blocks, 256, 0, c->stream>>>(G, x);
    CUDA_TRY(c, cudaGetLastError());
    const long long nb = (G.n_inst + kScanBlock - 1) / kScanBlock;
    if ((rc = grow(c, c->scan, (size_t)nb * 8))) return rc;
    long long *bs = reinterpret_cast<long long *>(c->scan.p);
    k_scan_blocks<<<(int)nb, kScanBlock, 0, c->stream>>>(x, G.n_inst, bs);
    k_scan_sums<<<1, kScanBlock, 0, c->stream>>>(bs, nb);
    k_scan_fix<<<(int)nb, kScanBlock, 0, c->stream>>>(x, G.n_inst, bs);
    CUDA_TRY(c, cudaGetLastError());
    c->launches += 4;
    return SCHED_OK;
}

int sched_gen_am2_fill(sched_ctx *c, const sched_gen_am2 *spec, const int64_t *req_offset, int32_t *req,
                       int32_t *mem_limit)
{
    if (!c) return SCHED_E_STATE;
    GenAm2 G;
    int rc = gen_params(c, spec, &G);
    if (rc) return rc;
    if (G.n_inst == 0) return SCHED_OK;
    if (!req_offset || !req || !mem_limit) return fail(c, SCHED_E_ARG, "null output");
    if (((uintptr_t)req) & 15u) return fail(c, SCHED_E_ARG, "req must be 16-byte aligned");
    DeviceGuard g(c->device);
    long long blocks = (G.n_inst + 3) / 4;
    if (blocks > 32LL * c->num_sms) blocks = 32LL * c->num_sms;
    k_gen_am2_fill<<<(int)blocks, 128, 0, c->stream>>>(G, reinterpret_cast<const long long *>(req_offset),
                                                        reinterpret_cast<int4 *>(req), mem_limit);
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

int sched_philox4x32_10(sched_ctx *c, int64_t n, const uint32_t *ctr, const uint32_t *key, uint32_t *out)
{
    if (!c) return SCHED_E_STATE;
    if (n < 0 || (n > 0 && (!ctr || !key || !out))) return fail(c, SCHED_E_ARG, "bad arguments");
    if (n == 0) return SCHED_OK;
    DeviceGuard g(c->device);
    k_philox<<<(int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024), 256, 0, c->stream>>>(
        n, reinterpret_cast<const uint4 *>(ctr), reinterpret_cast<const uint2 *>(key), reinterpret_cast<uint4 *>(out));
    CUDA_TRY(c, cudaGetLastError());
    c->launches++;
    return SCHED_OK;
}

int sched_set_timing(sched_ctx *c, int enable)
{
    if (!c) return SCHED_E_STATE;
    c->timing = enable != 0;
    return SCHED_OK;
}

static int drain_pending(sched_ctx *c)
{
    DeviceGuard g(c->device);
    for (auto &p : c->pending) {
        CUDA_TRY(c, cudaEventSynchronize(p.e1));
        float ms = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&ms, p.e0, p.e1));
        c->sim_ms += ms;
        bool found = false;
        for (auto &k : c->kstats)
            if (k.name == p.name || strcmp(k.name, p.name) == 0) {
                k.ms += ms;
                k.launches++;
                found = true;
                break;
            }
        if (!found) c->kstats.push_back({p.name, (double)ms, 1});
        c->free_events.push_back(p.e0);
        c->free_events.push_back(p.e1);
    }
    c->pending.clear();
    return SCHED_OK;
}

int sched_get_stats(sched_ctx *c, int64_t *launches, double *sim_kernel_ms, int64_t *sim_kernel_launches)
{
    if (!c) return SCHED_E_STATE;
    int rc = drain_pending(c);
    if (rc) return rc;
    if (launches) *launches = c->launches;
    if (sim_kernel_ms) *sim_kernel_ms = c->sim_ms;
    if (sim_kernel_launches) *sim_kernel_launches = c->sim_launches;
    return SCHED_OK;
}

int sched_get_kernel_stats(sched_ctx *c, int32_t i, const char **name, double *ms, int64_t *launches)
{
    if (!c) return SCHED_E_STATE;
    int rc = drain_pending(c);
    if (rc) return rc;
    if (i < 0 || (size_t)i >= c->kstats.size()) return fail(c, SCHED_E_ARG, "kernel stats index %d out of range", i);
    if (name) *name = c->kstats[i].name;
    if (ms) *ms = c->kstats[i].ms;
    if (launches) *launches = c->kstats[i].launches;
    return SCHED_OK;
}

int sched_reset_stats(sched_ctx *c)
{
    if (!c) return SCHED_E_STATE;
    double ms;
    int rc = sched_get_stats(c, nullptr, &ms, nullptr);
    c->launches = 0;
    c->sim_launches = 0;
    c->sim_ms = 0.0;
    c->kstats.clear();
    return rc;
}

const char *sched_last_kernel(const sched_ctx *c) { return c ? c->last_kernel : ""; }

int sched_finalize(sched_ctx *c)
{
    if (!c) return SCHED_E_STATE;
    {
        DeviceGuard g(c->device);
        cudaStreamSynchronize(c->stream);
        for (DevBuf *b : {&c->counter, &c->bounds, &c->rq, &c->arank, &c->pstart, &c->relnext, &c->total, &c->retry, &c->scan, &c->dec, &c->h_pk, &c->comp, &c->fkeys, &c->h_off,
                          &c->h_req, &c->h_mem, &c->h_out, &c->rq8, &c->arr8, &c->capv, &c->lpt})
            if (b->p) cudaFree(b->p);
        for (auto &p : c->pending) {
            cudaEventDestroy(p.e0);
            cudaEventDestroy(p.e1);
        }
        for (auto e : c->free_events) cudaEventDestroy(e);
        for (auto e : c->chunk_events) cudaEventDestroy(e);
        for (auto &r : c->extra) {
            for (DevBuf *b : {&r.counter, &r.bounds, &r.rq, &r.arank, &r.pstart, &r.relnext, &r.retry, &r.comp, &r.fkeys,
                              &r.rq8, &r.arr8, &r.capv, &r.lpt})
                if (b->p) cudaFree(b->p);
            if (r.stream) cudaStreamDestroy(r.stream);
        }
        if (c->s_side) cudaStreamDestroy(c->s_side);
        if (c->ev_split) cudaEventDestroy(c->ev_split);
        if (c->ev_side) cudaEventDestroy(c->ev_side);
        if (c->s_in) cudaStreamDestroy(c->s_in);
        if (c->s_out) cudaStreamDestroy(c->s_out);
    }
    delete c;
    return SCHED_OK;
}

const char *sched_last_error(const sched_ctx *c) { return c ? c->err : g_init_err; }

}  // extern "C"
