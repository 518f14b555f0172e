// kernel_clock.cuh -- NEXT-4: the wall clock of a schedule under an affine batch time.
//
// SPEC's DurationModel stand-in for the Vidur timing of P:459 (DESIGN Q28): feasibility stays
// in rounds; round r (first arrival r0 <= r < makespan) processes
//   tokens(r) = sum_{p_i = r} s_i  (prefill)  +  #{i : p_i < r < c_i}  (one decode token each)
// and lasts c0 + c1 tokens(r); W(r) is the start time of round r, W(r0) = 0.  Per instance:
//   tel_wall = sum_i W(c_i) - W(a_i),  makespan_wall = W(max c),
//   bins[b] += tokens(r) for b = floor(W(r) / bin_width) < n_bins        (Fig. 5)
//   mem[j]  = sum_{p_i <= r < c_i} (s_i + r + 1 - p_i), r = r0 + j      (Figs. 6 and 9)
// One warp per instance walks the instance's rounds in windows of kClockWin rounds: difference
// arrays in shared memory (prefill, decode activity, occupancy count and offset), warp scans
// for the activity and the clock, atomics for the bins.
#pragma once
#include "params.cuh"

namespace kv {

#ifndef KV_CLOCK_WIN
#define KV_CLOCK_WIN 256                       // measured: 256 is 11 % faster than 512 and 128 on C4
#endif
constexpr int kClockWin = KV_CLOCK_WIN;      // rounds per window (shared memory: 28 B per round)

struct ClockSmem {
    int pre[kClockWin];
    int dact[kClockWin + 1];
    int dcnt[kClockWin + 1];
    long long dsum[kClockWin + 1];
    long long W[kClockWin + 1];
};

struct ClockParams {
    long long n_inst;
    const long long *offset;
    const int4 *req;
    const int *start, *completion;
    long long c0, c1, bin_width;
    int n_bins, trace_len;
    long long *tel_wall, *makespan_wall, *bins;
    int *mem;
};

// inclusive warp scan of an int64 sequence in chunks of 32 with a running carry
__device__ __forceinline__ long long scan32_i64(long long x)
{
    const int lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const long long y = __shfl_up_sync(KV_FULL, x, d);
        if (lane >= d) x += y;
    }
    return x;
}

__global__ void __launch_bounds__(128) k_wallclock(const ClockParams C)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    ClockSmem &S = reinterpret_cast<ClockSmem *>(smem_raw)[wid];
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long k = blockIdx.x * (long long)(blockDim.x >> 5) + wid; k < C.n_inst; k += warps) {
        const long long off = C.offset[k];
        const int n = (int)(C.offset[k + 1] - off);
        long long *bins = C.bins ? C.bins + k * (long long)C.n_bins : nullptr;
        int *mem = C.mem ? C.mem + k * (long long)C.trace_len : nullptr;
        for (int b = lane; bins && b < C.n_bins; b += 32) bins[b] = 0;
        for (int j = lane; mem && j < C.trace_len; j += 32) mem[j] = 0;
        int rend = 0;
        bool unsched = false;
        for (int i = lane; i < n; i += 32) {
            const int c = C.completion[off + i], p = C.start[off + i];
            unsched |= c < 0 || p < 0;
            rend = max(rend, c);
        }
        unsched = __any_sync(KV_FULL, unsched);
        rend = warp_max_i32(rend);
        if (n == 0 || unsched) {
            if (lane == 0) {
                if (C.tel_wall) C.tel_wall[k] = n == 0 ? 0 : -1;
                if (C.makespan_wall) C.makespan_wall[k] = n == 0 ? 0 : -1;
            }
            continue;
        }
        const int r0 = C.req[off].x;
        long long Wc = 0, tel = 0;
        for (int w0 = r0; w0 < rend; w0 += kClockWin) {
            const int w1 = min(w0 + kClockWin, rend);          // rounds [w0, w1)
            const int len = w1 - w0;
            for (int j = lane; j <= kClockWin; j += 32) {
                if (j < kClockWin) S.pre[j] = 0;
                S.dact[j] = 0;
                S.dcnt[j] = 0;
                S.dsum[j] = 0;
            }
            __syncwarp();
            for (int i = lane; i < n; i += 32) {
                const int p = C.start[off + i], c = C.completion[off + i], s = C.req[off + i].y;
                if (p >= w0 && p < w1) atomicAdd(&S.pre[p - w0], s);
                int lo = max(p + 1, w0), hi = min(c - 1, w1 - 1);          // decode rounds
                if (lo <= hi) {
                    atomicAdd(&S.dact[lo - w0], 1);
                    atomicAdd(&S.dact[hi + 1 - w0], -1);
                }
                lo = max(p, w0);
                hi = min(c - 1, w1 - 1);                                    // occupancy rounds
                if (lo <= hi) {
                    atomicAdd(&S.dcnt[lo - w0], 1);
                    atomicAdd(&S.dcnt[hi + 1 - w0], -1);
                    const long long v = (long long)s + 1 - p;
                    atomicAdd(reinterpret_cast<unsigned long long *>(&S.dsum[lo - w0]), (unsigned long long)v);
                    atomicAdd(reinterpret_cast<unsigned long long *>(&S.dsum[hi + 1 - w0]), (unsigned long long)-v);
                }
            }
            __syncwarp();
            long long act_c = 0, cnt_c = 0, sum_c = 0, W_c = Wc;
            if (lane == 0) S.W[0] = Wc;
            for (int b = 0; b < len; b += 32) {
                const int j = b + lane;
                const bool in = j < len;
                const long long act = scan32_i64(in ? S.dact[j] : 0) + act_c;
                const long long cnt = scan32_i64(in ? S.dcnt[j] : 0) + cnt_c;
                const long long sum = scan32_i64(in ? S.dsum[j] : 0) + sum_c;
                const long long tokens = in ? S.pre[j] + act : 0;
                const long long dur = in ? C.c0 + C.c1 * tokens : 0;
                const long long Wend = scan32_i64(dur) + W_c;                // W(w0 + j + 1)
                const long long Wstart = Wend - dur;                          // W(w0 + j)
                if (in) S.W[j + 1] = Wend;
                const int r = w0 + j;
                if (in && mem && r - r0 < C.trace_len) mem[r - r0] = (int)(cnt * (r) + sum);
                if (bins && C.bin_width > 0 && in && tokens > 0) {
                    const long long bidx = Wstart / C.bin_width;
                    if (bidx < C.n_bins)
                        atomicAdd(reinterpret_cast<unsigned long long *>(&bins[bidx]), (unsigned long long)tokens);
                }
                act_c = __shfl_sync(KV_FULL, act, 31);
                cnt_c = __shfl_sync(KV_FULL, cnt, 31);
                sum_c = __shfl_sync(KV_FULL, sum, 31);
                W_c = __shfl_sync(KV_FULL, Wend, 31);
            }
            __syncwarp();
            long long part = 0;
            for (int i = lane; i < n; i += 32) {
                const int a = C.req[off + i].x, c = C.completion[off + i];
                if (c >= w0 && (c < w1 || (c == rend && w1 == rend))) part += S.W[c - w0];
                if (a >= w0 && a < w1) part -= S.W[a - w0];
            }
            tel += warp_sum_i64(part);
            Wc = W_c;
            __syncwarp();
        }
        if (lane == 0) {
            if (C.tel_wall) C.tel_wall[k] = tel;
            if (C.makespan_wall) C.makespan_wall[k] = Wc;
        }
    }
}

}  // namespace kv
