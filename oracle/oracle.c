/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, literal CPU transcription of the paper
 *   "Online Scheduling for LLM Inference with KV Cache Constraints" (arXiv 2502.07115)
 * used to prove the CUDA path correct.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with paper_2502_07115_b200/ (the product path) and
 * never imports it.
 *
 * Citations "P:<line>" are lines of the paper's LaTeX source; "DESIGN Qn" is
 * the reading adopted in DESIGN.md section "Readings" where the paper is silent.
 *
 * Everything is integer arithmetic: the model has integer sizes and unit-time
 * rounds, so there is no floating point anywhere on the path.
 *
 * Functions
 *   or_philox4x32_10        Philox4x32-10 (Salmon et al., SC'11), the alpha-beta RNG.
 *   or_projected_occupancy  LHS of Eq. 5 at one t'.
 *   or_is_feasible          Eq. 5 for all t' in [t+1, t_max(U)], exhaustive.
 *   or_simulate             one instance, one policy: Alg. 1, Alg. 2
 *                           (P:1076-1103), alpha-protection greedy,
 *                           alpha-protection beta-clearing, and MC-SF under
 *                           prediction error with a protection margin.
 *   or_simulate_batch       or_simulate over a CSR batch with a pthread pool.
 *   or_tel                  TEL = sum_i (c_i - a_i).
 *   or_opt_bruteforce       hindsight optimum of Eqs. 1-4 by exhaustive
 *                           branch-and-bound over start rounds (tiny instances only).
 *   or_lb_sorted            volume lower bound on OPT for all-at-0 instances (P:319 argument).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define OR_MCSF 0        /* Algorithm 1                       */
#define OR_MCBENCH 1     /* Algorithm 2                     */
#define OR_ALPHA 2       /* alpha-protection greedy           */
#define OR_ALPHA_BETA 3  /* alpha-protection beta-clearing        */
#define OR_MCSF_PROT 4   /* MC-SF on (1-alpha)M with clearing */
#define OR_MCSF_PROT_RAISE 5  /* the same; a cleared request's o~ is raised to the
                                 tokens it is known to need (DESIGN Q26b)          */
#define OR_IS_PROT(p) ((p) == OR_MCSF_PROT || (p) == OR_MCSF_PROT_RAISE)

/* at most this many beta passes per overflow (DESIGN Q29) */
#define OR_BETA_MAX_PASSES 65536

#define OR_OK 0
#define OR_INVALID 1
#define OR_LIVELOCK 2

/* ------------------------------------------------------------------------------------ */
/* Philox4x32-10.  Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as      */
/* 1, 2, 3", SC'11.  Round: (L0,R0,L1,R1) -> (hi(M1*R1)^L0^k0... ) as published.          */
/* ------------------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += W0; k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The alpha-beta eviction draw (DESIGN Q14): counter (t, pass, idx, 0), key from
 * K = seed ^ (gid * 0x9E3779B97F4A7C15 mod 2^64), output word 0.                         */
static uint32_t or_draw(uint64_t seed, uint64_t gid, int64_t t, int64_t pass, int64_t idx)
{
    uint64_t K = seed ^ (gid * 0x9E3779B97F4A7C15ull);
    uint32_t key[2] = { (uint32_t)K, (uint32_t)(K >> 32) };
    uint32_t ctr[4] = { (uint32_t)t, (uint32_t)pass, (uint32_t)idx, 0u };
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return out[0];
}

/* ------------------------------------------------------------------------------------ */
/* Eq. 5:                                                                        */
/*   sum_{i in S} (s_i + t' - p_i) 1{o~_i >= t' - p_i}                                   */
/* + sum_{i in U} (s_i + t' - t)   1{o~_i >= t' - t}          <= M,  t' in [t+1, t_max(U)] */
/* ------------------------------------------------------------------------------------ */
int64_t or_projected_occupancy(int64_t tp, int64_t t,
                               int64_t nS, const int32_t *S_s, const int32_t *S_p,
                               const int32_t *S_op,
                               int64_t nU, const int32_t *U_s, const int32_t *U_op)
{
    int64_t total = 0;
    for (int64_t j = 0; j < nS; j++)
        if ((int64_t)S_op[j] >= tp - S_p[j])
            total += (int64_t)S_s[j] + tp - S_p[j];
    for (int64_t j = 0; j < nU; j++)
        if ((int64_t)U_op[j] >= tp - t)
            total += (int64_t)U_s[j] + tp - t;
    return total;
}

/* Feasibility of U given S, by an exhaustive scan of every t' in [t+1, t_max(U)] where
 * t_max(U) = max_{i in U} (t + o~_i).  Returns 1 if feasible.                    */
int or_is_feasible(int64_t t, int64_t budget,
                   int64_t nS, const int32_t *S_s, const int32_t *S_p, const int32_t *S_op,
                   int64_t nU, const int32_t *U_s, const int32_t *U_op)
{
    int64_t tmax = t;
    for (int64_t j = 0; j < nU; j++)
        if (t + U_op[j] > tmax) tmax = t + U_op[j];
    for (int64_t tp = t + 1; tp <= tmax; tp++)
        if (or_projected_occupancy(tp, t, nS, S_s, S_p, S_op, nU, U_s, U_op) > budget)
            return 0;
    return 1;
}

/* ------------------------------------------------------------------------------------ */
/* One instance.                                                                         */
/* req is [n][4] = {a_i, s_i, o_i, o~_i} sorted by a; idx = row = tie-break.  */
/* stats[0..6] = tel, rounds, decision_rounds, makespan, peak, evictions, status.        */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int64_t n;
    const int32_t *a, *s, *o, *op;   /* views (stride 4) are copied into these arrays    */
} or_inst;

/* R is kept as an array of request indices in the policy's key order. */
static int or_key_less(const or_inst *I, int policy, int32_t x, int32_t y)
{
    if (policy == OR_MCSF || OR_IS_PROT(policy)) {       /* (o~, idx): P:175, DESIGN Q5 */
        if (I->op[x] != I->op[y]) return I->op[x] < I->op[y];
        return x < y;
    }
    return x < y;                                  /* arrival order: P:1089       */
}

static void or_insert_sorted(const or_inst *I, int policy, int32_t *R, int64_t *nR, int32_t i)
{
    int64_t pos = *nR;
    while (pos > 0 && or_key_less(I, policy, i, R[pos - 1])) {
        R[pos] = R[pos - 1];
        pos--;
    }
    R[pos] = i;
    (*nR)++;
}

static void or_remove_at(int32_t *arr, int64_t *n, int64_t pos)
{
    for (int64_t k = pos; k + 1 < *n; k++) arr[k] = arr[k + 1];
    (*n)--;
}

/* or_simulate: one instance under one policy.  Outputs
 *   completion[i] = c_i of the last admission of i that was not evicted, else -1;
 *   start[i]      = p_i likewise (may be NULL);
 *   stats[0] tel, [1] rounds, [2] decision_rounds, [3] makespan, [4] peak,
 *        [5] evictions, [6] status.   tel/rounds/makespan are -1 unless status OK.      */
int or_simulate(int64_t n, const int32_t *req, int32_t M,
                int32_t policy, int32_t alpha_num, int32_t alpha_den,
                uint64_t beta_thresh, uint64_t seed, int64_t round_cap, uint64_t gid,
                int32_t *completion, int32_t *start, int64_t *stats)
{
    for (int k = 0; k < 7; k++) stats[k] = 0;
    for (int64_t i = 0; i < n; i++) { completion[i] = -1; if (start) start[i] = -1; }
    if (policy < OR_MCSF || policy > OR_MCSF_PROT_RAISE) return -1;
    /* beta = beta_thresh / 2^32 must lie in (0, 1]: beta = 0 never clears (DESIGN Q29)    */
    if (policy == OR_ALPHA_BETA && (beta_thresh == 0 || beta_thresh > (1ull << 32))) return -1;

    size_t nb = sizeof(int32_t) * (size_t)(n + 2);
    int32_t *a = malloc(nb), *s = malloc(nb), *o = malloc(nb), *op = malloc(nb);
    int32_t *p = malloc(nb), *c = malloc(nb);
    int32_t *R = malloc(nb), *S = malloc(nb), *U = malloc(nb);
    int32_t *Ss = malloc(nb), *Sp = malloc(nb), *Sop = malloc(nb);
    int32_t *Us = malloc(nb), *Uop = malloc(nb);
    char *evict = malloc((size_t)n + 2);
    for (int64_t i = 0; i < n; i++) {
        a[i] = req[4 * i + 0]; s[i] = req[4 * i + 1];
        o[i] = req[4 * i + 2]; op[i] = req[4 * i + 3];
        p[i] = -1; c[i] = -1;
    }
    or_inst I = { n, a, s, o, op };
    int status = OR_OK;
    int64_t decision_rounds = 0, peak = 0, evictions = 0;

    /* ---- instance validation (DESIGN Q8) -------------------------------------------- */
    if (policy == OR_ALPHA || policy == OR_ALPHA_BETA || OR_IS_PROT(policy))
        if (alpha_den <= 0 || alpha_num < 0 || alpha_num >= alpha_den) status = OR_INVALID;
    for (int64_t i = 0; i < n; i++) {
        if (s[i] < 1 || o[i] < 1 || op[i] < 1 || a[i] < 0) status = OR_INVALID;
        if (i > 0 && a[i] < a[i - 1]) status = OR_INVALID;
        if (policy == OR_MCSF) {
            /* MC-SF projects with o~ >= o; a request with s+o~ > M could
             * never be admitted (Eq. 5 with S empty fails at t' = t + o~).              */
            if ((int64_t)s[i] + op[i] > M || op[i] < o[i]) status = OR_INVALID;
        } else {
            /* MC-Benchmark projects with the true o; the alpha policies and the
             * protected MC-SF (whose o~ may undershoot) cannot ever hold a request
             * whose peak s+o exceeds M.                                          */
            if ((int64_t)s[i] + o[i] > M) status = OR_INVALID;
        }
    }

    if (status == OR_OK && n > 0) {
        /* round cap (DESIGN Q23): past this absolute round the run is declared LIVELOCK */
        int64_t cap = round_cap;
        if (cap <= 0) {
            int64_t sum_o = 0;
            for (int64_t i = 0; i < n; i++) sum_o += o[i];
            cap = 16 * ((int64_t)a[n - 1] + sum_o) + 64;
            if (cap > (1ll << 30)) cap = 1ll << 30;
        }
        /* alpha budget B = floor((1 - alpha) M), alpha = num/den (DESIGN Q15) */
        int64_t B = 0;
        if (policy == OR_ALPHA || policy == OR_ALPHA_BETA || OR_IS_PROT(policy))
            B = ((int64_t)(alpha_den - alpha_num) * M) / alpha_den;
        /* Eq. 5's right-hand side: M, or (1-alpha)M for the protected MC-SF ("run MC-SF as
         * if the effective budget were (1-alpha)M")                               */
        const int64_t budget = OR_IS_PROT(policy) ? B : M;
        const int use_pred = (policy == OR_MCSF || OR_IS_PROT(policy));

        int64_t nR = 0, nS = 0, next = 0;
        int64_t t = a[0];
        /* alpha-greedy cycle detection (DESIGN Q24): state at the last clear-all */
        int64_t have_clear = 0, next_at_clear = 0, completed_since_clear = 0;
        /* "for each round t" */
        while (next < n || nR > 0 || nS > 0) {
            if (nR == 0 && nS == 0) t = a[next];           /* idle: jump to next arrival */
            if (t > cap) { status = OR_LIVELOCK; break; }

            /* requests with a_i <= t are revealed and join R^(t) */
            while (next < n && a[next] <= t) {
                or_insert_sorted(&I, policy, R, &nR, (int32_t)next);
                next++;
            }
            /* release: j completes at c_j = p_j + o_j; its KV cache clears */
            for (int64_t k = 0; k < nS;) {
                if (c[S[k]] <= t) { or_remove_at(S, &nS, k); completed_since_clear++; } else k++;
            }
            if (nR > 0) decision_rounds++;

            if (policy == OR_MCSF || policy == OR_MCBENCH || OR_IS_PROT(policy)) {
                /* Alg. 1 / Alg. 2: walk R in key order, add i
                 * to U while Eq. 5 holds for S and U+{i}; break at the first failure.    */
                const int64_t idle_before = (nS == 0);
                for (int64_t k = 0; k < nS; k++) {
                    Ss[k] = s[S[k]]; Sp[k] = p[S[k]];
                    Sop[k] = use_pred ? op[S[k]] : o[S[k]];
                }
                int64_t nU = 0;
                for (int64_t k = 0; k < nR; k++) {
                    int32_t i = R[k];
                    Us[nU] = s[i];
                    Uop[nU] = use_pred ? op[i] : o[i];
                    if (!or_is_feasible(t, budget, nS, Ss, Sp, Sop, nU + 1, Us, Uop)) break;
                    U[nU] = i;
                    nU++;
                }
                /* "Process the requests in S u U": every i in U starts now */
                for (int64_t k = 0; k < nU; k++) {
                    int32_t i = U[k];
                    p[i] = (int32_t)t;
                    c[i] = (int32_t)(t + o[i]);
                    S[nS++] = i;
                }
                for (int64_t k = 0; k + nU < nR; k++) R[k] = R[k + nU];
                nR -= nU;
                if (OR_IS_PROT(policy)) {
                    /* an underestimate o~ < o lets the realised KV growth pass M; "such an
                     * overflow triggers a clearing event, where all active requests are
                     * evicted and re-queued", with the cycle rule of DESIGN Q24   */
                    int64_t mem = 0;
                    for (int64_t k = 0; k < nS; k++) mem += (int64_t)s[S[k]] + t + 1 - p[S[k]];
                    if (mem > M) {
                        for (int64_t k = 0; k < nS; k++) {
                            int32_t j = S[k];
                            /* Q26b: j ran rounds p_j..t-1 and is not complete (c_j > t),
                             * so o_j >= t - p_j + 1                                       */
                            if (policy == OR_MCSF_PROT_RAISE && op[j] < t - p[j] + 1)
                                op[j] = (int32_t)(t - p[j] + 1);
                            p[j] = -1; c[j] = -1;
                            or_insert_sorted(&I, policy, R, &nR, j);
                            evictions++;
                        }
                        nS = 0;
                        /* DESIGN Q24: only once every request has arrived is the run from
                         * here a repeat of the last cycle (a later arrival may sort first).
                         * Not under Q26b: every clearing raises some o~ (the overflow needs
                         * an active request past its predicted end), so no state repeats. */
                        if (policy == OR_MCSF_PROT && next == n && have_clear && next == next_at_clear &&
                            completed_since_clear == 0) {
                            status = OR_LIVELOCK;
                            break;
                        }
                        have_clear = 1;
                        next_at_clear = next;
                        completed_since_clear = 0;
                    }
                    /* a head with s + o~ > (1-alpha)M never fits an empty worker: nothing is
                     * ever admitted again unless a request still to arrive sorts before it
                     * (DESIGN Q25)                                                        */
                    if (idle_before && nU == 0 && nR > 0) {
                        int rescue = 0;
                        for (int64_t j = next; j < n; j++)
                            if (or_key_less(&I, policy, (int32_t)j, R[0])) rescue = 1;
                        if (!rescue) { status = OR_LIVELOCK; break; }
                    }
                }
            } else {
                /* alpha-protection: FCFS; admit i while the next-round occupancy
                 * of S, plus s+1 for each prompt already admitted, plus s_i+1, stays
                 * <= (1-alpha)M (DESIGN Q12); stop at the first failure.                 */
                int64_t L = 0;
                for (int64_t k = 0; k < nS; k++) L += (int64_t)s[S[k]] + t + 1 - p[S[k]];
                int64_t admitted = 0, idle_before = (nS == 0);
                while (nR > 0) {
                    int32_t i = R[0];
                    if (L + s[i] + 1 > B) break;
                    L += (int64_t)s[i] + 1;
                    p[i] = (int32_t)t;
                    c[i] = (int32_t)(t + o[i]);
                    S[nS++] = i;
                    or_remove_at(R, &nR, 0);
                    admitted++;
                }
                /* overflow: the batch of round t needs Mem(t+1) = sum (s_j + t+1 - p_j)
                 * over S u U, including requests finishing at t+1 (Eq. 3; DESIGN Q13).  */
                int64_t mem = 0;
                for (int64_t k = 0; k < nS; k++) mem += (int64_t)s[S[k]] + t + 1 - p[S[k]];
                if (mem > M) {
                    if (policy == OR_ALPHA) {
                        /* "clear all active requests sending them back to the waiting
                         * queue as unprocessed"                                  */
                        for (int64_t k = 0; k < nS; k++) {
                            int32_t j = S[k];
                            p[j] = -1; c[j] = -1;
                            or_insert_sorted(&I, policy, R, &nR, j);
                            evictions++;
                        }
                        nS = 0;
                        /* "infinite processing loops": after a clear-all the state is
                         * (S empty, R, zero memory).  If nothing completed and nothing arrived
                         * since the previous clear-all, R is the same set as then; once no
                         * request is left to arrive, the deterministic run from here repeats
                         * the last cycle for ever (DESIGN Q24).                             */
                        if (next == n && have_clear && next == next_at_clear &&
                            completed_since_clear == 0) {
                            status = OR_LIVELOCK;
                            break;
                        }
                        have_clear = 1;
                        next_at_clear = next;
                        completed_since_clear = 0;
                    } else {
                        /* "each active request is cleared and sent back to the scheduler
                         * with an independent probability beta", in whole passes
                         * until the batch fits (DESIGN Q14), at most OR_BETA_MAX_PASSES of
                         * them; a batch still over M after that is LIVELOCK (DESIGN Q29)  */
                        int64_t pass = 0;
                        for (; pass < OR_BETA_MAX_PASSES; pass++) {
                            for (int64_t k = 0; k < nS; k++)
                                evict[k] = (uint64_t)or_draw(seed, gid, t, pass, S[k]) < beta_thresh;
                            int64_t keep = 0;
                            for (int64_t k = 0; k < nS; k++) {
                                int32_t j = S[k];
                                if (evict[k]) {
                                    p[j] = -1; c[j] = -1;
                                    or_insert_sorted(&I, policy, R, &nR, j);
                                    evictions++;
                                } else {
                                    S[keep++] = j;
                                }
                            }
                            nS = keep;
                            mem = 0;
                            for (int64_t k = 0; k < nS; k++)
                                mem += (int64_t)s[S[k]] + t + 1 - p[S[k]];
                            if (mem <= M || nS == 0) break;
                        }
                        if (pass == OR_BETA_MAX_PASSES) { status = OR_LIVELOCK; break; }
                    }
                }
                /* head-of-line blocked for ever: nothing was running, the FCFS head does
                 * not fit an empty worker (s+1 > B), and no later event can change that */
                if (idle_before && admitted == 0 && nR > 0) { status = OR_LIVELOCK; break; }
            }

            /* memory of the batch processed in round t: sum over S u U of s_j+(t+1-p_j),
             * the occupancy Eq. 3 counts at time t+1                            */
            int64_t mem_now = 0;
            for (int64_t k = 0; k < nS; k++) mem_now += (int64_t)s[S[k]] + t + 1 - p[S[k]];
            if (mem_now > peak) peak = mem_now;
            t++;
        }
    }

    for (int64_t i = 0; i < n; i++) { completion[i] = c[i]; if (start) start[i] = p[i]; }
    stats[0] = stats[1] = stats[3] = -1;
    if (status == OR_OK) {
        /* TEL(I; A) = sum_i c_i - a_i */
        int64_t tel = 0, makespan = 0, rounds = 0;
        for (int64_t i = 0; i < n; i++) {
            tel += (int64_t)c[i] - a[i];
            if (c[i] > makespan) makespan = c[i];
        }
        /* rounds = | union_i [a_i, c_i) | (DESIGN Q11), by marking each round */
        if (n > 0) {
            int64_t lo = a[0];
            char *busy = calloc((size_t)(makespan - lo + 1), 1);
            for (int64_t i = 0; i < n; i++)
                for (int64_t r = a[i]; r < c[i]; r++) busy[r - lo] = 1;
            for (int64_t r = 0; r <= makespan - lo; r++) rounds += busy[r];
            free(busy);
        }
        stats[0] = tel; stats[1] = rounds; stats[3] = makespan;
    }
    stats[2] = decision_rounds;
    stats[4] = peak;
    stats[5] = evictions;
    stats[6] = status;

    free(a); free(s); free(o); free(op); free(p); free(c); free(R); free(S); free(U);
    free(Ss); free(Sp); free(Sop); free(Us); free(Uop); free(evict);
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Batch driver: CSR instances, each simulated independently on a pthread pool.          */
/* gid of instance k = gid0 + k (the alpha-beta RNG key, DESIGN Q14).                    */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int64_t n_inst; const int64_t *offset; const int32_t *req; const int32_t *mem;
    int32_t policy, alpha_num, alpha_den; uint64_t beta_thresh, seed; int64_t round_cap;
    uint64_t gid0;
    int32_t *completion, *start;
    int64_t *tel, *rounds, *decision_rounds, *evictions;
    int32_t *makespan, *peak, *status;
    int64_t next;           /* shared work counter */
    pthread_mutex_t lock;
} or_batch;

static void *or_batch_worker(void *arg)
{
    or_batch *B = (or_batch *)arg;
    for (;;) {
        pthread_mutex_lock(&B->lock);
        int64_t k = B->next++;
        pthread_mutex_unlock(&B->lock);
        if (k >= B->n_inst) break;
        int64_t lo = B->offset[k], hi = B->offset[k + 1];
        int64_t st[7];
        or_simulate(hi - lo, B->req + 4 * lo, B->mem[k], B->policy, B->alpha_num,
                    B->alpha_den, B->beta_thresh, B->seed, B->round_cap, B->gid0 + (uint64_t)k,
                    B->completion + lo, B->start ? B->start + lo : NULL, st);
        B->tel[k] = st[0]; B->rounds[k] = st[1]; B->decision_rounds[k] = st[2];
        B->makespan[k] = (int32_t)st[3]; B->peak[k] = (int32_t)st[4];
        B->evictions[k] = st[5]; B->status[k] = (int32_t)st[6];
    }
    return NULL;
}

int or_simulate_batch(int64_t n_inst, const int64_t *offset, const int32_t *req,
                      const int32_t *mem, int32_t policy, int32_t alpha_num, int32_t alpha_den,
                      uint64_t beta_thresh, uint64_t seed, int64_t round_cap, uint64_t gid0,
                      int32_t nthreads,
                      int32_t *completion, int32_t *start, int64_t *tel, int64_t *rounds,
                      int64_t *decision_rounds, int32_t *makespan, int32_t *peak,
                      int64_t *evictions, int32_t *status)
{
    if (policy < OR_MCSF || policy > OR_MCSF_PROT_RAISE) return -1;
    if (policy == OR_ALPHA_BETA && (beta_thresh == 0 || beta_thresh > (1ull << 32))) return -1;
    or_batch B = { n_inst, offset, req, mem, policy, alpha_num, alpha_den, beta_thresh, seed,
                   round_cap, gid0, completion, start, tel, rounds, decision_rounds, evictions,
                   makespan, peak, status, 0, PTHREAD_MUTEX_INITIALIZER };
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int k = 0; k < nthreads; k++) pthread_create(&th[k], NULL, or_batch_worker, &B);
    for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th);
    return 0;
}

/* TEL(I; A) = sum_i (c_i - a_i); -1 if any request is unfinished (c_i < 0). */
int64_t or_tel(int64_t n, const int32_t *req, const int32_t *completion)
{
    int64_t tel = 0;
    for (int64_t i = 0; i < n; i++) {
        if (completion[i] < 0) return -1;
        tel += (int64_t)completion[i] - req[4 * i + 0];
    }
    return tel;
}

/* ------------------------------------------------------------------------------------ */
/* Hindsight optimum of the IP, Eqs. 1-4, for tiny instances.                */
/* Exhaustive search over start rounds: at every round t the search tries every subset   */
/* of the arrived, unstarted requests as the set starting at t (x_{i,t} = 1, Eq. 2), and */
/* keeps the absolute-round memory profile of Eq. 3 <= M.  Branch-and-bound: a branch is */
/* cut when its partial TEL plus, for each unstarted request, its earliest possible       */
/* latency max(a_i, t+1) + o_i - a_i cannot beat the incumbent.  The incumbent starts at */
/* `ub` (any feasible TEL, e.g. MC-SF's), so the result is min(OPT, ub) = OPT.           */
/* ------------------------------------------------------------------------------------ */
typedef struct {
    int n; int32_t M;
    const int32_t *a, *s, *o;
    int64_t H;            /* profile length (absolute rounds 0..H-1) */
    int64_t *prof;        /* Eq. 3 LHS by absolute round             */
    int32_t *p, *bestp;
    int64_t best;
    int64_t nodes;
} or_opt;

static int or_opt_add(or_opt *X, int i, int64_t k, int sign)
{
    /* started at k, request i holds s_i + t - k at t = k+1..k+o_i (Eq. 3) */
    int ok = 1;
    for (int64_t tt = k + 1; tt <= k + X->o[i]; tt++) {
        X->prof[tt] += sign * ((int64_t)X->s[i] + tt - k);
        if (X->prof[tt] > X->M) ok = 0;
    }
    return ok;
}

static void or_opt_round(or_opt *X, int64_t t, uint32_t unstarted, int64_t partial);

/* choose, among the arrived unstarted requests with index >= from, which start at t */
static void or_opt_subset(or_opt *X, int64_t t, uint32_t unstarted, uint32_t avail,
                          int from, int64_t partial)
{
    for (int i = from; i < X->n; i++) {
        if (!(avail & (1u << i))) continue;
        /* option: i starts at t (then continue choosing among i+1..) */
        int ok = or_opt_add(X, i, t, +1);
        if (ok) {
            X->p[i] = (int32_t)t;
            or_opt_subset(X, t, unstarted & ~(1u << i), avail, i + 1,
                          partial + t + X->o[i] - X->a[i]);
            X->p[i] = -1;
        }
        or_opt_add(X, i, t, -1);
        /* option: i does not start at t -> handled by the loop moving to the next i */
    }
    /* the chosen subset is final; go to round t+1 */
    or_opt_round(X, t + 1, unstarted, partial);
}

static void or_opt_round(or_opt *X, int64_t t, uint32_t unstarted, int64_t partial)
{
    X->nodes++;
    if (unstarted == 0) {
        if (partial < X->best) {
            X->best = partial;
            for (int i = 0; i < X->n; i++) X->bestp[i] = X->p[i];
        }
        return;
    }
    /* bound: every unstarted request starts at >= max(a_i, t) */
    int64_t lb = partial;
    int64_t tmin_arr = INT64_MAX;
    for (int i = 0; i < X->n; i++)
        if (unstarted & (1u << i)) {
            int64_t st = X->a[i] > t ? X->a[i] : t;
            lb += st + X->o[i] - X->a[i];
            if (X->a[i] < tmin_arr) tmin_arr = X->a[i];
        }
    if (lb >= X->best) return;
    if (t + X->M + 1 >= X->H) return;         /* unreachable: lb < best bounds t (below) */
    if (tmin_arr > t) t = tmin_arr;           /* nothing can start before it arrives */
    uint32_t avail = 0;
    for (int i = 0; i < X->n; i++)
        if ((unstarted & (1u << i)) && X->a[i] <= t) avail |= 1u << i;
    or_opt_subset(X, t, unstarted, avail, 0, partial);
}

/* Returns OPT (<= ub); best_start receives an optimal start vector when OPT < ub and is
 * left untouched otherwise.  n <= 20.  -1 on bad arguments.                              */
int64_t or_opt_bruteforce(int64_t n, const int32_t *req, int32_t M, int64_t ub,
                          int32_t *best_start, int64_t *nodes_out)
{
    if (n < 0 || n > 20) return -1;
    if (n == 0) return 0;
    int32_t a[20], s[20], o[20], p[20], bp[20];
    int64_t sum_o = 0, amax = 0;
    for (int i = 0; i < n; i++) {
        a[i] = req[4 * i]; s[i] = req[4 * i + 1]; o[i] = req[4 * i + 2];
        if (s[i] + o[i] > M) return -1;
        p[i] = -1; bp[i] = best_start ? best_start[i] : -1;
        sum_o += o[i];
        if (a[i] > amax) amax = a[i];
    }
    /* horizon: lb < best <= ub forces t + o_i - a_i < ub for every unstarted i, so a start
     * round t < amax + ub and every profile write lands below amax + ub + M (DESIGN Q22) */
    or_opt X;
    X.n = (int)n; X.M = M; X.a = a; X.s = s; X.o = o;
    X.H = amax + ub + M + 2;
    X.prof = calloc((size_t)X.H + 1, sizeof(int64_t));
    X.p = p; X.bestp = bp; X.best = ub; X.nodes = 0;
    or_opt_round(&X, 0, (n == 32) ? 0xffffffffu : ((1u << n) - 1u), 0);
    if (best_start && X.best < ub)
        for (int i = 0; i < n; i++) best_start[i] = bp[i];
    if (nodes_out) *nodes_out = X.nodes;
    free(X.prof);
    return X.best;
}

/* ------------------------------------------------------------------------------------ */
/* LB_sorted for all-at-0 instances.  The k requests that finish first occupy            */
/* vol_i = s_i o_i + o_i(o_i+1)/2 slot-rounds each inside rounds 1..c_(k) with    */
/* capacity M per round (the volume argument of P:319), so c_(k) >= ceil(V_k / M), V_k = */
/* the sum of the k smallest volumes; also c_(k) >= o_(k), the k-th smallest o.          */
/* TEL = sum_k c_(k) >= sum_k max(ceil(V_k/M), o_(k)).                                   */
/* ------------------------------------------------------------------------------------ */
static int or_cmp_i64(const void *x, const void *y)
{
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return (a > b) - (a < b);
}

int64_t or_lb_sorted(int64_t n, const int32_t *req, int32_t M)
{
    int64_t *vol = malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t *os = malloc(sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; i++) {
        int64_t s = req[4 * i + 1], o = req[4 * i + 2];
        vol[i] = s * o + o * (o + 1) / 2;
        os[i] = o;
    }
    qsort(vol, (size_t)n, sizeof(int64_t), or_cmp_i64);
    qsort(os, (size_t)n, sizeof(int64_t), or_cmp_i64);
    int64_t lb = 0, V = 0;
    for (int64_t k = 0; k < n; k++) {
        V += vol[k];
        int64_t c1 = (V + M - 1) / M;
        lb += c1 > os[k] ? c1 : os[k];
    }
    free(vol); free(os);
    return lb;
}

/* ------------------------------------------------------------------------------------ */
/* NEXT-4: the wall clock of a schedule under an affine batch time (SPEC's DurationModel, */
/* the stand-in for the Vidur timing of P:459; DESIGN Q28).  Feasibility stays in rounds; */
/* round r (r0 = a_0 <= r < makespan) processes tokens(r) = sum_{p_i = r} s_i (prefill) + */
/* #{i : p_i < r < c_i} (one decode token each) and lasts c0 + c1 tokens(r).  W(r) = the  */
/* start time of round r, W(r0) = 0.  Outputs: tel_wall = sum_i W(c_i) - W(a_i),        */
/* makespan_wall = W(max c); tokens of round r counted in bin floor(W(r) / bin_width)     */
/* (bins >= n_bins dropped); mem[j] = sum_{i: p_i <= r < c_i} (s_i + r + 1 - p_i) for     */
/* r = r0 + j (the batch memory of round r), j < trace_len.  Plain round-by-round loop.   */
/* Returns -1 if some request is unscheduled (c < 0).                                     */
/* ------------------------------------------------------------------------------------ */
int or_wallclock(int64_t n, const int32_t *req, const int32_t *start, const int32_t *completion,
                 int64_t c0, int64_t c1, int64_t bin_width, int32_t n_bins, int32_t trace_len,
                 int64_t *tel_wall, int64_t *makespan_wall, int64_t *bins, int32_t *mem)
{
    for (int32_t b = 0; b < n_bins; b++) bins[b] = 0;
    for (int32_t j = 0; j < trace_len; j++) mem[j] = 0;
    *tel_wall = 0;
    *makespan_wall = 0;
    if (n == 0) return 0;
    int64_t r0 = req[0], rend = 0;
    for (int64_t i = 0; i < n; i++) {
        if (completion[i] < 0 || start[i] < 0) return -1;
        if (completion[i] > rend) rend = completion[i];
    }
    /* W(r) for r0 <= r <= rend */
    int64_t *W = malloc(sizeof(int64_t) * (size_t)(rend - r0 + 2));
    W[0] = 0;
    for (int64_t r = r0; r < rend; r++) {
        int64_t tokens = 0, m = 0;
        for (int64_t i = 0; i < n; i++) {
            int64_t p = start[i], c = completion[i], s = req[4 * i + 1];
            if (p == r) tokens += s;                       /* prefill */
            else if (p < r && r < c) tokens += 1;          /* one decode token */
            if (p <= r && r < c) m += s + r + 1 - p;       /* batch memory (Eq. 3 at r+1) */
        }
        W[r - r0 + 1] = W[r - r0] + c0 + c1 * tokens;
        if (bin_width > 0) {
            int64_t b = W[r - r0] / bin_width;
            if (b < n_bins) bins[b] += tokens;
        }
        if (r - r0 < trace_len) mem[r - r0] = (int32_t)m;
    }
    for (int64_t i = 0; i < n; i++)
        *tel_wall += W[completion[i] - r0] - W[req[4 * i] - r0];
    *makespan_wall = W[rend - r0];
    free(W);
    return 0;
}
