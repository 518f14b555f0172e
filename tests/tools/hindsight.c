/* tests/tools/hindsight.c -- NEXT-2: best-known hindsight schedules for the
 * paper's synthetic experiments by large-neighbourhood search.  CPU analysis
 * code (test infrastructure), not the product path.
 *
 * The hindsight optimum is the IP of Eqs. 1-4: choose start rounds p_i >= a_i
 * minimising sum_i (p_i + o_i - a_i) subject to, for every round r,
 *     sum_{i : p_i < r <= p_i + o_i} (s_i + r - p_i) <= M.
 * The paper solves it with Gurobi; neither Gurobi nor an exact solver for n = 40-60 is
 * available here (HiGHS does not solve one instance in 15 min), so this searches
 * feasible schedules from MC-SF's: TEL(best found) >= OPT, hence
 *     TEL(MC-SF) / TEL(best found) <= TEL(MC-SF) / OPT,
 * a lower bound on each trial's ratio.
 *
 * Search: remove k requests (k in 2..8: random, adjacent in start order, or overlapping a
 * random one), re-insert them in a random or shortest-first order, each at the earliest
 * round >= a_i at which its ramp fits the profile of the others; keep the result if TEL does
 * not increase (ties accepted, so the search drifts across plateaus); restart from the best
 * every 2000 rejected moves.  Every accepted schedule is re-validated against Eq. 3.
 *
 *   int hs_search(n, req[n][4] {a,s,o,o~}, M, start[n] (in: a feasible schedule, out: the
 *                 best found), iters, seed) -> best TEL, or -1 if the input is infeasible
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int n, M, H;
    const int32_t *a, *s, *o;
    int64_t *prof;
} hs_inst;

static uint64_t hs_rng(uint64_t *x)
{
    *x ^= *x << 13; *x ^= *x >> 7; *x ^= *x << 17;
    return *x;
}

static void hs_apply(hs_inst *I, int i, int p, int sign)
{
    for (int r = p + 1; r <= p + I->o[i]; r++) I->prof[r] += sign * (int64_t)(I->s[i] + r - p);
}

static int hs_fits(const hs_inst *I, int i, int p)
{
    if (p + I->o[i] >= I->H) return 0;
    for (int r = p + 1; r <= p + I->o[i]; r++)
        if (I->prof[r] + I->s[i] + r - p > I->M) return 0;
    return 1;
}

static int hs_earliest(const hs_inst *I, int i)
{
    for (int p = I->a[i]; p + I->o[i] < I->H; p++)
        if (hs_fits(I, i, p)) return p;
    return -1;
}

static inline int64_t hs_tel(const hs_inst *I, const int32_t *p)
{
    int64_t t = 0;
    for (int i = 0; i < I->n; i++) t += (int64_t)p[i] + I->o[i] - I->a[i];
    return t;
}

static int hs_valid(hs_inst *I, const int32_t *p)
{
    memset(I->prof, 0, sizeof(int64_t) * (size_t)I->H);
    for (int i = 0; i < I->n; i++) {
        if (p[i] < I->a[i] || p[i] + I->o[i] >= I->H) return 0;
        hs_apply(I, i, p[i], +1);
    }
    for (int r = 0; r < I->H; r++)
        if (I->prof[r] > I->M) return 0;
    return 1;
}

int64_t hs_search(int n, const int32_t *req, int M, int32_t *start, int64_t iters, uint64_t seed)
{
    int32_t *a = malloc(sizeof(int32_t) * n), *s = malloc(sizeof(int32_t) * n), *o = malloc(sizeof(int32_t) * n);
    int64_t amax = 0, so = 0;
    for (int i = 0; i < n; i++) {
        a[i] = req[4 * i]; s[i] = req[4 * i + 1]; o[i] = req[4 * i + 2];
        if (a[i] > amax) amax = a[i];
        so += o[i];
    }
    hs_inst I = {n, M, 0, a, s, o, NULL};
    int64_t tel0 = 0;
    for (int i = 0; i < n; i++) tel0 += (int64_t)start[i] + o[i] - a[i];
    I.H = (int)(amax + tel0 + M + 2);
    I.prof = calloc((size_t)I.H + 1, sizeof(int64_t));
    int32_t *cur = malloc(sizeof(int32_t) * n), *best = malloc(sizeof(int32_t) * n);
    int32_t *sel = malloc(sizeof(int32_t) * n), *ord = malloc(sizeof(int32_t) * n), *save = malloc(sizeof(int32_t) * n);
    int32_t *save_by = malloc(sizeof(int32_t) * n);
    memcpy(cur, start, sizeof(int32_t) * n);
    if (!hs_valid(&I, cur)) { tel0 = -1; goto done; }
    memcpy(best, cur, sizeof(int32_t) * n);
    int64_t tcur = tel0, tbest = tel0;
    uint64_t x = seed * 0x9E3779B97F4A7C15ull + 1;
    int64_t rejected = 0;
    for (int64_t it = 0; it < iters && n > 1; it++) {
        /* choose the neighbourhood */
        int k = 2 + (int)(hs_rng(&x) % 7);
        if (k > n) k = n;
        const int mode = (int)(hs_rng(&x) % 3);
        int m = 0;
        char *in = calloc((size_t)n, 1);
        if (mode == 0) {                                   /* random */
            while (m < k) { int i = (int)(hs_rng(&x) % n); if (!in[i]) { in[i] = 1; sel[m++] = i; } }
        } else if (mode == 1) {                            /* adjacent in start order */
            for (int i = 0; i < n; i++) ord[i] = i;
            for (int i = 1; i < n; i++) {                  /* insertion sort by start */
                int v = ord[i], j = i - 1;
                while (j >= 0 && cur[ord[j]] > cur[v]) { ord[j + 1] = ord[j]; j--; }
                ord[j + 1] = v;
            }
            int b = (int)(hs_rng(&x) % (n - k + 1));
            for (int j = 0; j < k; j++) { sel[m++] = ord[b + j]; in[ord[b + j]] = 1; }
        } else {                                           /* overlapping a random request */
            int c = (int)(hs_rng(&x) % n);
            sel[m++] = c; in[c] = 1;
            for (int t = 0; t < 4 * n && m < k; t++) {
                int i = (int)(hs_rng(&x) % n);
                if (in[i]) continue;
                if (cur[i] < cur[c] + o[c] && cur[c] < cur[i] + o[i]) { in[i] = 1; sel[m++] = i; }
            }
        }
        free(in);
        /* remove, then re-insert in a random or shortest-first order */
        for (int j = 0; j < m; j++) { save[j] = cur[sel[j]]; save_by[sel[j]] = cur[sel[j]]; hs_apply(&I, sel[j], cur[sel[j]], -1); }
        if (hs_rng(&x) & 1) {
            for (int j = m - 1; j > 0; j--) { int r = (int)(hs_rng(&x) % (j + 1)); int t = sel[j]; sel[j] = sel[r]; sel[r] = t; }
        } else {
            for (int j = 1; j < m; j++) {
                int v = sel[j], q = j - 1;
                while (q >= 0 && (o[sel[q]] > o[v] || (o[sel[q]] == o[v] && a[sel[q]] > a[v]))) { sel[q + 1] = sel[q]; q--; }
                sel[q + 1] = v;
            }
        }
        int ok = 1, placed = 0;
        int64_t tnew = tcur;
        for (int j = 0; j < m; j++) tnew -= save[j];
        for (int j = 0; j < m; j++) {
            int p = hs_earliest(&I, sel[j]);
            if (p < 0) { ok = 0; break; }
            cur[sel[j]] = p;
            hs_apply(&I, sel[j], p, +1);
            tnew += p;
            placed++;
        }
        if (ok && tnew <= tcur) {                          /* accept (ties: plateau moves) */
            tcur = tnew;
            if (tcur < tbest) { tbest = tcur; memcpy(best, cur, sizeof(int32_t) * n); rejected = 0; }
            else rejected++;
        } else {                                           /* exact undo */
            for (int j = 0; j < placed; j++) hs_apply(&I, sel[j], cur[sel[j]], -1);
            for (int j = 0; j < m; j++) { cur[sel[j]] = save_by[sel[j]]; hs_apply(&I, sel[j], cur[sel[j]], +1); }
            rejected++;
        }
        if (rejected > 5000) {                             /* restart from the best */
            memcpy(cur, best, sizeof(int32_t) * n);
            tcur = tbest;
            hs_valid(&I, cur);
            rejected = 0;
        }
    }
    if (!hs_valid(&I, best)) { tbest = -1; }
    memcpy(start, best, sizeof(int32_t) * n);
    tel0 = tbest;
done:
    free(a); free(s); free(o); free(I.prof); free(cur); free(best); free(sel); free(ord); free(save); free(save_by);
    return tel0;
}
