/* tests/native/oracle_san_driver.c -- TEST INFRASTRUCTURE ONLY: runs oracle/oracle.c, built
 * with -fsanitize=address,undefined, over batches written by tests/test_oracle_sanitize.py.
 *
 *   oracle_san_driver <batch.bin> <policy> <alpha_num> <alpha_den> <beta_thresh> <seed> <out.bin>
 *
 * batch.bin: int64 n_inst, int64 offset[n_inst+1], int32 req[n_req][4], int32 mem[n_inst].
 * out.bin:   int32 completion[n_req], int32 start[n_req], int64 stats[n_inst][7]
 *            (or_simulate, one instance at a time, single thread), then for MC-SF also
 *            int64 lb and opt for the first instances with n <= 8 (or_lb_sorted,
 *            or_opt_bruteforce) and int64 tel (or_tel) per instance.                     */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

int or_simulate(int64_t n, const int32_t *req, int32_t M, int32_t policy, int32_t alpha_num,
                int32_t alpha_den, uint64_t beta_thresh, uint64_t seed, int64_t round_cap,
                uint64_t gid, int32_t *completion, int32_t *start, int64_t *stats);
int64_t or_tel(int64_t n, const int32_t *req, const int32_t *completion);
int64_t or_lb_sorted(int64_t n, const int32_t *req, int32_t M);
int64_t or_opt_bruteforce(int64_t n, const int32_t *req, int32_t M, int64_t ub, int32_t *best_start,
                          int64_t *nodes_out);
int or_wallclock(int64_t n, const int32_t *req, const int32_t *start, const int32_t *completion,
                 int64_t c0, int64_t c1, int64_t bin_width, int32_t n_bins, int32_t trace_len,
                 int64_t *tel_wall, int64_t *makespan_wall, int64_t *bins, int32_t *mem);

static void *rd(FILE *f, size_t bytes)
{
    void *p = malloc(bytes ? bytes : 1);
    if (bytes && fread(p, 1, bytes, f) != bytes) { fprintf(stderr, "short read\n"); exit(3); }
    return p;
}

int main(int argc, char **argv)
{
    if (argc != 8) return 2;
    FILE *f = fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t ni;
    if (fread(&ni, 8, 1, f) != 1) return 3;
    int64_t *off = rd(f, 8 * (size_t)(ni + 1));
    int64_t nr = off[ni];
    int32_t *req = rd(f, 16 * (size_t)nr);
    int32_t *mem = rd(f, 4 * (size_t)ni);
    fclose(f);
    int policy = atoi(argv[2]);
    int an = atoi(argv[3]), ad = atoi(argv[4]);
    uint64_t bt = strtoull(argv[5], 0, 10), seed = strtoull(argv[6], 0, 10);
    int32_t *comp = malloc(4 * (size_t)(nr + 1)), *start = malloc(4 * (size_t)(nr + 1));
    int64_t *stats = malloc(8 * 7 * (size_t)(ni + 1));
    int64_t *tel = malloc(8 * (size_t)(ni + 1));
    for (int64_t k = 0; k < ni; k++) {
        int64_t lo = off[k], n = off[k + 1] - off[k];
        if (or_simulate(n, req + 4 * lo, mem[k], policy, an, ad, bt, seed, 0, (uint64_t)k,
                        comp + lo, start + lo, stats + 7 * k) != 0) return 4;
        tel[k] = or_tel(n, req + 4 * lo, comp + lo);
        if (stats[7 * k + 6] == 0 && n > 0) {           /* exercise the wall-clock model too */
            int64_t tw, mw, bins[16];
            int32_t trace[64];
            or_wallclock(n, req + 4 * lo, start + lo, comp + lo, 3, 1, 7, 16, 64, &tw, &mw, bins, trace);
        }
    }
    FILE *o = fopen(argv[7], "wb");
    fwrite(comp, 4, (size_t)nr, o);
    fwrite(start, 4, (size_t)nr, o);
    fwrite(stats, 8, 7 * (size_t)ni, o);
    fwrite(tel, 8, (size_t)ni, o);
    if (policy == 0) {
        for (int64_t k = 0; k < ni && k < 40; k++) {
            int64_t lo = off[k], n = off[k + 1] - off[k];
            int64_t lb = or_lb_sorted(n, req + 4 * lo, mem[k]), opt = -1, nodes = 0;
            if (n > 0 && n <= 8 && mem[k] <= 20 && stats[7 * k + 6] == 0) {
                int32_t bs[8];
                opt = or_opt_bruteforce(n, req + 4 * lo, mem[k], stats[7 * k], bs, &nodes);
            }
            fwrite(&lb, 8, 1, o);
            fwrite(&opt, 8, 1, o);
        }
    }
    fclose(o);
    free(off); free(req); free(mem); free(comp); free(start); free(stats); free(tel);
    return 0;
}
