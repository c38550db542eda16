/*
 * oracle/c/di_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, sequential float64 C implementation of the D-Iteration (DI)
 * algorithm of Hong, Huynh & Mathieu, "D-Iteration: diffusion approach for
 * solving PageRank" (arxiv 1501.06350, /root/reference/PAPER.md).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this code.  It shares no code, header or constant
 * with the CUDA product path (paper_1501_06350_b200/csrc/).
 *
 * Graph representation used by every function here: the columns of the
 * diffusion matrix P (§2.1, Eq. (1)), stored source-major:
 *   col_ptr[j] .. col_ptr[j+1]-1   entries of column j of P
 *   row_idx[e]                     the row i of entry e (a target node)
 *   pval[e]                        the value P_{i,j} = w_{j,i} / sum_k w_{j,k}
 * Parallel entries (same i twice in one column) are allowed and simply add,
 * which is the same as merging w_{j,i} by summation.  A column with no entry
 * is a dangling node (§2.1: "0 if i is a dangling node").
 *
 * No blocking, no reordering, no fusion: each loop follows the paper's
 * equation it cites, in the paper's order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------------
 * One elementary diffusion of node i (§3.1, Eqs. (8) and (10)):
 *   H_k = H_{k-1} + F_{k-1}(i) e_i
 *   F_k = F_{k-1} + d F_{k-1}(i) P e_i - F_{k-1}(i) e_i
 * The "- F(i) e_i" term is applied before the push so that a self-loop
 * (P_{i,i} > 0) leaves d F(i) P_{i,i} at i, exactly as Eq. (8) states.
 * If column i is empty (dangling) the fluid leaves the system; the leak
 * l_k of §3.3 ("the total amount of fluid that has left the system when a
 * diffusion was applied on a dangling node") is increased by F_{k-1}(i).
 * ---------------------------------------------------------------------- */
static void diffuse_one(int64_t i, const int64_t *col_ptr, const int32_t *row_idx,
                        const double *pval, double d, double *F, double *H,
                        double *leak, int64_t *edges)
{
    double f = F[i];                       /* F_{k-1}(i_k) */
    H[i] += f;                             /* Eq. (10) */
    F[i] -= f;                             /* third term of Eq. (8) */
    int64_t b = col_ptr[i], e = col_ptr[i + 1];
    if (b == e) {                          /* dangling column: fluid lost */
        *leak += f;
        return;
    }
    for (int64_t k = b; k < e; ++k)        /* second term of Eq. (8): d F(i) P e_i */
        F[row_idx[k]] += d * f * pval[k];
    *edges += e - b;
}

static double l1_norm(int64_t n, const double *F, double *fmax)
{
    double s = 0.0, m = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        s += fabs(F[i]);
        if (fabs(F[i]) > m) m = fabs(F[i]);
    }
    if (fmax) *fmax = m;
    return s;
}

/* ------------------------------------------------------------------------
 * Sequential DI with a scheduler (§3.4):
 *   sched 0 = DI-cyc    "a Round-Robin (RR) one, where a given permutation of
 *                        nodes is repeated" (identity permutation here);
 *   sched 1 = DI-argmax "we run through the scheduler until we find a node
 *                        that possesses a fluid greater or equal to the
 *                        average fluid in the whole graph".
 * The average fluid uses |F|_1 / n, recomputed from scratch before every
 * choice (slow and obviously correct; magnitude |F(i)| so that the signed
 * fluid of a Theorem-4 restart is handled, reading R6).
 * Stops as soon as |F|_1 <= tol or after max_steps diffusions.
 * Returns the number of diffusions performed (k).
 * ---------------------------------------------------------------------- */
int64_t orc_seq_run(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                    const double *pval, double d, int sched, double tol,
                    int64_t max_steps, double *F, double *H, double *leak,
                    int64_t *edges, int64_t *cursor_io)
{
    int64_t k = 0;
    int64_t cursor = cursor_io ? *cursor_io : 0;
    double fmax = 0.0;
    double r = l1_norm(n, F, &fmax);
    while (k < max_steps && r > tol) {
        int64_t i;
        if (sched == 0) {
            i = cursor;
            cursor = (cursor + 1) % n;
        } else {
            double avg = r / (double)n;
            /* the max-fluid node always qualifies, so this terminates (the
             * min() only guards against rounding of r / n above max |F|) */
            if (avg > fmax) avg = fmax;
            for (;;) {
                i = cursor;
                cursor = (cursor + 1) % n;
                if (fabs(F[i]) >= avg && F[i] != 0.0) break;
            }
        }
        diffuse_one(i, col_ptr, row_idx, pval, d, F, H, leak, edges);
        ++k;
        r = l1_norm(n, F, &fmax);
    }
    if (cursor_io) *cursor_io = cursor;
    return k;
}

/* ------------------------------------------------------------------------
 * The data-parallel sweep (reading R1): one sweep diffuses, at the
 * same time, every node of the frontier
 *     S = { i : |F(i)| >= T, F(i) != 0 },   T = min(theta |F|_1 / n, max_i |F(i)|)
 * using the fluid values read before the sweep.  Step by step:
 *   1. r = |F|_1 (and max |F(i)|); stop if r <= tol.
 *   2. T as above (theta = 1 is DI-argmax's "average fluid" rule, theta = 0
 *      diffuses every node holding fluid).
 *   3. snapshot f_i = F(i) for i in S; H(i) += f_i; F(i) -= f_i   (Eq. (10),
 *      third term of Eq. (8))
 *   4. for i in S in ascending order: F += d f_i P e_i, or leak += f_i if i is
 *      dangling (second term of Eq. (8); §3.3 leak).
 * This is a composition of Eq. (8)-style updates that each move the snapshot
 * amount f_i, so Eq. (12) H + F = F_0 + dPH holds after every sweep.
 * Returns the number of sweeps performed.  residual_out = |F|_1 at exit.
 * ---------------------------------------------------------------------- */
int64_t orc_sweep_run(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                      const double *pval, double d, double theta, double tol,
                      int64_t max_sweeps, double *F, double *H, double *leak,
                      int64_t *edges, int64_t *nodes, double *residual_out)
{
    int64_t sweeps = 0;
    double *f = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t *S = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double r = 0.0;
    for (;;) {
        /* step 1 */
        double fmax = 0.0;
        r = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double a = fabs(F[i]);
            r += a;
            if (a > fmax) fmax = a;
        }
        if (r <= tol || sweeps >= max_sweeps) break;
        /* step 2 */
        double T = theta * r / (double)n;
        if (T > fmax) T = fmax;
        /* step 3 */
        int64_t s = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (F[i] != 0.0 && fabs(F[i]) >= T) {
                S[s] = i;
                f[s] = F[i];
                H[i] += F[i];
                F[i] -= f[s];
                ++s;
            }
        }
        /* step 4 */
        for (int64_t t = 0; t < s; ++t) {
            int64_t i = S[t];
            int64_t b = col_ptr[i], e = col_ptr[i + 1];
            if (b == e) {
                *leak += f[t];
                continue;
            }
            for (int64_t k = b; k < e; ++k)
                F[row_idx[k]] += d * f[t] * pval[k];
            *edges += e - b;
        }
        *nodes += s;
        ++sweeps;
    }
    free(f);
    free(S);
    if (residual_out) *residual_out = r;
    return sweeps;
}

/* ------------------------------------------------------------------------
 * Power Iteration (§2.2, Eq. (5)):  x_{k+1} = d P x_k + (1-d) Z,
 * run until |x_{k+1} - x_k|_1 <= eps ("until the change between two
 * consecutive vectors is negligible") or max_iter.  x holds x_0 on entry.
 * Returns the number of iterations; *last_delta = |x_K - x_{K-1}|_1.
 * ---------------------------------------------------------------------- */
int64_t orc_power_iteration(int64_t n, const int64_t *col_ptr, const int32_t *row_idx,
                            const double *pval, double d, const double *Z, double eps,
                            int64_t max_iter, double *x, double *last_delta)
{
    double *y = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int64_t it = 0;
    double delta = INFINITY;
    while (it < max_iter) {
        for (int64_t i = 0; i < n; ++i) y[i] = (1.0 - d) * Z[i];
        for (int64_t j = 0; j < n; ++j)          /* y += d P x, column by column */
            for (int64_t k = col_ptr[j]; k < col_ptr[j + 1]; ++k)
                y[row_idx[k]] += d * pval[k] * x[j];
        delta = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            delta += fabs(y[i] - x[i]);
            x[i] = y[i];
        }
        ++it;
        if (delta <= eps) break;
    }
    free(y);
    if (last_delta) *last_delta = delta;
    return it;
}

/* ------------------------------------------------------------------------
 * Tile-local sweeps (readings R12, R15), a D-Iteration schedule
 * ("freedom in the choice of a scheduler", §3.4), step by step:
 *   1. r = |F|_1; stop if r <= tol.
 *   2. for each wave c = 0 .. waves-1 (tile index mod waves = c):
 *      a. for each tile [a, a+tile) of the wave, in ascending order, starting
 *         from the tile's fluid f = F[a..): `rounds` times: every tile node i
 *         with f(i) != 0 is diffused (Eqs. (8), (10)): D(i) += f(i), and
 *         d f(i) P_{t,i} is pushed to its out-neighbours t INSIDE the tile (the
 *         new f); F[a..) = f.
 *      b. then, for every node i of the wave, the pushes of all its diffusions
 *         to targets OUTSIDE its tile: F(t) += d D(i) P_{t,i} (Eq. (8) is
 *         linear in the diffused amount) -- a tile of a later wave takes them
 *         in during this sweep, any other tile in the next one.
 *      c. H += D; l += D(i) for dangling i (§3.3).
 *   3. (partitions, R16) with nb > 1 partition bounds
 *      bounds[0] = 0 < bounds[1] < ... < bounds[nb-1] = n, a push of step 2b
 *      whose source and target lie in different partitions is held back and
 *      added to F after the sweep's last wave (the ranks exchange once a sweep).
 * waves = 1, rounds = 1 is the theta = 0 sweep of orc_sweep_run.
 * ---------------------------------------------------------------------- */
static int64_t part_of(const int64_t *bounds, int64_t nb, int64_t x)
{
    int64_t p = 0;                                /* largest p with bounds[p] <= x */
    while (p + 1 < nb - 1 && bounds[p + 1] <= x) ++p;
    return p;
}

int64_t orc_tiled_sweep_run(int64_t n, const int64_t *col_ptr, const int32_t *row_idx, const double *pval,
                            double d, int64_t tile, int rounds, int waves, double tol, int64_t max_sweeps,
                            double *F, double *H, double *leak, int64_t *edges, int64_t *nodes,
                            double *residual_out, const int64_t *bounds, int64_t nb)
{
    int64_t sweeps = 0;
    double *D = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *f = (double *)malloc(sizeof(double) * (size_t)(tile > 0 ? tile : 1));
    double *fn = (double *)malloc(sizeof(double) * (size_t)(tile > 0 ? tile : 1));
    double *Fx = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));   /* held-back cross-partition pushes */
    int64_t *pt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    const int parted = bounds != NULL && nb > 2;
    for (int64_t i = 0; i < n; ++i) pt[i] = parted ? part_of(bounds, nb, i) : 0;
    double r = 0.0;
    if (waves < 1) waves = 1;
    for (;;) {
        r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += fabs(F[i]);
        if (r <= tol || sweeps >= max_sweeps) break;
        for (int c = 0; c < waves; ++c) {
            for (int64_t i = 0; i < n; ++i) D[i] = 0.0;
            for (int64_t a = (int64_t)c * tile; a < n; a += (int64_t)waves * tile) {
                int64_t z = a + tile < n ? a + tile : n;
                for (int64_t i = a; i < z; ++i) f[i - a] = F[i];
                for (int k = 0; k < rounds; ++k) {
                    for (int64_t i = a; i < z; ++i) fn[i - a] = 0.0;
                    for (int64_t i = a; i < z; ++i) {
                        double fi = f[i - a];
                        if (fi == 0.0) continue;
                        D[i] += fi;
                        *nodes += 1;
                        *edges += col_ptr[i + 1] - col_ptr[i];
                        for (int64_t e = col_ptr[i]; e < col_ptr[i + 1]; ++e) {
                            int64_t t = row_idx[e];
                            if (t >= a && t < z) fn[t - a] += d * fi * pval[e];
                        }
                    }
                    for (int64_t i = a; i < z; ++i) f[i - a] = fn[i - a];
                }
                for (int64_t i = a; i < z; ++i) F[i] = f[i - a];
            }
            for (int64_t i = 0; i < n; ++i) {
                if (D[i] == 0.0) continue;
                int64_t a = (i / tile) * tile, z = a + tile;
                if (col_ptr[i] == col_ptr[i + 1]) *leak += D[i];
                for (int64_t e = col_ptr[i]; e < col_ptr[i + 1]; ++e) {
                    int64_t t = row_idx[e];
                    if (t >= a && t < z) continue;
                    if (pt[t] != pt[i]) Fx[t] += d * D[i] * pval[e];
                    else F[t] += d * D[i] * pval[e];
                }
                H[i] += D[i];
            }
        }
        if (parted)
            for (int64_t i = 0; i < n; ++i) {
                F[i] += Fx[i];
                Fx[i] = 0.0;
            }
        ++sweeps;
    }
    free(Fx);
    free(pt);
    free(D);
    free(f);
    free(fn);
    if (residual_out) *residual_out = r;
    return sweeps;
}
