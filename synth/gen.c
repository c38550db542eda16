/*
 * synth/gen.c -- seeded synthetic graph generator shared by tests, bench.py
 * and the oracle.  Holds NONE of the D-Iteration arithmetic: it only emits a
 * CSR edge list by source (row_ptr int64[n+1], col int32[m]) and optional raw
 * edge weights (float32, exactly representable), reproducing the workload
 * shapes named in BASELINE.json's configs (see DESIGN.md §"Input recipe").
 *
 * Counter-based: every random draw is mix64(seed, stream, node, k), so the
 * output is identical for any thread count and any node range [lo, hi)
 * (multi-GPU ranks generate only their own rows).
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <omp.h>

static inline uint64_t mix64(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline uint64_t rnd(uint64_t seed, uint64_t stream, uint64_t node, uint64_t k)
{
    return mix64(mix64(mix64(seed ^ (stream << 56)) ^ node) + k);
}

static inline double unit(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

enum { DEG_UNIFORM = 0, DEG_GEOMETRIC = 1, DEG_POWERLAW = 2 };
enum { TGT_UNIFORM = 0, TGT_HOSTZIPF = 1 };

typedef struct {
    uint64_t seed;
    int64_t n;
    int deg_kind;          /* DEG_* */
    double deg_a;          /* uniform: max degree; geometric: mean; powerlaw: exponent */
    double deg_b;          /* powerlaw: x_min */
    int64_t deg_cap;
    double p_dangling;
    int tgt_kind;          /* TGT_* */
    int64_t block;         /* host block size (ids) */
    double p_local;        /* probability a target falls in the host block */
    double zipf_s;         /* Zipf exponent (1.0 supported: log-uniform rank) */
} synth_params;

/* -------- out-degree of node i -------- */
static int64_t degree_of(const synth_params *P, int64_t i)
{
    if (unit(rnd(P->seed, 1, (uint64_t)i, 0)) < P->p_dangling) return 0;
    double u = unit(rnd(P->seed, 2, (uint64_t)i, 0));
    int64_t k;
    switch (P->deg_kind) {
    case DEG_UNIFORM:       /* uniform on 1..deg_a */
        k = 1 + (int64_t)(rnd(P->seed, 2, (uint64_t)i, 1) % (uint64_t)P->deg_a);
        break;
    case DEG_GEOMETRIC: {   /* geometric on {1,2,...} with mean deg_a */
        double p = 1.0 / P->deg_a;
        k = 1 + (int64_t)floor(log1p(-u) / log1p(-p));
        break;
    }
    default: {              /* Pareto(x_min = deg_b, exponent deg_a), floored */
        double x = P->deg_b * pow(1.0 - u, -1.0 / (P->deg_a - 1.0));
        k = x > 1e18 ? (int64_t)1e18 : (int64_t)floor(x);
        if (k < 1) k = 1;
    }
    }
    if (k > P->deg_cap) k = P->deg_cap;
    return k;
}

/* -------- seeded bijection on [0, n): 4-round Feistel + cycle walking -------- */
static inline uint64_t feistel(uint64_t x, int half, uint64_t seed)
{
    uint64_t mask = (1ULL << half) - 1, L = x >> half, R = x & mask;
    for (int r = 0; r < 4; ++r) {
        uint64_t F = mix64(R ^ (seed + 0x1234567ULL * (uint64_t)(r + 1))) & mask;
        uint64_t nL = R, nR = L ^ F;
        L = nL; R = nR;
    }
    return (L << half) | R;
}

static inline int64_t permute(int64_t x, int64_t n, uint64_t seed)
{
    int half = 1;
    while ((1ULL << (2 * half)) < (uint64_t)n) ++half;
    uint64_t y = (uint64_t)x;
    do { y = feistel(y, half, seed); } while (y >= (uint64_t)n);
    return (int64_t)y;
}

/* -------- target of the k-th out-edge of node i -------- */
static int32_t target_of(const synth_params *P, int64_t i, int64_t k, uint64_t stream)
{
    int64_t n = P->n;
    if (n <= 1) return 0;
    uint64_t r0 = rnd(P->seed, stream, (uint64_t)i, (uint64_t)(2 * k));
    uint64_t r1 = rnd(P->seed, stream, (uint64_t)i, (uint64_t)(2 * k + 1));
    int64_t t;
    if (P->tgt_kind == TGT_UNIFORM) {               /* uniform, no self-loop */
        t = (int64_t)(r0 % (uint64_t)(n - 1));
        if (t >= i) ++t;
        return (int32_t)t;
    }
    if (unit(r0) < P->p_local) {                    /* inside the host block */
        int64_t b0 = (i / P->block) * P->block;
        int64_t bs = P->block;
        if (b0 + bs > n) bs = n - b0;
        if (bs > 1) {
            t = b0 + (int64_t)(r1 % (uint64_t)(bs - 1));
            if (t >= i) ++t;
            return (int32_t)t;
        }
    }
    /* Zipf(s = 1) rank by inverse CDF of the continuous log-uniform law on
     * [1, n+1): rank = floor((n+1)^u) - 1, P(rank = r) ~ ln((r+2)/(r+1)),
     * then a seeded permutation scatters the ranks over the node ids */
    double u = unit(r1);
    int64_t rank = (int64_t)floor(exp(u * log((double)n + 1.0))) - 1;
    if (rank < 0) rank = 0;
    if (rank >= n) rank = n - 1;
    t = permute(rank, n, P->seed ^ 0xabcdef12345ULL);
    if (t == i) t = (t + 1) % n;
    return (int32_t)t;
}

/* degrees of nodes [lo, hi) into deg[0 .. hi-lo) */
void synth_degrees(const synth_params *P, int64_t lo, int64_t hi, int64_t *deg)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = lo; i < hi; ++i) deg[i - lo] = degree_of(P, i);
}

/* edges of nodes [lo, hi); row_ptr (hi-lo+1 entries, local offsets from 0)
 * must already hold the exclusive prefix sum of synth_degrees.  w may be NULL. */
void synth_edges(const synth_params *P, int64_t lo, int64_t hi, const int64_t *row_ptr,
                 int32_t *col, float *w)
{
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = lo; i < hi; ++i) {
        int64_t b = row_ptr[i - lo], e = row_ptr[i - lo + 1];
        for (int64_t k = 0; k < e - b; ++k) {
            col[b + k] = target_of(P, i, k, 3);
            if (w) {
                uint64_t j = rnd(P->seed, 4, (uint64_t)i, (uint64_t)k) >> 42;   /* 22 bits */
                w[b + k] = (float)(0.5 + 3.0 * (double)j / 8388608.0);        /* [0.5, 2.0), exact in f32 */
            }
        }
    }
}

/* targets for (src[q], k[q]) pairs drawn from a separate stream (used for the
 * dynamic-update insertions of config 4) */
void synth_targets(const synth_params *P, int64_t count, const int64_t *src, const int64_t *k,
                   uint64_t stream, int32_t *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < count; ++q) out[q] = target_of(P, src[q], k[q], 16 + stream);
}

int synth_num_threads(void) { return omp_get_max_threads(); }
