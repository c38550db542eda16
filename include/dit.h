/*
 * dit.h -- C ABI of the B200 D-Iteration engine (libdit.so).
 *
 * D-Iteration (DI): Hong, Huynh, Mathieu, "D-Iteration: diffusion approach for
 * solving PageRank", arxiv 1501.06350.  The engine solves
 *
 *     x = d P x + (1-d) Z                                   (§2.1, Eq. (3))
 *
 * by fluid diffusion (§3.1, Eqs. (7)-(10)): fluid F starts at F_0 = (1-d) Z,
 * history H at 0; diffusing node i adds F(i) to H(i), clears F(i) and pushes
 * d F(i) P_{j,i} to every out-neighbour j.  The GPU engine diffuses a whole
 * frontier { i : |F(i)| >= T } per sweep (reading R1) and repeats
 * until |F|_1 <= tol; Theorem 1 (Eq. (11)) then bounds |x - H|_1 <= |F|_1/(1-d).
 *
 * Conventions for every entry point
 *  - Return value: DI_OK (0) on success, a DI_ERR_* code otherwise; the text
 *    of the last error of the calling thread is returned by di_last_error().
 *    On error no output argument is written and the graph handle keeps its
 *    previous, consistent state (except DI_ERR_CUDA, after which the handle
 *    should only be destroyed).
 *  - `mem` arguments say where a pointer lives: DI_MEM_HOST (pageable or
 *    pinned host memory; copied by the call) or DI_MEM_DEVICE (device memory
 *    on the graph's CUDA device; read on the graph's stream, never retained).
 *  - Node ids are int32 in [0, n); CSR offsets are int64.  All fluid and
 *    history arithmetic is float64.
 *  - Calls are synchronous with respect to the host: when one returns, its
 *    outputs are written.  A handle must not be used by two threads at once.
 *  - Ownership: the library copies every input; the caller owns all buffers
 *    it passes and the library owns the handle until di_graph_destroy().
 */
#ifndef DIT_H
#define DIT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define DI_OK                 0
#define DI_ERR_INVALID        1   /* bad argument (null pointer, size, id out of range, d not in (0,1)) */
#define DI_ERR_CUDA           2   /* CUDA runtime error (message has the CUDA error string) */
#define DI_ERR_OOM            3   /* device allocation failed */
#define DI_ERR_EDGE_NOT_FOUND 4   /* di_update_edges: a removal names an absent edge */
#define DI_ERR_STATE          5   /* di_resume / di_get_state before any solve */

/* ---- memory kinds ---- */
#define DI_MEM_HOST   0
#define DI_MEM_DEVICE 1

/* ---- edge-weight dtypes ---- */
#define DI_W_NONE 0               /* unweighted: P_{i,j} = 1/out(j)              (§2.1) */
#define DI_W_F32  1               /* float32 raw weights w_{j,i} > 0              (Eq. (1)) */
#define DI_W_F64  2               /* float64 raw weights (stored as f32 when every value is
                                     exactly representable, else as f64)        */

/* ---- dangling-node handling (§2.1 "dangling node", §3.3 implicit completion) ---- */
#define DI_DANGLING_DROP     0    /* P stays substochastic; fluid reaching a dangling node
                                     leaves the system; H -> x of Eq. (3) */
#define DI_DANGLING_COMPLETE 1    /* Z-completion (1/n completion for uniform Z) computed
                                     implicitly, §3.3: H is returned multiplied by
                                     (1-d)/(1-d-d l) and the bound is |F|_1/(1-d-d l) */

/* ---- diffusion-kernel variant ---- */
#define DI_VARIANT_AUTO 0         /* per sweep: pull when the frontier is dense, else push */
#define DI_VARIANT_PUSH 1         /* push-scatter over the CSR with float64 atomic adds */
#define DI_VARIANT_PULL 2         /* deterministic pull-gather over the transpose (CSC) */
#define DI_VARIANT_TILED 3        /* tile-local schedule (R12): per node tile of
                                     DI_TILE_NODES ids, `local_rounds` diffusion rounds in shared
                                     memory over the tile's internal edges; the pushes along the
                                     other edges are gathered by their targets at the start of
                                     the next sweep (deterministic); every node holding fluid
                                     diffuses (theta is not used). */
#define DI_TILE_NODES 512         /* node ids per tile of DI_VARIANT_TILED */
#define DI_TILE_WAVES 3           /* DI_VARIANT_TILED: the tiles of a sweep run in this many
                                     waves (tile index mod waves); a wave's pushes to tiles of
                                     later waves are taken in during the same sweep (DESIGN.md
                                     R15).  Shards number waves from their first tile; pushes to
                                     other ranks land after the sweep's exchange (R16). */

typedef struct di_graph di_graph;  /* opaque: device CSR + derived arrays + DI state */

typedef struct {
    double  theta;       /* frontier threshold factor: T = min(theta |F|_1 / n, max|F|).
                            1.0 = DI-argmax's "average fluid" rule (§3.4); 0 = every node
                            holding fluid.  Must be in [0, 1]. Default 1.0. */
    int32_t variant;     /* DI_VARIANT_*, default DI_VARIANT_AUTO */
    int32_t dangling;    /* DI_DANGLING_*, default DI_DANGLING_DROP */
    int64_t max_sweeps;  /* stop after this many sweeps even if |F|_1 > tol; <= 0: 10^7 */
    double  pull_frac;   /* AUTO: use pull when frontier out-edges > pull_frac * m; default 0.25 */
    int32_t local_rounds;/* TILED: diffusion rounds per tile per sweep (>= 1), default 4 */
    int32_t reserved;
} di_solve_opts;

typedef struct {
    double  residual_l1;    /* |F|_1 at return (Theorem 1's "remaining fluid") */
    double  bound;          /* L1 distance bound of the returned H to the solution:
                               |F|_1/(1-d) (Eq. (11)) or |F|_1/(1-d-d l) (§3.3) */
    double  leak;           /* l: fluid consumed at dangling nodes = sum_{dangling j} H(j) */
    double  norm_factor;    /* factor applied to H on output: 1 or (1-d)/(1-d-d l) */
    int64_t sweeps;         /* sweeps performed by this call */
    int64_t diffused_nodes; /* elementary diffusions (frontier sizes summed) */
    int64_t diffused_edges; /* out-edges of the diffused nodes, summed */
    int64_t push_sweeps;    /* sweeps that ran the push variant */
    int64_t pull_sweeps;    /* sweeps that ran the pull variant */
    int32_t converged;      /* 1 if |F|_1 <= tol at return */
    int32_t reserved;
} di_result;

/* Fill `o` with the defaults listed above. */
void di_solve_opts_default(di_solve_opts *o);

/*
 * di_graph_create -- build the engine's graph from a CSR edge list by source.
 *   n        number of nodes (>= 0, < 2^31)
 *   m        number of edges (= row_ptr[n])
 *   row_ptr  int64[n+1], non-decreasing, row_ptr[0] = 0; out-edges of node j are
 *            col[row_ptr[j] .. row_ptr[j+1]-1]
 *   col      int32[m], targets in [0, n).  Parallel edges are allowed and
 *            merge by weight summation; self-loops are allowed (Eq. (1)).
 *   weights  NULL (w_dtype DI_W_NONE) or w_dtype[m] raw weights, each > 0
 *   mem      DI_MEM_HOST / DI_MEM_DEVICE for row_ptr, col and weights
 *   device   CUDA device ordinal
 *   stream   cudaStream_t every call on this handle runs on (NULL = the CUDA
 *            default stream, the usual CUDA convention)
 * Builds on the device (Eq. (1)): the per-source scale
 * 1/sum_k w_{j,k} (1/out(j) unweighted; 0 marks a dangling node).  The
 * transpose of the pull / push variants and the tile plan of DI_VARIANT_TILED
 * (built straight from the CSR) are built lazily on first use --
 * except that a graph of 2^24 edges or more given in PINNED host memory
 * (float32 or no weights) gets its tile plan during this call, chunk by chunk
 * while its edges upload (the plan is the same bits either way).
 * Errors: DI_ERR_INVALID (sizes, null pointers, ids out of range, w <= 0),
 *         DI_ERR_OOM, DI_ERR_CUDA.
 */
int di_graph_create(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                    const void *weights, int32_t w_dtype, int32_t mem, int32_t device,
                    void *stream, di_graph **out);

/* Free every device buffer of the handle.  NULL is a no-op. */
int di_graph_destroy(di_graph *g);

/* n, m and the storage of the weights (DI_W_*) of the graph. */
int di_graph_info(const di_graph *g, int64_t *n, int64_t *m, int32_t *w_storage);

/*
 * di_solve -- cold DI solve (§3.1): F_0 = (1-d) Z, H_0 = 0, sweep until
 * |F|_1 <= tol or opts->max_sweeps.
 *   d      damping, 0 < d < 1
 *   Z      float64[n] default distribution (entries >= 0; not renormalised)
 *          or NULL for uniform 1/n; Z_mem says where it lives
 *   tol    stop when |F|_1 <= tol (>= 0)
 *   opts   NULL for defaults
 *   H_out  NULL or float64[n] receiving H (times res->norm_factor), H_mem
 *   res    NULL or receives the di_result
 * The (F, H, l, d) state stays in the handle for di_resume / di_update_edges.
 */
int di_solve(di_graph *g, double d, const double *Z, int32_t Z_mem, double tol,
             const di_solve_opts *opts, double *H_out, int32_t H_mem, di_result *res);

/*
 * di_resume -- continue sweeping from the state left by di_solve / di_resume
 * / di_update_edges (warm restart, Theorem 4) until |F|_1 <= tol.
 * Errors: DI_ERR_STATE if no state exists.
 */
int di_resume(di_graph *g, double tol, const di_solve_opts *opts, double *H_out,
              int32_t H_mem, di_result *res);

/*
 * di_update_edges -- dynamic-graph update (§3.5, Theorem 4).
 * Removes every edge (rem_src[q] -> rem_dst[q]) (all parallel copies) and
 * appends the edges (add_src[q] -> add_dst[q], weight add_w[q]); the
 * per-source scales of the touched sources are recomputed.  If a DI state
 * exists, the corrective fluid of Theorem 4 is injected,
 *     F'_0 = F + d (P' - P) H,   H'_0 = H,
 * touching only the changed columns of P, so that di_resume converges to the
 * solution of x' = d P' x' + (1-d) Z.  F may become negative (§3.5).
 *   add_w   NULL (unit weights) or w_dtype[n_add]; must be NULL for an
 *           unweighted graph unless every value is 1
 *   mem     where add_* and rem_* live
 * Errors: DI_ERR_INVALID (ids out of range, w <= 0), DI_ERR_EDGE_NOT_FOUND
 * (a removal names no existing edge; the graph and state are unchanged).
 */
int di_update_edges(di_graph *g, int64_t n_add, const int32_t *add_src, const int32_t *add_dst,
                    const void *add_w, int32_t w_dtype, int64_t n_rem, const int32_t *rem_src,
                    const int32_t *rem_dst, int32_t mem);

/*
 * di_get_state / di_set_state -- copy the raw DI state out of / into the
 * handle: F, H (float64[n], not normalised), the damping d and the leak l.
 * di_set_state lets a caller start sweeps from any (F, H) (e.g. a saved
 * state); its d must be in (0,1).  NULL F/H pointers are skipped by get.
 */
int di_get_state(const di_graph *g, double *F, double *H, int32_t mem, double *d, double *leak);
int di_set_state(di_graph *g, double d, const double *F, const double *H, int32_t mem, double leak);

/*
 * Profiling (bench.py's roofline): when enabled on a handle, every sweep of
 * the next di_solve / di_resume is bracketed by CUDA events on the handle's
 * stream and the per-sweep frontier sizes are recorded on the device.
 * di_profile_get returns, per kernel class, the summed event durations and the
 * ALGORITHMIC bytes of the launches that did work.
 */
typedef struct {
    double  select_ms, push_ms, pull_ms, reduce_ms;
    double  select_bytes, push_bytes, pull_bytes, reduce_bytes;
    int64_t select_launches, push_launches, pull_launches, reduce_launches;
    int64_t sweeps;
    double  tile_ms, tile_bytes;      /* TILED: the tile-local kernel (pull_* = remote pull) */
    int64_t tile_launches;
} di_profile;

int di_profile_enable(di_graph *g, int32_t on);
int di_profile_get(const di_graph *g, di_profile *out);

/*
 * Per-sweep frontier history of the last di_solve / di_resume call: for sweep
 * s < *count (at most cap), the frontier size nodes[s], its out-edges
 * edges[s], the push entries entries[s] and variant[s] (1 = pull).  Any
 * output pointer may be NULL.  Up to 65536 sweeps are recorded.
 */
int di_sweep_history(const di_graph *g, int64_t cap, int64_t *nodes, int64_t *edges, int64_t *entries,
                     int32_t *variant, int64_t *count);

/*
 * ---- Multi-GPU shards ----
 * One process per GPU owns the contiguous node range [lo, hi) of a graph with
 * n_global nodes: its out-edges (CSR rows lo..hi-1, `col` holding GLOBAL ids)
 * and the fluid / history of its nodes.  Fluid pushed to a node of another
 * rank accumulates in a "ghost" slot (one per distinct remote target, in
 * ascending global id); after every sweep the caller moves the ghost fluid
 * to its owners (an all-to-all, e.g. NCCL over NVLink) and adds what it
 * received with di_shard_apply; the residual and max fluid are all-reduced
 * (sum / max) by the caller between di_shard_reduce and di_shard_control.
 * Every di_shard_* call except create/info/ghost_ids/set_recv/poll/finish is
 * asynchronous on the handle's stream.  DESIGN.md reading R1 covers why the
 * exchange after the sweep is still an exact D-Iteration.
 */
int di_shard_create(int64_t n_global, int64_t lo, int64_t hi, int64_t m, const int64_t *row_ptr,
                    const int32_t *col, const void *weights, int32_t w_dtype, int32_t mem, int32_t device,
                    void *stream, di_graph **out);
/* owned nodes (hi - lo), ghost slots, lo */
int di_shard_info(const di_graph *g, int64_t *n_local, int64_t *n_ghost, int64_t *lo);
/* global ids of the ghost slots, ascending (int32[n_ghost]) */
int di_shard_ghost_ids(const di_graph *g, int32_t *ids, int32_t mem);
/* receive map: local_idx[total] (owned ids - lo) in the order values arrive,
 * cut into nseg consecutive segments of seg_counts[k] values (one per source
 * rank; ids are distinct within a segment) */
int di_shard_set_recv(di_graph *g, int64_t total, const int32_t *local_idx, int32_t nseg,
                      const int64_t *seg_counts, int32_t mem);
/* F_0 = (1-d) Z on owned nodes (Z: owned slice or NULL = 1/n_global), H_0 = 0;
 * local {|F|_1, max|F|, leak, frontier edges} -> stats (device double[4],
 * retained until di_shard_finish) */
int di_shard_begin(di_graph *g, double d, const double *Z, int32_t Z_mem, double tol,
                   const di_solve_opts *opts, double *stats);
/* next threshold / done flag from every rank's stats, gathered in rank order:
 * gathered = device double[4 * nranks] (an all-gather of the stats buffers).
 * The device sums |F|_1 and the leak and takes max |F| over ranks in rank order
 * (deterministic, one collective per sweep); the global leak l (PAPER §3.3)
 * sets di_shard_finish's completion factor and bound. */
int di_shard_control(di_graph *g, const double *gathered, int32_t nranks);
/* one sweep (select + diffusion); ghost fluid moved to ghost_out (device double[n_ghost]) */
int di_shard_sweep(di_graph *g, double *ghost_out);
/* DI_VARIANT_TILED: the sweep's heavy gather of the rank's own wave-0 targets
 * (PAPER §3.1 Eq. (8) pushes of the previous sweep), which does
 * not depend on the exchange: call it after starting the all-to-all of the
 * ghost fluid di_shard_sweep wrote, so the two overlap.  Optional (di_shard_apply
 * runs it first when it was not called); a no-op for the other variants. */
int di_shard_heavy_local(di_graph *g);
/* F[local_idx[q]] += recv[q] (device double[total]), segment by segment */
int di_shard_apply(di_graph *g, const double *recv);
/* local statistics of the current F into the stats buffer given to di_shard_begin */
int di_shard_reduce(di_graph *g);
/* After the sweeps (poll says done): the pushes still pending (DI_VARIANT_TILED
 * completes a sweep's remote pushes at the start of the next one, DESIGN.md
 * R13) exchanged like a sweep: di_shard_flush writes the ghost fluid to
 * ghost_out (zeros for the other variants), the caller runs the all-to-all,
 * di_shard_flush_apply adds what it received, gathers the local pending pushes
 * into F and takes the exact local |F|_1 into stats; after the all-reduce,
 * di_shard_control re-derives `done` from the exact residual (the sweeps
 * continue if it is above tol). */
int di_shard_flush(di_graph *g, double *ghost_out);
int di_shard_flush_apply(di_graph *g, const double *recv);
/* host-synchronous: 1 once the control block says done */
int di_shard_poll(di_graph *g, int32_t *done);
/* local H (owned nodes) and local counters; residual_l1 / bound are global */
int di_shard_finish(di_graph *g, double tol, const di_solve_opts *opts, double *H_out, int32_t H_mem,
                    di_result *res);

/*
 * Sizes of the graph's DI_VARIANT_TILED plan (built by the first tiled solve;
 * DESIGN.md §5), written to stats[0 .. min(cap, DI_PLAN_STATS)-1] in this order:
 * node tiles, local in-edges, sliced-ELL slots (local edges + padding), light
 * remote in-edges, heavy remote in-edges, heavy targets, heavy segments, heavy
 * runs, heavy chunks, source stripes.  All zero before the plan exists.
 */
#define DI_PLAN_STATS 10
int di_plan_stats(const di_graph *g, int64_t *stats, int32_t cap);

/* Text of the last error raised on the calling thread ("" if none). */
const char *di_last_error(void);

/* Number of kernel launches issued by the library since load (for bench). */
int64_t di_kernel_launches(void);

/*
 * Give the device memory the library keeps cached back to the driver.  The
 * engine allocates from the device's stream-ordered default pool with an
 * unlimited release threshold, reserves it once for the plan builder's peak
 * (about 40 B per edge + 256 B per node) and keeps the transpose's sort
 * buffers (24 B per edge) and CUB's scratch outside the pool:
 * repeated graph builds then reuse mapped memory.  Call this (with no
 * solve running on the device) when other allocators in the process need
 * that memory.  device: CUDA ordinal.  Returns DI_OK or DI_ERR_CUDA.
 */
int di_release_memory(int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* DIT_H */
