// dit_internal.cuh -- internal types and device helpers of libdit (B200, sm_100a).
// The C ABI is include/dit.h; DESIGN.md describes the data layout and kernels.
#pragma once

#include <functional>
#include <mutex>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dit.h"

namespace dit {

constexpr int kThreads = 256;           // block size of every grid-stride kernel
constexpr int kWarps = kThreads / 32;
constexpr int64_t kSplit = 512;         // a frontier row is split into entries of <= kSplit edges
constexpr int kSplitShift = 9;
constexpr int kLenBits = 24;            // entry: begin (40 bits) | len (24 bits)
constexpr int64_t kNodeTile = 512;      // TILED: node ids per tile (= DI_TILE_NODES)
// ctrl->use_pull: which diffusion kernels run this sweep
constexpr int kUsePush = 0, kUsePull = 1, kUseTiled = 2;

// One record per sweep, written by the last block of k_reduce.
struct SweepRec {
    unsigned long long entries, edges, nodes_cum;
    int use_pull, pad;
};
constexpr int64_t kHistCap = 1 << 16;
constexpr int kEvPerSweep = 17;         // profiling events per sweep (tiled: 2 W + 1; waves > 8 not timed)

// Device-resident control block: the solver loop runs without host round
// trips; the host polls `done` once per chunk of sweeps.
struct Ctrl {
    double resid;            // |F|_1 of the current F (from the last reduce)
    double fmax;             // max_i |F(i)|
    double T;                // frontier threshold of the next select
    double leak;             // l, fluid consumed at dangling nodes
    double d, theta, tol;
    double pull_edges;       // AUTO: pull when frontier edges > pull_edges
    unsigned long long n_entries;       // frontier entries written this sweep
    unsigned long long sel_edges;       // out-edges of this sweep's frontier
    unsigned long long sweeps;          // sweeps done in the current call
    unsigned long long max_sweeps;
    unsigned long long diffused_nodes;  // cumulative over the current call
    unsigned long long diffused_edges;
    unsigned long long push_sweeps, pull_sweeps;
    SweepRec *hist;                     // per-sweep records (device), kHistCap entries
    double n_global;                    // n of the whole graph (threshold denominator)
    double *stats_out;                  // shard mode: local {r, fmax, leak, sel_edges} go here
    double gleak;                       // shard mode: leak summed over ranks (k_control), -1 before
    unsigned long long last_sel_edges;  // frontier out-edges of the last sweep
    int stats_is_init;
    unsigned int done;
    unsigned int sel_blocks;            // last-block counters
    unsigned int red_blocks;
    int variant;                        // DI_VARIANT_* requested
    int use_pull;                       // decision for the current sweep
    int gather;                         // TILED: remote pushes of the last sweep are pending in A
};

// A CSC (targets -> in-edges, ascending source) and its pull work plan:
// pieces of <= 64 in-edges that never cross a 2048-edge tile, split targets.
struct PullPlan {
    bool built = false;            // CSC ready
    bool pieces_built = false;     // pull work plan ready (built on the first pull-variant call)
    int64_t nt = 0, m = 0;         // targets, edges
    int64_t *ptr = nullptr;        // [nt+1]
    int32_t *src = nullptr;        // [m] source row of each in-edge
    void *w = nullptr;             // [m] raw weight (graph storage kind) or null
    uint4 *pieces = nullptr;       // {begin<<24 | len, target, split}
    int64_t npieces = 0;
    int4 *fix = nullptr;           // split targets: {j, first piece lo, hi, count}
    int64_t nfix = 0;
    double *pbuf = nullptr;        // [npieces] partial sums of split targets
    int64_t *tile_start = nullptr; // [ntiles+1] first piece of each 2048-edge tile
    int64_t ntiles = 0;
};

// Tile-local schedule (R12, §5): node tiles of kNodeTile ids.  An
// in-edge is LOCAL when its source is in the target's tile (u16 tile-relative
// source), otherwise REMOTE.  Remote in-edges of "light" targets sit per tile
// in a {source, weight} record array that the tile kernel stages with TMA and
// gathers itself; "heavy" targets (many remote in-edges, or tiles whose light
// records would overflow kLightCap) are gathered by k_heavy over fixed chunks
// of the heavy edge array (segments = target ∩ chunk), deterministic.
#ifndef DIT_LIGHT_CAP
#define DIT_LIGHT_CAP 1344
#endif
constexpr int64_t kLightCap = DIT_LIGHT_CAP;   // light remote records per tile (shared memory)
#ifndef DIT_HEAVY_TH
#define DIT_HEAVY_TH 16
#endif
constexpr int64_t kHeavyTh = DIT_HEAVY_TH;       // remote in-degree above which a target is heavy
#ifndef DIT_HEAVY_CHUNK
#define DIT_HEAVY_CHUNK 1024
#endif
constexpr int64_t kHeavyChunk = DIT_HEAVY_CHUNK;   // heavy edges per k_heavy chunk
#ifndef DIT_HEAVY_THREADS
#define DIT_HEAVY_THREADS 256
#endif
constexpr int kHeavyThreads = DIT_HEAVY_THREADS;   // block size of k_heavy_chunks

constexpr int32_t kDegLocalDelta = 1 << 30;     // TilePlan::deg: the node has in-round delta in-edges
constexpr int32_t kDegMask = kDegLocalDelta - 1;

struct TilePlan {
    bool built = false;
    int64_t ntile = 0;             // node tiles
    // per node [n]
    uint32_t *rrel = nullptr;      // light remote in-edge start, relative to rtile[tile]
    int32_t *hidx = nullptr;       // heavy index of the target or -1
    float *wr = nullptr;           // share of node i's outflow that leaves its tile: sum_remote w * inv
    int32_t *deg = nullptr;        // out-degree (diffused-edge accounting)
    // per tile [ntile+1]
    int64_t *ltile = nullptr, *rtile = nullptr;
    // local in-edges in a balanced sliced-ELL layout per tile: each target's
    // local in-edge list is cut into pieces of <= cap edges (cap chosen so the
    // tile has <= 2 x kNodeTile pieces); pieces are ranked by length (longest
    // first) and cut into 32 virtual warps of 32; real warp w runs virtual
    // warps w and 31-w (longest with shortest).  Slot s of the piece of rank r
    // sits at ltile[t] + vofs[t*33 + r/32] + ell_slot(s, r%32, K) (dit_tile.cu:
    // runs of 4 slots per lane for s < K - K%4, then 32 s + r%32; padding: source
    // kNodeTile, weight 0).  A target's pieces, in edge order, are the ranks
    // plist[t*1024 + vfirst[t*513 + i] ...  vfirst[t*513 + i + 1]).
    uint32_t *vofs = nullptr;      // [ntile*33]
    uint16_t *vfirst = nullptr;    // [ntile*513]
    uint16_t *plist = nullptr;     // [ntile*1024]
    uint16_t *lsrc = nullptr;      // [mpad] source - tile base (+16 B for aligned TMA supersets)
    void *lw = nullptr;            // [mpad] raw weight (graph storage kind) or null
    int64_t mloc = 0, mpad = 0;    // local in-edges, padded slots
    // light remote in-edges: per target tile, CSC order, {int32 src, weight}
    // records (8 B for f32/unweighted, 16 B for f64), gathered by the tile kernel
    void *rrec = nullptr;          // [mlight] (+16 B)
    int64_t mlight = 0;
    // heavy targets: remote in-edges sorted by (source stripe, target, source);
    // one stripe's slice of the outflow A stays in L2 while its edges are
    // gathered.  Segments = (stripe, target) runs cut at the stripe's 2048-edge
    // chunks; hsum(h) accumulates the runs stripe by stripe (fixed order).
    int64_t nh = 0, mh = 0, nseg = 0, nchunk = 0, nrun = 0;
    int64_t stripe_nodes = 0;
    void *hrec = nullptr;          // [mh] records
    int64_t *chunk_start = nullptr;  // [nchunk+1] first heavy edge of each chunk
    int64_t *seg_start = nullptr;  // [nseg+1] first heavy edge of each segment
    int64_t *cfirst = nullptr;     // [nchunk+1] first segment of each chunk
    int32_t *run_h = nullptr;      // [nrun] heavy index of each run
    int64_t *run_seg = nullptr;    // [nrun+1] first segment of each run
    // fold order: heavy targets grouped by wave (wave_slot), each with its runs in
    // stripe order: runs fold_run[fold_ptr[i] .. fold_ptr[i+1]) of target fold_h[i]
    int64_t *fold_ptr = nullptr;   // [nh+1]
    int32_t *fold_h = nullptr;     // [nh]
    uint32_t *fold_run = nullptr;  // [nrun]
    std::vector<int64_t> wave_slot;   // [waves+1]
    std::vector<int64_t> s_chunk;  // per (wave, stripe) group [W S + 1]: first chunk
    int waves = 1;                 // tile waves per sweep (R15): wave of tile t = t % waves
    int groups = 1;                // heavy groups: the waves, + the ghost slots (group `waves`) on a shard
    int64_t nstripe = 0;           // source stripes S
    double *tpart = nullptr;       // k_tile partials [2][waves][grid]
    double *part = nullptr;        // [nseg] segment partial sums
    double *hsum = nullptr;        // [nh] remote inflow of each heavy target
    int64_t max_tile_edges = 0;    // most local in-edges of one tile
    int32_t *lstage = nullptr;     // [ntile] first slot (relative to ltile) that k_tile stages in shared memory
    // delta in-edges of edge updates since the build (dit_delta.cu, R18):
    // +w added / -w removed, sorted by (target wave, target, source)
    int64_t nd = 0;
    int32_t *dsrc = nullptr, *dtgt = nullptr;
    double *dw = nullptr;
    std::vector<int64_t> dwave;    // [waves+1] first entry of each target wave
    int64_t *dseg = nullptr;       // [segments+1] first entry of each target's run
    std::vector<int64_t> dsegw;    // [waves+1] first segment of each target wave
    double *dval = nullptr;        // [nd] per-sweep scratch: A(s) w of each entry
    // kept delta entries inside one tile (no padding slot), pushed in k_tile's rounds:
    // per node t dl_ptr[t] .. dl_ptr[t+1] {source - tile base, w}; deg bit 30 flags t
    int32_t *dl_ptr = nullptr;     // [n+1] or null (none)
    uint16_t *dl_src = nullptr;
    double *dl_w = nullptr;
    int64_t *dbig = nullptr;       // segments of > 4096 entries (a block each), ascending
    std::vector<int64_t> dbigw;    // [waves+1] first big segment of each wave
    double *rw0 = nullptr;         // [n] plan-time pending out-weight (set at the first update)
};

// removed CSR entries of one update (-w), collected before the CSR swap
struct DeltaBatch {
    int64_t nrem = 0;
    int32_t *s = nullptr, *t = nullptr;
    double *w = nullptr;
};

// Chunks of whole tiles for the plan builder (dit_plan.cu): chunk c is tiles
// [tile_lo[c], tile_lo[c+1]), edges [edge_lo[c], edge_lo[c+1]); with a feed
// (graph create overlapping the upload) its targets / weights are resident once
// col_ready[c] / w_ready[c] fired, and on_col / on_w run right after the waits
// (validation and scales of the chunk, on the build's stream).
struct PlanFeed {
    std::vector<int64_t> tile_lo, edge_lo;
    std::vector<cudaEvent_t> col_ready, w_ready;
    std::function<void(int)> on_col, on_w;
};
constexpr int64_t kPlanChunkEdges = (int64_t)1 << 26;   // plan chunk of the pipelined create (~9 ms of upload)
constexpr int64_t kPlanChunkEdgesLazy = (int64_t)1 << 28; // plan chunk of a build from resident data (fewer syncs)

// Per-node weight-scale storage and raw weights.
struct DevGraph {
    int64_t n = 0, m = 0;          // rows (owned nodes) and edges
    int64_t nt = 0;                // fluid slots = n, + ghost slots for a shard
    int64_t n_global = 0;          // nodes of the whole graph (= n unless shard)
    int64_t lo = 0;                // shard: first owned global id
    bool shard = false;
    int32_t *ghost_ids = nullptr;  // shard: global id of each ghost slot (ascending)
    int32_t *recv_idx = nullptr;   // shard: local target of each received value
    std::vector<int64_t> recv_seg; // shard: received values per source rank
    int64_t *row_ptr = nullptr;    // [n+1]
    int32_t *col = nullptr;        // [m]
    void *w = nullptr;             // [m] float or double raw weights, or null
    int w_kind = DI_W_NONE;        // storage: DI_W_NONE / DI_W_F32 / DI_W_F64
    double *inv = nullptr;         // [n] 1/sum_k w_{j,k} (0: dangling)
    // transpose (built lazily for the pull variant)
    PullPlan t;
    // tile-local schedule (built lazily for DI_VARIANT_TILED)
    TilePlan tl;
};

struct State {
    bool valid = false;
    SweepRec *hist = nullptr;            // [kHistCap] device
    bool profile = false;
    std::vector<cudaEvent_t> events;     // profiling: 5 per sweep
    di_profile last_prof{};
    int64_t launched = 0;                // sweeps enqueued in the current call
    int rounds = 4;                      // TILED local rounds of the current call
    bool tiled_call = false;
    bool flushing = false;               // shard: the next control follows a flush
    bool local_pending = false;          // shard (tiled): this sweep's local wave-0 heavy gather not run yet
    int64_t last_sweeps = 0;
    double d = 0.85;
    double *F = nullptr, *H = nullptr;   // [n]
    double *A = nullptr;                 // [n] pull: outflow amount per node
    double *A2 = nullptr;                // [n] TILED: second outflow buffer (ping-pong by sweep parity)
    uint4 *ent = nullptr;                // frontier entries (16 B each)
    int64_t ent_cap = 0;
    Ctrl *ctrl = nullptr;                // device
    Ctrl *ctrl_host = nullptr;           // pinned mirror
    double *part = nullptr;              // per-block partials (2 per block)
    int grid = 0;                        // grid of the grid-stride kernels
};

}  // namespace dit

struct di_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    dit::DevGraph g;
    dit::State s;
    int num_sms = 148;
};

namespace dit {

// ---- error plumbing (thread-local message) ----
void set_error(const std::string &msg);
struct Fail {
    int code;
};
void check_cuda(cudaError_t e, const char *what);   // throws Fail{DI_ERR_CUDA / DI_ERR_OOM}
#define DI_CUDA(x) ::dit::check_cuda((x), #x)
void count_launch(int k = 1);

// ---- builders / solver (dit_graph.cu, dit_solve.cu) ----
void build_scales(di_graph *h);
void build_transpose(di_graph *h);
void free_graph(DevGraph &g, cudaStream_t st);   // stream-ordered frees (back to the pool, no device sync)
void ensure_state(di_graph *h);
void free_state(State &s, cudaStream_t st);
void run_sweeps(di_graph *h, double tol, const di_solve_opts &o, di_result *res);
void prepare_call(di_graph *h, double tol, const di_solve_opts &o, double *stats_out);
void launch_sweep(di_graph *h);
void launch_sweep_reduce(di_graph *h);
void launch_reduce(di_graph *h, int is_init);
void launch_select(di_graph *h, bool pull);
void launch_push(di_graph *h);
void launch_pull(di_graph *h);
void launch_pull_plan(di_graph *h, const PullPlan &p, const double *A, int want);
void build_plan_pieces(di_graph *h, PullPlan &p);
void free_plan(PullPlan &p, cudaStream_t st);
// feed: chunks arriving during create (then `bad` = the create's validation flags:
// nonzero after the chunks stops the build before its remote part)
void build_tiles(di_graph *h, const PlanFeed *feed = nullptr, const int *bad = nullptr);
void free_tiles(TilePlan &t, cudaStream_t st);
void launch_tile_sweep(di_graph *h, int rounds);
void launch_tile_flush(di_graph *h);
bool delta_enabled(const di_graph *h);
void delta_collect_removed(di_graph *h, const unsigned char *del, const unsigned char *chg, DeltaBatch &out,
                           bool plan);
void delta_batch_free(DeltaBatch &b, cudaStream_t st);
void delta_commit(di_graph *h, DeltaBatch &rem, const int32_t *as, const int32_t *ad, const double *aw, int64_t nadd,
                  const unsigned char *chg);
void launch_delta(di_graph *h, int wave, int force);
void *cub_scratch(int device, size_t bytes);   // dit_pull.cu: CUB scratch cached per device
void release_cub_scratch(int device);
std::mutex &scratch_mutex(int device);         // builds on one device take turns on the cached scratch
void launch_tile_heavy(di_graph *h, int force, int wave = 0, int group = -1);
void launch_tile_kernel(di_graph *h, int rounds, int wave = 0);
int tile_waves(const di_graph *h);
void launch_take_ghost_sums(di_graph *h, double *out, int force);
void launch_reduce_exact(di_graph *h);
void mark_event(di_graph *h, int64_t sweep, int k);
bool poll_done(di_graph *h);
void fill_result(di_graph *h, const di_solve_opts &o, double tol, di_result *res);
void init_state(di_graph *h, double d, const double *Z_dev);
void write_H(di_graph *h, double factor, double *H_out, int mem);
void set_leak_from_history(di_graph *h);
void create_graph(di_graph *h, int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                  const void *weights, int w_dtype, int mem, int64_t col_bound);
int grid_for(di_graph *h, int64_t count);
void create_shard(di_graph *h, int64_t n_global, int64_t lo, int64_t hi, int64_t m, const int64_t *row_ptr,
                  const int32_t *col, const void *weights, int w_dtype, int mem);
void shard_set_recv(di_graph *h, int64_t total, const int32_t *local_idx, int nseg, const int64_t *seg_counts,
                    int mem);
void shard_sweep(di_graph *h, double *ghost_out);
void shard_heavy_local(di_graph *h);
void shard_apply(di_graph *h, const double *recv, int force);
void shard_control(di_graph *h, const double *gathered, int nranks, int force);
void shard_reduce(di_graph *h);
void shard_flush(di_graph *h, double *ghost_out);
void shard_flush_apply(di_graph *h, const double *recv);
void update_edges(di_graph *h, int64_t n_add, const int32_t *add_src, const int32_t *add_dst,
                  const void *add_w, int w_dtype, int64_t n_rem, const int32_t *rem_src,
                  const int32_t *rem_dst, int mem);
void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t count, cudaStream_t st);
std::pair<uint32_t *, uint32_t *> radix_sort_u32(uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1,
                                                 int64_t count, int bits, cudaStream_t st);
std::pair<uint32_t *, uint64_t *> radix_sort_u32_u64(uint32_t *k0, uint64_t *v0, uint32_t *k1, uint64_t *v1,
                                                     int64_t count, int bits, cudaStream_t st);

// ---- DIT_BUILD_TIMING (debug): host-side phase timer, stream-synchronised ----
void phase_mark(cudaStream_t st, const char *name);

// ---- device helpers ----
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if ((int)lane_id() >= o) v += u;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Fire-and-forget float64 add at L2 (RED.E.ADD.F64).
__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Streaming 32-bit load that does not allocate in L1 (index/weight streams).
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t *p) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream_f32(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double ld_stream_f64(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <typename W>
__device__ __forceinline__ double load_w(const W *w, int64_t e);
template <>
__device__ __forceinline__ double load_w<float>(const float *w, int64_t e) { return (double)ld_stream_f32(w + e); }
template <>
__device__ __forceinline__ double load_w<double>(const double *w, int64_t e) { return ld_stream_f64(w + e); }

struct NoW {};

// Next-sweep control from the (global) residual r and max fluid fm.
__device__ __forceinline__ void finalize_control(Ctrl *ctrl, double r, double fm, int is_init, int64_t m) {
    ctrl->resid = r;
    ctrl->fmax = fm;
    const double T = ctrl->theta * r / ctrl->n_global;
    ctrl->T = T < fm ? T : fm;
    ctrl->done = (r <= ctrl->tol || ctrl->sweeps >= ctrl->max_sweeps) ? 1u : 0u;
    // direction of the next sweep: AUTO takes this sweep's frontier out-edges
    // as the estimate of the next one's (the first sweep from a uniform F_0
    // takes every node)
    const unsigned long long fe = is_init ? (unsigned long long)m : ctrl->last_sel_edges;
    if (ctrl->variant == DI_VARIANT_TILED) ctrl->use_pull = kUseTiled;
    else if (ctrl->variant == DI_VARIANT_PULL) ctrl->use_pull = kUsePull;
    else if (ctrl->variant == DI_VARIANT_PUSH) ctrl->use_pull = kUsePush;
    else ctrl->use_pull = ((double)fe > ctrl->pull_edges) ? kUsePull : kUsePush;
}

// End-of-sweep bookkeeping (last block of the sweep's final kernel): leak,
// per-sweep record, counters, per-sweep accumulators reset.
__device__ __forceinline__ void end_sweep(Ctrl *ctrl, double lk) {
    ctrl->leak += lk;
    if (ctrl->hist && ctrl->sweeps < (unsigned long long)kHistCap) {
        SweepRec rec;
        rec.entries = ctrl->n_entries;
        rec.edges = ctrl->sel_edges;
        rec.nodes_cum = ctrl->diffused_nodes;
        rec.use_pull = ctrl->use_pull;
        rec.pad = 0;
        ctrl->hist[ctrl->sweeps] = rec;
    }
    ctrl->sweeps += 1;
    ctrl->diffused_edges += ctrl->sel_edges;
    if (ctrl->use_pull == kUsePush) ctrl->push_sweeps += 1; else ctrl->pull_sweeps += 1;
    ctrl->last_sel_edges = ctrl->sel_edges;
}

}  // namespace dit
