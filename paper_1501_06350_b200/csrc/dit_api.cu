// dit_api.cu -- the extern "C" boundary of libdit (include/dit.h).
// Argument validation, error codes and thread-local error text; every compute
// step is a kernel in dit_graph.cu / dit_solve.cu / dit_pull.cu / dit_scan.cu.
#include "dit_internal.cuh"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>

namespace dit {

static thread_local std::string t_err;
static std::atomic<long long> g_launches{0};

void set_error(const std::string &msg) { t_err = msg; }

void count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

void check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return;
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    cudaGetLastError();   // clear a sticky-free error
    throw Fail{e == cudaErrorMemoryAllocation ? DI_ERR_OOM : DI_ERR_CUDA};
}

template <typename Fn>
static int guarded(Fn &&fn) {
    try {
        fn();
        return DI_OK;
    } catch (const Fail &f) {
        return f.code;
    } catch (const std::exception &ex) {
        t_err = ex.what();
        return DI_ERR_CUDA;
    }
}

static void fail(int code, const char *msg) {
    t_err = msg;
    throw Fail{code};
}

static void use_device(const di_graph *g) { DI_CUDA(cudaSetDevice(g->device)); }

// The builders' temporaries come from the device's default stream-ordered pool;
// keep freed blocks cached there (release threshold = max) so that a second
// build on the device does not remap gigabytes of memory.
static void keep_pool_memory(int device) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// One up-front reservation of the pool for the graph builder's peak (about 40 B
// per edge + 256 B per node, at most 60% of the free memory): the builders then
// carve their temporaries out of one mapped chunk instead of growing the pool
// piecemeal (which costs ~0.1 s of mapping whenever fragmentation forces it).
static std::atomic<bool> g_reserved[64] = {};   // reserve_pool done (reset by di_release_memory)

static void reserve_pool(int device, int64_t n, int64_t m, cudaStream_t st) {
    std::atomic<bool> *done = g_reserved;
    if (device < 0 || device >= 64 || done[device].load() || getenv("DIT_NO_POOL_RESERVE")) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return;
    uint64_t cur = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &cur);
    const uint64_t want = std::min<uint64_t>((uint64_t)(40 * (double)m + 256 * (double)n), (uint64_t)(0.6 * (double)fr));
    if (want < ((uint64_t)1 << 30)) return;         // small graphs: a later big one may still reserve
    if (done[device].exchange(true)) return;        // another thread reserved it meanwhile
    if (want <= cur) return;
    void *p = nullptr;
    if (cudaMallocAsync(&p, want, st) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
}

static di_solve_opts resolve(const di_solve_opts *o) {
    di_solve_opts r;
    di_solve_opts_default(&r);
    if (o) r = *o;
    if (!(r.theta >= 0.0 && r.theta <= 1.0)) fail(DI_ERR_INVALID, "opts.theta must be in [0, 1]");
    if (r.variant < DI_VARIANT_AUTO || r.variant > DI_VARIANT_TILED) fail(DI_ERR_INVALID, "opts.variant");
    if (r.local_rounds < 1 || r.local_rounds > 1000) fail(DI_ERR_INVALID, "opts.local_rounds must be in [1, 1000]");
    if (r.dangling != DI_DANGLING_DROP && r.dangling != DI_DANGLING_COMPLETE) fail(DI_ERR_INVALID, "opts.dangling");
    if (!(r.pull_frac >= 0.0)) fail(DI_ERR_INVALID, "opts.pull_frac must be >= 0");
    return r;
}

static void finish(di_graph *g, const di_solve_opts &o, double tol, double *H_out, int H_mem, di_result *res) {
    di_result r;
    run_sweeps(g, tol, o, &r);
    write_H(g, r.norm_factor, H_out, H_mem);
    if (res) *res = r;
}

}  // namespace dit

using namespace dit;

extern "C" {

void di_solve_opts_default(di_solve_opts *o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->theta = 1.0;
    o->variant = DI_VARIANT_AUTO;
    o->dangling = DI_DANGLING_DROP;
    o->max_sweeps = 10000000;
    o->pull_frac = 0.25;
    o->local_rounds = 4;
}

const char *di_last_error(void) { return t_err.c_str(); }

int64_t di_kernel_launches(void) { return (int64_t)g_launches.load(); }

int di_release_memory(int32_t device) {
    return guarded([&] {
        DI_CUDA(cudaSetDevice(device));
        DI_CUDA(cudaDeviceSynchronize());
        release_cub_scratch(device);
        if (device >= 0 && device < 64) g_reserved[device].store(false);
        cudaMemPool_t pool;
        DI_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        DI_CUDA(cudaMemPoolTrimTo(pool, 0));
    });
}

int di_graph_create(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col, const void *weights,
                    int32_t w_dtype, int32_t mem, int32_t device, void *stream, di_graph **out) {
    return guarded([&] {
        if (!out) fail(DI_ERR_INVALID, "out is NULL");
        if (n < 0 || n >= (1LL << 31) || m < 0) fail(DI_ERR_INVALID, "need 0 <= n < 2^31 and m >= 0");
        if (!row_ptr || (m > 0 && !col)) fail(DI_ERR_INVALID, "row_ptr / col is NULL");
        if (w_dtype != DI_W_NONE && w_dtype != DI_W_F32 && w_dtype != DI_W_F64) fail(DI_ERR_INVALID, "w_dtype");
        if (w_dtype != DI_W_NONE && m > 0 && !weights) fail(DI_ERR_INVALID, "weights is NULL");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        if (mem == DI_MEM_HOST && row_ptr[n] != m) fail(DI_ERR_INVALID, "row_ptr[n] != m");
        if (m >= (1LL << 40)) fail(DI_ERR_INVALID, "m must be < 2^40");
        DI_CUDA(cudaSetDevice(device));
        keep_pool_memory(device);
        di_graph *g = new di_graph();
        g->device = device;
        try {
            cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);
            g->stream = (cudaStream_t)stream;   // NULL = the CUDA default stream
            reserve_pool(device, n, m, g->stream);
            create_graph(g, n, m, row_ptr, col, weights, w_dtype, mem, n);
        } catch (...) {
            free_graph(g->g, g->stream);
            cudaStreamSynchronize(g->stream);
            if (g->own_stream) cudaStreamDestroy(g->stream);
            delete g;
            throw;
        }
        *out = g;
    });
}

int di_graph_destroy(di_graph *g) {
    if (!g) return DI_OK;
    return guarded([&] {
        cudaSetDevice(g->device);
        free_state(g->s, g->stream);                 // stream-ordered: the memory goes back to the pool
        free_graph(g->g, g->stream);
        cudaStreamSynchronize(g->stream);
        if (g->own_stream) cudaStreamDestroy(g->stream);
        delete g;
    });
}

int di_graph_info(const di_graph *g, int64_t *n, int64_t *m, int32_t *w_storage) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        if (n) *n = g->g.n;
        if (m) *m = g->g.m;
        if (w_storage) *w_storage = g->g.w_kind;
    });
}

int di_solve(di_graph *g, double d, const double *Z, int32_t Z_mem, double tol, const di_solve_opts *opts,
             double *H_out, int32_t H_mem, di_result *res) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        if (g->g.shard) fail(DI_ERR_INVALID, "di_solve on a shard handle: use the di_shard_* protocol");
        if (!(d > 0.0 && d < 1.0)) fail(DI_ERR_INVALID, "d must be in (0, 1)");
        if (!(tol >= 0.0)) fail(DI_ERR_INVALID, "tol must be >= 0");
        if ((Z || H_out) && (Z_mem != DI_MEM_HOST && Z_mem != DI_MEM_DEVICE)) fail(DI_ERR_INVALID, "Z_mem");
        if (H_out && H_mem != DI_MEM_HOST && H_mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "H_mem");
        const di_solve_opts o = resolve(opts);
        use_device(g);
        double *Zd = nullptr;
        if (Z && g->g.n > 0) {
            if (Z_mem == DI_MEM_HOST) {
                DI_CUDA(cudaMallocAsync(&Zd, g->g.n * sizeof(double), g->stream));
                DI_CUDA(cudaMemcpyAsync(Zd, Z, g->g.n * sizeof(double), cudaMemcpyHostToDevice, g->stream));
            } else {
                Zd = const_cast<double *>(Z);
            }
        }
        init_state(g, d, Zd);
        if (Zd && Z_mem == DI_MEM_HOST) DI_CUDA(cudaFreeAsync(Zd, g->stream));
        finish(g, o, tol, H_out, H_mem, res);
    });
}

int di_resume(di_graph *g, double tol, const di_solve_opts *opts, double *H_out, int32_t H_mem, di_result *res) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        if (g->g.shard) fail(DI_ERR_INVALID, "di_resume on a shard handle");
        if (!g->s.valid) fail(DI_ERR_STATE, "di_resume: no DI state (call di_solve or di_set_state first)");
        if (!(tol >= 0.0)) fail(DI_ERR_INVALID, "tol must be >= 0");
        if (H_out && H_mem != DI_MEM_HOST && H_mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "H_mem");
        const di_solve_opts o = resolve(opts);
        use_device(g);
        finish(g, o, tol, H_out, H_mem, res);
    });
}

int di_update_edges(di_graph *g, int64_t n_add, const int32_t *add_src, const int32_t *add_dst, const void *add_w,
                    int32_t w_dtype, int64_t n_rem, const int32_t *rem_src, const int32_t *rem_dst, int32_t mem) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        if (g->g.shard) fail(DI_ERR_INVALID, "di_update_edges is not supported on shards");
        if (n_add < 0 || n_rem < 0) fail(DI_ERR_INVALID, "negative counts");
        if (n_add > 0 && (!add_src || !add_dst)) fail(DI_ERR_INVALID, "add_src / add_dst is NULL");
        if (n_rem > 0 && (!rem_src || !rem_dst)) fail(DI_ERR_INVALID, "rem_src / rem_dst is NULL");
        if (add_w && w_dtype != DI_W_F32 && w_dtype != DI_W_F64) fail(DI_ERR_INVALID, "w_dtype");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        use_device(g);
        update_edges(g, n_add, add_src, add_dst, add_w, w_dtype, n_rem, rem_src, rem_dst, mem);
    });
}

int di_get_state(const di_graph *gc, double *F, double *H, int32_t mem, double *d, double *leak) {
    return guarded([&] {
        if (!gc) fail(DI_ERR_INVALID, "graph is NULL");
        di_graph *g = const_cast<di_graph *>(gc);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_get_state: no DI state");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        use_device(g);
        const int64_t n = g->g.n;
        const cudaMemcpyKind k = mem == DI_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (F && n) DI_CUDA(cudaMemcpyAsync(F, g->s.F, n * sizeof(double), k, g->stream));
        if (H && n) DI_CUDA(cudaMemcpyAsync(H, g->s.H, n * sizeof(double), k, g->stream));
        double lk = 0.0;
        DI_CUDA(cudaMemcpyAsync(&lk, &g->s.ctrl->leak, sizeof(double), cudaMemcpyDeviceToHost, g->stream));
        DI_CUDA(cudaStreamSynchronize(g->stream));
        if (d) *d = g->s.d;
        if (leak) *leak = lk;
    });
}

int di_set_state(di_graph *g, double d, const double *F, const double *H, int32_t mem, double leak) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        if (!(d > 0.0 && d < 1.0)) fail(DI_ERR_INVALID, "d must be in (0, 1)");
        if (g->g.n > 0 && (!F || !H)) fail(DI_ERR_INVALID, "F / H is NULL");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        use_device(g);
        ensure_state(g);
        const int64_t n = g->g.n;
        const cudaMemcpyKind k = mem == DI_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        if (n) {
            DI_CUDA(cudaMemcpyAsync(g->s.F, F, n * sizeof(double), k, g->stream));
            DI_CUDA(cudaMemcpyAsync(g->s.H, H, n * sizeof(double), k, g->stream));
        }
        DI_CUDA(cudaMemsetAsync(g->s.ctrl, 0, sizeof(Ctrl), g->stream));
        DI_CUDA(cudaMemcpyAsync(&g->s.ctrl->leak, &leak, sizeof(double), cudaMemcpyHostToDevice, g->stream));
        DI_CUDA(cudaStreamSynchronize(g->stream));
        g->s.d = d;
        g->s.valid = true;
    });
}

int di_profile_enable(di_graph *g, int32_t on) {
    return guarded([&] {
        if (!g) fail(DI_ERR_INVALID, "graph is NULL");
        g->s.profile = on != 0;
    });
}

int di_profile_get(const di_graph *g, di_profile *out) {
    return guarded([&] {
        if (!g || !out) fail(DI_ERR_INVALID, "NULL argument");
        *out = g->s.last_prof;
    });
}

int di_plan_stats(const di_graph *g, int64_t *stats, int32_t cap) {
    return guarded([&] {
        if (!g || !stats || cap < 0) fail(DI_ERR_INVALID, "bad argument");
        const TilePlan &t = g->g.tl;
        const int64_t v[DI_PLAN_STATS] = {t.ntile, t.mloc, t.mpad, t.mlight, t.mh, t.nh, t.nseg, t.nrun, t.nchunk,
                                          t.built ? (int64_t)t.s_chunk.size() - 1 : 0};
        for (int k = 0; k < cap && k < DI_PLAN_STATS; ++k) stats[k] = t.built ? v[k] : 0;
    });
}

int di_sweep_history(const di_graph *gc, int64_t cap, int64_t *nodes, int64_t *edges, int64_t *entries,
                     int32_t *variant, int64_t *count) {
    return guarded([&] {
        if (!gc || cap < 0) fail(DI_ERR_INVALID, "bad argument");
        di_graph *g = const_cast<di_graph *>(gc);
        if (!g->s.hist) fail(DI_ERR_STATE, "di_sweep_history: no solve yet");
        use_device(g);
        const int64_t S = std::min<int64_t>(std::min<int64_t>(g->s.last_sweeps, kHistCap), cap);
        std::vector<SweepRec> hs(S > 0 ? S : 1);
        if (S > 0) {
            DI_CUDA(cudaMemcpyAsync(hs.data(), g->s.hist, S * sizeof(SweepRec), cudaMemcpyDeviceToHost, g->stream));
            DI_CUDA(cudaStreamSynchronize(g->stream));
        }
        unsigned long long prev = 0;
        for (int64_t k = 0; k < S; ++k) {
            if (nodes) nodes[k] = (int64_t)(hs[k].nodes_cum - prev);
            prev = hs[k].nodes_cum;
            if (edges) edges[k] = (int64_t)hs[k].edges;
            if (entries) entries[k] = (int64_t)hs[k].entries;
            if (variant) variant[k] = hs[k].use_pull;
        }
        if (count) *count = S;
    });
}

// ---------------------------------------------------------------- shards
int di_shard_create(int64_t n_global, int64_t lo, int64_t hi, int64_t m, const int64_t *row_ptr, const int32_t *col,
                    const void *weights, int32_t w_dtype, int32_t mem, int32_t device, void *stream, di_graph **out) {
    return guarded([&] {
        if (!out) fail(DI_ERR_INVALID, "out is NULL");
        if (n_global < 0 || n_global >= (1LL << 31) || lo < 0 || hi < lo || hi > n_global || m < 0)
            fail(DI_ERR_INVALID, "need 0 <= lo <= hi <= n_global < 2^31, m >= 0");
        if (!row_ptr || (m > 0 && !col)) fail(DI_ERR_INVALID, "row_ptr / col is NULL");
        if (w_dtype != DI_W_NONE && w_dtype != DI_W_F32 && w_dtype != DI_W_F64) fail(DI_ERR_INVALID, "w_dtype");
        if (w_dtype != DI_W_NONE && m > 0 && !weights) fail(DI_ERR_INVALID, "weights is NULL");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        if (mem == DI_MEM_HOST && row_ptr[hi - lo] != m) fail(DI_ERR_INVALID, "row_ptr[hi-lo] != m");
        if (m >= (1LL << 40)) fail(DI_ERR_INVALID, "m must be < 2^40");
        DI_CUDA(cudaSetDevice(device));
        keep_pool_memory(device);
        di_graph *g = new di_graph();
        g->device = device;
        try {
            cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);
            g->stream = (cudaStream_t)stream;   // NULL = the CUDA default stream
            reserve_pool(device, hi - lo, m, g->stream);
            create_shard(g, n_global, lo, hi, m, row_ptr, col, weights, w_dtype, mem);
        } catch (...) {
            free_graph(g->g, g->stream);
            cudaStreamSynchronize(g->stream);
            if (g->own_stream) cudaStreamDestroy(g->stream);
            delete g;
            throw;
        }
        *out = g;
    });
}

static void need_shard(const di_graph *g) {
    if (!g) fail(DI_ERR_INVALID, "graph is NULL");
    if (!g->g.shard) fail(DI_ERR_INVALID, "not a shard handle (use di_shard_create)");
}

int di_shard_info(const di_graph *g, int64_t *n_local, int64_t *n_ghost, int64_t *lo) {
    return guarded([&] {
        need_shard(g);
        if (n_local) *n_local = g->g.n;
        if (n_ghost) *n_ghost = g->g.nt - g->g.n;
        if (lo) *lo = g->g.lo;
    });
}

int di_shard_ghost_ids(const di_graph *gc, int32_t *ids, int32_t mem) {
    return guarded([&] {
        need_shard(gc);
        di_graph *g = const_cast<di_graph *>(gc);
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        use_device(g);
        const int64_t ng = g->g.nt - g->g.n;
        if (ng > 0) {
            if (!ids) fail(DI_ERR_INVALID, "ids is NULL");
            DI_CUDA(cudaMemcpyAsync(ids, g->g.ghost_ids, ng * sizeof(int32_t),
                                    mem == DI_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                    g->stream));
        }
        DI_CUDA(cudaStreamSynchronize(g->stream));
    });
}

int di_shard_set_recv(di_graph *g, int64_t total, const int32_t *local_idx, int32_t nseg, const int64_t *seg_counts,
                      int32_t mem) {
    return guarded([&] {
        need_shard(g);
        if (total < 0 || nseg < 0 || (nseg > 0 && !seg_counts) || (total > 0 && !local_idx))
            fail(DI_ERR_INVALID, "bad receive map");
        int64_t sum = 0;
        for (int k = 0; k < nseg; ++k) {
            if (seg_counts[k] < 0) fail(DI_ERR_INVALID, "negative segment");
            sum += seg_counts[k];
        }
        if (sum != total) fail(DI_ERR_INVALID, "segment counts do not add up to total");
        if (mem != DI_MEM_HOST && mem != DI_MEM_DEVICE) fail(DI_ERR_INVALID, "mem");
        use_device(g);
        shard_set_recv(g, total, local_idx, nseg, seg_counts, mem);
    });
}

int di_shard_begin(di_graph *g, double d, const double *Z, int32_t Z_mem, double tol, const di_solve_opts *opts,
                   double *stats) {
    return guarded([&] {
        need_shard(g);
        if (!(d > 0.0 && d < 1.0)) fail(DI_ERR_INVALID, "d must be in (0, 1)");
        if (!(tol >= 0.0)) fail(DI_ERR_INVALID, "tol must be >= 0");
        if (!stats) fail(DI_ERR_INVALID, "stats is NULL");
        const di_solve_opts o = resolve(opts);
        use_device(g);
        double *Zd = nullptr;
        if (Z && g->g.n > 0) {
            if (Z_mem == DI_MEM_HOST) {
                DI_CUDA(cudaMallocAsync(&Zd, g->g.n * sizeof(double), g->stream));
                DI_CUDA(cudaMemcpyAsync(Zd, Z, g->g.n * sizeof(double), cudaMemcpyHostToDevice, g->stream));
            } else {
                Zd = const_cast<double *>(Z);
            }
        }
        init_state(g, d, Zd);
        if (Zd && Z_mem == DI_MEM_HOST) DI_CUDA(cudaFreeAsync(Zd, g->stream));
        prepare_call(g, tol, o, stats);
        launch_reduce(g, 1);
        DI_CUDA(cudaGetLastError());
    });
}

int di_shard_control(di_graph *g, const double *gathered, int32_t nranks) {
    return guarded([&] {
        need_shard(g);
        if (!gathered || nranks < 1) fail(DI_ERR_INVALID, "gathered stats: NULL or nranks < 1");
        use_device(g);
        shard_control(g, gathered, nranks, g->s.flushing ? 1 : 0);
        g->s.flushing = false;
    });
}

int di_shard_sweep(di_graph *g, double *ghost_out) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        if (g->g.nt > g->g.n && !ghost_out) fail(DI_ERR_INVALID, "ghost_out is NULL");
        use_device(g);
        shard_sweep(g, ghost_out);
    });
}

int di_shard_heavy_local(di_graph *g) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        use_device(g);
        shard_heavy_local(g);
    });
}

int di_shard_apply(di_graph *g, const double *recv) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        int64_t tot = 0;
        for (int64_t c : g->g.recv_seg) tot += c;
        if (tot > 0 && !recv) fail(DI_ERR_INVALID, "recv is NULL");
        use_device(g);
        shard_apply(g, recv, 0);
    });
}

int di_shard_flush(di_graph *g, double *ghost_out) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        if (g->g.nt > g->g.n && !ghost_out) fail(DI_ERR_INVALID, "ghost_out is NULL");
        use_device(g);
        shard_flush(g, ghost_out);
        DI_CUDA(cudaGetLastError());
    });
}

int di_shard_flush_apply(di_graph *g, const double *recv) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        int64_t tot = 0;
        for (int64_t c : g->g.recv_seg) tot += c;
        if (tot > 0 && !recv) fail(DI_ERR_INVALID, "recv is NULL");
        use_device(g);
        shard_flush_apply(g, recv);
        DI_CUDA(cudaGetLastError());
    });
}

int di_shard_reduce(di_graph *g) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        use_device(g);
        shard_reduce(g);
        DI_CUDA(cudaGetLastError());
    });
}

int di_shard_poll(di_graph *g, int32_t *done) {
    return guarded([&] {
        need_shard(g);
        use_device(g);
        const bool d = poll_done(g);
        if (done) *done = d ? 1 : 0;
    });
}

int di_shard_finish(di_graph *g, double tol, const di_solve_opts *opts, double *H_out, int32_t H_mem,
                    di_result *res) {
    return guarded([&] {
        need_shard(g);
        if (!g->s.valid) fail(DI_ERR_STATE, "di_shard_begin first");
        const di_solve_opts o = resolve(opts);
        use_device(g);
        poll_done(g);
        di_result r;
        fill_result(g, o, tol, &r);
        write_H(g, r.norm_factor, H_out, H_mem);
        if (res) *res = r;
    });
}

}  // extern "C"
