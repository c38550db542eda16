// dit_graph.cu -- graph builder and dynamic update (B200, sm_100a).
//
// Builder (§2.1, Eq. (1)): the CSR by source IS the column structure
// of P; the only derived per-node array needed by the sweep is
//     inv(j) = 1 / sum_k w_{j,k}   (1/out(j) unweighted, 0 for a dangling j)
// so that P_{i,j} = w_{j,i} inv(j) is formed on the fly from the raw weight.
// Raw float64 weights are stored as float32 when every value converts exactly
// (then the arithmetic is identical and the edge stream is 4 B smaller).
//
// Update (§3.5, Theorem 4): F'_0 = F + d (P' - P) H touches only the changed
// columns: the old column of each changed source j is withdrawn
// (F(t) -= d H(j) P_{t,j}), the CSR is rebuilt with the removals dropped and
// the additions appended, the scales recomputed, and the new column injected
// (F(t) += d H(j) P'_{t,j}).
#include "dit_internal.cuh"

#include <algorithm>
#include <vector>

namespace dit {

// ---------------------------------------------------------------- validation
__global__ void k_check_rows(const int64_t *__restrict__ row_ptr, int64_t n, int64_t m, int *__restrict__ bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = row_ptr[i];
        if ((i == 0 && v != 0) || (i == n && v != m) || (i < n && row_ptr[i + 1] < v)) atomicOr(bad, 1);
    }
}

template <typename Wt>
__global__ void k_check_edges(const int32_t *__restrict__ col, const Wt *__restrict__ w, int64_t m, int64_t n,
                              int *__restrict__ bad, int *__restrict__ not_f32) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = col[e];
        if (c < 0 || (int64_t)c >= n) atomicOr(bad, 2);
        if (w) {
            const double x = (double)w[e];
            if (!(x > 0.0) || !isfinite(x)) atomicOr(bad, 4);
            if ((double)(float)x != x) atomicOr(not_f32, 1);
        }
    }
}

__global__ void k_f64_to_f32(const double *__restrict__ a, float *__restrict__ b, int64_t m) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        b[e] = (float)a[e];
}

// ---------------------------------------------------------------- scales (Eq. (1))
template <typename Wt>
__global__ void k_scales(const int64_t *__restrict__ row_ptr, const Wt *__restrict__ w, int64_t n,
                         double *__restrict__ inv, const unsigned char *__restrict__ only) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        if (only && !only[j]) continue;
        const int64_t b = row_ptr[j], e = row_ptr[j + 1];
        if (b == e) {
            inv[j] = 0.0;                     // dangling: null column of P
            continue;
        }
        if (!w) {
            inv[j] = 1.0 / (double)(e - b);   // P_{i,j} = 1/out(j)
            continue;
        }
        double s = 0.0;                       // sum_k w_{j,k}, in edge order
        for (int64_t k = b; k < e; ++k) s += (double)w[k];
        inv[j] = 1.0 / s;
    }
}

static void launch_scales(di_graph *h, const unsigned char *only) {
    DevGraph &g = h->g;
    if (g.n == 0) return;
    const int grid = (int)std::min<int64_t>((g.n + 255) / 256, (int64_t)h->num_sms * 16);
    if (g.w_kind == DI_W_F32)
        k_scales<float><<<grid, 256, 0, h->stream>>>(g.row_ptr, (const float *)g.w, g.n, g.inv, only);
    else if (g.w_kind == DI_W_F64)
        k_scales<double><<<grid, 256, 0, h->stream>>>(g.row_ptr, (const double *)g.w, g.n, g.inv, only);
    else
        k_scales<float><<<grid, 256, 0, h->stream>>>(g.row_ptr, nullptr, g.n, g.inv, only);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

void build_scales(di_graph *h) {
    DevGraph &g = h->g;
    if (!g.inv) DI_CUDA(cudaMallocAsync(&g.inv, (g.n > 0 ? g.n : 1) * sizeof(double) + 16, h->stream));   // +16: TMA tile rows
    launch_scales(h, nullptr);
}

int grid_for(di_graph *h, int64_t count) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)h->num_sms * 16));
}

static int read_flag(int *dflag, cudaStream_t st) {
    int v = 0;
    DI_CUDA(cudaMemcpyAsync(&v, dflag, sizeof(int), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    return v;
}

// scales of the rows [i0, i1) (pipelined create)
template <typename Wt>
__global__ void k_scales_rows(const int64_t *__restrict__ row_ptr, const Wt *__restrict__ w, int64_t i0, int64_t i1,
                              double *__restrict__ inv) {
    for (int64_t j = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < i1; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = row_ptr[j], e = row_ptr[j + 1];
        if (b == e) {
            inv[j] = 0.0;
            continue;
        }
        if (!w) {
            inv[j] = 1.0 / (double)(e - b);
            continue;
        }
        double s = 0.0;                       // sum_k w_{j,k}, in edge order (as k_scales)
        for (int64_t k = b; k < e; ++k) s += (double)w[k];
        inv[j] = 1.0 / s;
    }
}

static bool pinned_host(const void *p) {
    cudaPointerAttributes a;
    if (!p || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Create from pinned host buffers with the tile plan built while the edges
// upload: row_ptr first, then the targets chunk by chunk (plan
// phase 1 of each chunk as it lands), then the weights chunk by chunk (phase
// 2: validation, scales, ELL); the remote part of the plan after the last chunk.
static void create_graph_pipelined(di_graph *h, int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                                   const void *weights, int w_dtype) {
    DevGraph &g = h->g;
    cudaStream_t st = h->stream;
    g.n = n;
    g.m = m;
    g.nt = n;
    g.n_global = n;
    phase_mark(st, "create: start");
    DI_CUDA(cudaMallocAsync(&g.row_ptr, (n + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&g.col, m * sizeof(int32_t), st));
    if (w_dtype == DI_W_F32) DI_CUDA(cudaMallocAsync(&g.w, m * sizeof(float), st));
    DI_CUDA(cudaMallocAsync(&g.inv, n * sizeof(double) + 16, st));
    g.w_kind = w_dtype == DI_W_F32 ? DI_W_F32 : DI_W_NONE;
    int *flags = nullptr;
    DI_CUDA(cudaMallocAsync(&flags, 2 * sizeof(int), st));
    DI_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
    // chunks of whole tiles, ~kPlanChunkEdges edges each (host row_ptr)
    PlanFeed feed;
    const int64_t ntile = (n + kNodeTile - 1) / kNodeTile;
    feed.tile_lo.push_back(0);
    feed.edge_lo.push_back(0);
    for (int64_t t = 1; t <= ntile; ++t) {
        // (clamped: a malformed row_ptr is rejected below, after the copies are issued)
        const int64_t e = std::min(m, std::max(feed.edge_lo.back(), row_ptr[std::min(n, t * kNodeTile)]));
        if (t == ntile || e - feed.edge_lo.back() >= kPlanChunkEdges) {
            feed.tile_lo.push_back(t);
            feed.edge_lo.push_back(e);
        }
    }
    const int nch = (int)feed.tile_lo.size() - 1;
    cudaStream_t cs = nullptr;
    DI_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaEvent_t go = nullptr;
    std::vector<cudaEvent_t> evs;
    auto cleanup = [&]() {
        if (cs) cudaStreamSynchronize(cs);
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
        if (go) cudaEventDestroy(go);
        if (cs) cudaStreamDestroy(cs);
        cs = nullptr;
        go = nullptr;
        evs.clear();
    };
    try {
        DI_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
        DI_CUDA(cudaEventRecord(go, st));                // the buffers exist before the copies land
        DI_CUDA(cudaStreamWaitEvent(cs, go, 0));
        // row_ptr first on the copy stream (copies on one engine run in issue order)
        DI_CUDA(cudaMemcpyAsync(g.row_ptr, row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, cs));
        cudaEvent_t rows_ready;
        DI_CUDA(cudaEventCreateWithFlags(&rows_ready, cudaEventDisableTiming));
        evs.push_back(rows_ready);
        DI_CUDA(cudaEventRecord(rows_ready, cs));
        for (int pass = 0; pass < (w_dtype == DI_W_F32 ? 2 : 1); ++pass)
            for (int c = 0; c < nch; ++c) {
                const int64_t e0 = feed.edge_lo[c], e1 = feed.edge_lo[c + 1];
                if (e1 > e0) {
                    if (pass == 0)
                        DI_CUDA(cudaMemcpyAsync(g.col + e0, col + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, cs));
                    else
                        DI_CUDA(cudaMemcpyAsync((float *)g.w + e0, (const float *)weights + e0, (e1 - e0) * 4,
                                                cudaMemcpyHostToDevice, cs));
                }
                cudaEvent_t ev;
                DI_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                evs.push_back(ev);
                DI_CUDA(cudaEventRecord(ev, cs));
                (pass == 0 ? feed.col_ready : feed.w_ready).push_back(ev);
            }
        if (w_dtype != DI_W_F32) feed.w_ready = feed.col_ready;   // unweighted: phase 2 needs the targets only
        // row_ptr validated before the plan uses it
        DI_CUDA(cudaStreamWaitEvent(st, rows_ready, 0));
        k_check_rows<<<grid_for(h, n + 1), 256, 0, st>>>(g.row_ptr, n, m, flags);
        count_launch();
        if (read_flag(flags, st)) {
            set_error("row_ptr must be non-decreasing with row_ptr[0]=0 and row_ptr[n]=m");
            throw Fail{DI_ERR_INVALID};
        }
        feed.on_col = [&](int c) {                       // target ids of the chunk in [0, n)
            const int64_t e0 = feed.edge_lo[c], e1 = feed.edge_lo[c + 1];
            if (e1 > e0) {
                k_check_edges<float><<<grid_for(h, e1 - e0), 256, 0, st>>>(g.col + e0, nullptr, e1 - e0, n, flags,
                                                                          flags + 1);
                count_launch();
            }
        };
        feed.on_w = [&](int c) {                         // weights of the chunk, then the scales of its rows
            const int64_t e0 = feed.edge_lo[c], e1 = feed.edge_lo[c + 1];
            const int64_t i0 = std::min(n, feed.tile_lo[c] * kNodeTile), i1 = std::min(n, feed.tile_lo[c + 1] * kNodeTile);
            if (w_dtype == DI_W_F32 && e1 > e0) {
                k_check_edges<float><<<grid_for(h, e1 - e0), 256, 0, st>>>(g.col + e0, (const float *)g.w + e0, e1 - e0,
                                                                          n, flags, flags + 1);
                count_launch();
            }
            if (i1 > i0) {
                k_scales_rows<float><<<grid_for(h, i1 - i0), 256, 0, st>>>(
                    g.row_ptr, w_dtype == DI_W_F32 ? (const float *)g.w : nullptr, i0, i1, g.inv);
                count_launch();
            }
        };
        phase_mark(st, "create: row_ptr + launch the upload");
        build_tiles(h, &feed, flags);
        cleanup();
    } catch (...) {
        cleanup();
        cudaFreeAsync(flags, st);
        throw;
    }
    int fl[2] = {0, 0};
    DI_CUDA(cudaMemcpyAsync(fl, flags, sizeof(fl), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaFreeAsync(flags, st));
    DI_CUDA(cudaStreamSynchronize(st));
    if (fl[0]) {
        set_error(fl[0] & 1 ? "row_ptr must be non-decreasing with row_ptr[0]=0 and row_ptr[n]=m"
                            : (fl[0] & 2 ? "col ids must be in [0, n) (n_global for a shard)" : "weights must be finite and > 0"));
        throw Fail{DI_ERR_INVALID};
    }
}

// Copy + validate the caller's CSR into the handle.
void create_graph(di_graph *h, int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                  const void *weights, int w_dtype, int mem, int64_t col_bound) {
    DevGraph &g = h->g;
    cudaStream_t st = h->stream;
    // host graphs of 16M+ edges from pinned memory: the tile plan is built during the upload
    if (mem == DI_MEM_HOST && col_bound == n && m >= ((int64_t)1 << 24) && w_dtype != DI_W_F64 && n > 0 &&
        !getenv("DIT_NO_EAGER_PLAN") && pinned_host(col) && pinned_host(row_ptr) &&
        (w_dtype == DI_W_NONE || pinned_host(weights))) {
        create_graph_pipelined(h, n, m, row_ptr, col, weights, w_dtype);
        return;
    }
    g.n = n;
    phase_mark(st, "create: start");
    g.m = m;
    g.nt = n;
    g.n_global = n;
    const cudaMemcpyKind kind = mem == DI_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    DI_CUDA(cudaMallocAsync(&g.row_ptr, (n + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&g.col, (m > 0 ? m : 1) * sizeof(int32_t), st));
    DI_CUDA(cudaMemcpyAsync(g.row_ptr, row_ptr, (n + 1) * sizeof(int64_t), kind, st));
    if (m > 0) DI_CUDA(cudaMemcpyAsync(g.col, col, m * sizeof(int32_t), kind, st));
    void *wtmp = nullptr;
    if (w_dtype != DI_W_NONE && m > 0) {
        const size_t es = w_dtype == DI_W_F32 ? 4 : 8;
        DI_CUDA(cudaMallocAsync(&wtmp, m * es, st));
        DI_CUDA(cudaMemcpyAsync(wtmp, weights, m * es, kind, st));
    }
    int *flags = nullptr;
    DI_CUDA(cudaMallocAsync(&flags, 2 * sizeof(int), st));
    DI_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
    phase_mark(st, "create: upload");
    k_check_rows<<<grid_for(h, n + 1), 256, 0, st>>>(g.row_ptr, n, m, flags);
    count_launch();
    if (m > 0) {
        if (w_dtype == DI_W_F32)
            k_check_edges<float><<<grid_for(h, m), 256, 0, st>>>(g.col, (const float *)wtmp, m, col_bound, flags, flags + 1);
        else if (w_dtype == DI_W_F64)
            k_check_edges<double><<<grid_for(h, m), 256, 0, st>>>(g.col, (const double *)wtmp, m, col_bound, flags, flags + 1);
        else
            k_check_edges<float><<<grid_for(h, m), 256, 0, st>>>(g.col, nullptr, m, col_bound, flags, flags + 1);
        count_launch();
    }
    DI_CUDA(cudaGetLastError());
    int fl[2] = {0, 0};
    DI_CUDA(cudaMemcpyAsync(fl, flags, sizeof(fl), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaFreeAsync(flags, st));
    DI_CUDA(cudaStreamSynchronize(st));
    if (fl[0]) {
        cudaFreeAsync(wtmp, st);
        set_error(fl[0] & 1 ? "row_ptr must be non-decreasing with row_ptr[0]=0 and row_ptr[n]=m"
                            : (fl[0] & 2 ? "col ids must be in [0, n) (n_global for a shard)" : "weights must be finite and > 0"));
        throw Fail{DI_ERR_INVALID};
    }
    if (w_dtype == DI_W_F32 && m > 0) {
        g.w = wtmp;
        g.w_kind = DI_W_F32;
    } else if (w_dtype == DI_W_F64 && m > 0) {
        if (fl[1]) {
            g.w = wtmp;
            g.w_kind = DI_W_F64;
        } else {   // every weight is exactly a float: store 4 bytes per edge
            DI_CUDA(cudaMallocAsync(&g.w, m * sizeof(float), st));
            k_f64_to_f32<<<grid_for(h, m), 256, 0, st>>>((const double *)wtmp, (float *)g.w, m);
            count_launch();
            DI_CUDA(cudaFreeAsync(wtmp, st));
            g.w_kind = DI_W_F32;
        }
    }

    phase_mark(st, "create: check + scales");    build_scales(h);
}

static void free_transpose(DevGraph &g, cudaStream_t st) {
    free_plan(g.t, st);
    free_tiles(g.tl, st);
}

void free_graph(DevGraph &g, cudaStream_t st) {
    free_transpose(g, st);
    for (void *p : {(void *)g.ghost_ids, (void *)g.recv_idx, (void *)g.row_ptr, (void *)g.col, g.w, (void *)g.inv})
        if (p) cudaFreeAsync(p, st);
    g = DevGraph();
}

// ---------------------------------------------------------------- update (Theorem 4)
__global__ void k_check_ids(const int32_t *__restrict__ a, const int32_t *__restrict__ b, int64_t cnt, int64_t n,
                            int *__restrict__ bad) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        if (a[q] < 0 || a[q] >= n || b[q] < 0 || b[q] >= n) atomicOr(bad, 1);
}

// flags[0] |= invalid weight, flags[1] |= not exactly a float, flags[2] |= not 1
__global__ void k_check_w(const double *__restrict__ w, int64_t cnt, int *__restrict__ fl) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        const double x = w[q];
        if (!(x > 0.0) || !isfinite(x)) atomicOr(fl, 1);
        if ((double)(float)x != x) atomicOr(fl + 1, 1);
        if (x != 1.0) atomicOr(fl + 2, 1);
    }
}

// mark every CSR entry matched by a removal; count matches per removal / row
__global__ void k_mark_removals(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                const int32_t *__restrict__ rs, const int32_t *__restrict__ rd, int64_t nrem,
                                unsigned char *__restrict__ del, unsigned char *__restrict__ chg,
                                int *__restrict__ notfound) {
    // a thread per removal in a row of <= 32 entries, the warp for a longer row
    const unsigned lane = lane_id();
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nrem; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = base + threadIdx.x;
        int32_t s = 0, t = 0;
        int64_t b = 0, e = 0;
        if (q < nrem) {
            s = rs[q];
            t = rd[q];
            b = row_ptr[s];
            e = row_ptr[s + 1];
            chg[s] = 1;
        }
        if (q < nrem && e - b <= 32) {
            int found = 0;
            for (int64_t k = b; k < e; ++k)
                if (col[k] == t) {
                    del[k] = 1;
                    found = 1;
                }
            if (!found) atomicOr(notfound, 1);
        }
        for (unsigned big = __ballot_sync(0xffffffffu, q < nrem && e - b > 32); big; big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int32_t tl = __shfl_sync(0xffffffffu, t, l);
            const int64_t bl = __shfl_sync(0xffffffffu, b, l), el = __shfl_sync(0xffffffffu, e, l);
            int found = 0;
            for (int64_t k = bl + lane; k < el; k += 32)
                if (col[k] == tl) {
                    del[k] = 1;
                    found = 1;
                }
            if (!__any_sync(0xffffffffu, found) && lane == 0) atomicOr(notfound, 1);
        }
    }
}

__global__ void k_mark_adds(const int32_t *__restrict__ as, int64_t nadd, unsigned char *__restrict__ chg,
                            int64_t *__restrict__ addcnt) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nadd; q += (int64_t)gridDim.x * blockDim.x) {
        chg[as[q]] = 1;
        atomicAdd((unsigned long long *)&addcnt[as[q]], 1ull);
    }
}

// F(t) += sign * d * H(j) * w_{j,t} * inv(j) over the out-edges of changed sources j
// Theorem 4 in one pass over the NEW changed rows (after the CSR swap):
// F += d H(j) (P' - P) e_j.  Kept entries (the row's prefix) move by
// d H(j) w (inv'(j) - inv(j)), added ones (the suffix) by d H(j) w inv'(j); the
// removed entries (k_removed_fluid) by -d H(j) w inv(j).  (float64 atomics: the
// summation order into F varies run to run, R14.)
template <typename Wt>
__global__ void k_column_fluid_new(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                   const Wt *__restrict__ w, const double *__restrict__ inv_old,
                                   const double *__restrict__ inv_new, const unsigned char *__restrict__ chg,
                                   const int64_t *__restrict__ addcnt, const double *__restrict__ H,
                                   double *__restrict__ F, int64_t n, double d) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = warp; j < n; j += nw) {
        if (!chg[j] || H[j] == 0.0) continue;
        const double an = d * H[j] * inv_new[j], ak = an - d * H[j] * inv_old[j];
        const int64_t b = row_ptr[j], e = row_ptr[j + 1], ke = e - addcnt[j];
        for (int64_t q = b + lane_id(); q < e; q += 32) {
            const double a = q < ke ? ak : an;
            red_add(F + col[q], w ? a * (double)w[q] : a);
        }
    }
}

__global__ void k_removed_fluid(const int32_t *__restrict__ rs, const int32_t *__restrict__ rt,
                                const double *__restrict__ rw, int64_t cnt, const double *__restrict__ inv_old,
                                const double *__restrict__ H, double *__restrict__ F, double d) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = rs[q];
        const double h = H[j];
        if (h != 0.0) red_add(F + rt[q], d * h * inv_old[j] * rw[q]);   // rw = -w
    }
}

// new out-degree = old - removed + added
__global__ void k_new_deg(const int64_t *__restrict__ row_ptr, const unsigned char *__restrict__ del,
                          const unsigned char *__restrict__ chg, const int64_t *__restrict__ addcnt, int64_t n,
                          int64_t *__restrict__ deg) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = warp; j < n; j += nw) {
        const int64_t b = row_ptr[j], e = row_ptr[j + 1];
        int64_t kept = e - b;
        if (chg[j]) {
            int64_t r = 0;
            for (int64_t k = b + lane_id(); k < e; k += 32) r += del[k];
            kept -= warp_sum(r);
            kept += addcnt[j];
        }
        if (lane_id() == 0) deg[j] = kept;
    }
}

// copy kept entries of every row in order: a thread per row of <= 32 entries
// (32 rows per warp step), a warp per longer one (ballot compaction)
template <typename Wt>
__global__ void k_copy_kept(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const Wt *__restrict__ w, const unsigned char *__restrict__ del,
                            const unsigned char *__restrict__ chg, const int64_t *__restrict__ nrp, int64_t n,
                            int32_t *__restrict__ ncol, Wt *__restrict__ nw_, int64_t *__restrict__ cursor) {
    const unsigned lane = lane_id();
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = base + threadIdx.x;
        int64_t b = 0, e = 0, out = 0;
        bool c = false;
        if (j < n) {
            b = row_ptr[j];
            e = row_ptr[j + 1];
            out = nrp[j];
            c = chg[j] != 0;
        }
        if (j < n && e - b <= 32) {
            for (int64_t k = b; k < e; ++k)
                if (!(c && del[k])) {
                    ncol[out] = col[k];
                    if (w) nw_[out] = w[k];
                    ++out;
                }
            cursor[j] = out;                          // additions of row j go from here
        }
        for (unsigned big = __ballot_sync(0xffffffffu, j < n && e - b > 32); big; big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int64_t jl = __shfl_sync(0xffffffffu, j, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            int64_t o = __shfl_sync(0xffffffffu, out, l);
            const bool cl = __shfl_sync(0xffffffffu, c, l);
            for (int64_t k0 = bl; k0 < el; k0 += 32) {
                const int64_t k = k0 + lane;
                const bool keep = k < el && !(cl && del[k]);
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep) {
                    const int64_t at = o + __popc(bal & ((1u << lane) - 1u));
                    ncol[at] = col[k];
                    if (w) nw_[at] = w[k];
                }
                o += __popc(bal);
            }
            if (lane == 0) cursor[jl] = o;
        }
    }
}

template <typename Wt>
__global__ void k_place_adds(const int32_t *__restrict__ as, const int32_t *__restrict__ ad,
                             const double *__restrict__ aw, int64_t nadd, int64_t *__restrict__ cursor,
                             int32_t *__restrict__ ncol, Wt *__restrict__ nw_) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nadd; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = (int64_t)atomicAdd((unsigned long long *)&cursor[as[q]], 1ull);
        ncol[o] = ad[q];
        if (nw_) nw_[o] = (Wt)(aw ? aw[q] : 1.0);
    }
}

template <typename T>
static T *to_device(const T *p, int64_t cnt, int mem, cudaStream_t st) {
    if (cnt == 0 || !p) return nullptr;
    T *d = nullptr;
    DI_CUDA(cudaMallocAsync(&d, cnt * sizeof(T), st));
    DI_CUDA(cudaMemcpyAsync(d, p, cnt * sizeof(T), mem == DI_MEM_HOST ? cudaMemcpyHostToDevice
                                                                      : cudaMemcpyDeviceToDevice, st));
    return d;
}

__global__ void k_f32_to_f64(const float *__restrict__ a, double *__restrict__ b, int64_t m) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        b[e] = (double)a[e];
}


void update_edges(di_graph *h, int64_t n_add, const int32_t *add_src, const int32_t *add_dst, const void *add_w,
                  int w_dtype, int64_t n_rem, const int32_t *rem_src, const int32_t *rem_dst, int mem) {
    DevGraph &g = h->g;
    cudaStream_t st = h->stream;
    const int64_t n = g.n;
    std::vector<void *> tmp;
    auto track = [&](void *p) { tmp.push_back(p); return p; };
    DeltaBatch rem;                                  // removed entries (-w), Theorem 4 and the kept plan
    auto release = [&]() {
        for (void *p : tmp) cudaFreeAsync(p, st);
        tmp.clear();
        delta_batch_free(rem, st);
    };
    try {
        int32_t *as = (int32_t *)track(to_device(add_src, n_add, mem, st));
        int32_t *ad = (int32_t *)track(to_device(add_dst, n_add, mem, st));
        int32_t *rs = (int32_t *)track(to_device(rem_src, n_rem, mem, st));
        int32_t *rd = (int32_t *)track(to_device(rem_dst, n_rem, mem, st));
        double *aw = nullptr;
        if (add_w && n_add > 0) {
            if (w_dtype == DI_W_F64) {
                aw = (double *)track(to_device((const double *)add_w, n_add, mem, st));
            } else {
                float *f = (float *)track(to_device((const float *)add_w, n_add, mem, st));
                DI_CUDA(cudaMallocAsync(&aw, n_add * sizeof(double), st));
                track(aw);
                k_f32_to_f64<<<grid_for(h, n_add), 256, 0, st>>>(f, aw, n_add);
                count_launch();
            }
        }
        int *flags = nullptr;   // [0] bad id, [1..3] weight checks, [4] removal not found
        DI_CUDA(cudaMallocAsync(&flags, 5 * sizeof(int), st));
        track(flags);
        DI_CUDA(cudaMemsetAsync(flags, 0, 5 * sizeof(int), st));
        if (n_add) {
            k_check_ids<<<grid_for(h, n_add), 256, 0, st>>>(as, ad, n_add, n, flags);
            count_launch();
        }
        if (n_rem) {
            k_check_ids<<<grid_for(h, n_rem), 256, 0, st>>>(rs, rd, n_rem, n, flags);
            count_launch();
        }
        if (aw) {
            k_check_w<<<grid_for(h, n_add), 256, 0, st>>>(aw, n_add, flags + 1);
            count_launch();
        }
        phase_mark(st, "update: upload + checks");
        int fl[5];
        DI_CUDA(cudaMemcpyAsync(fl, flags, sizeof(fl), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        if (fl[0] || fl[1]) {
            set_error("di_update_edges: node id out of range or weight not finite and > 0");
            throw Fail{DI_ERR_INVALID};
        }
        if (aw && g.w_kind == DI_W_NONE && fl[3]) {   // the graph stays unweighted only for unit weights
            set_error("di_update_edges: weighted additions on an unweighted graph");
            throw Fail{DI_ERR_INVALID};
        }
        unsigned char *del = nullptr, *chg = nullptr;
        int64_t *addcnt = nullptr;
        DI_CUDA(cudaMallocAsync(&del, (g.m > 0 ? g.m : 1), st));
        track(del);
        DI_CUDA(cudaMallocAsync(&chg, (n > 0 ? n : 1), st));
        track(chg);
        DI_CUDA(cudaMallocAsync(&addcnt, (n > 0 ? n : 1) * sizeof(int64_t), st));
        track(addcnt);
        DI_CUDA(cudaMemsetAsync(del, 0, (g.m > 0 ? g.m : 1), st));
        DI_CUDA(cudaMemsetAsync(chg, 0, (n > 0 ? n : 1), st));
        DI_CUDA(cudaMemsetAsync(addcnt, 0, (n > 0 ? n : 1) * sizeof(int64_t), st));
        if (n_rem) {
            k_mark_removals<<<grid_for(h, n_rem), 256, 0, st>>>(g.row_ptr, g.col, rs, rd, n_rem, del, chg, flags + 4);
            count_launch();
        }
        if (read_flag(flags + 4, st)) {
            set_error("di_update_edges: a removal names an edge absent from the graph");
            throw Fail{DI_ERR_EDGE_NOT_FOUND};
        }
        if (n_add) {
            k_mark_adds<<<grid_for(h, n_add), 256, 0, st>>>(as, n_add, chg, addcnt);
            count_launch();
        }
        phase_mark(st, "update: marks");
        const bool state = h->s.valid;
        const double d = h->s.d;
        // the tile plan stays, corrected by delta in-edges (dit_delta.cu, DESIGN.md
        // R18), unless the weight storage changes under it
        bool keep_plan = delta_enabled(h) && !(g.w_kind == DI_W_F32 && aw && fl[2]);
        // f32 weight storage must stay exact: promote to f64 if an added weight is not a float
        if (g.w_kind == DI_W_F32 && aw && fl[2]) {
            double *w64 = nullptr;
            DI_CUDA(cudaMallocAsync(&w64, (g.m > 0 ? g.m : 1) * sizeof(double), st));
            if (g.m > 0) {
                k_f32_to_f64<<<grid_for(h, g.m), 256, 0, st>>>((const float *)g.w, w64, g.m);
                count_launch();
            }
            DI_CUDA(cudaFreeAsync(g.w, st));
            g.w = w64;
            g.w_kind = DI_W_F64;
        }
        // the transpose and tile plan are derived from the old CSR: free them first
        // (rebuilt by the next call that needs them), then allocate every buffer of
        // the new CSR before the state is touched, so that a failure (OOM) leaves
        // graph and fluid as they were
        if (keep_plan) free_plan(g.t, st);
        else free_transpose(g, st);
        int64_t *deg = nullptr, *nrp = nullptr, *cursor = nullptr;
        DI_CUDA(cudaMallocAsync(&deg, (n > 0 ? n : 1) * sizeof(int64_t), st));
        track(deg);
        DI_CUDA(cudaMallocAsync(&cursor, (n > 0 ? n : 1) * sizeof(int64_t), st));
        track(cursor);
        DI_CUDA(cudaMallocAsync(&nrp, (n + 1) * sizeof(int64_t), st));
        track(nrp);
        if (n > 0) {
            k_new_deg<<<h->num_sms * 8, 256, 0, st>>>(g.row_ptr, del, chg, addcnt, n, deg);
            count_launch();
        }
        exclusive_scan_i64(deg, nrp, n, st);
        int64_t m2 = 0;
        DI_CUDA(cudaMemcpyAsync(&m2, nrp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        phase_mark(st, "update: new degrees");
        int32_t *ncol = nullptr;
        void *nwt = nullptr;
        DI_CUDA(cudaMallocAsync(&ncol, (m2 > 0 ? m2 : 1) * sizeof(int32_t), st));
        track(ncol);
        const size_t es = g.w_kind == DI_W_F64 ? 8 : (g.w_kind == DI_W_F32 ? 4 : 0);
        if (es) {
            DI_CUDA(cudaMallocAsync(&nwt, (m2 > 0 ? m2 : 1) * es, st));
            track(nwt);
        }
        // the scales of the old graph (Theorem 4 needs P and P')
        double *inv_old = nullptr;
        if (state && n > 0) {
            DI_CUDA(cudaMallocAsync(&inv_old, n * sizeof(double), st));
            track(inv_old);
        }
        // every allocation done: nothing of graph or state has changed yet
        phase_mark(st, "update: CSR alloc");
        if (n > 0) {
            if (g.w_kind == DI_W_F64)
                k_copy_kept<double><<<h->num_sms * 8, 256, 0, st>>>(g.row_ptr, g.col, (const double *)g.w, del, chg,
                                                                     nrp, n, ncol, (double *)nwt, cursor);
            else
                k_copy_kept<float><<<h->num_sms * 8, 256, 0, st>>>(g.row_ptr, g.col, (const float *)g.w, del, chg, nrp,
                                                                    n, ncol, (float *)nwt, cursor);
            count_launch();
        }
        if (n_add) {
            if (g.w_kind == DI_W_F64)
                k_place_adds<double><<<grid_for(h, n_add), 256, 0, st>>>(as, ad, aw, n_add, cursor, ncol, (double *)nwt);
            else
                k_place_adds<float><<<grid_for(h, n_add), 256, 0, st>>>(as, ad, aw, n_add, cursor, ncol, (float *)nwt);
            count_launch();
        }
        DI_CUDA(cudaGetLastError());
        DI_CUDA(cudaStreamSynchronize(st));
        phase_mark(st, "update: new CSR");
        // the removed entries (-w) from the old CSR; any failure of the delta path
        // drops the plan instead (rebuilt from the new CSR on the next tiled call)
        auto drop_plan = [&]() {
            free_tiles(g.tl, st);
            keep_plan = false;
        };
        // (a failure here leaves graph and fluid as they were)
        if (keep_plan || state) delta_collect_removed(h, del, chg, rem, keep_plan);
        phase_mark(st, "update: collect removed");
        // swap in the new CSR (no longer temporaries), recompute the scales of changed rows
        tmp.erase(std::remove_if(tmp.begin(), tmp.end(), [&](void *p) { return p == nrp || p == ncol || p == nwt; }),
                  tmp.end());
        cudaFreeAsync(g.row_ptr, st);
        cudaFreeAsync(g.col, st);
        if (g.w) cudaFreeAsync(g.w, st);
        g.row_ptr = nrp;
        g.col = ncol;
        g.w = nwt;
        g.m = m2;
        if (inv_old) DI_CUDA(cudaMemcpyAsync(inv_old, g.inv, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (n > 0) launch_scales(h, chg);
        if (keep_plan) {
            try {
                delta_commit(h, rem, as, ad, aw, n_add, chg);
            } catch (const Fail &) {
                drop_plan();
            }
        }
        phase_mark(st, "update: scales + delta commit");
        // Theorem 4: the corrective fluid d (P' - P) H over the changed columns
        if (state && n > 0) {
            if (g.w_kind == DI_W_F64)
                k_column_fluid_new<double><<<h->num_sms * 8, 256, 0, st>>>(
                    g.row_ptr, g.col, (const double *)g.w, inv_old, g.inv, chg, addcnt, h->s.H, h->s.F, n, d);
            else
                k_column_fluid_new<float><<<h->num_sms * 8, 256, 0, st>>>(
                    g.row_ptr, g.col, (const float *)g.w, inv_old, g.inv, chg, addcnt, h->s.H, h->s.F, n, d);
            count_launch();
            if (rem.nrem > 0) {
                k_removed_fluid<<<grid_for(h, rem.nrem), 256, 0, st>>>(rem.s, rem.t, rem.w, rem.nrem, inv_old, h->s.H,
                                                                      h->s.F, d);
                count_launch();
            }
        }
        delta_batch_free(rem, st);
        DI_CUDA(cudaGetLastError());
        DI_CUDA(cudaStreamSynchronize(st));
        phase_mark(st, "update: inject");
        // the entry buffer is sized by m
        if (state) {
            State &s = h->s;
            const int64_t need = n + g.m / kSplit + 1;
            if (need > s.ent_cap) {
                cudaFreeAsync(s.ent, st);
                s.ent = nullptr;
                DI_CUDA(cudaMallocAsync(&s.ent, need * sizeof(uint4), st));
                s.ent_cap = need;
            }
            // l as a function of the state (R5): sum of H over the
            // dangling nodes of the new graph
            set_leak_from_history(h);
        }
        phase_mark(st, "update: leak done");
        release();
    } catch (...) {
        release();
        throw;
    }
}

}  // namespace dit
