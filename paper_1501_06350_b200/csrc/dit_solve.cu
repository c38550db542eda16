// dit_solve.cu -- the D-Iteration sweep on B200 (sm_100a).
//
// One sweep (reading R1; §3.1 Eqs. (8), (10)) =
//   k_select  frontier S = { i : F(i) != 0, |F(i)| >= T }: H(i) += F(i), F(i) = 0,
//             emit (edge range, amount d F(i) / sum_k w_{i,k}) entries (push) or
//             the dense outflow A(i) (pull); warp-ballot/scan compaction with one
//             atomic per warp; dangling nodes add their fluid to the leak l (§3.3)
//   k_push    edge-balanced scatter: a warp takes 32 entries, scans their lengths
//             and walks the union of their edges 32 at a time, RED.ADD.F64 into F
//   k_pull    (dit_pull.cu) deterministic gather over the transpose
//   k_reduce  |F|_1 and max|F| (Theorem 1's remaining fluid), deterministic
//             block partials; the last block sets the next threshold
//             T = min(theta |F|_1 / n, max|F|) and the `done` flag.
// Every kernel has a fixed grid and returns at once when ctrl->done is set, so
// a chunk of sweeps can be enqueued (or graph-launched) without host syncs.
#include "dit_internal.cuh"

#include <chrono>
#include <cmath>
#include <cstdio>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace dit {

// ---------------------------------------------------------------- init
__global__ void __launch_bounds__(kThreads) k_init(double *__restrict__ F, double *__restrict__ H,
                                                   const double *__restrict__ Z, int64_t n, int64_t nt,
                                                   double n_global, double d) {
    const double u = (1.0 - d) / n_global;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nt; i += (int64_t)gridDim.x * kThreads) {
        if (i < n) {
            F[i] = Z ? (1.0 - d) * Z[i] : u;     // Eq. (7): F_0 = (1-d) Z
            H[i] = 0.0;                          //          H_0 = 0
        } else {
            F[i] = 0.0;                          // shard: ghost fluid slots
        }
    }
}

// ---------------------------------------------------------------- select
// Entry = { (begin << 24) | len , amount } in 16 bytes.
__device__ __forceinline__ void store_entry(uint4 *p, int64_t begin, int64_t len, double a) {
    unsigned long long packed = ((unsigned long long)begin << kLenBits) | (unsigned long long)len;
    unsigned long long ab = (unsigned long long)__double_as_longlong(a);
    *p = make_uint4((unsigned)packed, (unsigned)(packed >> 32), (unsigned)ab, (unsigned)(ab >> 32));
}

template <bool kPull>
__global__ void __launch_bounds__(kThreads) k_select(const int64_t *__restrict__ row_ptr,
                                                     const double *__restrict__ inv, double *__restrict__ F,
                                                     double *__restrict__ H, double *__restrict__ A,
                                                     uint4 *__restrict__ ent, int64_t n, Ctrl *__restrict__ ctrl,
                                                     double *__restrict__ part_sel) {
    __shared__ double s_leak[kWarps];
    __shared__ unsigned long long s_cnt[kWarps][2];
    if (ctrl->done) return;
    if (ctrl->use_pull != (kPull ? kUsePull : kUsePush)) return;
    const double T = ctrl->T, d = ctrl->d;
    const unsigned lane = lane_id();
    double leak = 0.0;
    unsigned long long nodes = 0, edges = 0;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t base = (int64_t)blockIdx.x * kThreads + (threadIdx.x & ~31u); base < n; base += stride) {
        const int64_t i = base + lane;
        const bool valid = i < n;
        const double f = valid ? F[i] : 0.0;
        const bool sel = valid && f != 0.0 && fabs(f) >= T;
        int64_t b = 0, deg = 0;
        double a = 0.0;
        if (sel) {
            H[i] += f;                       // Eq. (10)
            F[i] = 0.0;                      // third term of Eq. (8)
            b = row_ptr[i];
            deg = row_ptr[i + 1] - b;
            nodes += 1;
            edges += (unsigned long long)deg;
            if (deg == 0) leak += f;         // dangling: fluid leaves (§3.3 l_k)
            else a = d * f * inv[i];         // d F(i) / sum_k w_{i,k}
        }
        if (kPull) {
            if (valid) A[i] = a;
        } else {
            const unsigned nch = (unsigned)((deg + kSplit - 1) >> kSplitShift);
            const unsigned incl = warp_incl_scan(nch);
            const unsigned tot = __shfl_sync(0xffffffffu, incl, 31);
            if (tot) {
                unsigned long long pos = 0;
                if (lane == 31) pos = atomicAdd(&ctrl->n_entries, (unsigned long long)tot);
                pos = __shfl_sync(0xffffffffu, pos, 31) + (incl - nch);
                for (unsigned c = 0; c < nch; ++c) {
                    const int64_t cb = b + ((int64_t)c << kSplitShift);
                    const int64_t len = min((int64_t)kSplit, deg - ((int64_t)c << kSplitShift));
                    store_entry(ent + pos + c, cb, len, a);
                }
            }
        }
    }
    // deterministic block reduction of the leak; integer counters by atomics
    leak = warp_sum(leak);
    nodes = warp_sum(nodes);
    edges = warp_sum(edges);
    const unsigned w = threadIdx.x >> 5;
    if (lane == 0) {
        s_leak[w] = leak;
        s_cnt[w][0] = nodes;
        s_cnt[w][1] = edges;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        unsigned long long nn = 0, ee = 0;
        for (int k = 0; k < kWarps; ++k) {
            l += s_leak[k];
            nn += s_cnt[k][0];
            ee += s_cnt[k][1];
        }
        part_sel[blockIdx.x] = l;
        if (nn) {
            atomicAdd(&ctrl->diffused_nodes, nn);
            atomicAdd(&ctrl->sel_edges, ee);
        }
    }
}

// ---------------------------------------------------------------- push
template <typename W>
__global__ void __launch_bounds__(kThreads) k_push(const int32_t *__restrict__ col, const W *__restrict__ w,
                                                   double *__restrict__ F, const uint4 *__restrict__ ent,
                                                   const Ctrl *__restrict__ ctrl) {
    if (ctrl->done || ctrl->use_pull != kUsePush) return;
    const unsigned long long N = ctrl->n_entries;
    const unsigned lane = lane_id();
    const unsigned long long warp = ((unsigned long long)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const unsigned long long nwarps = ((unsigned long long)gridDim.x * kThreads) >> 5;
    for (unsigned long long cbase = warp * 32; cbase < N; cbase += nwarps * 32) {
        const unsigned long long j = cbase + lane;
        int len = 0;
        long long beg = 0;
        double a = 0.0;
        if (j < N) {
            const uint4 e = ent[j];
            const unsigned long long packed = ((unsigned long long)e.y << 32) | e.x;
            len = (int)(packed & ((1ull << kLenBits) - 1));
            beg = (long long)(packed >> kLenBits);
            a = __longlong_as_double((long long)(((unsigned long long)e.w << 32) | e.z));
        }
        const int incl = warp_incl_scan(len);
        const int E = __shfl_sync(0xffffffffu, incl, 31);
        for (int k0 = 0; k0 < E; k0 += 32) {
            const int k = k0 + (int)lane;
            // entry of edge k: number of lanes whose inclusive end is <= k
            int pos = 0;
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, pos + s - 1);
                if (v <= k) pos += s;
            }
            const int src = min(pos, 31);
            const int excl = __shfl_sync(0xffffffffu, incl, src) - __shfl_sync(0xffffffffu, len, src);
            const long long bL = __shfl_sync(0xffffffffu, beg, src);
            const double aL = __shfl_sync(0xffffffffu, a, src);
            if (k < E) {
                const int64_t e = bL + (k - excl);
                const int32_t t = ld_stream_i32(col + e);
                double v = aL;
                if constexpr (!std::is_same<W, NoW>::value) v *= load_w(w, e);   // P_{t,i} = w_{i,t} inv_i
                red_add(F + t, v);                                                // Eq. (8) push
            }
        }
    }
}

// ---------------------------------------------------------------- reduce
__global__ void __launch_bounds__(kThreads) k_reduce(const double *__restrict__ F, int64_t n, int64_t m,
                                                     Ctrl *__restrict__ ctrl, double *__restrict__ part,
                                                     const double *__restrict__ part_sel, int is_init,
                                                     int force) {
    __shared__ double s_sum[kWarps], s_max[kWarps];
    __shared__ bool s_last;
    if (ctrl->done && !force) return;
    // two independent 16-byte streams per thread (F is 256-byte aligned)
    double s0 = 0.0, s1 = 0.0, mx = 0.0;
    const int64_t n2 = n >> 1;
    const double2 *F2 = reinterpret_cast<const double2 *>(F);
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    for (; i + stride < n2; i += 2 * stride) {
        const double2 a = F2[i], b = F2[i + stride];
        s0 += fabs(a.x) + fabs(a.y);
        s1 += fabs(b.x) + fabs(b.y);
        mx = fmax(mx, fmax(fmax(fabs(a.x), fabs(a.y)), fmax(fabs(b.x), fabs(b.y))));
    }
    for (; i < n2; i += stride) {
        const double2 a = F2[i];
        s0 += fabs(a.x) + fabs(a.y);
        mx = fmax(mx, fmax(fabs(a.x), fabs(a.y)));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        s1 += fabs(F[n - 1]);
        mx = fmax(mx, fabs(F[n - 1]));
    }
    double s = warp_sum(s0 + s1);
    mx = warp_max(mx);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s_sum[w] = s;
        s_max[w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < kWarps; ++k) {
            a += s_sum[k];
            b = fmax(b, s_max[k]);
        }
        part[2 * blockIdx.x] = a;
        part[2 * blockIdx.x + 1] = b;
        __threadfence();
        const unsigned v = atomicAdd(&ctrl->red_blocks, 1u);
        s_last = (v == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    // last block: ordered final sums (deterministic), sweep bookkeeping
    __threadfence();
    const volatile double *vp = part;
    const volatile double *vs = part_sel;
    double r = 0.0, fm = 0.0, lk = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
        r += vp[2 * b];
        fm = fmax(fm, vp[2 * b + 1]);
    }
    if (!is_init) {
        for (unsigned b = 0; b < gridDim.x; ++b) lk += vs[b];
        end_sweep(ctrl, lk);
    }
    if (force) ctrl->gather = 0;        // TILED flush: the pending remote pushes are now in F
    ctrl->n_entries = 0;
    ctrl->sel_edges = 0;
    ctrl->red_blocks = 0;
    if (ctrl->stats_out) {              // shard: the global values come back through k_control
        ctrl->stats_out[0] = r;
        ctrl->stats_out[1] = fm;
        ctrl->stats_out[2] = ctrl->leak;
        ctrl->stats_out[3] = (double)ctrl->last_sel_edges;
        ctrl->stats_is_init = is_init;
        return;
    }
    finalize_control(ctrl, r, fm, is_init, m);
}

// shard mode: control from every rank's {r, fmax, leak, sel_edges}, gathered in
// rank order: sum r, max fmax, sum leak (fixed order: every rank gets the same bits)
__global__ void k_control(Ctrl *__restrict__ ctrl, const double *__restrict__ gathered, int nranks, int64_t m,
                          int force) {
    if (threadIdx.x != 0 || (ctrl->done && !force)) return;
    double r = 0.0, fm = 0.0, lk = 0.0;
    for (int q = 0; q < nranks; ++q) {
        r += gathered[4 * q];
        fm = fmax(fm, gathered[4 * q + 1]);
        lk += gathered[4 * q + 2];
    }
    ctrl->gleak = lk;
    finalize_control(ctrl, r, fm, ctrl->stats_is_init, m);
}

// ---------------------------------------------------------------- output helpers
__global__ void k_scale_copy(const double *__restrict__ H, double *__restrict__ out, int64_t n, double f) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = H[i] * f;
}

// sum of H over dangling nodes (l of §3.3 as a function of the state, R5)
__global__ void __launch_bounds__(kThreads) k_dangling_hist(const int64_t *__restrict__ row_ptr,
                                                            const double *__restrict__ H, int64_t n,
                                                            double *__restrict__ part) {
    __shared__ double s[kWarps];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
        if (row_ptr[i + 1] == row_ptr[i]) acc += H[i];
    acc = warp_sum(acc);
    if (lane_id() == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int k = 0; k < kWarps; ++k) a += s[k];
        part[blockIdx.x] = a;
    }
}

// pull-variant kernels live in dit_pull.cu
void launch_pull(di_graph *h);

// ---------------------------------------------------------------- host side
// pinned host mirrors of the control block, recycled across handles (cudaMallocHost /
// cudaFreeHost per graph cost milliseconds and synchronise the device)
static std::mutex g_ctrl_mu;
static std::vector<Ctrl *> g_ctrl_free;
static Ctrl *pinned_ctrl_get() {
    {
        std::lock_guard<std::mutex> lock(g_ctrl_mu);
        if (!g_ctrl_free.empty()) {
            Ctrl *c = g_ctrl_free.back();
            g_ctrl_free.pop_back();
            return c;
        }
    }
    Ctrl *c = nullptr;
    DI_CUDA(cudaMallocHost(&c, sizeof(Ctrl)));
    return c;
}
static void pinned_ctrl_put(Ctrl *c) {
    std::lock_guard<std::mutex> lock(g_ctrl_mu);
    g_ctrl_free.push_back(c);
}

void ensure_state(di_graph *h) {
    State &s = h->s;
    const int64_t n = h->g.n;
    if (s.F) return;
    const int64_t nn = n > 0 ? n : 1;
    DI_CUDA(cudaMallocAsync(&s.F, (h->g.nt > 0 ? h->g.nt : 1) * sizeof(double) + 16, h->stream));   // +16: TMA tile rows
    DI_CUDA(cudaMallocAsync(&s.H, nn * sizeof(double) + 16, h->stream));
    s.ent_cap = n + h->g.m / kSplit + 1;
    DI_CUDA(cudaMallocAsync(&s.ent, s.ent_cap * sizeof(uint4), h->stream));
    DI_CUDA(cudaMallocAsync(&s.ctrl, sizeof(Ctrl), h->stream));
    s.ctrl_host = pinned_ctrl_get();
    std::memset(s.ctrl_host, 0, sizeof(Ctrl));
    // fixed grid for every grid-stride kernel: 8 resident 256-thread blocks per SM
    const int64_t want = (n + kThreads - 1) / kThreads;
    s.grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)h->num_sms * 8));
    DI_CUDA(cudaMallocAsync(&s.part, (size_t)s.grid * 3 * sizeof(double), h->stream));
    DI_CUDA(cudaMallocAsync(&s.hist, kHistCap * sizeof(SweepRec), h->stream));
    DI_CUDA(cudaMemsetAsync(s.ctrl, 0, sizeof(Ctrl), h->stream));
}

void free_state(State &s, cudaStream_t st) {
    for (cudaEvent_t e : s.events) cudaEventDestroy(e);
    for (void *p : {(void *)s.hist, (void *)s.F, (void *)s.H, (void *)s.A, (void *)s.A2, (void *)s.ent, (void *)s.ctrl,
                    (void *)s.part})
        if (p) cudaFreeAsync(p, st);
    if (s.ctrl_host) pinned_ctrl_put(s.ctrl_host);
    s = State();
}

void init_state(di_graph *h, double d, const double *Z_dev) {
    ensure_state(h);
    State &s = h->s;
    const int64_t n = h->g.n;
    if (n > 0) {
        k_init<<<s.grid, kThreads, 0, h->stream>>>(s.F, s.H, Z_dev, n, h->g.nt, (double)h->g.n_global, d);
        count_launch();
        DI_CUDA(cudaGetLastError());
    }
    s.d = d;
    s.valid = true;
    // leak restarts with the state
    DI_CUDA(cudaMemsetAsync(s.ctrl, 0, sizeof(Ctrl), h->stream));
}

void launch_select(di_graph *h, bool pull) {
    State &s = h->s;
    DevGraph &g = h->g;
    if (pull)
        k_select<true><<<s.grid, kThreads, 0, h->stream>>>(g.row_ptr, g.inv, s.F, s.H, s.A, s.ent, g.n, s.ctrl,
                                                            s.part + 2 * s.grid);
    else
        k_select<false><<<s.grid, kThreads, 0, h->stream>>>(g.row_ptr, g.inv, s.F, s.H, s.A, s.ent, g.n, s.ctrl,
                                                             s.part + 2 * s.grid);
    count_launch();
}

void launch_push(di_graph *h) {
    State &s = h->s;
    DevGraph &g = h->g;
    const int grid = h->num_sms * 8;
    switch (g.w_kind) {
    case DI_W_F32:
        k_push<float><<<grid, kThreads, 0, h->stream>>>(g.col, (const float *)g.w, s.F, s.ent, s.ctrl);
        break;
    case DI_W_F64:
        k_push<double><<<grid, kThreads, 0, h->stream>>>(g.col, (const double *)g.w, s.F, s.ent, s.ctrl);
        break;
    default:
        k_push<NoW><<<grid, kThreads, 0, h->stream>>>(g.col, nullptr, s.F, s.ent, s.ctrl);
    }
    count_launch();
}

void launch_reduce(di_graph *h, int is_init) {
    State &s = h->s;
    k_reduce<<<s.grid, kThreads, 0, h->stream>>>(s.F, h->g.n, h->g.m, s.ctrl, s.part, s.part + 2 * s.grid, is_init,
                                                 0);
    count_launch();
}

// exact |F|_1 / max|F| of the current F even when `done` is set (after a TILED
// flush): no sweep is counted; `done` is re-derived from the exact residual
void launch_reduce_exact(di_graph *h) {
    State &s = h->s;
    k_reduce<<<s.grid, kThreads, 0, h->stream>>>(s.F, h->g.n, h->g.m, s.ctrl, s.part, s.part + 2 * s.grid, 1, 1);
    count_launch();
}

// Algorithmic bytes per launch: every index / weight /
// entry read once, every fluid read-modify-write counted as 16 B.
static void collect_profile(di_graph *h, const Ctrl &r) {
    State &s = h->s;
    DevGraph &g = h->g;
    di_profile p{};
    const int64_t S = std::min<int64_t>((int64_t)r.sweeps, kHistCap);
    std::vector<SweepRec> hs(S > 0 ? S : 1);
    if (S > 0) {
        DI_CUDA(cudaMemcpyAsync(hs.data(), s.hist, S * sizeof(SweepRec), cudaMemcpyDeviceToHost, h->stream));
        DI_CUDA(cudaStreamSynchronize(h->stream));
    }
    const double n = (double)g.n, m = (double)g.m;
    const double wb = g.w_kind == DI_W_F32 ? 4.0 : (g.w_kind == DI_W_F64 ? 8.0 : 0.0);
    unsigned long long prev_nodes = 0;
    for (int64_t k = 0; k < S; ++k) {
        float t[4];
        auto ev = [&](int q) { return s.events[kEvPerSweep * k + q]; };
        const SweepRec &rc = hs[k];
        const double nodes = (double)(rc.nodes_cum - prev_nodes);
        prev_nodes = rc.nodes_cum;
        if (rc.use_pull == kUseTiled) {
            // waves: [2c] -> [2c+1] heavy gather of wave c, [2c+1] -> [2c+2] its tile kernel
            // (per node 66 B, per local edge 2 + w, per light record rec + 8,
            // per heavy edge rec + 8, per heavy segment / run 24 B)
            const TilePlan &tp = g.tl;
            const double rec = g.w_kind == DI_W_F64 ? 16.0 : 8.0;
            for (int c = 0; c < tp.waves && 2 * c + 2 < kEvPerSweep; ++c) {
                float th, tt;
                DI_CUDA(cudaEventElapsedTime(&th, ev(2 * c), ev(2 * c + 1)));
                DI_CUDA(cudaEventElapsedTime(&tt, ev(2 * c + 1), ev(2 * c + 2)));
                p.pull_ms += th;
                p.tile_ms += tt;
            }
            p.pull_bytes += (double)tp.mh * (rec + 8.0) + 24.0 * (double)tp.nseg + 24.0 * (double)tp.nrun;
            p.pull_launches += 1;
            p.tile_bytes += 66.0 * n + (double)tp.mloc * (2.0 + wb) + (double)tp.mlight * (rec + 8.0) +
                            8.0 * (double)tp.nh;
            p.tile_launches += 1;
            continue;
        }
        for (int q = 0; q < 4; ++q) DI_CUDA(cudaEventElapsedTime(&t[q], ev(q), ev(q + 1)));
        p.select_ms += t[0];
        p.select_bytes += 8.0 * n + 48.0 * nodes + (rc.use_pull ? 8.0 * n : 16.0 * (double)rc.entries);
        p.select_launches += 1;
        if (rc.use_pull) {
            p.pull_ms += t[2];
            p.pull_bytes += 32.0 * (double)g.t.npieces + m * (12.0 + wb);
            p.pull_launches += 1;
        } else {
            p.push_ms += t[1];
            p.push_bytes += 16.0 * (double)rc.entries + (double)rc.edges * (20.0 + wb);
            p.push_launches += 1;
        }
        p.reduce_ms += t[3];
        p.reduce_bytes += 8.0 * n;
        p.reduce_launches += 1;
    }
    p.sweeps = S;
    s.last_prof = p;
}

// Per-call control block: leak persists with the state, everything else is reset.
void prepare_call(di_graph *h, double tol, const di_solve_opts &o, double *stats_out) {
    State &s = h->s;
    DevGraph &g = h->g;
    const bool want_pull = o.variant != DI_VARIANT_PUSH;
    if (want_pull && g.n > 0) {
        if (o.variant == DI_VARIANT_TILED) {
            build_tiles(h);                          // straight from the CSR (dit_plan.cu): no transpose
            if (!s.A2) DI_CUDA(cudaMallocAsync(&s.A2, g.n * sizeof(double), h->stream));
        } else {
            build_transpose(h);
            if (!g.t.pieces_built) {
                build_plan_pieces(h, g.t);
                phase_mark(h->stream, "transpose: pull pieces");
            }
        }
        if (!s.A) DI_CUDA(cudaMallocAsync(&s.A, g.n * sizeof(double), h->stream));
    }
    s.rounds = o.local_rounds > 0 ? o.local_rounds : 4;
    DI_CUDA(cudaMemcpyAsync(s.ctrl_host, s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
    DI_CUDA(cudaStreamSynchronize(h->stream));
    Ctrl c = *s.ctrl_host;
    const double leak = c.leak;
    std::memset(&c, 0, sizeof(Ctrl));
    c.leak = leak;
    c.d = s.d;
    c.theta = o.theta;
    c.tol = tol;
    c.max_sweeps = (unsigned long long)(o.max_sweeps > 0 ? o.max_sweeps : 10000000LL);
    c.variant = o.variant == DI_VARIANT_TILED ? (g.tl.built ? o.variant : DI_VARIANT_PUSH)
                                              : (g.t.built && g.t.pieces_built ? o.variant : DI_VARIANT_PUSH);
    c.pull_edges = o.pull_frac * (double)g.m;
    c.hist = s.hist;
    c.n_global = (double)(g.n_global > 0 ? g.n_global : 1);
    c.stats_out = stats_out;
    c.gleak = -1.0;
    *s.ctrl_host = c;
    DI_CUDA(cudaMemcpyAsync(s.ctrl, s.ctrl_host, sizeof(Ctrl), cudaMemcpyHostToDevice, h->stream));
    s.launched = 0;
    s.tiled_call = c.variant == DI_VARIANT_TILED;
}

void mark_event(di_graph *h, int64_t sweep, int k) {  // profiling events (declared in dit_internal.cuh)
    State &s = h->s;
    if (!s.profile || sweep >= kHistCap || k >= kEvPerSweep) return;
    const size_t idx = (size_t)sweep * kEvPerSweep + k;
    while (s.events.size() <= idx) {
        cudaEvent_t e;
        DI_CUDA(cudaEventCreate(&e));
        s.events.push_back(e);
    }
    DI_CUDA(cudaEventRecord(s.events[idx], h->stream));
}

// select + diffusion of one sweep (events 0..3 of the sweep when profiling)
void launch_sweep(di_graph *h) {
    State &s = h->s;
    const int64_t k = s.launched;
    mark_event(h, k, 0);
    if (s.tiled_call) {
        launch_tile_sweep(h, s.rounds);              // heavy gather (0..1), fused tile kernel (2..3)
        return;
    }
    launch_select(h, false);
    if (h->g.t.pieces_built) launch_select(h, true);
    mark_event(h, k, 1);
    launch_push(h);
    mark_event(h, k, 2);
    if (h->g.t.pieces_built) launch_pull(h);
    mark_event(h, k, 3);
}

void launch_sweep_reduce(di_graph *h) {
    if (!h->s.tiled_call) {                      // the tile kernel ends its own sweep (events 0..2W)
        launch_reduce(h, 0);
        mark_event(h, h->s.launched, 4);
    }
    h->s.launched += 1;
}

bool poll_done(di_graph *h) {
    State &s = h->s;
    DI_CUDA(cudaGetLastError());
    DI_CUDA(cudaMemcpyAsync(s.ctrl_host, s.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, h->stream));
    DI_CUDA(cudaStreamSynchronize(h->stream));
    return s.ctrl_host->done != 0;
}

void fill_result(di_graph *h, const di_solve_opts &o, double tol, di_result *res) {
    State &s = h->s;
    DevGraph &g = h->g;
    const Ctrl &r = *s.ctrl_host;
    s.last_sweeps = (int64_t)r.sweeps;
    if (s.profile) collect_profile(h, r);
    if (res) {
        std::memset(res, 0, sizeof(*res));
        res->residual_l1 = g.n > 0 ? r.resid : 0.0;
        // a shard's bound and completion factor use the leak of the whole graph (§3.3)
        const double leak = (g.shard && r.gleak >= 0.0) ? r.gleak : r.leak;
        res->leak = leak;
        const bool comp = o.dangling == DI_DANGLING_COMPLETE;
        const double den = comp ? (1.0 - s.d - s.d * leak) : (1.0 - s.d);
        res->bound = res->residual_l1 / den;
        res->norm_factor = comp ? (1.0 - s.d) / den : 1.0;
        res->sweeps = (int64_t)r.sweeps;
        res->diffused_nodes = (int64_t)r.diffused_nodes;
        res->diffused_edges = (int64_t)r.diffused_edges;
        res->push_sweeps = (int64_t)r.push_sweeps;
        res->pull_sweeps = (int64_t)r.pull_sweeps;
        res->converged = res->residual_l1 <= tol ? 1 : 0;
    }
}

// L2 fetch granularity for the sweep's random 8-byte gathers (experiment knob)
static void set_l2_fetch() {
    const char *e = getenv("DIT_L2_FETCH");
    if (e && *e) DI_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e)));
}

// DIT_SOLVE_TIMING=1 (debug): host-side phase times of a solve (stream synchronised)
static void solve_mark(cudaStream_t st, const char *name) {
    static const bool on = getenv("DIT_SOLVE_TIMING") != nullptr;
    if (!on) return;
    static auto last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[dit] solve %-22s %8.3f ms\n", name, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

void run_sweeps(di_graph *h, double tol, const di_solve_opts &o, di_result *res) {
    State &s = h->s;
    set_l2_fetch();
    solve_mark(h->stream, "init");
    prepare_call(h, tol, o, nullptr);
    if (h->g.n > 0) {
        launch_reduce(h, 1);
        solve_mark(h->stream, "prepare + reduce");
        int chunk = 2;
        double r_prev = -1.0;
        unsigned long long s_prev = 0;
        for (;;) {
            for (int k = 0; k < chunk; ++k) {
                launch_sweep(h);
                launch_sweep_reduce(h);
            }
            const bool dn = poll_done(h);
            if (getenv("DIT_SOLVE_TIMING"))
                fprintf(stderr, "[dit] chunk of %d: sweeps %llu resid %.3e done %d\n", chunk,
                        (unsigned long long)s.ctrl_host->sweeps, s.ctrl_host->resid, (int)dn);
            solve_mark(h->stream, "chunk");
            if (dn) {
                if (!s.tiled_call || !s.ctrl_host->gather) break;
                // TILED: the last sweep's remote pushes are still pending in A;
                // gather them into F and take the exact residual
                launch_tile_flush(h);
                launch_reduce_exact(h);
                const bool dn2 = poll_done(h);
                solve_mark(h->stream, "flush");
                if (dn2) break;
            }
            // next chunk: the sweeps the residual's decay over the last chunk still
            // needs to reach tol (doubling while no decay is measurable): a sweep
            // enqueued past convergence costs more (~0.5 ms of early-exit launches)
            // than one more poll when the estimate falls a sweep short
            const double r = s.ctrl_host->resid;
            const unsigned long long sw = s.ctrl_host->sweeps;
            int next = std::min(chunk * 2, 64);
            if (r_prev > 0.0 && r > 0.0 && r < r_prev && sw > s_prev && tol > 0.0) {
                const double rate = std::pow(r / r_prev, 1.0 / (double)(sw - s_prev));
                const double need = std::log(tol / r) / std::log(rate);
                if (std::isfinite(need)) next = (int)std::min(64.0, std::max(1.0, std::ceil(need - 1e-3)));
            }
            r_prev = r;
            s_prev = sw;
            chunk = next;
        }
    } else {
        s.ctrl_host->done = 1;
    }
    fill_result(h, o, tol, res);
    solve_mark(h->stream, "result");
}

void write_H(di_graph *h, double factor, double *H_out, int mem) {
    const int64_t n = h->g.n;
    if (!H_out || n == 0) return;
    State &s = h->s;
    double *dst = H_out;
    double *tmp = nullptr;
    if (mem == DI_MEM_HOST) {
        if (factor == 1.0) {
            DI_CUDA(cudaMemcpyAsync(H_out, s.H, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
            DI_CUDA(cudaStreamSynchronize(h->stream));
            return;
        }
        DI_CUDA(cudaMallocAsync(&tmp, n * sizeof(double), h->stream));
        dst = tmp;
    }
    k_scale_copy<<<s.grid, kThreads, 0, h->stream>>>(s.H, dst, n, factor);
    count_launch();
    DI_CUDA(cudaGetLastError());
    if (tmp) {
        DI_CUDA(cudaMemcpyAsync(H_out, tmp, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
        DI_CUDA(cudaFreeAsync(tmp, h->stream));
    }
    DI_CUDA(cudaStreamSynchronize(h->stream));
}

// l := sum of H over dangling nodes, summed on the device in a fixed order
__global__ void k_leak_final(const double *__restrict__ part, int nb, Ctrl *__restrict__ ctrl) {
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int b = 0; b < nb; ++b) a += part[b];
        ctrl->leak = a;
    }
}

void set_leak_from_history(di_graph *h) {
    State &s = h->s;
    const int64_t n = h->g.n;
    if (n == 0) return;
    k_dangling_hist<<<s.grid, kThreads, 0, h->stream>>>(h->g.row_ptr, s.H, n, s.part);
    k_leak_final<<<1, 32, 0, h->stream>>>(s.part, s.grid, s.ctrl);
    count_launch(2);
    DI_CUDA(cudaGetLastError());
}

}  // namespace dit
