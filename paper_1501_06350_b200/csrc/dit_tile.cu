// dit_tile.cu -- the tile-local D-Iteration sweep (reading R12).
//
// PAPER §3.4: DI converges for any fair diffusion sequence ("one strength of
// D-Iteration is the freedom in the choice of a scheduler").  This schedule
// exploits the locality of web graphs (most links stay inside a site) and the
// SM's shared memory: node ids are cut into tiles of kNodeTile; one CTA loads
// a tile's fluid and its LOCAL in-edges (source and target in the tile) into
// shared memory and runs `rounds` Jacobi diffusion rounds there (every node
// holding fluid is diffused each round, Eq. (8), local pushes applied
// immediately); the amount each node diffused over the rounds, D(i), is then
// pushed along its REMOTE edges by one deterministic pull over the remote CSC
// (linearity of Eq. (8) in the diffused amount).  rounds = 1 is exactly the
// theta = 0 sweep.  Deterministic: fixed summation orders everywhere.
#include "dit_internal.cuh"

namespace dit {

constexpr int kTileThreads = 1024;

// ---------------------------------------------------------------- build
__global__ void k_count_local(const int64_t *__restrict__ tptr, const int32_t *__restrict__ tsrc, int64_t n,
                              int64_t nt, int64_t *__restrict__ lc, int64_t *__restrict__ rc) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < nt; t += nw) {
        const int64_t b = tptr[t], e = tptr[t + 1];
        int64_t c = 0;
        if (t < n) {
            const int64_t tile = t / kNodeTile;
            for (int64_t k = b + lane_id(); k < e; k += 32) c += (tsrc[k] / kNodeTile == tile);
            c = warp_sum(c);
        }
        if (lane_id() == 0) {
            lc[t] = c;
            rc[t] = (e - b) - c;
        }
    }
}

template <typename Wt>
__global__ void k_split_local(const int64_t *__restrict__ tptr, const int32_t *__restrict__ tsrc,
                              const Wt *__restrict__ tw, int64_t n, int64_t nt, const int64_t *__restrict__ lptr,
                              const int64_t *__restrict__ rptr, uint16_t *__restrict__ lsrc, Wt *__restrict__ lw,
                              int32_t *__restrict__ rsrc, Wt *__restrict__ rw) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    for (int64_t t = warp; t < nt; t += nw) {
        const int64_t b = tptr[t], e = tptr[t + 1];
        const int64_t tile = t < n ? t / kNodeTile : -1;
        int64_t lo = lptr[t], ro = rptr[t];
        for (int64_t k0 = b; k0 < e; k0 += 32) {
            const int64_t k = k0 + lane;
            const bool ok = k < e;
            const int32_t s = ok ? tsrc[k] : 0;
            const bool loc = ok && (s / kNodeTile == tile);
            const unsigned bl = __ballot_sync(0xffffffffu, loc);
            const unsigned br = __ballot_sync(0xffffffffu, ok && !loc);
            const unsigned lt = (1u << lane) - 1u;
            if (loc) {
                const int64_t o = lo + __popc(bl & lt);
                lsrc[o] = (uint16_t)(s - tile * kNodeTile);
                if (tw) lw[o] = tw[k];
            } else if (ok) {
                const int64_t o = ro + __popc(br & lt);
                rsrc[o] = s;
                if (tw) rw[o] = tw[k];
            }
            lo += __popc(bl);
            ro += __popc(br);
        }
    }
}

__global__ void k_out_deg(const int64_t *__restrict__ row_ptr, int64_t n, int32_t *__restrict__ deg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        deg[i] = (int32_t)(row_ptr[i + 1] - row_ptr[i]);
}

__global__ void k_tile_edges(const int64_t *__restrict__ lptr, int64_t n, int64_t ntile,
                             unsigned long long *__restrict__ mx) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < ntile; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = b * kNodeTile, z = min(n, a + kNodeTile);
        atomicMax(mx, (unsigned long long)(lptr[z] - lptr[a]));
    }
}

void free_tiles(TilePlan &t) {
    cudaFree(t.lptr);
    cudaFree(t.lsrc);
    cudaFree(t.lw);
    cudaFree(t.deg);
    free_plan(t.rem);
    t = TilePlan();
}

void build_tiles(di_graph *h) {
    DevGraph &g = h->g;
    TilePlan &tp = g.tl;
    if (tp.built) return;
    build_transpose(h);
    cudaStream_t st = h->stream;
    const int64_t n = g.n, nt = g.nt, m = g.m;
    const size_t wsz = g.w_kind == DI_W_F32 ? 4 : (g.w_kind == DI_W_F64 ? 8 : 0);
    tp.ntile = (n + kNodeTile - 1) / kNodeTile;
    int64_t *lc, *rc;
    DI_CUDA(cudaMallocAsync(&lc, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&rc, (nt + 1) * sizeof(int64_t), st));
    const int grid = h->num_sms * 8;
    if (nt > 0) {
        k_count_local<<<grid, 256, 0, st>>>(g.t.ptr, g.t.src, n, nt, lc, rc);
        count_launch();
    }
    DI_CUDA(cudaMalloc(&tp.lptr, (nt + 1) * sizeof(int64_t)));
    DI_CUDA(cudaMalloc(&tp.rem.ptr, (nt + 1) * sizeof(int64_t)));
    exclusive_scan_i64(lc, tp.lptr, nt, st);
    exclusive_scan_i64(rc, tp.rem.ptr, nt, st);
    int64_t ml = 0, mr = 0;
    DI_CUDA(cudaMemcpyAsync(&ml, tp.lptr + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaMemcpyAsync(&mr, tp.rem.ptr + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    tp.mloc = ml;
    tp.rem.nt = nt;
    tp.rem.m = mr;
    DI_CUDA(cudaMalloc(&tp.lsrc, (ml > 0 ? ml : 1) * sizeof(uint16_t)));
    DI_CUDA(cudaMalloc(&tp.rem.src, (mr > 0 ? mr : 1) * sizeof(int32_t)));
    if (wsz) {
        DI_CUDA(cudaMalloc(&tp.lw, (ml > 0 ? ml : 1) * wsz));
        DI_CUDA(cudaMalloc(&tp.rem.w, (mr > 0 ? mr : 1) * wsz));
    }
    if (nt > 0 && m > 0) {
        if (g.w_kind == DI_W_F64)
            k_split_local<double><<<grid, 256, 0, st>>>(g.t.ptr, g.t.src, (const double *)g.t.w, n, nt, tp.lptr,
                                                         tp.rem.ptr, tp.lsrc, (double *)tp.lw, tp.rem.src,
                                                         (double *)tp.rem.w);
        else
            k_split_local<float><<<grid, 256, 0, st>>>(g.t.ptr, g.t.src, (const float *)g.t.w, n, nt, tp.lptr,
                                                        tp.rem.ptr, tp.lsrc, (float *)tp.lw, tp.rem.src,
                                                        (float *)tp.rem.w);
        count_launch();
    }
    DI_CUDA(cudaMalloc(&tp.deg, (n > 0 ? n : 1) * sizeof(int32_t)));
    if (n > 0) {
        k_out_deg<<<grid, 256, 0, st>>>(g.row_ptr, n, tp.deg);
        count_launch();
    }
    unsigned long long *mx;
    DI_CUDA(cudaMallocAsync(&mx, sizeof(unsigned long long), st));
    DI_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
    if (tp.ntile > 0) {
        k_tile_edges<<<grid_for(h, tp.ntile), 256, 0, st>>>(tp.lptr, n, tp.ntile, mx);
        count_launch();
    }
    unsigned long long mxh = 0;
    DI_CUDA(cudaMemcpyAsync(&mxh, mx, sizeof(mxh), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaFreeAsync(mx, st));
    DI_CUDA(cudaFreeAsync(lc, st));
    DI_CUDA(cudaFreeAsync(rc, st));
    DI_CUDA(cudaStreamSynchronize(st));
    tp.max_tile_edges = (int64_t)mxh;
    build_plan_pieces(h, tp.rem);
    tp.built = true;
}

// ---------------------------------------------------------------- tile-local sweep
// Shared memory: f and the round's outflow gq (8 B per node), the tile-relative
// local CSC offsets lp (4 B per node), then the staged local edges: sources
// (u16) and weights, each an aligned superset of the tile's range copied with
// 16-byte vector loads.  D (diffused amount), inv and the out-degree of the
// thread's own node stay in registers (thread i owns node i of the tile).
constexpr int kFixedSmem = kNodeTile * 16 + (kNodeTile + 4) * 4;
static_assert(kTileThreads == kNodeTile, "thread i owns node i of the tile");

__device__ __forceinline__ void copy_vec16(void *dst, const void *src, int64_t bytes) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    const int64_t n16 = bytes >> 4;
    for (int64_t k = threadIdx.x; k < n16; k += blockDim.x) d4[k] = __ldcs(s4 + k);
}

template <typename W>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tile_local(const int64_t *__restrict__ lptr, const uint16_t *__restrict__ lsrc, const W *__restrict__ lw,
                 const double *__restrict__ inv, const int32_t *__restrict__ deg, double *__restrict__ F,
                 double *__restrict__ H, double *__restrict__ A, int64_t n, int64_t ntile, int rounds,
                 int64_t edge_cap, Ctrl *__restrict__ ctrl, double *__restrict__ part_sel, int part_n) {
    extern __shared__ __align__(16) unsigned char smem[];
    double *f = reinterpret_cast<double *>(smem);
    double *gq = f + kNodeTile;
    int32_t *lp = reinterpret_cast<int32_t *>(gq + kNodeTile);
    unsigned char *ebuf = smem + kFixedSmem;                      // 16-byte aligned
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr int kWB = kW ? (int)sizeof(W) : 0;
    __shared__ double s_leak[kTileThreads / 32];
    __shared__ unsigned long long s_cnt[kTileThreads / 32][2];
    if (ctrl->done || ctrl->use_pull != kUseTiled) return;
    if (blockIdx.x == 0)
        for (int k = gridDim.x + threadIdx.x; k < part_n; k += kTileThreads) part_sel[k] = 0.0;
    const double d = ctrl->d;
    double leak = 0.0;
    unsigned long long nodes = 0, edges = 0;
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int64_t a = tile * kNodeTile;
        const int nn = (int)min((int64_t)kNodeTile, n - a);
        const int64_t e0 = lptr[a];
        const int64_t E = lptr[a + nn] - e0;
        // aligned supersets of the tile's source / weight ranges
        const int64_t sb0 = (e0 * 2) & ~int64_t(15), sb1 = ((e0 + E) * 2 + 15) & ~int64_t(15);
        const int64_t wb0 = (e0 * kWB) & ~int64_t(15), wb1 = ((e0 + E) * kWB + 15) & ~int64_t(15);
        const bool staged = (sb1 - sb0) + (kW ? (wb1 - wb0) : 0) <= edge_cap;
        const uint16_t *es = lsrc + e0;
        const W *ew = kW ? lw + e0 : nullptr;
        if (staged) {
            copy_vec16(ebuf, reinterpret_cast<const unsigned char *>(lsrc) + sb0, sb1 - sb0);
            es = reinterpret_cast<const uint16_t *>(ebuf) + ((e0 * 2 - sb0) >> 1);
            if constexpr (kW) {
                unsigned char *wbuf = ebuf + (sb1 - sb0);
                copy_vec16(wbuf, reinterpret_cast<const unsigned char *>(lw) + wb0, wb1 - wb0);
                ew = reinterpret_cast<const W *>(wbuf) + ((e0 * kWB - wb0) / kWB);
            }
        }
        const int i = threadIdx.x;                 // this thread's node (kTileThreads == kNodeTile)
        double Di = 0.0, ivi = 0.0;
        int dgi = 0;
        if (i < nn) {
            f[i] = F[a + i];
            ivi = inv[a + i];
            dgi = deg[a + i];
            lp[i] = (int32_t)(lptr[a + i] - e0);
        }
        if (i == 0) lp[nn] = (int32_t)E;
        __syncthreads();
        for (int r = 0; r < rounds; ++r) {
            // every node holding fluid is diffused (Eqs. (8), (10)); gq = d f / sum w
            if (i < nn) {
                const double fi = f[i];
                double q = 0.0;
                if (fi != 0.0) {
                    Di += fi;
                    nodes += 1;
                    edges += (unsigned long long)dgi;
                    q = d * fi * ivi;
                }
                gq[i] = q;
            }
            __syncthreads();
            // local pushes gathered per target (thread i owns target i), in edge order
            if (i < nn) {
                const int kb = lp[i], ke = lp[i + 1];
                double acc = 0.0;
                int k = kb;
                for (; k + 4 <= ke; k += 4) {
                    const int s0 = es[k], s1 = es[k + 1], s2 = es[k + 2], s3 = es[k + 3];
                    double v0 = gq[s0], v1 = gq[s1], v2 = gq[s2], v3 = gq[s3];
                    if constexpr (kW) {
                        v0 *= (double)ew[k];
                        v1 *= (double)ew[k + 1];
                        v2 *= (double)ew[k + 2];
                        v3 *= (double)ew[k + 3];
                    }
                    acc += v0;
                    acc += v1;
                    acc += v2;
                    acc += v3;
                }
                for (; k < ke; ++k) {
                    double v = gq[es[k]];
                    if constexpr (kW) v *= (double)ew[k];
                    acc += v;
                }
                f[i] = acc;      // only thread i writes f[i]; gq is read-only here
            }
            __syncthreads();
        }
        if (i < nn) {
            F[a + i] = f[i];
            if (Di != 0.0) H[a + i] += Di;
            A[a + i] = d * Di * ivi;                   // remote outflow (linearity of Eq. (8))
            if (dgi == 0) leak += Di;                  // dangling: fluid left the system (§3.3)
        }
        __syncthreads();
    }
    leak = warp_sum(leak);
    nodes = warp_sum(nodes);
    edges = warp_sum(edges);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s_leak[w] = leak;
        s_cnt[w][0] = nodes;
        s_cnt[w][1] = edges;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l = 0.0;
        unsigned long long x = 0, y = 0;
        for (int k = 0; k < kTileThreads / 32; ++k) {
            l += s_leak[k];
            x += s_cnt[k][0];
            y += s_cnt[k][1];
        }
        part_sel[blockIdx.x] = l;
        if (x) {
            atomicAdd(&ctrl->diffused_nodes, x);
            atomicAdd(&ctrl->sel_edges, y);
        }
    }
}

template <typename W>
static void launch_tile_t(di_graph *h, int rounds, const W *lw) {
    DevGraph &g = h->g;
    State &s = h->s;
    TilePlan &tp = g.tl;
    int optin = 0;
    DI_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    cudaFuncAttributes fa;
    DI_CUDA(cudaFuncGetAttributes(&fa, k_tile_local<W>));
    const size_t max_dyn = (size_t)optin - fa.sharedSizeBytes;
    const size_t wsz = std::is_same<W, NoW>::value ? 0 : sizeof(W);
    // staged bytes: both aligned supersets (+32 B of alignment slack)
    int64_t cap = (int64_t)(max_dyn - kFixedSmem) & ~int64_t(15);
    cap = std::min<int64_t>(cap, (std::max<int64_t>(tp.max_tile_edges, 1) * (int64_t)(2 + wsz) + 47) & ~int64_t(15));
    const size_t smem = kFixedSmem + cap;
    DI_CUDA(cudaFuncSetAttribute(k_tile_local<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>(tp.ntile, std::min(h->num_sms, s.grid));
    k_tile_local<W><<<grid, kTileThreads, smem, h->stream>>>(tp.lptr, tp.lsrc, lw, g.inv, tp.deg, s.F, s.H, s.A, g.n,
                                                             tp.ntile, rounds, cap, s.ctrl, s.part + 2 * s.grid,
                                                             s.grid);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

void launch_tile_local(di_graph *h, int rounds) {
    TilePlan &tp = h->g.tl;
    if (tp.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_tile_t<float>(h, rounds, (const float *)tp.lw); break;
    case DI_W_F64: launch_tile_t<double>(h, rounds, (const double *)tp.lw); break;
    default: launch_tile_t<NoW>(h, rounds, nullptr);
    }
}

}  // namespace dit
