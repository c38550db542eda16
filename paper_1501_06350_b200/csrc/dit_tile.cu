// dit_tile.cu -- the tile-local D-Iteration sweep (reading R12, §5).
//
// PAPER §3.4: DI converges for any fair diffusion sequence ("one strength of
// D-Iteration is the freedom in the choice of a scheduler").  This schedule
// exploits the locality of web graphs (most links stay inside a site) and the
// SM's shared memory.  Node ids are cut into tiles of kNodeTile; per sweep:
//
//   1. every tile first takes in the remote pushes of the previous sweep
//      (F(t) += d D(i) P_{t,i} for i outside t's tile: a gather of the
//      previous sweep's outflow A(i) = d D(i) / sum_k w_{i,k} over t's remote
//      in-edges, Eq. (8) being linear in the diffused amount);
//   2. then runs `rounds` Jacobi diffusion rounds over its LOCAL in-edges
//      (source and target in the tile) in shared memory: every node holding
//      fluid is diffused (Eqs. (8), (10)), local pushes applied at once;
//   3. writes F (what is left in the tile), H += D and the new outflow A.
//
// Step 1 of sweep k+1 completes the remote pushes of sweep k, so the sequence
// of Eq. (8) updates is exactly the oracle's (orc_tiled_sweep_run: rounds in
// every tile, then the remote pushes).  The stop test after sweep k uses
// |F|_1 = sum_t |f_t| + sum_i |A(i)| wr(i) (wr = share of i's outflow that leaves
// its tile): exact for non-negative fluid, an upper bound for signed fluid
// (§3.5), so stopping on it keeps Theorem 1's guarantee; after the last sweep
// the pending pushes are flushed into F and the exact |F|_1 is taken.
//
// Kernels (B200): k_tile -- one 512-thread CTA per tile, 2 CTAs per SM,
// the tile's local edges and light remote records staged by TMA bulk copies
// (cp.async.bulk + mbarrier) while the per-node state streams into registers;
// k_heavy / k_heavy_fix -- the remote gather of heavy targets over fixed
// 2048-edge chunks, warp-per-segment sums and warp-per-target fix-ups.  Every
// summation has a fixed order: bitwise reproducible run to run.
#include "dit_internal.cuh"

#include <algorithm>
#include <type_traits>

namespace dit {

constexpr int kTileThreads = (int)kNodeTile;     // thread i owns node i of the tile
constexpr int kTileWarps = kTileThreads / 32;

// remote record: source and raw weight of one remote in-edge
template <typename W>
struct RemRec {
    int32_t src;
    float w;
};
template <>
struct RemRec<double> {
    int32_t src;
    int32_t pad;
    double w;
};
template <typename W>
__device__ __forceinline__ double rec_w(const RemRec<W> &r) { return (double)r.w; }

template <typename W>
using StoreW = typename std::conditional<std::is_same<W, NoW>::value, float, W>::type;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    return ok != 0;
}
// bounded wait: a byte-count mismatch becomes a trap (an error), never a hung GPU
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    for (long long spin = 0; !mbar_try_wait(bar, phase); ++spin)
        if (spin > (1ll << 26)) __trap();
}
// bulk global -> shared copy (the TMA engine), completion counted on `bar`
__device__ __forceinline__ void tma_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// ---------------------------------------------------------------- build
// per target: local / remote in-edge counts from the transpose
__global__ void k_count_local(const int64_t *__restrict__ tptr, const int32_t *__restrict__ tsrc, int64_t n,
                              int64_t *__restrict__ lc, int64_t *__restrict__ rc) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < n; t += nw) {
        const int64_t b = tptr[t], e = tptr[t + 1];
        const int64_t tile = t / kNodeTile;
        int64_t c = 0;
        for (int64_t k = b + lane_id(); k < e; k += 32) c += (tsrc[k] / kNodeTile == tile);
        c = warp_sum(c);
        if (lane_id() == 0) {
            lc[t] = c;
            rc[t] = (e - b) - c;
        }
    }
}

// light / heavy split of the remote in-edges, one thread per tile
__global__ void k_classify(const int64_t *__restrict__ rc, int64_t n, int64_t ntile, int64_t *__restrict__ lrc,
                           int64_t *__restrict__ hc, int64_t *__restrict__ hflag) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntile; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = t * kNodeTile, z = min(n, a + kNodeTile);
        int64_t light = 0;
        for (int64_t j = a; j < z; ++j)
            if (rc[j] <= kHeavyTh) light += rc[j];
        const int64_t th = light > kLightCap ? 0 : kHeavyTh;   // overflowing tile: every remote target heavy
        for (int64_t j = a; j < z; ++j) {
            const bool heavy = rc[j] > th;
            lrc[j] = heavy ? 0 : rc[j];
            hc[j] = heavy ? rc[j] : 0;
            hflag[j] = heavy ? 1 : 0;
        }
    }
}

// tile-relative offsets, tile bases, heavy index, out-degree
__global__ void k_tile_rel(const int64_t *__restrict__ lptr, const int64_t *__restrict__ rptr,
                           const int64_t *__restrict__ hpos, const int64_t *__restrict__ hflag,
                           const int64_t *__restrict__ row_ptr, int64_t n, int64_t ntile, uint32_t *__restrict__ lrel,
                           uint32_t *__restrict__ rrel, int32_t *__restrict__ hidx, int32_t *__restrict__ hj,
                           int32_t *__restrict__ deg, int64_t *__restrict__ ltile, int64_t *__restrict__ rtile) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < n) {
            const int64_t b = (j / kNodeTile) * kNodeTile;
            lrel[j] = (uint32_t)(lptr[j] - lptr[b]);
            rrel[j] = (uint32_t)(rptr[j] - rptr[b]);
            const int32_t h = hflag[j] ? (int32_t)hpos[j] : -1;
            hidx[j] = h;
            if (h >= 0) hj[h] = (int32_t)j;
            deg[j] = (int32_t)(row_ptr[j + 1] - row_ptr[j]);
        }
        if (j % kNodeTile == 0 || j == n) {
            const int64_t t = (j + kNodeTile - 1) / kNodeTile;   // j == n: the end of the last tile
            if (t <= ntile) {
                ltile[t] = lptr[j];
                rtile[t] = rptr[j];
            }
        }
    }
}

// scatter every in-edge (ascending source within its target) to its class
template <typename W>
__global__ void k_split_edges(const int64_t *__restrict__ tptr, const int32_t *__restrict__ tsrc,
                              const StoreW<W> *__restrict__ tw, int64_t n, const int64_t *__restrict__ lptr,
                              const int64_t *__restrict__ rptr, const int64_t *__restrict__ hptr,
                              const int32_t *__restrict__ hidx, uint16_t *__restrict__ lsrc,
                              StoreW<W> *__restrict__ lw, RemRec<W> *__restrict__ rrec, RemRec<W> *__restrict__ hrec) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const unsigned lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    constexpr bool kW = !std::is_same<W, NoW>::value;
    for (int64_t t = warp; t < n; t += nw) {
        const int64_t b = tptr[t], e = tptr[t + 1];
        const int64_t tile = t / kNodeTile;
        const bool heavy = hidx[t] >= 0;
        int64_t lo = lptr[t];
        int64_t ro = heavy ? hptr[t] : rptr[t];
        RemRec<W> *dst = heavy ? hrec : rrec;
        for (int64_t k0 = b; k0 < e; k0 += 32) {
            const int64_t k = k0 + lane;
            const bool ok = k < e;
            const int32_t s = ok ? tsrc[k] : 0;
            const bool loc = ok && (s / kNodeTile == tile);
            const unsigned bl = __ballot_sync(0xffffffffu, loc);
            const unsigned br = __ballot_sync(0xffffffffu, ok && !loc);
            if (loc) {
                const int64_t o = lo + __popc(bl & lt);
                lsrc[o] = (uint16_t)(s - tile * kNodeTile);
                if (kW) lw[o] = tw[k];
            } else if (ok) {
                const int64_t o = ro + __popc(br & lt);
                RemRec<W> r{};
                r.src = s;
                if constexpr (kW) r.w = tw[k];
                else r.w = 1.0f;
                dst[o] = r;
            }
            lo += __popc(bl);
            ro += __popc(br);
        }
    }
}

// share of every source's outflow that leaves its tile (warp per source)
template <typename W>
__global__ void k_remote_share(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                               const StoreW<W> *__restrict__ w, const double *__restrict__ inv, int64_t n,
                               float *__restrict__ wr) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr bool kW = !std::is_same<W, NoW>::value;
    for (int64_t i = warp; i < n; i += nw) {
        const int64_t tile = i / kNodeTile;
        double s = 0.0;
        for (int64_t e = row_ptr[i] + lane_id(); e < row_ptr[i + 1]; e += 32)
            if (col[e] / kNodeTile != tile) s += kW ? (double)w[e] : 1.0;
        s = warp_sum(s);
        if (lane_id() == 0) wr[i] = (float)(s * inv[i]);
    }
}

// heavy segments: segments of heavy target h = its edge range cut at chunk boundaries
__global__ void k_seg_count(const int32_t *__restrict__ hj, const int64_t *__restrict__ hptr, int64_t nh,
                            int64_t *__restrict__ cnt) {
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = hptr[hj[h]], e = hptr[hj[h] + 1];
        cnt[h] = (e - 1) / kHeavyChunk - b / kHeavyChunk + 1;
    }
}

__global__ void k_seg_write(const int32_t *__restrict__ hj, const int64_t *__restrict__ hptr, int64_t nh,
                            const int64_t *__restrict__ hfirst, int64_t *__restrict__ seg_start,
                            int64_t *__restrict__ cfirst) {
    for (int64_t h = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; h < nh; h += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = hptr[hj[h]];
        const int64_t s0 = hfirst[h], s1 = hfirst[h + 1];
        for (int64_t q = 0; q < s1 - s0; ++q) {
            const int64_t p = q == 0 ? b : (b / kHeavyChunk + q) * kHeavyChunk;
            seg_start[s0 + q] = p;
            if (p % kHeavyChunk == 0) cfirst[p / kHeavyChunk] = s0 + q;   // every chunk starts a segment
        }
    }
}

__global__ void k_tile_max_edges(const int64_t *__restrict__ ltile, int64_t ntile, unsigned long long *__restrict__ mx) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntile; t += (int64_t)gridDim.x * blockDim.x)
        atomicMax(mx, (unsigned long long)(ltile[t + 1] - ltile[t]));
}

void free_tiles(TilePlan &t) {
    cudaFree(t.lrel);
    cudaFree(t.rrel);
    cudaFree(t.hidx);
    cudaFree(t.wr);
    cudaFree(t.deg);
    cudaFree(t.ltile);
    cudaFree(t.rtile);
    cudaFree(t.lsrc);
    cudaFree(t.lw);
    cudaFree(t.rrec);
    cudaFree(t.hrec);
    cudaFree(t.seg_start);
    cudaFree(t.cfirst);
    cudaFree(t.hfirst);
    cudaFree(t.part);
    cudaFree(t.hsum);
    t = TilePlan();
}

static int64_t read_i64(const int64_t *p, cudaStream_t st) {
    int64_t v = 0;
    DI_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    return v;
}

template <typename W>
static void build_tiles_t(di_graph *h) {
    DevGraph &g = h->g;
    TilePlan &tp = g.tl;
    cudaStream_t st = h->stream;
    const int64_t n = g.n;
    const int grid = h->num_sms * 8;
    using SW = StoreW<W>;
    constexpr bool kW = !std::is_same<W, NoW>::value;
    tp.ntile = (n + kNodeTile - 1) / kNodeTile;
    int64_t *lc, *rc, *lrc, *hc, *hflag, *lptr, *rptr, *hptr, *hpos;
    for (int64_t **p : {&lc, &rc, &lrc, &hc, &hflag, &lptr, &rptr, &hptr, &hpos})
        DI_CUDA(cudaMallocAsync(p, (n + 1) * sizeof(int64_t), st));
    k_count_local<<<grid, 256, 0, st>>>(g.t.ptr, g.t.src, n, lc, rc);
    k_classify<<<grid_for(h, tp.ntile), 256, 0, st>>>(rc, n, tp.ntile, lrc, hc, hflag);
    count_launch(2);
    exclusive_scan_i64(lc, lptr, n, st);
    exclusive_scan_i64(lrc, rptr, n, st);
    exclusive_scan_i64(hc, hptr, n, st);
    exclusive_scan_i64(hflag, hpos, n, st);
    tp.mloc = read_i64(lptr + n, st);
    tp.mlight = read_i64(rptr + n, st);
    tp.mh = read_i64(hptr + n, st);
    tp.nh = read_i64(hpos + n, st);
    const size_t rs = sizeof(RemRec<W>);
    DI_CUDA(cudaMalloc(&tp.lrel, n * sizeof(uint32_t)));
    DI_CUDA(cudaMalloc(&tp.rrel, n * sizeof(uint32_t)));
    DI_CUDA(cudaMalloc(&tp.hidx, n * sizeof(int32_t)));
    DI_CUDA(cudaMalloc(&tp.wr, n * sizeof(float)));
    DI_CUDA(cudaMalloc(&tp.deg, n * sizeof(int32_t)));
    DI_CUDA(cudaMalloc(&tp.ltile, (tp.ntile + 1) * sizeof(int64_t)));
    DI_CUDA(cudaMalloc(&tp.rtile, (tp.ntile + 1) * sizeof(int64_t)));
    // +16 B: aligned TMA supersets may read up to 15 bytes past the end
    DI_CUDA(cudaMalloc(&tp.lsrc, tp.mloc * sizeof(uint16_t) + 16));
    if (kW) DI_CUDA(cudaMalloc(&tp.lw, tp.mloc * sizeof(SW) + 16));
    DI_CUDA(cudaMalloc(&tp.rrec, tp.mlight * rs + 16));
    DI_CUDA(cudaMalloc(&tp.hrec, tp.mh * rs + 16));
    DI_CUDA(cudaMalloc(&tp.hsum, (tp.nh > 0 ? tp.nh : 1) * sizeof(double)));
    int32_t *hj;
    DI_CUDA(cudaMallocAsync(&hj, (tp.nh > 0 ? tp.nh : 1) * sizeof(int32_t), st));
    k_tile_rel<<<grid_for(h, n + 1), 256, 0, st>>>(lptr, rptr, hpos, hflag, g.row_ptr, n, tp.ntile, tp.lrel, tp.rrel,
                                                   tp.hidx, hj, tp.deg, tp.ltile, tp.rtile);
    k_split_edges<W><<<grid, 256, 0, st>>>(g.t.ptr, g.t.src, (const SW *)g.t.w, n, lptr, rptr, hptr, tp.hidx,
                                           tp.lsrc, (SW *)tp.lw, (RemRec<W> *)tp.rrec, (RemRec<W> *)tp.hrec);
    k_remote_share<W><<<grid, 256, 0, st>>>(g.row_ptr, g.col, (const SW *)g.w, g.inv, n, tp.wr);
    count_launch(3);
    // heavy segments
    tp.nchunk = (tp.mh + kHeavyChunk - 1) / kHeavyChunk;
    DI_CUDA(cudaMalloc(&tp.hfirst, (tp.nh + 1) * sizeof(int64_t)));
    DI_CUDA(cudaMalloc(&tp.cfirst, (tp.nchunk + 1) * sizeof(int64_t)));
    int64_t *cnt;
    DI_CUDA(cudaMallocAsync(&cnt, (tp.nh + 1) * sizeof(int64_t), st));
    if (tp.nh > 0) {
        k_seg_count<<<grid_for(h, tp.nh), 256, 0, st>>>(hj, hptr, tp.nh, cnt);
        count_launch();
    }
    exclusive_scan_i64(cnt, tp.hfirst, tp.nh, st);
    tp.nseg = read_i64(tp.hfirst + tp.nh, st);
    DI_CUDA(cudaMalloc(&tp.seg_start, (tp.nseg + 1) * sizeof(int64_t)));
    DI_CUDA(cudaMalloc(&tp.part, (tp.nseg > 0 ? tp.nseg : 1) * sizeof(double)));
    DI_CUDA(cudaMemcpyAsync(tp.seg_start + tp.nseg, &tp.mh, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    DI_CUDA(cudaMemcpyAsync(tp.cfirst + tp.nchunk, &tp.nseg, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (tp.nh > 0) {
        k_seg_write<<<grid_for(h, tp.nh), 256, 0, st>>>(hj, hptr, tp.nh, tp.hfirst, tp.seg_start, tp.cfirst);
        count_launch();
    }
    unsigned long long *mx;
    DI_CUDA(cudaMallocAsync(&mx, sizeof(unsigned long long), st));
    DI_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
    if (tp.ntile > 0) {
        k_tile_max_edges<<<grid_for(h, tp.ntile), 256, 0, st>>>(tp.ltile, tp.ntile, mx);
        count_launch();
    }
    unsigned long long mxh = 0;
    DI_CUDA(cudaMemcpyAsync(&mxh, mx, sizeof(mxh), cudaMemcpyDeviceToHost, st));
    for (int64_t *p : {lc, rc, lrc, hc, hflag, lptr, rptr, hptr, hpos, cnt}) DI_CUDA(cudaFreeAsync(p, st));
    DI_CUDA(cudaFreeAsync(hj, st));
    DI_CUDA(cudaFreeAsync(mx, st));
    DI_CUDA(cudaStreamSynchronize(st));
    DI_CUDA(cudaGetLastError());
    tp.max_tile_edges = (int64_t)mxh;
    tp.built = true;
}

void build_tiles(di_graph *h) {
    DevGraph &g = h->g;
    if (g.tl.built || g.n == 0) return;
    if (g.shard) {
        set_error("the tiled variant is not available on shards");
        throw Fail{DI_ERR_INVALID};
    }
    build_transpose(h);
    switch (g.w_kind) {
    case DI_W_F32: build_tiles_t<float>(h); break;
    case DI_W_F64: build_tiles_t<double>(h); break;
    default: build_tiles_t<NoW>(h);
    }
}

// ---------------------------------------------------------------- heavy remote gather
// hsum[h] = sum over heavy target h's remote in-edges of A(src) w, from the
// previous sweep's outflow.  CTA per 2048-edge chunk: products staged in
// shared memory, then one warp per segment (lane-strided + fixed butterfly).
template <typename W>
__global__ void __launch_bounds__(kThreads) k_heavy(const RemRec<W> *__restrict__ hrec, int64_t mh, int64_t nchunk,
                                                    const int64_t *__restrict__ seg_start,
                                                    const int64_t *__restrict__ cfirst, const double *__restrict__ A0,
                                                    const double *__restrict__ A1, double *__restrict__ part,
                                                    const Ctrl *__restrict__ ctrl, int force) {
    __shared__ double vals[kHeavyChunk];
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    if (!ctrl->gather) return;
    // the previous sweep wrote A[(sweeps - 1) & 1]
    const double *__restrict__ A = (ctrl->sweeps & 1) ? A0 : A1;
    const unsigned w = threadIdx.x >> 5, lane = lane_id();
    for (int64_t c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const int64_t e0 = c * kHeavyChunk;
        const int cnt = (int)min(kHeavyChunk, mh - e0);
#pragma unroll 4
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
            const RemRec<W> r = hrec[e0 + k];
            vals[k] = A[r.src] * rec_w(r);
        }
        __syncthreads();
        const int64_t s1 = cfirst[c + 1];
        for (int64_t s = cfirst[c] + w; s < s1; s += kWarps) {
            const int b = (int)(seg_start[s] - e0), e = (int)(seg_start[s + 1] - e0);
            double acc = 0.0;
            for (int k = b + (int)lane; k < e; k += 32) acc += vals[k];
            acc = warp_sum(acc);
            if (lane == 0) part[s] = acc;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_heavy_fix(const int64_t *__restrict__ hfirst, int64_t nh,
                                                        const double *__restrict__ part, double *__restrict__ hsum,
                                                        const Ctrl *__restrict__ ctrl, int force) {
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    if (!ctrl->gather) return;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t h = warp; h < nh; h += nw) {
        const int64_t s0 = hfirst[h], s1 = hfirst[h + 1];
        double acc = 0.0;
        for (int64_t s = s0 + lane_id(); s < s1; s += 32) acc += part[s];
        acc = warp_sum(acc);
        if (lane_id() == 0) hsum[h] = acc;
    }
}

// ---------------------------------------------------------------- tile kernel
template <typename W>
struct TileArgs {
    const uint32_t *lrel, *rrel;
    const int32_t *hidx, *deg;
    const float *wr;
    const double *inv;
    const int64_t *ltile, *rtile;
    const uint16_t *lsrc;
    const StoreW<W> *lw;
    const RemRec<W> *rrec;
    const double *hsum;
    double *F, *H, *A0, *A1;
    double *part;            // per-CTA partials: resid [grid], leak [grid]
    int64_t n, ntile, m;
    int rounds;
    int64_t edge_cap;        // bytes of shared memory for the staged local edges
};

template <typename W>
__device__ __forceinline__ double local_sum(const uint16_t *es, const StoreW<W> *ew, const double *gq, int kb, int ke) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
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
    return acc;
}

template <typename W>
__global__ void __launch_bounds__(kTileThreads, 2) k_tile(TileArgs<W> a, Ctrl *__restrict__ ctrl) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr int kWB = kW ? (int)sizeof(StoreW<W>) : 0;
    constexpr int kRS = (int)sizeof(RemRec<W>);
    constexpr int kRecBytes = (int)kLightCap * kRS + 32;
    double *gq = reinterpret_cast<double *>(smem);                       // [kNodeTile]
    unsigned char *rbuf = smem + kNodeTile * sizeof(double);             // light records (16-B aligned)
    unsigned char *ebuf = rbuf + kRecBytes;                              // local edges (16-B aligned)
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double s_r[kTileWarps], s_l[kTileWarps];
    __shared__ unsigned long long s_c[kTileWarps][2];
    __shared__ bool s_last;
    if (ctrl->done || ctrl->use_pull != kUseTiled) return;
    const double d = ctrl->d;
    const bool gather = ctrl->gather != 0;
    const unsigned long long sw = ctrl->sweeps;
    double *__restrict__ Anext = (sw & 1) ? a.A1 : a.A0;
    const double *__restrict__ Aprev = (sw & 1) ? a.A0 : a.A1;
    const uint32_t barp = smem_u32(&bar);
    const int i = threadIdx.x;
    if (i == 0) {
        mbar_init(barp, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    double resid = 0.0, leak = 0.0;
    unsigned long long nodes = 0, edges = 0;
    for (int64_t tile = blockIdx.x; tile < a.ntile; tile += gridDim.x) {
        const int64_t a0 = tile * kNodeTile;
        const int nn = (int)min(kNodeTile, a.n - a0);
        const int64_t l0 = a.ltile[tile], l1 = a.ltile[tile + 1];
        const int64_t r0 = gather ? a.rtile[tile] : 0, r1 = gather ? a.rtile[tile + 1] : 0;
        // aligned byte supersets of the tile's ranges
        const int64_t rb0 = (r0 * kRS) & ~int64_t(15), rb1 = (r1 * kRS + 15) & ~int64_t(15);
        const int64_t sb0 = (l0 * 2) & ~int64_t(15), sb1 = (l1 * 2 + 15) & ~int64_t(15);
        const int64_t wb0 = (l0 * kWB) & ~int64_t(15), wb1 = (l1 * kWB + 15) & ~int64_t(15);
        const bool staged = (sb1 - sb0) + (kW ? (wb1 - wb0) : 0) <= a.edge_cap;
        if (i == 0) {
            // order this CTA's earlier generic-proxy accesses of the buffers before the async writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            uint32_t bytes = (uint32_t)(rb1 - rb0);
            if (staged) bytes += (uint32_t)((sb1 - sb0) + (kW ? (wb1 - wb0) : 0));
            mbar_arrive_tx(barp, bytes);
            if (rb1 > rb0)
                tma_load(smem_u32(rbuf), reinterpret_cast<const unsigned char *>(a.rrec) + rb0, (uint32_t)(rb1 - rb0),
                         barp);
            if (staged) {
                if (sb1 > sb0)
                    tma_load(smem_u32(ebuf), reinterpret_cast<const unsigned char *>(a.lsrc) + sb0,
                             (uint32_t)(sb1 - sb0), barp);
                if (kW && wb1 > wb0)
                    tma_load(smem_u32(ebuf + (sb1 - sb0)), reinterpret_cast<const unsigned char *>(a.lw) + wb0,
                             (uint32_t)(wb1 - wb0), barp);
            }
        }
        // per-node state into registers while the bulk copies fly
        const bool valid = i < nn;
        const int64_t j = a0 + i;
        double Fi = 0.0, Hi = 0.0, ivi = 0.0, hs = 0.0;
        float wri = 0.f;
        int dgi = 0, lb = 0, le = 0, rb = 0, re = 0;
        if (valid) {
            Fi = a.F[j];
            Hi = a.H[j];
            ivi = a.inv[j];
            dgi = a.deg[j];
            wri = a.wr[j];
            lb = (int)a.lrel[j];
            le = i + 1 < nn ? (int)a.lrel[j + 1] : (int)(l1 - l0);
            if (gather) {
                rb = (int)a.rrel[j];
                re = i + 1 < nn ? (int)a.rrel[j + 1] : (int)(r1 - r0);
                const int32_t hx = a.hidx[j];
                if (hx >= 0) hs = a.hsum[hx];
            }
        }
        mbar_wait(barp, phase);
        phase ^= 1u;
        // 1. remote pushes of the previous sweep: light records -> products in place
        const int R = (int)(r1 - r0);
        RemRec<W> *recs = reinterpret_cast<RemRec<W> *>(rbuf + (r0 * kRS - rb0));
#pragma unroll 4
        for (int k = i; k < R; k += kTileThreads) {
            const RemRec<W> r = recs[k];
            *reinterpret_cast<double *>(&recs[k]) = Aprev[r.src] * rec_w(r);
        }
        __syncthreads();
        double f = Fi;
        if (valid) {
            double s = 0.0;
            for (int k = rb; k < re; ++k) s += *reinterpret_cast<const double *>(&recs[k]);
            f = Fi + s + hs;
        }
        // 2. local diffusion rounds in shared memory
        const uint16_t *es;
        const StoreW<W> *ew = nullptr;
        if (staged) {
            es = reinterpret_cast<const uint16_t *>(ebuf + (l0 * 2 - sb0));
            if constexpr (kW) ew = reinterpret_cast<const StoreW<W> *>(ebuf + (sb1 - sb0) + (l0 * kWB - wb0));
        } else {
            es = a.lsrc + l0;
            if constexpr (kW) ew = a.lw + l0;
        }
        double D = 0.0;
        for (int r = 0; r < a.rounds; ++r) {
            double q = 0.0;
            if (valid && f != 0.0) {
                D += f;                              // Eq. (10)
                nodes += 1;
                edges += (unsigned long long)dgi;
                q = d * f * ivi;                     // d F(i) / sum_k w_{i,k}
            }
            gq[i] = q;
            __syncthreads();
            if (valid) f = local_sum<W>(es, ew, gq, lb, le);   // Eq. (8) local pushes, edge order
            __syncthreads();
        }
        // 3. state out
        if (valid) {
            const double An = d * D * ivi;           // remote pushes, completed by the next sweep
            a.F[j] = f;
            if (D != 0.0) a.H[j] = Hi + D;
            Anext[j] = An;
            resid += fabs(f) + fabs(An) * (double)wri;
            if (dgi == 0) leak += D;                 // dangling: the fluid left the system (§3.3)
        }
        __syncthreads();                             // buffers free for the next tile's copies
    }
    // CTA partials (fixed order) and the last-block end of the sweep
    resid = warp_sum(resid);
    leak = warp_sum(leak);
    nodes = warp_sum(nodes);
    edges = warp_sum(edges);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s_r[w] = resid;
        s_l[w] = leak;
        s_c[w][0] = nodes;
        s_c[w][1] = edges;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double rr = 0.0, ll = 0.0;
        unsigned long long x = 0, y = 0;
        for (int k = 0; k < kTileWarps; ++k) {
            rr += s_r[k];
            ll += s_l[k];
            x += s_c[k][0];
            y += s_c[k][1];
        }
        a.part[blockIdx.x] = rr;
        a.part[gridDim.x + blockIdx.x] = ll;
        if (x) {
            atomicAdd(&ctrl->diffused_nodes, x);
            atomicAdd(&ctrl->sel_edges, y);
        }
        __threadfence();
        const unsigned v = atomicAdd(&ctrl->red_blocks, 1u);
        s_last = (v == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    const volatile double *vp = a.part;
    double r = 0.0, lk = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) {
        r += vp[b];
        lk += vp[gridDim.x + b];
    }
    end_sweep(ctrl, lk);
    ctrl->gather = 1;                                // this sweep's remote pushes are pending in A
    ctrl->n_entries = 0;
    ctrl->sel_edges = 0;
    ctrl->red_blocks = 0;
    finalize_control(ctrl, r, 0.0, 0, a.m);
}

// The pending remote pushes of the last sweep into F (same arithmetic and
// order as step 1 of k_tile), thread per node.
template <typename W>
__global__ void __launch_bounds__(kThreads) k_tile_flush(TileArgs<W> a, const Ctrl *__restrict__ ctrl) {
    if (!ctrl->gather) return;
    const double *__restrict__ Aprev = (ctrl->sweeps & 1) ? a.A0 : a.A1;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = j / kNodeTile;
        const int64_t base = a.rtile[t];
        const int64_t b = base + a.rrel[j];
        const int64_t e = (j + 1 < a.n && (j + 1) % kNodeTile != 0) ? base + a.rrel[j + 1] : a.rtile[t + 1];
        double s = 0.0;
        for (int64_t k = b; k < e; ++k) {
            const RemRec<W> r = a.rrec[k];
            s += Aprev[r.src] * rec_w(r);
        }
        const int32_t hx = a.hidx[j];
        const double hs = hx >= 0 ? a.hsum[hx] : 0.0;
        a.F[j] = a.F[j] + s + hs;
    }
}

template <typename W>
static TileArgs<W> tile_args(di_graph *h, int rounds) {
    DevGraph &g = h->g;
    State &s = h->s;
    TilePlan &tp = g.tl;
    TileArgs<W> a;
    a.lrel = tp.lrel;
    a.rrel = tp.rrel;
    a.hidx = tp.hidx;
    a.deg = tp.deg;
    a.wr = tp.wr;
    a.inv = g.inv;
    a.ltile = tp.ltile;
    a.rtile = tp.rtile;
    a.lsrc = tp.lsrc;
    a.lw = (const StoreW<W> *)tp.lw;
    a.rrec = (const RemRec<W> *)tp.rrec;
    a.hsum = tp.hsum;
    a.F = s.F;
    a.H = s.H;
    a.A0 = s.A;
    a.A1 = s.A2;
    a.part = s.part;
    a.n = g.n;
    a.ntile = tp.ntile;
    a.m = g.m;
    a.rounds = rounds;
    a.edge_cap = 0;
    return a;
}

template <typename W>
static void launch_heavy_t(di_graph *h, int force) {
    TilePlan &tp = h->g.tl;
    State &s = h->s;
    if (tp.nh == 0) return;
    const int grid = (int)std::min<int64_t>(tp.nchunk, (int64_t)h->num_sms * 8);
    k_heavy<W><<<grid, kThreads, 0, h->stream>>>((const RemRec<W> *)tp.hrec, tp.mh, tp.nchunk, tp.seg_start, tp.cfirst,
                                                 s.A, s.A2, tp.part, s.ctrl, force);
    k_heavy_fix<<<(unsigned)std::min<int64_t>((tp.nh + kWarps - 1) / kWarps, (int64_t)h->num_sms * 8), kThreads, 0,
                  h->stream>>>(tp.hfirst, tp.nh, tp.part, tp.hsum, s.ctrl, force);
    count_launch(2);
}

template <typename W>
static void launch_tile_t(di_graph *h, int rounds) {
    DevGraph &g = h->g;
    State &s = h->s;
    TilePlan &tp = g.tl;
    const int64_t k = s.launched;
    launch_heavy_t<W>(h, 0);
    mark_event(h, k, 1);
    mark_event(h, k, 2);
    // two CTAs per SM: each takes half of the SM's shared memory
    int per_sm = 0;
    DI_CUDA(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device));
    cudaFuncAttributes fa;
    DI_CUDA(cudaFuncGetAttributes(&fa, k_tile<W>));
    constexpr bool kW = !std::is_same<W, NoW>::value;
    const int64_t fixed = kNodeTile * (int64_t)sizeof(double) + (int64_t)kLightCap * sizeof(RemRec<W>) + 32;
    const int64_t budget = (int64_t)per_sm / 2 - 1024 - (int64_t)fa.sharedSizeBytes;
    const int64_t wsz = kW ? (int64_t)sizeof(StoreW<W>) : 0;
    int64_t cap = (budget - fixed) & ~int64_t(15);
    cap = std::min<int64_t>(cap, (std::max<int64_t>(tp.max_tile_edges, 1) * (2 + wsz) + 47) & ~int64_t(15));
    const size_t smem = (size_t)(fixed + cap);
    DI_CUDA(cudaFuncSetAttribute(k_tile<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TileArgs<W> a = tile_args<W>(h, rounds);
    a.edge_cap = cap;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tp.ntile, (int64_t)h->num_sms * 2));
    k_tile<W><<<grid, kTileThreads, smem, h->stream>>>(a, s.ctrl);
    count_launch();
    DI_CUDA(cudaGetLastError());
    mark_event(h, k, 3);
}

void launch_tile_sweep(di_graph *h, int rounds) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_tile_t<float>(h, rounds); break;
    case DI_W_F64: launch_tile_t<double>(h, rounds); break;
    default: launch_tile_t<NoW>(h, rounds);
    }
}

template <typename W>
static void launch_flush_t(di_graph *h) {
    launch_heavy_t<W>(h, 1);
    k_tile_flush<W><<<grid_for(h, h->g.n), kThreads, 0, h->stream>>>(tile_args<W>(h, 0), h->s.ctrl);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

void launch_tile_flush(di_graph *h) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_flush_t<float>(h); break;
    case DI_W_F64: launch_flush_t<double>(h); break;
    default: launch_flush_t<NoW>(h);
    }
}

}  // namespace dit
