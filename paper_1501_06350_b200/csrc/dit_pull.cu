// dit_pull.cu -- transpose builder and the deterministic pull-gather sweep.
//
// Transpose (CSC of the edge list = rows of P): a stable LSD radix sort of the
// edge indices by target (8-bit digits, per-tile histograms, digit-major
// offsets, warp match_any ranking), so the in-edges of every target appear in
// ascending source order.  The pull sweep then computes, for every target j,
//     F(j) += sum_{i -> j} A(i) w_{i,j},   A(i) = d F(i) / sum_k w_{i,k}  (i in S, else 0)
// which is the push of Eq. (8) written as a gather.  Each target is cut into
// pieces of <= kPullSplit in-edges; a warp walks 32 pieces' edges 32 at a time
// and reduces them with a segmented warp scan, in a fixed order: the result is
// bitwise reproducible run to run on a given graph.
#include "dit_internal.cuh"


namespace dit {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortItems = 16;                       // items per lane
constexpr int kWarpItems = 32 * kSortItems;          // 512 items per warp
constexpr int kSortTile = kWarps * kWarpItems;       // 4096 items per block
constexpr int64_t kPullSplit = 256;

// ---------------------------------------------------------------- radix sort
__global__ void __launch_bounds__(kThreads) k_radix_hist(const uint32_t *__restrict__ keys, int64_t count,
                                                         int shift, int64_t ntiles, int64_t *__restrict__ cnt) {
    __shared__ unsigned h[kWarps][kRadix];
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const unsigned w = threadIdx.x >> 5, lane = lane_id();
    const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)w * kWarpItems;
#pragma unroll 4
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < count) atomicAdd(&h[w][(keys[i] >> shift) & (kRadix - 1)], 1u);
    }
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < kRadix; dgt += kThreads) {
        unsigned s = 0;
        for (int k = 0; k < kWarps; ++k) s += h[k][dgt];
        cnt[(int64_t)dgt * ntiles + blockIdx.x] = s;
    }
}

template <typename V>
__global__ void __launch_bounds__(kThreads) k_radix_scatter(const uint32_t *__restrict__ keys,
                                                            const V *__restrict__ vals, int64_t count, int shift,
                                                            int64_t ntiles, const int64_t *__restrict__ off,
                                                            uint32_t *__restrict__ okeys, V *__restrict__ ovals) {
    __shared__ unsigned wc[kWarps][kRadix];
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&wc[0][0])[i] = 0;
    __syncthreads();
    const unsigned w = threadIdx.x >> 5, lane = lane_id();
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)w * kWarpItems;
    unsigned dg[kSortItems], rk[kSortItems];
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = base + k * 32 + lane;
        const bool ok = i < count;
        const unsigned d = ok ? ((keys[i] >> shift) & (kRadix - 1)) : kRadix;   // kRadix = "no item"
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned before = __popc(peers & lt);
        unsigned r = 0;
        if (ok) r = wc[w][d] + before;
        __syncwarp();
        if (ok && before == 0) wc[w][d] += __popc(peers);
        __syncwarp();
        dg[k] = d;
        rk[k] = r;
    }
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < kRadix; dgt += kThreads) {
        unsigned run = 0;
        for (int k = 0; k < kWarps; ++k) {
            const unsigned t = wc[k][dgt];
            wc[k][dgt] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kSortItems; ++k) {
        const int64_t i = base + k * 32 + lane;
        if (i < count) {
            const unsigned d = dg[k];
            const int64_t pos = off[(int64_t)d * ntiles + blockIdx.x] + wc[w][d] + rk[k];
            okeys[pos] = keys[i];
            ovals[pos] = vals[i];
        }
    }
}

// ---------------------------------------------------------------- transpose helpers
__global__ void k_iota_keys(const int32_t *__restrict__ col, int64_t m, uint32_t *__restrict__ keys,
                            void *__restrict__ vals, int wide) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = (uint32_t)col[e];
        if (wide) ((uint64_t *)vals)[e] = (uint64_t)e;
        else ((uint32_t *)vals)[e] = (uint32_t)e;
    }
}

// source id of every edge (warp per row)
__global__ void k_edge_src(const int64_t *__restrict__ row_ptr, int64_t n, int32_t *__restrict__ src) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < n; i += nw)
        for (int64_t e = row_ptr[i] + lane_id(); e < row_ptr[i + 1]; e += 32) src[e] = (int32_t)i;
}

// in-degree from the sorted keys: run ends minus run starts
__global__ void k_run_bounds(const uint32_t *__restrict__ sk, int64_t m, int64_t *__restrict__ cnt) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = sk[p];
        if (p == 0 || sk[p - 1] != k) atomicAdd((unsigned long long *)&cnt[k], (unsigned long long)(-p));
        if (p == m - 1 || sk[p + 1] != k) atomicAdd((unsigned long long *)&cnt[k], (unsigned long long)(p + 1));
    }
}

template <typename V, typename Wt>
__global__ void k_gather_t(const V *__restrict__ sv, int64_t m, const int32_t *__restrict__ esrc,
                           const Wt *__restrict__ w, int32_t *__restrict__ t_src, Wt *__restrict__ t_w) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = (int64_t)sv[p];
        t_src[p] = esrc[e];
        if (w) t_w[p] = w[e];
    }
}

__global__ void k_piece_count(const int64_t *__restrict__ t_ptr, int64_t n, int64_t *__restrict__ pc) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        pc[j] = (t_ptr[j + 1] - t_ptr[j] + kPullSplit - 1) / kPullSplit;
}

// piece = { begin<<24 | len, target, first-piece-of-split-target index or -1 }
__global__ void k_piece_write(const int64_t *__restrict__ t_ptr, int64_t n, const int64_t *__restrict__ po,
                              uint4 *__restrict__ pieces, int4 *__restrict__ fix, unsigned long long *__restrict__ nfix) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t_ptr[j], deg = t_ptr[j + 1] - b;
        const int64_t np = po[j + 1] - po[j];
        const bool split = np > 1;
        for (int64_t c = 0; c < np; ++c) {
            const int64_t cb = b + c * kPullSplit;
            const int64_t len = min(kPullSplit, deg - c * kPullSplit);
            const unsigned long long packed = ((unsigned long long)cb << kLenBits) | (unsigned long long)len;
            pieces[po[j] + c] = make_uint4((unsigned)packed, (unsigned)(packed >> 32), (unsigned)j, split ? 1u : 0u);
        }
        if (split) {
            const unsigned long long q = atomicAdd(nfix, 1ull);
            fix[q] = make_int4((int)j, (int)(po[j] & 0xffffffff), (int)(po[j] >> 32), (int)np);
        }
    }
}

static void radix_sort_pass_launch(const uint32_t *k, const void *v, uint32_t *ok, void *ov, int64_t m, int shift,
                                   int64_t ntiles, int64_t *cnt, int64_t *off, bool wide, cudaStream_t st) {
    k_radix_hist<<<(unsigned)ntiles, kThreads, 0, st>>>(k, m, shift, ntiles, cnt);
    count_launch();
    exclusive_scan_i64(cnt, off, (int64_t)kRadix * ntiles, st);
    if (wide)
        k_radix_scatter<uint64_t><<<(unsigned)ntiles, kThreads, 0, st>>>(k, (const uint64_t *)v, m, shift, ntiles, off,
                                                                           ok, (uint64_t *)ov);
    else
        k_radix_scatter<uint32_t><<<(unsigned)ntiles, kThreads, 0, st>>>(k, (const uint32_t *)v, m, shift, ntiles, off,
                                                                           ok, (uint32_t *)ov);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

void build_transpose(di_graph *h) {
    DevGraph &g = h->g;
    if (g.has_t) return;
    cudaStream_t st = h->stream;
    const int64_t n = g.n, m = g.m;
    const bool wide = m >= (int64_t)0xffffffffLL;
    const size_t vsz = wide ? 8 : 4;
    DI_CUDA(cudaMalloc(&g.t_ptr, (n + 1) * sizeof(int64_t)));
    DI_CUDA(cudaMalloc(&g.t_src, (m > 0 ? m : 1) * sizeof(int32_t)));
    const size_t wsz = g.w_kind == DI_W_F32 ? 4 : (g.w_kind == DI_W_F64 ? 8 : 0);
    if (wsz) DI_CUDA(cudaMalloc(&g.t_w, (m > 0 ? m : 1) * wsz));
    int64_t *cnt = nullptr;
    DI_CUDA(cudaMallocAsync(&cnt, (n + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int64_t), st));
    if (m > 0) {
        uint32_t *k0, *k1;
        void *v0, *v1;
        int32_t *esrc;
        DI_CUDA(cudaMallocAsync(&k0, m * 4, st));
        DI_CUDA(cudaMallocAsync(&k1, m * 4, st));
        DI_CUDA(cudaMallocAsync(&v0, m * vsz, st));
        DI_CUDA(cudaMallocAsync(&v1, m * vsz, st));
        const int grid = h->num_sms * 8;
        k_iota_keys<<<grid, kThreads, 0, st>>>(g.col, m, k0, v0, wide);
        count_launch();
        const int64_t ntiles = (m + kSortTile - 1) / kSortTile;
        int64_t *hc, *ho;
        DI_CUDA(cudaMallocAsync(&hc, (int64_t)kRadix * ntiles * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&ho, ((int64_t)kRadix * ntiles + 1) * sizeof(int64_t), st));
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) < n) ++bits;
        for (int shift = 0; shift < bits; shift += kRadixBits) {
            radix_sort_pass_launch(k0, v0, k1, v1, m, shift, ntiles, hc, ho, wide, st);
            std::swap(k0, k1);
            std::swap(v0, v1);
        }
        DI_CUDA(cudaFreeAsync(hc, st));
        DI_CUDA(cudaFreeAsync(ho, st));
        // in-degrees -> t_ptr
        k_run_bounds<<<grid, kThreads, 0, st>>>(k0, m, cnt);
        count_launch();
        DI_CUDA(cudaMallocAsync(&esrc, m * 4, st));
        k_edge_src<<<grid, kThreads, 0, st>>>(g.row_ptr, n, esrc);
        count_launch();
        if (wide) {
            if (g.w_kind == DI_W_F64)
                k_gather_t<uint64_t, double><<<grid, kThreads, 0, st>>>((const uint64_t *)v0, m, esrc, (const double *)g.w, g.t_src, (double *)g.t_w);
            else
                k_gather_t<uint64_t, float><<<grid, kThreads, 0, st>>>((const uint64_t *)v0, m, esrc, (const float *)g.w, g.t_src, (float *)g.t_w);
        } else {
            if (g.w_kind == DI_W_F64)
                k_gather_t<uint32_t, double><<<grid, kThreads, 0, st>>>((const uint32_t *)v0, m, esrc, (const double *)g.w, g.t_src, (double *)g.t_w);
            else
                k_gather_t<uint32_t, float><<<grid, kThreads, 0, st>>>((const uint32_t *)v0, m, esrc, (const float *)g.w, g.t_src, (float *)g.t_w);
        }
        count_launch();
        DI_CUDA(cudaFreeAsync(esrc, st));
        DI_CUDA(cudaFreeAsync(k0, st));
        DI_CUDA(cudaFreeAsync(k1, st));
        DI_CUDA(cudaFreeAsync(v0, st));
        DI_CUDA(cudaFreeAsync(v1, st));
    }
    exclusive_scan_i64(cnt, g.t_ptr, n, st);
    // pieces
    DevGraph &pd = g;
    int64_t *pc, *po;
    DI_CUDA(cudaMallocAsync(&pc, (n + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&po, (n + 1) * sizeof(int64_t), st));
    const int grid = h->num_sms * 8;
    if (n > 0) {
        k_piece_count<<<grid, kThreads, 0, st>>>(g.t_ptr, n, pc);
        count_launch();
    }
    exclusive_scan_i64(pc, po, n, st);
    int64_t np = 0;
    DI_CUDA(cudaMemcpyAsync(&np, po + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    pd.npieces = np;
    DI_CUDA(cudaMalloc(&pd.pieces, (np > 0 ? np : 1) * sizeof(uint4)));
    DI_CUDA(cudaMalloc(&pd.pbuf, (np > 0 ? np : 1) * sizeof(double)));
    DI_CUDA(cudaMalloc(&pd.fix, (n > 0 ? n : 1) * sizeof(int4)));
    unsigned long long *nf;
    DI_CUDA(cudaMallocAsync(&nf, sizeof(unsigned long long), st));
    DI_CUDA(cudaMemsetAsync(nf, 0, sizeof(unsigned long long), st));
    if (n > 0) {
        k_piece_write<<<grid, kThreads, 0, st>>>(g.t_ptr, n, po, pd.pieces, pd.fix, nf);
        count_launch();
    }
    unsigned long long nfix = 0;
    DI_CUDA(cudaMemcpyAsync(&nfix, nf, sizeof(nfix), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaFreeAsync(nf, st));
    DI_CUDA(cudaFreeAsync(pc, st));
    DI_CUDA(cudaFreeAsync(po, st));
    DI_CUDA(cudaFreeAsync(cnt, st));
    DI_CUDA(cudaStreamSynchronize(st));
    pd.nfix = (int64_t)nfix;
    g.has_t = true;
}

// ---------------------------------------------------------------- pull sweep
template <typename W>
__global__ void __launch_bounds__(kThreads) k_pull(const int32_t *__restrict__ t_src, const W *__restrict__ t_w,
                                                   const double *__restrict__ A, double *__restrict__ F,
                                                   const uint4 *__restrict__ pieces, int64_t npieces,
                                                   double *__restrict__ pbuf, const Ctrl *__restrict__ ctrl) {
    __shared__ double acc[kWarps][33];
    if (ctrl->done || !ctrl->use_pull) return;
    const unsigned lane = lane_id(), wi = threadIdx.x >> 5;
    const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
    for (int64_t cbase = warp * 32; cbase < npieces; cbase += nwarps * 32) {
        const int64_t pi = cbase + lane;
        int len = 0;
        long long beg = 0;
        unsigned tgt = 0, split = 0;
        if (pi < npieces) {
            const uint4 p = pieces[pi];
            const unsigned long long packed = ((unsigned long long)p.y << 32) | p.x;
            len = (int)(packed & ((1ull << kLenBits) - 1));
            beg = (long long)(packed >> kLenBits);
            tgt = p.z;
            split = p.w;
        }
        acc[wi][lane] = 0.0;
        __syncwarp();
        const int incl = warp_incl_scan(len);
        const int E = __shfl_sync(0xffffffffu, incl, 31);
        for (int k0 = 0; k0 < E; k0 += 32) {
            const int k = k0 + (int)lane;
            int pos = 0;
#pragma unroll
            for (int s = 16; s; s >>= 1) {
                const int v = __shfl_sync(0xffffffffu, incl, pos + s - 1);
                if (v <= k) pos += s;
            }
            const int excl = __shfl_sync(0xffffffffu, incl, pos) - __shfl_sync(0xffffffffu, len, pos);
            const long long bL = __shfl_sync(0xffffffffu, beg, pos);
            const bool ok = k < E;
            const int seg = ok ? pos : 32;
            double v = 0.0;
            if (ok) {
                const int64_t e = bL + (k - excl);
                const int32_t s = ld_stream_i32(t_src + e);
                v = A[s];
                if constexpr (!std::is_same<W, NoW>::value) v *= load_w(t_w, e);
            }
            // segmented inclusive scan by piece (fixed order -> deterministic)
            const int prev = __shfl_up_sync(0xffffffffu, seg, 1);
            bool head = lane == 0 || prev != seg;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double u = __shfl_up_sync(0xffffffffu, v, o);
                const int hu = __shfl_up_sync(0xffffffffu, (int)head, o);
                if ((int)lane >= o && !head) {
                    v += u;
                    head = hu != 0;
                }
            }
            const int next = __shfl_down_sync(0xffffffffu, seg, 1);
            const bool tail = lane == 31 || next != seg;
            if (ok && tail) acc[wi][seg] += v;
            __syncwarp();
        }
        if (pi < npieces) {
            const double a = acc[wi][lane];
            if (split) pbuf[pi] = a;
            else F[tgt] += a;
        }
        __syncwarp();
    }
}

__global__ void k_pull_fix(const int4 *__restrict__ fix, int64_t nfix, const double *__restrict__ pbuf,
                           double *__restrict__ F, const Ctrl *__restrict__ ctrl) {
    if (ctrl->done || !ctrl->use_pull) return;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nfix; q += (int64_t)gridDim.x * blockDim.x) {
        const int4 f = fix[q];
        const int64_t p0 = (int64_t)(unsigned)f.y | ((int64_t)f.z << 32);
        double s = 0.0;
        for (int c = 0; c < f.w; ++c) s += pbuf[p0 + c];
        F[f.x] += s;
    }
}

void launch_pull(di_graph *h) {
    DevGraph &g = h->g;
    State &s = h->s;
    DevGraph &pd = g;
    const int grid = h->num_sms * 8;
    if (pd.npieces > 0) {
        switch (g.w_kind) {
        case DI_W_F32:
            k_pull<float><<<grid, kThreads, 0, h->stream>>>(g.t_src, (const float *)g.t_w, s.A, s.F, pd.pieces,
                                                             pd.npieces, pd.pbuf, s.ctrl);
            break;
        case DI_W_F64:
            k_pull<double><<<grid, kThreads, 0, h->stream>>>(g.t_src, (const double *)g.t_w, s.A, s.F, pd.pieces,
                                                              pd.npieces, pd.pbuf, s.ctrl);
            break;
        default:
            k_pull<NoW><<<grid, kThreads, 0, h->stream>>>(g.t_src, nullptr, s.A, s.F, pd.pieces, pd.npieces, pd.pbuf,
                                                           s.ctrl);
        }
        count_launch();
    }
    if (pd.nfix > 0) {
        k_pull_fix<<<(unsigned)std::min<int64_t>((pd.nfix + 255) / 256, 4096), 256, 0, h->stream>>>(pd.fix, pd.nfix,
                                                                                                    pd.pbuf, s.F, s.ctrl);
        count_launch();
    }
}

}  // namespace dit
