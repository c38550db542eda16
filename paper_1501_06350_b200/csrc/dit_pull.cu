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

#include <cub/device/device_radix_sort.cuh>
#include <cstdlib>
#include <mutex>

#include <utility>


namespace dit {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortItems = 16;                       // items per lane
constexpr int kWarpItems = 32 * kSortItems;          // 512 items per warp
constexpr int kSortTile = kWarps * kWarpItems;       // 4096 items per block
constexpr int64_t kPullSplit = 64;     // max in-edges per piece (one thread sums a piece)
constexpr int64_t kPullTile = 2048;    // edges staged in shared memory per pull tile

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

// Pieces: the in-edge range of each target cut at every kPullTile boundary of
// the edge index and after kPullSplit edges, so that every pull tile (edges
// [t kPullTile, (t+1) kPullTile)) is a whole number of pieces.
__device__ __forceinline__ int64_t piece_end(int64_t b, int64_t e) {
    const int64_t tile_end = (b / kPullTile + 1) * kPullTile;
    return min(e, min(b + kPullSplit, tile_end));
}

__global__ void k_piece_count(const int64_t *__restrict__ t_ptr, int64_t n, int64_t *__restrict__ pc) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = t_ptr[j], c = 0;
        const int64_t e = t_ptr[j + 1];
        while (b < e) {
            b = piece_end(b, e);
            ++c;
        }
        pc[j] = c;
    }
}

// piece = { begin<<24 | len, target, split flag }; tile_start[t] = first piece of tile t
__global__ void k_piece_write(const int64_t *__restrict__ t_ptr, int64_t n, const int64_t *__restrict__ po,
                              uint4 *__restrict__ pieces, int4 *__restrict__ fix, unsigned long long *__restrict__ nfix,
                              int64_t *__restrict__ tile_start) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = t_ptr[j + 1];
        const int64_t np = po[j + 1] - po[j];
        const bool split = np > 1;
        int64_t b = t_ptr[j];
        for (int64_t c = 0; c < np; ++c) {
            const int64_t pe = piece_end(b, e);
            const unsigned long long packed = ((unsigned long long)b << kLenBits) | (unsigned long long)(pe - b);
            pieces[po[j] + c] = make_uint4((unsigned)packed, (unsigned)(packed >> 32), (unsigned)j, split ? 1u : 0u);
            if (b % kPullTile == 0) tile_start[b / kPullTile] = po[j] + c;
            b = pe;
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

// Stable LSD radix sort of (keys, u32 values) on the low `bits` bits of the
// keys; k1/v1 are scratch of the same size.  Returns the buffers holding the
// result (either the inputs or the scratch).
std::pair<uint32_t *, uint32_t *> radix_sort_u32(uint32_t *k0, uint32_t *v0, uint32_t *k1, uint32_t *v1,
                                                 int64_t count, int bits, cudaStream_t st) {
    if (count <= 0) return {k0, v0};
    const int64_t ntiles = (count + kSortTile - 1) / kSortTile;
    int64_t *hc, *ho;
    DI_CUDA(cudaMallocAsync(&hc, (int64_t)kRadix * ntiles * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&ho, ((int64_t)kRadix * ntiles + 1) * sizeof(int64_t), st));
    for (int shift = 0; shift < bits; shift += kRadixBits) {
        radix_sort_pass_launch(k0, v0, k1, v1, count, shift, ntiles, hc, ho, false, st);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    DI_CUDA(cudaFreeAsync(hc, st));
    DI_CUDA(cudaFreeAsync(ho, st));
    return {k0, v0};
}

// the same with u64 values (the tile plan's packed {source, weight} payloads)
std::pair<uint32_t *, uint64_t *> radix_sort_u32_u64(uint32_t *k0, uint64_t *v0, uint32_t *k1, uint64_t *v1,
                                                     int64_t count, int bits, cudaStream_t st) {
    if (count <= 0) return {k0, v0};
    const int64_t ntiles = (count + kSortTile - 1) / kSortTile;
    int64_t *hc, *ho;
    DI_CUDA(cudaMallocAsync(&hc, (int64_t)kRadix * ntiles * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&ho, ((int64_t)kRadix * ntiles + 1) * sizeof(int64_t), st));
    for (int shift = 0; shift < bits; shift += kRadixBits) {
        radix_sort_pass_launch(k0, v0, k1, v1, count, shift, ntiles, hc, ho, true, st);
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    DI_CUDA(cudaFreeAsync(hc, st));
    DI_CUDA(cudaFreeAsync(ho, st));
    return {k0, v0};
}

// Work plan of a CSC (pieces, tiles, split-target fixups) for k_pull.
void build_plan_pieces(di_graph *h, PullPlan &pd) {
    cudaStream_t st = h->stream;
    const int64_t nt = pd.nt, m = pd.m;
    int64_t *pc, *po;
    DI_CUDA(cudaMallocAsync(&pc, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&po, (nt + 1) * sizeof(int64_t), st));
    const int grid = h->num_sms * 8;
    if (nt > 0) {
        k_piece_count<<<grid, kThreads, 0, st>>>(pd.ptr, nt, pc);
        count_launch();
    }
    exclusive_scan_i64(pc, po, nt, st);
    int64_t np = 0;
    DI_CUDA(cudaMemcpyAsync(&np, po + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    pd.npieces = np;
    DI_CUDA(cudaMallocAsync(&pd.pieces, (np > 0 ? np : 1) * sizeof(uint4), st));
    DI_CUDA(cudaMallocAsync(&pd.pbuf, (np > 0 ? np : 1) * sizeof(double), st));
    DI_CUDA(cudaMallocAsync(&pd.fix, (nt > 0 ? nt : 1) * sizeof(int4), st));
    pd.ntiles = (m + kPullTile - 1) / kPullTile;
    DI_CUDA(cudaMallocAsync(&pd.tile_start, (pd.ntiles + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemcpyAsync(pd.tile_start + pd.ntiles, &pd.npieces, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    unsigned long long *nf;
    DI_CUDA(cudaMallocAsync(&nf, sizeof(unsigned long long), st));
    DI_CUDA(cudaMemsetAsync(nf, 0, sizeof(unsigned long long), st));
    if (nt > 0) {
        k_piece_write<<<grid, kThreads, 0, st>>>(pd.ptr, nt, po, pd.pieces, pd.fix, nf, pd.tile_start);
        count_launch();
    }
    unsigned long long nfix = 0;
    DI_CUDA(cudaMemcpyAsync(&nfix, nf, sizeof(nfix), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaFreeAsync(nf, st));
    DI_CUDA(cudaFreeAsync(pc, st));
    DI_CUDA(cudaFreeAsync(po, st));
    DI_CUDA(cudaStreamSynchronize(st));
    pd.nfix = (int64_t)nfix;
    pd.pieces_built = true;
}

void free_plan(PullPlan &p, cudaStream_t st) {
    for (void *q : {(void *)p.ptr, (void *)p.src, p.w, (void *)p.pieces, (void *)p.fix, (void *)p.pbuf,
                    (void *)p.tile_start})
        if (q) cudaFreeAsync(q, st);
    p = PullPlan();
}

// sort payload (source id, f32 weight bits) of every edge, keys = targets
__global__ void k_pack_keys(const int32_t *__restrict__ col, const int32_t *__restrict__ esrc,
                            const float *__restrict__ w, int64_t m, uint32_t *__restrict__ keys,
                            unsigned long long *__restrict__ vals) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        keys[e] = (uint32_t)col[e];
        vals[e] = ((unsigned long long)(uint32_t)esrc[e] << 32) | (w ? __float_as_uint(w[e]) : 0u);
    }
}

__global__ void k_unpack_t(const unsigned long long *__restrict__ vals, int64_t m, int32_t *__restrict__ src,
                           float *__restrict__ w) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long v = vals[k];
        src[k] = (int32_t)(v >> 32);
        if (w) w[k] = __uint_as_float((uint32_t)v);
    }
}

// CUB's sort scratch: one buffer per device kept for the process (grown on demand,
// outside the stream-ordered pool so the builders' temporaries keep a stable
// layout there; a cudaMalloc / cudaFree pair per build cost up to 0.6 s when the
// driver had to make room).
// slot 0: CUB scratch; slot 1: the packed transpose's sort buffers
static void *g_cub_buf[2][64] = {};
static size_t g_cub_cap[2][64] = {};

void release_cub_scratch(int device) {
    if (device < 0 || device >= 64) return;
    std::lock_guard<std::mutex> lock(scratch_mutex(device));   // no build on this device uses it meanwhile
    for (int sl = 0; sl < 2; ++sl) {
        if (g_cub_buf[sl][device]) cudaFree(g_cub_buf[sl][device]);
        g_cub_buf[sl][device] = nullptr;
        g_cub_cap[sl][device] = 0;
    }
}

static void *cached_scratch(int slot, int device, size_t bytes) {
    void **buf = g_cub_buf[slot];
    size_t *cap = g_cub_cap[slot];
    if (device < 0 || device >= 64) device = 0;
    if (bytes > cap[device]) {
        if (buf[device]) DI_CUDA(cudaFree(buf[device]));
        buf[device] = nullptr;
        cap[device] = 0;
        DI_CUDA(cudaMalloc(&buf[device], bytes));
        cap[device] = bytes;
    }
    return buf[device];
}

void *cub_scratch(int device, size_t bytes) { return cached_scratch(0, device, bytes); }

std::mutex &scratch_mutex(int device) {
    static std::mutex mu[64];
    return mu[(device >= 0 && device < 64) ? device : 0];
}

// Transpose with the sources and f32 weights riding in the sort (CUB, m < 2^31):
// no gather through the permutation afterwards.
static void build_transpose_packed(di_graph *h, int64_t *cnt) {
    DevGraph &g = h->g;
    PullPlan &T = g.t;
    cudaStream_t st = h->stream;
    const int64_t n = g.n, m = g.m, nt = g.nt;
    const int grid = h->num_sms * 8;
    // the four sort buffers: one block cached per device outside the pool (a 24 GB
    // request at configs[2]; from the pool it sometimes cost 20-50 ms of mapping).
    // Builds on one device take turns on it (and on the CUB scratch).
    const size_t mv = ((size_t)m * 8 + 255) & ~(size_t)255, mk = ((size_t)m * 4 + 255) & ~(size_t)255;
    std::lock_guard<std::mutex> lock(scratch_mutex(h->device));
    unsigned char *blk = (unsigned char *)cached_scratch(1, h->device, 2 * mv + 2 * mk);
    unsigned long long *v0 = (unsigned long long *)blk, *v1 = (unsigned long long *)(blk + mv);
    uint32_t *k0 = (uint32_t *)(blk + 2 * mv), *k1 = (uint32_t *)(blk + 2 * mv + mk);
    int32_t *esrc = (int32_t *)k1;                   // the second key buffer is free until the sort
    k_edge_src<<<grid, kThreads, 0, st>>>(g.row_ptr, n, esrc);
    k_pack_keys<<<grid, kThreads, 0, st>>>(g.col, esrc, (const float *)g.w, m, k0, v0);
    count_launch(2);
    phase_mark(st, "transpose: pack");
    int bits = 1;
    while (bits < 31 && ((int64_t)1 << bits) < nt) ++bits;
    cub::DoubleBuffer<uint32_t> kb(k0, k1);
    cub::DoubleBuffer<unsigned long long> vb(v0, v1);
    size_t tmp_bytes = 0;
    DI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, (int)m, 0, bits, st));
    DI_CUDA(cub::DeviceRadixSort::SortPairs(cub_scratch(h->device, tmp_bytes), tmp_bytes, kb, vb, (int)m, 0, bits, st));
    phase_mark(st, "transpose: radix sort");
    k_run_bounds<<<grid, kThreads, 0, st>>>(kb.Current(), m, cnt);
    k_unpack_t<<<grid, kThreads, 0, st>>>(vb.Current(), m, T.src, (float *)T.w);
    count_launch(2);
    DI_CUDA(cudaStreamSynchronize(st));              // the block is free for the next build
}

void build_transpose(di_graph *h) {
    DevGraph &g = h->g;
    PullPlan &T = g.t;
    if (T.built) return;
    cudaStream_t st = h->stream;
    const int64_t n = g.n, m = g.m, nt = g.nt;   // rows = owned sources, targets = fluid slots
    T.nt = nt;
    T.m = m;
    const bool wide = m >= (int64_t)0xffffffffLL;
    const size_t vsz = wide ? 8 : 4;
    DI_CUDA(cudaMallocAsync(&T.ptr, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&T.src, (m > 0 ? m : 1) * sizeof(int32_t), st));
    const size_t wsz = g.w_kind == DI_W_F32 ? 4 : (g.w_kind == DI_W_F64 ? 8 : 0);
    if (wsz) DI_CUDA(cudaMallocAsync(&T.w, (m > 0 ? m : 1) * wsz, st));
    int64_t *cnt = nullptr;
    DI_CUDA(cudaMallocAsync(&cnt, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemsetAsync(cnt, 0, (nt + 1) * sizeof(int64_t), st));
    if (m > 0 && m < (int64_t)0x7fffffff && g.w_kind != DI_W_F64 && !getenv("DIT_OWN_RADIX") &&
        !getenv("DIT_TRANSPOSE_GATHER")) {
        build_transpose_packed(h, cnt);
    } else if (m > 0) {
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
        int bits = 1;
        while (bits < 31 && ((int64_t)1 << bits) < nt) ++bits;
        if (m < (int64_t)0x7fffffff && !getenv("DIT_OWN_RADIX")) {
            // graph-builder plumbing: the toolkit's (CUB) stable radix sort of the edge
            // indices by target -- the sweep kernels are all our own
            cub::DoubleBuffer<uint32_t> kb(k0, k1);
            cub::DoubleBuffer<uint32_t> vb((uint32_t *)v0, (uint32_t *)v1);
            size_t tmp_bytes = 0;
            DI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, (int)m, 0, bits, st));
            {
                std::lock_guard<std::mutex> lock(scratch_mutex(h->device));
                DI_CUDA(cub::DeviceRadixSort::SortPairs(cub_scratch(h->device, tmp_bytes), tmp_bytes, kb, vb, (int)m,
                                                        0, bits, st));
                DI_CUDA(cudaStreamSynchronize(st));
            }
            if (kb.Current() != k0) {
                std::swap(k0, k1);
                std::swap(v0, v1);
            }
        } else {
            const int64_t ntiles = (m + kSortTile - 1) / kSortTile;
            int64_t *hc, *ho;
            DI_CUDA(cudaMallocAsync(&hc, (int64_t)kRadix * ntiles * sizeof(int64_t), st));
            DI_CUDA(cudaMallocAsync(&ho, ((int64_t)kRadix * ntiles + 1) * sizeof(int64_t), st));
            for (int shift = 0; shift < bits; shift += kRadixBits) {
                radix_sort_pass_launch(k0, v0, k1, v1, m, shift, ntiles, hc, ho, wide, st);
                std::swap(k0, k1);
                std::swap(v0, v1);
            }
            DI_CUDA(cudaFreeAsync(hc, st));
            DI_CUDA(cudaFreeAsync(ho, st));
        }
        // in-degrees -> ptr
        phase_mark(st, "transpose: radix sort");
        k_run_bounds<<<grid, kThreads, 0, st>>>(k0, m, cnt);
        count_launch();
        DI_CUDA(cudaMallocAsync(&esrc, m * 4, st));
        k_edge_src<<<grid, kThreads, 0, st>>>(g.row_ptr, n, esrc);
        count_launch();
        if (wide) {
            if (g.w_kind == DI_W_F64)
                k_gather_t<uint64_t, double><<<grid, kThreads, 0, st>>>((const uint64_t *)v0, m, esrc, (const double *)g.w, T.src, (double *)T.w);
            else
                k_gather_t<uint64_t, float><<<grid, kThreads, 0, st>>>((const uint64_t *)v0, m, esrc, (const float *)g.w, T.src, (float *)T.w);
        } else {
            if (g.w_kind == DI_W_F64)
                k_gather_t<uint32_t, double><<<grid, kThreads, 0, st>>>((const uint32_t *)v0, m, esrc, (const double *)g.w, T.src, (double *)T.w);
            else
                k_gather_t<uint32_t, float><<<grid, kThreads, 0, st>>>((const uint32_t *)v0, m, esrc, (const float *)g.w, T.src, (float *)T.w);
        }
        count_launch();
        DI_CUDA(cudaFreeAsync(esrc, st));
        DI_CUDA(cudaFreeAsync(k0, st));
        DI_CUDA(cudaFreeAsync(k1, st));
        DI_CUDA(cudaFreeAsync(v0, st));
        DI_CUDA(cudaFreeAsync(v1, st));
    }

    phase_mark(st, "transpose: gather");    exclusive_scan_i64(cnt, T.ptr, nt, st);
    DI_CUDA(cudaFreeAsync(cnt, st));
    T.built = true;                      // the pull work plan follows on first use (build_plan_pieces)
}

// ---------------------------------------------------------------- pull sweep
// One CTA per tile of kPullTile consecutive in-edges (grid-stride):
//   phase 1: v_e = A(src_e) w_e for the tile's edges -> shared memory
//            (coalesced index/weight streams, gathers of A, no shuffles)
//   phase 2: one thread per piece sums its slice of v in edge order and adds
//            it to F(target), or parks it in pbuf for targets cut into pieces.
// Fixed summation order everywhere: bitwise reproducible on a given graph.
template <typename W>
__global__ void __launch_bounds__(kThreads) k_pull(const int32_t *__restrict__ t_src, const W *__restrict__ t_w,
                                                   const double *__restrict__ A, double *__restrict__ F,
                                                   const uint4 *__restrict__ pieces,
                                                   const int64_t *__restrict__ tile_start, int64_t ntiles, int64_t m,
                                                   double *__restrict__ pbuf, const Ctrl *__restrict__ ctrl,
                                                   int want) {
    __shared__ double vals[kPullTile];
    if (ctrl->done || ctrl->use_pull != want) return;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t e0 = t * kPullTile;
        const int cnt = (int)min((int64_t)kPullTile, m - e0);
#pragma unroll 8
        for (int k = threadIdx.x; k < cnt; k += kThreads) {
            const int64_t e = e0 + k;
            double v = A[ld_stream_i32(t_src + e)];
            if constexpr (!std::is_same<W, NoW>::value) v *= load_w(t_w, e);
            vals[k] = v;
        }
        __syncthreads();
        const int64_t p1 = tile_start[t + 1];
        for (int64_t p = tile_start[t] + threadIdx.x; p < p1; p += kThreads) {
            const uint4 pc = pieces[p];
            const unsigned long long packed = ((unsigned long long)pc.y << 32) | pc.x;
            const int len = (int)(packed & ((1ull << kLenBits) - 1));
            const int off = (int)((int64_t)(packed >> kLenBits) - e0);
            double s = 0.0;
            for (int k = 0; k < len; ++k) s += vals[off + k];
            if (pc.w) pbuf[p] = s;
            else F[pc.z] += s;
        }
        __syncthreads();
    }
}

// Targets cut into several pieces.  A warp takes 32 fix entries: entries with
// fewer than 32 pieces are summed by their own lane (in piece order), the
// others by the whole warp (lane-strided, then a fixed butterfly).  Every sum
// has a fixed order: deterministic.
__global__ void k_pull_fix(const int4 *__restrict__ fix, int64_t nfix, const double *__restrict__ pbuf,
                           double *__restrict__ F, const Ctrl *__restrict__ ctrl, int want) {
    if (ctrl->done || ctrl->use_pull != want) return;
    const unsigned lane = lane_id();
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32; base < nfix; base += nw * 32) {
        const int64_t q = base + lane;
        int4 f = make_int4(0, 0, 0, 0);
        if (q < nfix) f = fix[q];
        const int64_t p0 = (int64_t)(unsigned)f.y | ((int64_t)f.z << 32);
        if (f.w > 0 && f.w < 32) {
            double s = 0.0;
            for (int c = 0; c < f.w; ++c) s += pbuf[p0 + c];
            F[f.x] += s;
        }
        unsigned big = __ballot_sync(0xffffffffu, f.w >= 32);
        while (big) {
            const int b = __ffs(big) - 1;
            big &= big - 1;
            const int j = __shfl_sync(0xffffffffu, f.x, b);
            const int np = __shfl_sync(0xffffffffu, f.w, b);
            const int64_t pb = __shfl_sync(0xffffffffu, p0, b);
            double s = 0.0;
            for (int c = (int)lane; c < np; c += 32) s += pbuf[pb + c];
            s = warp_sum(s);
            if (lane == 0) F[j] += s;
        }
    }
}

void launch_pull_plan(di_graph *h, const PullPlan &pd, const double *A, int want) {
    DevGraph &g = h->g;
    State &s = h->s;
    if (pd.ntiles > 0) {
        const unsigned grid = (unsigned)std::min<int64_t>(pd.ntiles, (int64_t)h->num_sms * 8);
        switch (g.w_kind) {
        case DI_W_F32:
            k_pull<float><<<grid, kThreads, 0, h->stream>>>(pd.src, (const float *)pd.w, A, s.F, pd.pieces,
                                                             pd.tile_start, pd.ntiles, pd.m, pd.pbuf, s.ctrl, want);
            break;
        case DI_W_F64:
            k_pull<double><<<grid, kThreads, 0, h->stream>>>(pd.src, (const double *)pd.w, A, s.F, pd.pieces,
                                                              pd.tile_start, pd.ntiles, pd.m, pd.pbuf, s.ctrl, want);
            break;
        default:
            k_pull<NoW><<<grid, kThreads, 0, h->stream>>>(pd.src, nullptr, A, s.F, pd.pieces, pd.tile_start,
                                                           pd.ntiles, pd.m, pd.pbuf, s.ctrl, want);
        }
        count_launch();
    }
    if (pd.nfix > 0) {
        k_pull_fix<<<(unsigned)std::min<int64_t>((pd.nfix + 255) / 256, (int64_t)h->num_sms * 8), 256, 0, h->stream>>>(
            pd.fix, pd.nfix, pd.pbuf, s.F, s.ctrl, want);
        count_launch();
    }
}

void launch_pull(di_graph *h) { launch_pull_plan(h, h->g.t, h->s.A, kUsePull); }

}  // namespace dit
