// dit_tile.cu -- the tile-local D-Iteration sweep (reading R12, §5).
//
// PAPER §3.4: DI converges for any fair diffusion sequence ("one strength of
// D-Iteration is the freedom in the choice of a scheduler").  This schedule
// exploits the locality of web graphs (most links stay inside a site) and the
// SM's shared memory.  Node ids are cut into tiles of kNodeTile; per sweep:
//
//   1. every tile first takes in the remote pushes of the previous sweep
//      (F(t) += d D(i) P_{t,i} for i outside t's tile, Eq. (8) being linear in
//      the diffused amount D);
//   2. then runs `rounds` Jacobi diffusion rounds over its LOCAL in-edges
//      (source and target in the tile) in shared memory: every node holding
//      fluid is diffused (Eqs. (8), (10)), local pushes applied at once;
//   3. writes F (what is left in the tile) and H += D, and emits the remote
//      pushes d D(i) P_{t,i} of its sources.
//
// Step 1 of sweep k+1 completes the remote pushes of sweep k, so the sequence
// of Eq. (8) updates is exactly the oracle's (orc_tiled_sweep_run: rounds in
// every tile, then the remote pushes).  The stop test after sweep k uses
// |F|_1 = sum_t |f_t| + sum_i |d D(i)| wr(i) (wr = share of i's out-weight whose
// pushes are still pending): exact for non-negative fluid, an upper bound for
// signed fluid (§3.5), so stopping on it keeps Theorem 1's guarantee; after the
// last sweep the pending pushes are flushed into F and the exact |F|_1 taken.
//
// Remote pushes are gathered by their targets.  Light targets (few remote
// in-edges) are gathered inside the tile kernel from the previous sweep's
// outflow A(i) = d D(i) inv(i), over {source, weight} records staged by TMA.
// Heavy targets' in-edges are sorted by (source stripe, target, source) and
// gathered stripe by stripe, so that the slice of A being read stays in L2
// (a random 8-byte read from HBM costs a 64-byte DRAM access on B200).
//
// Kernels (B200): k_tile -- one 512-thread CTA per tile, 2 CTAs per SM; the
// tile's per-node state, piece layout and light records staged by TMA bulk
// copies (cp.async.bulk + mbarrier, double-buffered), its local edges
// (sliced-ELL, runs of four slots per lane) prefetched into L2 and read
// through L1 by the rounds (staged in shared memory too with one 1024-thread
// CTA per SM, DIT_TILE_BLOCK=1024).  k_heavy_s -- per stripe: CTA per
// 2048-edge chunk, warp per segment; then the stripe's runs folded into
// hsum in stripe order.  Every summation has a fixed order: bitwise
// reproducible run to run.
#include "dit_internal.cuh"

#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace dit {

constexpr int kTileThreads = (int)kNodeTile;     // build kernels: thread i owns node i of the tile
// k_tile: one 1024-thread CTA per SM, 16 round warps (thread i owns node i) and
// 16 prep warps (the next tile's inflow)
constexpr int kRW = (int)kNodeTile;
constexpr int kPWt = (int)kNodeTile / 2;           // two nodes per prep thread
constexpr int kPN = (int)kNodeTile / kPWt;
constexpr int kTileBlock = kRW + kPWt;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kVRows = 2 * (int)kNodeTile;       // local-edge pieces per tile (at most)
constexpr int kVWarps = kVRows / 32;             // virtual warps: round warp w runs w and kVWarps-1-w
constexpr int kVofsStride = 36;                  // u32 per tile (kVWarps + 1, padded to 16 B)
constexpr int kVfStride = 520;                   // u16 per tile (kNodeTile + 1, padded to 16 B)
constexpr int kMetaBytes = kVofsStride * 4 + kVfStride * 2 + kVRows * 2;   // per-tile layout, TMA-staged
constexpr int64_t kGqSlots = kNodeTile + 16;     // outflow per node + one zero slot per bank pair (ELL padding)
constexpr int kTileSmemBudget = 227 * 1024 - 2048;   // dynamic shared memory of k_tile (static arrays aside)
static_assert(kVWarps == 2 * kTileWarps, "two virtual warps per round warp");

template <typename W>
using StoreW = typename std::conditional<std::is_same<W, NoW>::value, float, W>::type;

// sliced-ELL slot groups: the first K - K % 4 slots of a lane sit in runs of four
// (one 8-byte source load, one 16-byte weight load), the rest one per row of 32
constexpr int kSlotGroup = 4;
// offset of slot s of lane `lane` in a virtual warp of K slots per lane
__host__ __device__ __forceinline__ int64_t ell_slot(int64_t s, int lane, int64_t K) {
    const int64_t Kg = K - K % kSlotGroup;
    return s < Kg ? 32 * kSlotGroup * (s / kSlotGroup) + kSlotGroup * lane + (s % kSlotGroup) : 32 * s + lane;
}

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

// Shared memory of k_tile (one CTA per SM, everything double-buffered by tile
// parity): gq / psum of the rounds, the prepared per-node rows P, the light
// records R (prep warps) and the edge bundles E = {layout, staged slots} (round warps).
struct PrepRow {
    double f, ivi, H;        // inflow-completed fluid, 1/sum w, history
    float wr;                // pending share of the out-weight (R13)
    int32_t deg;             // out-degree
};
static_assert(sizeof(PrepRow) == 32, "32-byte prepared rows");
constexpr int kOffPsum = ((int)kGqSlots * 8 + 127) & ~127;
constexpr int kOffP = kOffPsum + kVRows * 8;
constexpr int kOffR = kOffP + 2 * (int)kNodeTile * (int)sizeof(PrepRow);
template <typename W>
constexpr int tile_rec_buf() { return (((int)kLightCap * (int)sizeof(RemRec<W>) + 32) + 127) & ~127; }
template <typename W>
constexpr int tile_off_e() { return kOffR + 2 * tile_rec_buf<W>(); }
template <typename W>
constexpr int tile_e_buf() { return ((kTileSmemBudget - tile_off_e<W>()) / 2) & ~127; }
template <typename W>
constexpr int tile_smem_bytes() { return tile_off_e<W>() + 2 * tile_e_buf<W>(); }
static_assert(kOffP % 16 == 0 && kOffR % 128 == 0 && kMetaBytes % 16 == 0, "aligned shared buffers");

#ifndef DIT_STRIPE_MB
#define DIT_STRIPE_MB 48
#endif
constexpr int64_t kStripeBytes = (int64_t)DIT_STRIPE_MB << 20;   // outflow slice per heavy stripe (L2-resident)
#ifndef DIT_TILE_WAVES
#define DIT_TILE_WAVES 2
#endif
constexpr int kTileWaves = DIT_TILE_WAVES;      // tile waves per sweep (R15), single GPU
__device__ __forceinline__ int tile_wave(int64_t node, int waves) { return (int)((node / kNodeTile) % waves); }

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
    for (long long spin = 0; !mbar_try_wait(bar, phase); ++spin) {
        if (spin > 8) __nanosleep(64);               // long waits: leave the issue slots to others
        if (spin > (1ll << 26)) __trap();
    }
}
// bulk global -> shared copy (the TMA engine), completion counted on `bar`
__device__ __forceinline__ void tma_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

// bulk prefetch of a global range into L2 (the TMA engine; no completion tracking)
__device__ __forceinline__ void tma_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------- build
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

// shard ghost slots: heavy targets whose sums leave through the all-to-all
__global__ void k_classify_ghosts(const int64_t *__restrict__ rc, int64_t n, int64_t nt, int64_t *__restrict__ lrc,
                                  int64_t *__restrict__ hc, int64_t *__restrict__ hflag) {
    for (int64_t t = n + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
        lrc[t] = 0;
        hc[t] = rc[t];
        hflag[t] = rc[t] > 0;
    }
}

// balanced sliced-ELL layout of a tile's local in-edges: CTA per tile
// 512-thread block reductions for the layout kernel (fixed order: deterministic)
__device__ __forceinline__ int64_t block_sum_512(int64_t v, int64_t *red) {
    v = warp_sum(v);
    if (lane_id() == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t s = 0;
    for (int w = 0; w < (int)kNodeTile / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}
__device__ __forceinline__ int block_exscan_512(int v, int *sc) {
    const int lane = (int)lane_id(), w = (int)(threadIdx.x >> 5);
    int x = v;                                       // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sc[w] = x;
    __syncthreads();
    int base = 0;
    for (int q = 0; q < w; ++q) base += sc[q];
    __syncthreads();
    return base + x - v;
}

__global__ void __launch_bounds__(kTileThreads) k_tile_layout(const int64_t *__restrict__ lc, int64_t n,
                                                               int64_t ntile, int eb, int64_t stage_cap,
                                                               uint32_t *__restrict__ vofs,
                                                               uint16_t *__restrict__ vfirst,
                                                               uint16_t *__restrict__ plist, int32_t *__restrict__ vcap,
                                                               int64_t *__restrict__ pcnt, int32_t *__restrict__ lstage) {
    __shared__ int64_t d_s[kNodeTile];
    __shared__ int32_t len_s[kVRows], lenr_s[kVRows];
    __shared__ uint16_t vf_s[kNodeTile + 1], rank_s[kVRows];
    __shared__ int s_V;
    __shared__ int64_t s_red[kNodeTile / 32 + 1];
    __shared__ int s_scan[kNodeTile / 32 + 1];
    const int k = threadIdx.x;
    for (int64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
        const int64_t a0 = t * kNodeTile;
        const int nn = (int)min(kNodeTile, n - a0);
        const int64_t dk = k < nn ? lc[a0 + k] : 0;
        d_s[k] = dk;
        // cap: at most kVRows pieces (E / cap + nonzero rows <= kVRows); block sums
        const int64_t E = block_sum_512(dk, s_red), nz = block_sum_512((int64_t)(dk > 0), s_red);
        const int64_t cap = nz ? std::max<int64_t>(1, (E + (kVRows - nz) - 1) / (kVRows - nz)) : 1;
        // node k's pieces: its slots in node order (exclusive scan of the piece counts)
        const int np = (int)((dk + cap - 1) / cap);
        const int first = block_exscan_512(np, s_scan);
        vf_s[k] = (uint16_t)first;
        for (int q = 0; q < np; ++q) len_s[first + q] = (int32_t)min(cap, dk - (int64_t)q * cap);
        if (k == kNodeTile - 1) {
            vf_s[kNodeTile] = (uint16_t)(first + np);
            s_V = first + np;
            vcap[t] = (int32_t)cap;
        }
        __syncthreads();
        const int V = s_V;
        for (int p = k; p < V; p += kTileThreads) {   // rank: longest first, ties by piece order
            const int lp = len_s[p];
            int r = 0;
            for (int q = 0; q < V; ++q) {
                const int lq = len_s[q];
                r += (lq > lp) || (lq == lp && q < p);
            }
            rank_s[p] = (uint16_t)r;
            lenr_s[r] = lp;
        }
        __syncthreads();
        for (int p = k; p < kVRows; p += kTileThreads) plist[t * kVRows + p] = p < V ? rank_s[p] : 0;
        for (int i = k; i < kVfStride; i += kTileThreads) vfirst[t * kVfStride + i] = vf_s[min(i, (int)kNodeTile)];
        if (k == 0) {
            uint32_t off = 0;
            for (int vw = 0; vw < kVWarps; ++vw) {
                vofs[t * kVofsStride + vw] = off;
                off += 32u * (uint32_t)(32 * vw < V ? lenr_s[32 * vw] : 0);   // the virtual warp's longest piece
            }
            for (int vw = kVWarps; vw < kVofsStride; ++vw) vofs[t * kVofsStride + vw] = off;
            pcnt[t] = off;
            // shared-memory staging (k_tile): the longest suffix of virtual warps whose
            // slots (eb bytes each) fit the edge buffer; the others are read from L2
            int v = 0;
            while (v < kVWarps && (int64_t)(off - vofs[t * kVofsStride + v]) * eb > stage_cap) ++v;
            lstage[t] = (int32_t)(v < kVWarps ? vofs[t * kVofsStride + v] : off);
        }
        __syncthreads();
    }
}

// light offsets relative to the tile, tile bases, heavy index, out-degree
__global__ void k_tile_rel(const int64_t *__restrict__ rptr, const int64_t *__restrict__ hpos,
                           const int64_t *__restrict__ hflag, const int64_t *__restrict__ row_ptr, int64_t n,
                           int64_t nt, int64_t ntile, uint32_t *__restrict__ rrel, int32_t *__restrict__ hidx,
                           int32_t *__restrict__ deg, int64_t *__restrict__ rtile) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j <= nt; j += (int64_t)gridDim.x * blockDim.x) {
        if (j < nt) hidx[j] = hflag[j] ? (int32_t)hpos[j] : -1;
        if (j < n) {
            const int64_t b = (j / kNodeTile) * kNodeTile;
            rrel[j] = (uint32_t)(rptr[j] - rptr[b]);
            deg[j] = (int32_t)(row_ptr[j + 1] - row_ptr[j]);
        }
        if (j <= n && (j % kNodeTile == 0 || j == n)) {
            const int64_t t = (j + kNodeTile - 1) / kNodeTile;   // j == n: the end of the last tile
            if (t <= ntile) rtile[t] = rptr[j];
        }
    }
}

template <typename W>
__global__ void k_fill_pad(uint16_t *__restrict__ lsrc, StoreW<W> *__restrict__ lw, int64_t cnt) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
        lsrc[e] = (uint16_t)kNodeTile;     // the always-zero outflow slot
        if (lw) lw[e] = StoreW<W>(0);
    }
}

// ---- edge-parallel plan build (hub targets with millions of in-edges must not
// serialise on one warp): target of every CSC position, local flags, their
// exclusive scan L, so that a local in-edge's rank within its target is
// L[k] - L[tptr[t]] and a remote one's (k - tptr[t]) minus that.
__global__ void k_fill_tkey(const int64_t *__restrict__ tptr, int64_t nt, uint32_t *__restrict__ tkey) {
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < nt; t += nw)
        for (int64_t k = tptr[t] + lane_id(); k < tptr[t + 1]; k += 32) tkey[k] = (uint32_t)t;
}

template <typename LT>
__global__ void k_local_flags(const uint32_t *__restrict__ tkey, const int32_t *__restrict__ tsrc, int64_t m,
                              int64_t n, LT *__restrict__ flag) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= m; k += (int64_t)gridDim.x * blockDim.x) {
        if (k == m) {
            flag[k] = 0;
            continue;
        }
        const int64_t t = tkey[k];
        flag[k] = (t < n && tsrc[k] / kNodeTile == t / kNodeTile) ? 1 : 0;
    }
}

template <typename LT>
__global__ void k_counts_from_scan(const int64_t *__restrict__ tptr, const LT *__restrict__ L, int64_t nt,
                                   int64_t *__restrict__ lc, int64_t *__restrict__ rc) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = tptr[t], e = tptr[t + 1];
        lc[t] = L[e] - L[b];
        rc[t] = (e - b) - lc[t];
    }
}

// every in-edge to its class, one thread per CSC position (see k_split_edges)
template <typename W, typename LT>
__global__ void k_split_flat(const int64_t *__restrict__ tptr, const uint32_t *__restrict__ tkey,
                             const int32_t *__restrict__ tsrc, const StoreW<W> *__restrict__ tw,
                             const LT *__restrict__ L, int64_t m, int64_t n, const int64_t *__restrict__ ltile,
                             const uint32_t *__restrict__ vofs, const uint16_t *__restrict__ vfirst,
                             const uint16_t *__restrict__ plist, const int32_t *__restrict__ vcap,
                             const int64_t *__restrict__ rptr, const int64_t *__restrict__ hptr,
                             const int32_t *__restrict__ hidx, int64_t stripe_nodes, int64_t nstripe, int waves,
                             uint16_t *__restrict__ lsrc, StoreW<W> *__restrict__ lw, RemRec<W> *__restrict__ rrec,
                             RemRec<W> *__restrict__ htmp, uint32_t *__restrict__ hkey, uint32_t *__restrict__ hval,
                             uint32_t *__restrict__ hof) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = tkey[k];
        const int32_t s = tsrc[k];
        const int64_t b = tptr[t];
        const int64_t lrank = (int64_t)(L[k] - L[b]);
        const bool owned = t < n;
        const int64_t tile = owned ? t / kNodeTile : -1;
        if (owned && s / kNodeTile == tile) {
            // balanced sliced-ELL: local in-edge q of t is slot q % cap of its piece q / cap
            const int64_t cap = vcap[tile];
            const int pf = vfirst[tile * kVfStride + (t - tile * kNodeTile)];
            const int r = plist[tile * kVRows + pf + (int)(lrank / cap)];
            const uint32_t v0 = vofs[tile * kVofsStride + r / 32], v1 = vofs[tile * kVofsStride + r / 32 + 1];
            const int64_t o = ltile[tile] + v0 + ell_slot(lrank % cap, r % 32, (v1 - v0) / 32);
            lsrc[o] = (uint16_t)(s - tile * kNodeTile);
            if constexpr (kW) lw[o] = tw[k];
        } else {
            const int32_t hx = hidx[t];
            const int64_t o = (hx >= 0 ? hptr[t] : rptr[t]) + (k - b) - lrank;
            RemRec<W> r{};
            r.src = s;
            if constexpr (kW) r.w = tw[k];
            else r.w = 1.0f;
            if (hx >= 0) {
                htmp[o] = r;
                // heavy edges grouped by (wave of the target, stripe of the source)
                hkey[o] = (uint32_t)((owned ? tile_wave(t, waves) : 0) * nstripe + s / stripe_nodes);
                hval[o] = (uint32_t)o;
                hof[o] = (uint32_t)hx;
            } else {
                rrec[o] = r;
            }
        }
    }
}

// heavy edges in (stripe, target, source) order: records, stripe and target of each
template <typename W>
__global__ void k_heavy_gather(const uint32_t *__restrict__ skey, const uint32_t *__restrict__ sval, int64_t mh,
                               const RemRec<W> *__restrict__ htmp, const uint32_t *__restrict__ hof,
                               RemRec<W> *__restrict__ hrec, uint32_t *__restrict__ hh) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t q = sval[p];
        hrec[p] = htmp[q];
        hh[p] = hof[q];
    }
}

// run / segment / chunk flags: run = (stripe, target); chunk = 2048 edges from
// the stripe's start; segment = run cut at chunk starts
__global__ void k_heavy_flags(const uint32_t *__restrict__ st, const uint32_t *__restrict__ hh, int64_t mh,
                              const int64_t *__restrict__ sbeg, int64_t *__restrict__ runf, int64_t *__restrict__ segf,
                              int64_t *__restrict__ chkf) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = st[p];
        const bool run = p == 0 || st[p - 1] != s || hh[p - 1] != hh[p];
        const bool chk = (p - sbeg[s]) % kHeavyChunk == 0;
        runf[p] = run;
        chkf[p] = chk;
        segf[p] = run || chk;
    }
}

__global__ void k_heavy_index(const int64_t *__restrict__ runf, const int64_t *__restrict__ segf,
                              const int64_t *__restrict__ chkf, const int64_t *__restrict__ runid,
                              const int64_t *__restrict__ segid, const int64_t *__restrict__ chkid,
                              const uint32_t *__restrict__ hh, const uint32_t *__restrict__ st, int64_t mh,
                              int64_t nstripe, int64_t nh, int64_t *__restrict__ seg_start,
                              int64_t *__restrict__ chunk_start, int64_t *__restrict__ cfirst,
                              int32_t *__restrict__ run_h, int64_t *__restrict__ run_seg,
                              uint32_t *__restrict__ rkey, uint32_t *__restrict__ rval) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x) {
        if (segf[p]) seg_start[segid[p]] = p;
        if (chkf[p]) {
            chunk_start[chkid[p]] = p;
            cfirst[chkid[p]] = segid[p];
        }
        if (runf[p]) {
            const int64_t r = runid[p];
            run_h[r] = (int32_t)hh[p];
            run_seg[r] = segid[p];
            // fold order: by (wave of the target, heavy index); a stable sort keeps stripe order
            rkey[r] = (uint32_t)((int64_t)(st[p] / nstripe) * nh + hh[p]);
            rval[r] = (uint32_t)r;
        }
    }
}

// fold index: target slot of every sorted run position (flags on key changes)
__global__ void k_fold_flags(const uint32_t *__restrict__ skey, int64_t nrun, int64_t *__restrict__ flag) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nrun; p += (int64_t)gridDim.x * blockDim.x)
        flag[p] = (p == 0 || skey[p - 1] != skey[p]) ? 1 : 0;
}

__global__ void k_fold_index(const uint32_t *__restrict__ skey, const int64_t *__restrict__ flag,
                             const int64_t *__restrict__ slot, int64_t nrun, int64_t nh, int64_t *__restrict__ fold_ptr,
                             int32_t *__restrict__ fold_h, unsigned long long *__restrict__ wave_first) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nrun; p += (int64_t)gridDim.x * blockDim.x)
        if (flag[p]) {
            fold_ptr[slot[p]] = p;
            fold_h[slot[p]] = (int32_t)(skey[p] % (uint32_t)nh);
            atomicMin(&wave_first[skey[p] / (uint32_t)nh], (unsigned long long)slot[p]);
        }
}

__global__ void k_fill_u64(unsigned long long *__restrict__ p, int64_t cnt, unsigned long long v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// share of every source's out-weight that leaves its tile: a thread per source
// (rows of more than 32 edges by the whole warp)
template <typename W>
__global__ void k_remote_share(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                               const StoreW<W> *__restrict__ w, const double *__restrict__ inv, int64_t n,
                               int waves, float *__restrict__ wr) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    const int lane = lane_id();
    // leaves the tile and is still pending after the sweep (a later wave takes its
    // pushes in during the sweep, R15); ghost targets always pending
    auto pending = [&](int64_t i, int64_t e) {
        const int64_t t = col[e];
        return t >= n || (t / kNodeTile != i / kNodeTile && tile_wave(t, waves) <= tile_wave(i, waves));
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        if (i < n) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        const bool big = e - b > 32;
        if (i < n && !big) {
            double s = 0.0;
            for (int64_t q = b; q < e; ++q)
                if (pending(i, q)) s += kW ? (double)w[q] : 1.0;
            wr[i] = (float)(s * inv[i]);
        }
        unsigned m = __ballot_sync(0xffffffffu, big);
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const int64_t il = __shfl_sync(0xffffffffu, i, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            double s = 0.0;
            for (int64_t q = bl + lane; q < el; q += 32)
                if (pending(il, q)) s += kW ? (double)w[q] : 1.0;
            s = warp_sum(s);
            if (lane == 0) wr[il] = (float)(s * inv[il]);
        }
    }
}

// Bank-aware slot order: the rounds gather gq[src] for 32
// pieces at once, one slot row per load; a 64-bit shared load is served per
// half-warp, one wavefront per distinct bank pair (src mod 16) hit twice.  The
// order of a piece's slots is free (any fixed order is a valid summation
// order, R14), so each virtual warp's rows are refilled greedily: per row, the
// lanes of a half-warp claim distinct bank pairs, the most frequent remaining
// ones first; padding slots (zero outflow) take a free pair.  One warp per
// virtual warp of <= kBalMaxK slots per lane (longer ones keep edge order).
constexpr int kBalMaxK = 32, kBalWarps = 4;
template <typename W>
__global__ void __launch_bounds__(kBalWarps * 32) k_ell_balance(const int64_t *__restrict__ ltile,
                                                                const uint32_t *__restrict__ vofs, int64_t ntile,
                                                                uint16_t *__restrict__ lsrc,
                                                                StoreW<W> *__restrict__ lw) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    __shared__ uint16_t es[kBalWarps][kBalMaxK][32];
    __shared__ StoreW<W> ew[kBalWarps][kW ? kBalMaxK : 1][32];
    __shared__ uint8_t ord[kBalWarps][kBalMaxK][32];
    __shared__ int cnt[kBalWarps][2][16];
    const int wb = threadIdx.x >> 5, lane = lane_id(), half = lane >> 4;
    const int64_t nitem = ntile * kVWarps;
    for (int64_t item = (int64_t)blockIdx.x * kBalWarps + wb; item < nitem; item += (int64_t)gridDim.x * kBalWarps) {
        const int64_t tile = item / kVWarps;
        const int vw = (int)(item % kVWarps);
        const uint32_t o0 = vofs[tile * kVofsStride + vw];
        const int K = (int)((vofs[tile * kVofsStride + vw + 1] - o0) >> 5);
        if (K < 2 || K > kBalMaxK) continue;           // warp-uniform
        const int64_t base = ltile[tile] + o0;
        if (lane < 16) cnt[wb][0][lane] = cnt[wb][1][lane] = 0;
        __syncwarp();
        for (int s = 0; s < K; ++s) {
            const int64_t pos = base + ell_slot(s, lane, K);
            const int src = lsrc[pos];
            es[wb][s][lane] = (uint16_t)src;
            if constexpr (kW) ew[wb][s][lane] = lw[pos];
            if (src < (int)kNodeTile) atomicAdd(&cnt[wb][half][src & 15], 1);
        }
        __syncwarp();
        uint32_t rem = K == 32 ? 0xffffffffu : ((1u << K) - 1u);
        for (int r = 0; r < K; ++r) {
            unsigned used = 0;
            int choice = -1, cb = -1;
            for (int it = 0; it < 4; ++it) {
                int best = -1, bb = -1, bc = -1;
                if (choice < 0)
                    for (uint32_t m = rem; m; m &= m - 1) {
                        const int e = __ffs(m) - 1;
                        const int src = es[wb][e][lane];
                        if (src >= (int)kNodeTile) continue;
                        const int b = src & 15;
                        if ((used >> b) & 1u) continue;
                        const int c = cnt[wb][half][b];
                        if (c > bc) {
                            bc = c;
                            best = e;
                            bb = b;
                        }
                    }
                const bool prop = choice < 0 && best >= 0;
                const unsigned peers = __match_any_sync(0xffffffffu, prop ? half * 16 + bb : 64 + lane);
                const bool win = prop && lane == __ffs(peers) - 1;
                if (win) {
                    choice = best;
                    cb = bb;
                }
                unsigned bits = win ? (1u << bb) : 0u;
                for (int o = 8; o; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
                used |= bits;
            }
            // left over: a padding slot takes a free bank pair, else the most frequent remaining entry
            int pad = -1;
            if (choice < 0)
                for (uint32_t m = rem; m; m &= m - 1) {
                    const int e = __ffs(m) - 1;
                    if (es[wb][e][lane] >= (int)kNodeTile) {
                        pad = e;
                        break;
                    }
                }
            const unsigned padl = __ballot_sync(0xffffffffu, pad >= 0) & (half ? 0xffff0000u : 0x0000ffffu);
            if (pad >= 0) {
                int k = __popc(padl & ((1u << lane) - 1u));
                unsigned fr = ~used & 0xffffu;
                int b = 0;
                for (; fr && k > 0; --k) fr &= fr - 1;
                if (fr) b = __ffs(fr) - 1;
                choice = pad;
                es[wb][pad][lane] = (uint16_t)(kNodeTile + b);
            } else if (choice < 0) {
                int bc = -1;
                for (uint32_t m = rem; m; m &= m - 1) {
                    const int e = __ffs(m) - 1;
                    const int b = es[wb][e][lane] & 15;
                    if (cnt[wb][half][b] > bc) {
                        bc = cnt[wb][half][b];
                        choice = e;
                        cb = b;
                    }
                }
            }
            __syncwarp();
            if (pad < 0) atomicSub(&cnt[wb][half][cb], 1);
            ord[wb][r][lane] = (uint8_t)choice;
            rem &= ~(1u << choice);
            __syncwarp();
        }
        for (int r = 0; r < K; ++r) {
            const int e = ord[wb][r][lane];
            const int64_t pos = base + ell_slot(r, lane, K);
            lsrc[pos] = es[wb][e][lane];
            if constexpr (kW) lw[pos] = ew[wb][e][lane];
        }
        __syncwarp();
    }
}

__global__ void k_tile_max_edges(const int64_t *__restrict__ ltile, int64_t ntile, unsigned long long *__restrict__ mx) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntile; t += (int64_t)gridDim.x * blockDim.x)
        atomicMax(mx, (unsigned long long)(ltile[t + 1] - ltile[t]));
}

void free_tiles(TilePlan &t) {
    for (void *p : {(void *)t.rrel, (void *)t.hidx, (void *)t.wr, (void *)t.deg, (void *)t.ltile, (void *)t.rtile,
                    (void *)t.vofs, (void *)t.lstage, (void *)t.vfirst, (void *)t.plist, (void *)t.lsrc, t.lw, t.rrec, t.hrec, (void *)t.chunk_start,
                    (void *)t.seg_start, (void *)t.cfirst, (void *)t.run_h, (void *)t.run_seg, (void *)t.part,
                    (void *)t.hsum, (void *)t.tpart, (void *)t.fold_ptr, (void *)t.fold_h, (void *)t.fold_run})
        cudaFree(p);
    t = TilePlan();
}

static int64_t read_i64(const int64_t *p, cudaStream_t st) {
    int64_t v = 0;
    DI_CUDA(cudaMemcpyAsync(&v, p, sizeof(v), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    return v;
}

static int bits_for(int64_t x) {
    int b = 1;
    while (b < 32 && ((int64_t)1 << b) < x) ++b;
    return b;
}

__global__ void k_u32_to_i64(const uint32_t *__restrict__ a, int64_t *__restrict__ b, int64_t cnt) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}

// per-stripe edge counts of the sorted stripe keys
__global__ void k_stripe_count(const uint32_t *__restrict__ st, int64_t mh, unsigned long long *__restrict__ cnt) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x)
        if (p == mh - 1 || st[p + 1] != st[p]) atomicAdd(&cnt[st[p]], (unsigned long long)(p + 1));
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
    const size_t rs = sizeof(RemRec<W>);
    const int64_t nt = g.nt;                         // owned nodes + shard ghost slots
    phase_mark(st, "tiles: start");
    tp.ntile = (n + kNodeTile - 1) / kNodeTile;
    tp.stripe_nodes = std::max<int64_t>(kNodeTile, kStripeBytes / (int64_t)sizeof(double));
    if (const char *e = getenv("DIT_STRIPE_NODES")) tp.stripe_nodes = std::max<int64_t>(kNodeTile, atoll(e));   // tests
    const int64_t nS = (n + tp.stripe_nodes - 1) / tp.stripe_nodes;
    tp.nstripe = nS;
    tp.waves = kTileWaves;                           // shards too (R16: cross-rank pushes wait a sweep)
    if (const char *e = getenv("DIT_TILE_WAVES_RT")) tp.waves = std::max(1, atoi(e));
    // empty waves dropped; at most 32 (the per-wave totals of k_tile's partials array)
    tp.waves = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(tp.waves, 32), tp.ntile));
    const int64_t S = tp.waves * nS;                 // heavy groups (wave, stripe)
    // ---- classes of the in-edges
    int64_t *lc, *rc, *lrc, *hc, *hflag, *rptr, *hptr, *hpos;
    for (int64_t **p : {&lc, &rc, &lrc, &hc, &hflag, &rptr, &hptr, &hpos})
        DI_CUDA(cudaMallocAsync(p, (nt + 1) * sizeof(int64_t), st));
    const int64_t m = g.m;
    uint32_t *tkey = g.t.tkey;                       // the transpose's sorted keys when it kept them
    g.t.tkey = nullptr;
    if (!tkey) {
        DI_CUDA(cudaMallocAsync(&tkey, (m > 0 ? m : 1) * sizeof(uint32_t), st));
        k_fill_tkey<<<grid, 256, 0, st>>>(g.t.ptr, nt, tkey);
        count_launch();
    }
    // local rank of every CSC position among its target's local in-edges: a scan of
    // local flags (32-bit through CUB when m < 2^31, else 64-bit)
    const bool l32 = m < (int64_t)0x7fffffff && !getenv("DIT_FORCE_L64");   // DIT_FORCE_L64: tests of the 64-bit path
    void *L = nullptr;
    {
        const size_t ls = l32 ? sizeof(uint32_t) : sizeof(int64_t);
        void *lflag = nullptr;
        DI_CUDA(cudaMallocAsync(&lflag, (m + 1) * ls, st));
        DI_CUDA(cudaMallocAsync(&L, (m + 1) * ls, st));
        if (l32) {
            k_local_flags<uint32_t><<<grid_for(h, m + 1), 256, 0, st>>>(tkey, g.t.src, m, n, (uint32_t *)lflag);
            size_t tb = 0;
            DI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (uint32_t *)lflag, (uint32_t *)L, (int)(m + 1), st));
            {
                std::lock_guard<std::mutex> lock(scratch_mutex(h->device));
                DI_CUDA(cub::DeviceScan::ExclusiveSum(cub_scratch(h->device, tb), tb, (uint32_t *)lflag, (uint32_t *)L,
                                                      (int)(m + 1), st));
                DI_CUDA(cudaStreamSynchronize(st));
            }
            k_counts_from_scan<uint32_t><<<grid_for(h, nt), 256, 0, st>>>(g.t.ptr, (const uint32_t *)L, nt, lc, rc);
        } else {
            k_local_flags<int64_t><<<grid_for(h, m + 1), 256, 0, st>>>(tkey, g.t.src, m, n, (int64_t *)lflag);
            exclusive_scan_i64((const int64_t *)lflag, (int64_t *)L, m, st);
            k_counts_from_scan<int64_t><<<grid_for(h, nt), 256, 0, st>>>(g.t.ptr, (const int64_t *)L, nt, lc, rc);
        }
        count_launch(2);
        DI_CUDA(cudaFreeAsync(lflag, st));
    }
    k_classify<<<grid_for(h, tp.ntile), 256, 0, st>>>(rc, n, tp.ntile, lrc, hc, hflag);
    count_launch(2);
    if (nt > n) {
        k_classify_ghosts<<<grid_for(h, nt - n), 256, 0, st>>>(rc, n, nt, lrc, hc, hflag);
        count_launch();
    }
    exclusive_scan_i64(lrc, rptr, nt, st);
    exclusive_scan_i64(hc, hptr, nt, st);
    exclusive_scan_i64(hflag, hpos, nt, st);
    tp.mlight = read_i64(rptr + nt, st);
    tp.mh = read_i64(hptr + nt, st);
    tp.nh = read_i64(hpos + nt, st);
    if (tp.mh >= (int64_t)0xffffffffLL) {
        set_error("tiled plan: too many heavy remote edges for one graph handle");
        throw Fail{DI_ERR_INVALID};
    }
    phase_mark(st, "tiles: classify");
    // ---- sliced-ELL layout of the local in-edges
    int32_t *vcap;
    int64_t *pcnt;
    DI_CUDA(cudaMallocAsync(&vcap, (tp.ntile + 1) * sizeof(int32_t), st));
    DI_CUDA(cudaMallocAsync(&pcnt, (tp.ntile + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&tp.vofs, tp.ntile * kVofsStride * sizeof(uint32_t), st));
    DI_CUDA(cudaMallocAsync(&tp.vfirst, tp.ntile * kVfStride * sizeof(uint16_t), st));
    DI_CUDA(cudaMallocAsync(&tp.plist, tp.ntile * kVRows * sizeof(uint16_t), st));
    DI_CUDA(cudaMallocAsync(&tp.ltile, (tp.ntile + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&tp.lstage, (tp.ntile + 1) * sizeof(int32_t), st));
    k_tile_layout<<<(unsigned)std::min<int64_t>(tp.ntile, (int64_t)h->num_sms * 4), kTileThreads, 0, st>>>(
        lc, n, tp.ntile, (int)(2 + (kW ? sizeof(SW) : 0)), (int64_t)(tile_e_buf<W>() - kMetaBytes), tp.vofs,
        tp.vfirst, tp.plist, vcap, pcnt, tp.lstage);
    count_launch();
    exclusive_scan_i64(pcnt, tp.ltile, tp.ntile, st);
    tp.mpad = read_i64(tp.ltile + tp.ntile, st);
    tp.mloc = g.m - tp.mlight - tp.mh;
    // +16 B: aligned TMA supersets may read up to 15 bytes past the end
    DI_CUDA(cudaMallocAsync(&tp.lsrc, tp.mpad * sizeof(uint16_t) + 16, st));
    if (kW) DI_CUDA(cudaMallocAsync(&tp.lw, tp.mpad * sizeof(SW) + 16, st));
    if (tp.mpad > 0) {
        k_fill_pad<W><<<grid_for(h, tp.mpad), 256, 0, st>>>(tp.lsrc, (SW *)tp.lw, tp.mpad);
        count_launch();
    }
    phase_mark(st, "tiles: ELL layout");
    // ---- per-node arrays, tile bases
    DI_CUDA(cudaMallocAsync(&tp.rrel, n * sizeof(uint32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.hidx, nt * sizeof(int32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.wr, n * sizeof(float) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.deg, n * sizeof(int32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.rtile, (tp.ntile + 1) * sizeof(int64_t), st));
    k_tile_rel<<<grid_for(h, nt + 1), 256, 0, st>>>(rptr, hpos, hflag, g.row_ptr, n, nt, tp.ntile, tp.rrel, tp.hidx,
                                                    tp.deg, tp.rtile);
    k_remote_share<W><<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, g.col, (const SW *)g.w, g.inv, n, tp.waves, tp.wr);
    count_launch(2);
    phase_mark(st, "tiles: node arrays");
    // ---- edges to their classes
    DI_CUDA(cudaMallocAsync(&tp.rrec, tp.mlight * rs + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.hrec, tp.mh * rs + 16, st));
    const int64_t mh1 = tp.mh > 0 ? tp.mh : 1;
    RemRec<W> *htmp;
    uint32_t *k0, *v0, *k1, *v1, *hof, *hh;
    DI_CUDA(cudaMallocAsync(&htmp, mh1 * rs, st));
    for (uint32_t **p : {&k0, &v0, &k1, &v1, &hof, &hh}) DI_CUDA(cudaMallocAsync(p, mh1 * sizeof(uint32_t), st));
    if (m > 0 && l32)
        k_split_flat<W, uint32_t><<<grid_for(h, m), 256, 0, st>>>(
            g.t.ptr, tkey, g.t.src, (const SW *)g.t.w, (const uint32_t *)L, m, n, tp.ltile, tp.vofs, tp.vfirst,
            tp.plist, vcap, rptr, hptr, tp.hidx, tp.stripe_nodes, nS, tp.waves, tp.lsrc, (SW *)tp.lw,
            (RemRec<W> *)tp.rrec, htmp, k0, v0, hof);
    else if (m > 0)
        k_split_flat<W, int64_t><<<grid_for(h, m), 256, 0, st>>>(
            g.t.ptr, tkey, g.t.src, (const SW *)g.t.w, (const int64_t *)L, m, n, tp.ltile, tp.vofs, tp.vfirst,
            tp.plist, vcap, rptr, hptr, tp.hidx, tp.stripe_nodes, nS, tp.waves, tp.lsrc, (SW *)tp.lw,
            (RemRec<W> *)tp.rrec, htmp, k0, v0, hof);
    DI_CUDA(cudaFreeAsync(tkey, st));
    DI_CUDA(cudaFreeAsync(L, st));
    count_launch();
    if (tp.mpad > 0 && getenv("DIT_BANK_ORDER")) {   // opt-in: ~1% faster rounds for ~55 ms of build (configs[2])
        k_ell_balance<W><<<(int)std::min<int64_t>(tp.ntile * kVWarps / kBalWarps + 1, (int64_t)h->num_sms * 16),
                           kBalWarps * 32, 0, st>>>(
            tp.ltile, tp.vofs, tp.ntile, tp.lsrc, (SW *)tp.lw);
        count_launch();
    }
    phase_mark(st, "tiles: split edges");
    // ---- heavy edges by (stripe, target, source): a stable sort on the stripe
    tp.s_chunk.assign(S + 1, 0);
    if (tp.mh > 0) {
        auto sorted = radix_sort_u32(k0, v0, k1, v1, tp.mh, bits_for(S + 1), st);
        uint32_t *skey = sorted.first, *sval = sorted.second;
        k_heavy_gather<W><<<grid_for(h, tp.mh), 256, 0, st>>>(skey, sval, tp.mh, htmp, hof, (RemRec<W> *)tp.hrec, hh);
        count_launch();
        phase_mark(st, "heavy: stripe sort");
        // stripe starts
        unsigned long long *scnt;
        DI_CUDA(cudaMallocAsync(&scnt, (S + 1) * sizeof(unsigned long long), st));
        DI_CUDA(cudaMemsetAsync(scnt, 0, (S + 1) * sizeof(unsigned long long), st));
        k_stripe_count<<<grid_for(h, tp.mh), 256, 0, st>>>(skey, tp.mh, scnt);
        count_launch();
        std::vector<unsigned long long> ends(S + 1);
        DI_CUDA(cudaMemcpyAsync(ends.data(), scnt, (S + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> sbeg(S + 1, 0);
        for (int64_t s = 0, last = 0; s < S; ++s) {   // ends[s] = one past the stripe's last edge (0 if empty)
            sbeg[s] = last;
            if (ends[s]) last = (int64_t)ends[s];
            sbeg[s + 1] = last;
        }
        for (int64_t s = 0; s < S; ++s)
            tp.s_chunk[s + 1] = tp.s_chunk[s] + (sbeg[s + 1] - sbeg[s] + kHeavyChunk - 1) / kHeavyChunk;
        tp.nchunk = tp.s_chunk[S];
        int64_t *sbeg_d;
        DI_CUDA(cudaMallocAsync(&sbeg_d, (S + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMemcpyAsync(sbeg_d, sbeg.data(), (S + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        // flags -> ids
        int64_t *runf, *segf, *chkf, *runid, *segid, *chkid;
        for (int64_t **p : {&runf, &segf, &chkf, &runid, &segid, &chkid})
            DI_CUDA(cudaMallocAsync(p, (tp.mh + 1) * sizeof(int64_t), st));
        k_heavy_flags<<<grid_for(h, tp.mh), 256, 0, st>>>(skey, hh, tp.mh, sbeg_d, runf, segf, chkf);
        count_launch();
        exclusive_scan_i64(runf, runid, tp.mh, st);
        exclusive_scan_i64(segf, segid, tp.mh, st);
        exclusive_scan_i64(chkf, chkid, tp.mh, st);
        phase_mark(st, "heavy: flags + scans");
        tp.nrun = read_i64(runid + tp.mh, st);
        tp.nseg = read_i64(segid + tp.mh, st);
        if (read_i64(chkid + tp.mh, st) != tp.nchunk) {
            set_error("tiled plan: heavy chunk count mismatch");
            throw Fail{DI_ERR_CUDA};
        }
        DI_CUDA(cudaMallocAsync(&tp.seg_start, (tp.nseg + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.chunk_start, (tp.nchunk + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.cfirst, (tp.nchunk + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.run_h, tp.nrun * sizeof(int32_t), st));
        DI_CUDA(cudaMallocAsync(&tp.run_seg, (tp.nrun + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.part, tp.nseg * sizeof(double), st));
        uint32_t *rk0, *rv0, *rk1, *rv1;
        for (uint32_t **p : {&rk0, &rv0, &rk1, &rv1}) DI_CUDA(cudaMallocAsync(p, tp.nrun * sizeof(uint32_t), st));
        k_heavy_index<<<grid_for(h, tp.mh), 256, 0, st>>>(runf, segf, chkf, runid, segid, chkid, hh, skey, tp.mh, nS,
                                                          tp.nh, tp.seg_start, tp.chunk_start, tp.cfirst, tp.run_h,
                                                          tp.run_seg, rk0, rv0);
        count_launch();
        if ((int64_t)tp.waves * tp.nh >= (int64_t)0xffffffffLL) {
            set_error("tiled plan: too many heavy targets for one graph handle");
            throw Fail{DI_ERR_INVALID};
        }
        // the heavy targets of each wave, each with its runs in stripe order (k_heavy_fold)
        {
            auto fs = radix_sort_u32(rk0, rv0, rk1, rv1, tp.nrun, bits_for((int64_t)tp.waves * tp.nh + 1), st);
            int64_t *ff, *fslot;
            DI_CUDA(cudaMallocAsync(&ff, (tp.nrun + 1) * sizeof(int64_t), st));
            DI_CUDA(cudaMallocAsync(&fslot, (tp.nrun + 1) * sizeof(int64_t), st));
            k_fold_flags<<<grid_for(h, tp.nrun), 256, 0, st>>>(fs.first, tp.nrun, ff);
            exclusive_scan_i64(ff, fslot, tp.nrun, st);
            const int64_t nslot = read_i64(fslot + tp.nrun, st);
            DI_CUDA(cudaMallocAsync(&tp.fold_ptr, (nslot + 1) * sizeof(int64_t), st));
            DI_CUDA(cudaMallocAsync(&tp.fold_h, (nslot + 1) * sizeof(int32_t), st));
            DI_CUDA(cudaMallocAsync(&tp.fold_run, tp.nrun * sizeof(uint32_t), st));
            unsigned long long *wf;
            DI_CUDA(cudaMallocAsync(&wf, (tp.waves + 1) * sizeof(unsigned long long), st));
            k_fill_u64<<<1, 64, 0, st>>>(wf, tp.waves + 1, (unsigned long long)nslot);
            k_fold_index<<<grid_for(h, tp.nrun), 256, 0, st>>>(fs.first, ff, fslot, tp.nrun, tp.nh, tp.fold_ptr,
                                                               tp.fold_h, wf);
            count_launch(3);
            DI_CUDA(cudaMemcpyAsync(tp.fold_run, fs.second, tp.nrun * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(tp.fold_ptr + nslot, &tp.nrun, sizeof(int64_t), cudaMemcpyHostToDevice, st));
            std::vector<unsigned long long> w(tp.waves + 1);
            DI_CUDA(cudaMemcpyAsync(w.data(), wf, (tp.waves + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                    st));
            DI_CUDA(cudaStreamSynchronize(st));
            tp.wave_slot.assign(tp.waves + 1, nslot);
            for (int c = tp.waves - 1; c >= 0; --c) tp.wave_slot[c] = std::min<int64_t>((int64_t)w[c], tp.wave_slot[c + 1]);
            for (void *p : {(void *)ff, (void *)fslot, (void *)wf, (void *)rk0, (void *)rv0, (void *)rk1, (void *)rv1})
                DI_CUDA(cudaFreeAsync(p, st));
        }
        DI_CUDA(cudaMemcpyAsync(tp.seg_start + tp.nseg, &tp.mh, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.chunk_start + tp.nchunk, &tp.mh, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.cfirst + tp.nchunk, &tp.nseg, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.run_seg + tp.nrun, &tp.nseg, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        phase_mark(st, "heavy: index");
        for (int64_t *p : {runf, segf, chkf, runid, segid, chkid, sbeg_d}) DI_CUDA(cudaFreeAsync(p, st));
        DI_CUDA(cudaFreeAsync(scnt, st));
    }
    phase_mark(st, "tiles: heavy sort + index");
    DI_CUDA(cudaMallocAsync(&tp.hsum, (tp.nh > 0 ? tp.nh : 1) * sizeof(double), st));
    DI_CUDA(cudaMallocAsync(&tp.tpart, (2 * (size_t)tp.waves * 4096 + 64) * sizeof(double), st));
    unsigned long long *mx;
    DI_CUDA(cudaMallocAsync(&mx, sizeof(unsigned long long), st));
    DI_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
    if (tp.ntile > 0) {
        k_tile_max_edges<<<grid_for(h, tp.ntile), 256, 0, st>>>(tp.ltile, tp.ntile, mx);
        count_launch();
    }
    unsigned long long mxh = 0;
    DI_CUDA(cudaMemcpyAsync(&mxh, mx, sizeof(mxh), cudaMemcpyDeviceToHost, st));
    for (int64_t *p : {lc, rc, lrc, hc, hflag, rptr, hptr, hpos, pcnt}) DI_CUDA(cudaFreeAsync(p, st));
    for (uint32_t *p : {k0, v0, k1, v1, hof, hh}) DI_CUDA(cudaFreeAsync(p, st));
    DI_CUDA(cudaFreeAsync(htmp, st));
    DI_CUDA(cudaFreeAsync(vcap, st));
    DI_CUDA(cudaFreeAsync(mx, st));
    DI_CUDA(cudaStreamSynchronize(st));
    DI_CUDA(cudaGetLastError());
    tp.max_tile_edges = (int64_t)mxh;
    tp.built = true;
    phase_mark(st, "tiles: free + done");
}

void build_tiles(di_graph *h) {
    DevGraph &g = h->g;
    if (g.tl.built || g.n == 0) return;
    build_transpose(h);
    switch (g.w_kind) {
    case DI_W_F32: build_tiles_t<float>(h); break;
    case DI_W_F64: build_tiles_t<double>(h); break;
    default: build_tiles_t<NoW>(h);
    }
}

// ---------------------------------------------------------------- heavy remote sums
// Heavy targets' remote inflow, per wave, in two launches:
//   k_heavy_chunks -- one launch per source stripe (the gathered slice of the
//     outflow A stays L2-resident), CTAs stride over the stripe's 2048-edge
//     chunks (a shared ticket counter was measured 2x slower: 40K same-address
//     atomics per wave serialise at one L2 slice); a CTA stages A(src) w of its
//     chunk in shared memory, then one thread per short segment (target within
//     chunk) / one warp per long one sums it into part;
//   k_heavy_fold -- per heavy target of the wave, its runs (one per source
//     stripe) and their segments summed in stripe / edge order into hsum.
// Every sum has a fixed order whatever CTA takes which chunk: bitwise reproducible.

// the chunks [c0, c1) of one stripe; CTA per chunk at a time
template <typename W>
__global__ void __launch_bounds__(kThreads) k_heavy_chunks(const RemRec<W> *__restrict__ hrec,
                                                           const int64_t *__restrict__ chunk_start,
                                                           const int64_t *__restrict__ seg_start,
                                                           const int64_t *__restrict__ cfirst, int64_t c0, int64_t c1,
                                                           const double *__restrict__ A0, const double *__restrict__ A1,
                                                           double *__restrict__ part, int wave, int waves,
                                                           const Ctrl *__restrict__ ctrl, int force) {
    __shared__ double vals[kHeavyChunk];
    __shared__ int sbnd[kHeavyChunk + 1];
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool gather = ctrl->gather != 0;
    if (force ? !gather : (!gather && wave == 0)) return;
    // the previous sweep wrote A[(sweeps - 1) & 1], this sweep's earlier waves A[sweeps & 1]
    const double *__restrict__ Aprev = (ctrl->sweeps & 1) ? A0 : A1;
    const double *__restrict__ Afresh = (ctrl->sweeps & 1) ? A1 : A0;
    const unsigned w = threadIdx.x >> 5, lane = lane_id();
    for (int64_t c = c0 + blockIdx.x; c < c1; c += gridDim.x) {
        const int64_t e0 = chunk_start[c];
        const int cnt = (int)(chunk_start[c + 1] - e0);
        const int64_t sg0 = cfirst[c];
        const int ns = (int)(cfirst[c + 1] - sg0);
        for (int q = threadIdx.x; q < ns; q += kThreads) sbnd[q] = (int)(seg_start[sg0 + q] - e0);
        if (threadIdx.x == 0) sbnd[ns] = cnt;
        // all of this thread's records first, then all their gathers (kPer loads in flight each)
        constexpr int kPer = (int)kHeavyChunk / kThreads;
        RemRec<W> rr[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int k = threadIdx.x + u * kThreads;
            if (k < cnt) rr[u] = hrec[e0 + k];
        }
        double vv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            // a source of an earlier wave pushed this sweep; the others in the previous
            // one (still pending); in the flush only the pending pushes are left (R15)
            const int k = threadIdx.x + u * kThreads;
            vv[u] = 0.0;
            if (k < cnt) {
                const bool early = tile_wave(rr[u].src, waves) < wave;
                if (force ? !early : (early || gather)) vv[u] = (early && !force ? Afresh : Aprev)[rr[u].src];
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int k = threadIdx.x + u * kThreads;
            if (k < cnt) vals[k] = vv[u] * rec_w(rr[u]);
        }
        __syncthreads();
        for (int q0 = (int)(w * 32); q0 < ns; q0 += kThreads) {
            const int q = q0 + (int)lane;
            int b = 0, e = 0;
            if (q < ns) {
                b = sbnd[q];
                e = sbnd[q + 1];
            }
            if (e - b < 64 && e > b) {
                double acc = 0.0;
                for (int k = b; k < e; ++k) acc += vals[k];
                part[sg0 + q] = acc;
            }
            unsigned big = __ballot_sync(0xffffffffu, e - b >= 64);
            while (big) {
                const int l = __ffs(big) - 1;
                big &= big - 1;
                const int bb = __shfl_sync(0xffffffffu, b, l), be = __shfl_sync(0xffffffffu, e, l);
                double acc = 0.0;
                for (int k = bb + (int)lane; k < be; k += 32) acc += vals[k];
                acc = warp_sum(acc);
                if (lane == 0) part[sg0 + q0 + l] = acc;
            }
        }
        __syncthreads();
    }
}

// hsum of the wave's heavy targets [t0, t1) (fold slots): lane per target, a
// warp per target of more than 64 segments
__global__ void __launch_bounds__(kThreads) k_heavy_fold(const int64_t *__restrict__ fold_ptr,
                                                         const int32_t *__restrict__ fold_h,
                                                         const uint32_t *__restrict__ fold_run,
                                                         const int64_t *__restrict__ run_seg,
                                                         const double *__restrict__ part, double *__restrict__ hsum,
                                                         int64_t t0, int64_t t1, int wave, const Ctrl *__restrict__ ctrl,
                                                         int force) {

    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool gather = ctrl->gather != 0;
    if (force ? !gather : (!gather && wave == 0)) return;
    const unsigned lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = t0 + gw * 32; base < t1; base += nw * 32) {
        const int64_t i = base + lane;
        int64_t r0 = 0, r1 = 0, nseg = 0;
        if (i < t1) {
            r0 = fold_ptr[i];
            r1 = fold_ptr[i + 1];
            for (int64_t r = r0; r < r1; ++r) nseg += run_seg[fold_run[r] + 1] - run_seg[fold_run[r]];
        }
        if (i < t1 && nseg <= 64) {
            double acc = 0.0;
            for (int64_t r = r0; r < r1; ++r) {
                const uint32_t q = fold_run[r];
                double rs = 0.0;
                for (int64_t s = run_seg[q]; s < run_seg[q + 1]; ++s) rs += part[s];
                acc += rs;
            }
            hsum[fold_h[i]] = acc;
        }
        unsigned big = __ballot_sync(0xffffffffu, i < t1 && nseg > 64);
        while (big) {
            const int l = __ffs(big) - 1;
            big &= big - 1;
            const int64_t b0 = __shfl_sync(0xffffffffu, r0, l), b1 = __shfl_sync(0xffffffffu, r1, l);
            double acc = 0.0;
            for (int64_t r = b0; r < b1; ++r) {
                const uint32_t q = fold_run[r];
                double rs = 0.0;
                for (int64_t s = run_seg[q] + lane; s < run_seg[q + 1]; s += 32) rs += part[s];
                acc += warp_sum(rs);
            }
            if (lane == 0) hsum[fold_h[base + l]] = acc;
        }
    }
}

// ---------------------------------------------------------------- tile kernel
// DIT_TILE_TIMING (debug): per-CTA phase cycle counters of k_tile
static unsigned long long *g_tile_dbg = nullptr;
constexpr int kDbg = 48;                         // counters per CTA (see di_debug_tile_timing)

template <typename W>
struct TileArgs {
    const uint32_t *vofs;
    const uint16_t *vfirst, *plist;
    const uint32_t *rrel;
    const int32_t *hidx, *deg, *lstage;
    const float *wr;
    const double *inv;
    const int64_t *ltile, *rtile;
    const uint16_t *lsrc;
    const StoreW<W> *lw;
    const RemRec<W> *rrec;
    const double *hsum;
    double *F, *H, *A0, *A1;
    double *part;            // per-CTA partials: resid [grid], leak [grid]
    unsigned long long *dbg; // optional per-CTA phase cycle counters [grid][kDbg] (DIT_TILE_TIMING)
    int64_t n, ntile, m;
    int rounds;
    int wave, waves;         // this launch runs tiles wave, wave + waves, ... (R15)
    int64_t ntw;             // tiles of the wave
};

// one target's local pushes in its sliced-ELL column: slots base, base+32, ...
// (coalesced across the warp); es / ew point into shared memory (staged
// virtual warps) or global memory (the rest), each call site one of them
template <typename W>
__device__ __forceinline__ double local_sum(const uint16_t *es, const StoreW<W> *ew, const double *gq, int base,
                                            int K) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    // four partial sums (slot mod 4), combined in a fixed order at the end: no
    // serial chain of dependent adds (R14: a fixed, deterministic order)
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int s = 0;
    // grouped slots: four sources (and weights) per vector load
    const int lane = base & 31, o0 = base - lane;
    const int Kg = K - K % kSlotGroup;
#pragma unroll 2
    for (; s < Kg; s += kSlotGroup) {
        const int k = o0 + 32 * s + kSlotGroup * lane;
        const uint2 e = *reinterpret_cast<const uint2 *>(es + k);
        const double v0 = gq[e.x & 0xffffu], v1 = gq[e.x >> 16], v2 = gq[e.y & 0xffffu], v3 = gq[e.y >> 16];
        if constexpr (kW) {
            if constexpr (sizeof(StoreW<W>) == 4) {
                const float4 w4 = *reinterpret_cast<const float4 *>(ew + k);
                a0 = fma(v0, (double)w4.x, a0);
                a1 = fma(v1, (double)w4.y, a1);
                a2 = fma(v2, (double)w4.z, a2);
                a3 = fma(v3, (double)w4.w, a3);
            } else {
                a0 = fma(v0, (double)ew[k], a0);
                a1 = fma(v1, (double)ew[k + 1], a1);
                a2 = fma(v2, (double)ew[k + 2], a2);
                a3 = fma(v3, (double)ew[k + 3], a3);
            }
        } else {
            a0 += v0;
            a1 += v1;
            a2 += v2;
            a3 += v3;
        }
    }
    // the last K % 4 slots (one per row of 32): their loads issued together
    const int t = K - s;
    if (t > 0) {
        const int k = base + 32 * s;
        const int s0 = es[k], s1 = t > 1 ? es[k + 32] : (int)kNodeTile, s2 = t > 2 ? es[k + 64] : (int)kNodeTile;
        const double v0 = gq[s0], v1 = gq[s1], v2 = gq[s2];
        if constexpr (kW) {
            a0 = fma(v0, (double)ew[k], a0);
            if (t > 1) a1 = fma(v1, (double)ew[k + 32], a1);
            if (t > 2) a2 = fma(v2, (double)ew[k + 64], a2);
        } else {
            a0 += v0;
            a1 += v1;
            a2 += v2;                                 // padding slot reads a zero
        }
    }
    return (a0 + a1) + (a2 + a3);
}

struct TileScalars {
    int64_t l0, l1;
    int32_t st, pad;
};

// named barriers (0 is __syncthreads): 1 = the round warps, 2 = the prep warps,
// 3 + x = "P[x] full" (prep arrives, rounds sync), 5 + x = "P[x] read" (rounds
// arrive, prep syncs): a warp waiting at a hardware barrier issues nothing
constexpr int kBarRW = 1, kBarPW = 2, kBarPFull = 3, kBarPEmpty = 5;

__device__ __forceinline__ void bar_sync_n(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// round-warp thread 0: tile `tile`'s edge bundle {layout, staged slots} into E buffer `buf`
template <typename W>
__device__ __forceinline__ void issue_edges(const TileArgs<W> &a, int64_t tile, const TileScalars &ts,
                                            unsigned char *buf, uint32_t bar) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr int kWB = kW ? (int)sizeof(StoreW<W>) : 0;
    const int64_t cnt = ts.l1 - ts.l0 - ts.st;       // staged slots: multiples of 32 (16-byte aligned)
    const uint32_t bytes = (uint32_t)(kMetaBytes + cnt * (2 + kWB));
    // order this CTA's earlier generic-proxy reads of the buffer before the async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(bar, bytes);
    const uint32_t sb = smem_u32(buf);
    tma_load(sb, a.vofs + tile * kVofsStride, kVofsStride * 4, bar);
    tma_load(sb + kVofsStride * 4, a.vfirst + tile * kVfStride, kVfStride * 2, bar);
    tma_load(sb + kVofsStride * 4 + kVfStride * 2, a.plist + tile * kVRows, kVRows * 2, bar);
    if (cnt > 0) {
        tma_load(sb + kMetaBytes, a.lsrc + ts.l0 + ts.st, (uint32_t)(cnt * 2), bar);
        if constexpr (kW) tma_load(sb + kMetaBytes + (uint32_t)(cnt * 2), a.lw + ts.l0 + ts.st, (uint32_t)(cnt * kWB), bar);
    }
    // the unstaged (longest) virtual warps are read through L2 by the rounds
    if (ts.st > 0) {
        tma_prefetch_l2(a.lsrc + ts.l0, (uint32_t)(ts.st * 2));
        if constexpr (kW) tma_prefetch_l2(a.lw + ts.l0, (uint32_t)(ts.st * kWB));
    }
}

// prep-warp thread 0: the light records [r0, r1) (16-byte aligned superset) into R buffer `buf`
template <typename W>
__device__ __forceinline__ void issue_records(const TileArgs<W> &a, int64_t r0, int64_t r1, unsigned char *buf,
                                              uint32_t bar) {
    constexpr int kRS = (int)sizeof(RemRec<W>);
    const int64_t rb0 = (r0 * kRS) & ~int64_t(15), rb1 = (r1 * kRS + 15) & ~int64_t(15);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(bar, (uint32_t)(rb1 - rb0));
    if (rb1 > rb0)
        tma_load(smem_u32(buf), reinterpret_cast<const unsigned char *>(a.rrec) + rb0, (uint32_t)(rb1 - rb0), bar);
}

// Persistent kernel, one 1024-thread CTA per SM, warp-specialised:
//   round warps 0-15 -- thread i owns node i of the current tile: the `rounds`
//     Jacobi rounds over the tile's local in-edges (Eq. (8) pushes, sliced-ELL
//     slots from shared memory), then F, H += D, A = d D inv out;
//   prep warps 16-31 -- meanwhile the NEXT tile's inflow: the remote pushes still
//     pending (heavy sums, light records' gathered outflow) added to F, into P.
// TMA bulk copies bring each tile's edge bundle (round warps) and light records
// (prep warps) into the buffer of its parity; mbarriers hand P between the groups.
template <typename W, bool kProf>
__global__ void __launch_bounds__(kTileBlock, 1) k_tile(TileArgs<W> a, Ctrl *__restrict__ ctrl) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr int kWB = kW ? (int)sizeof(StoreW<W>) : 0;
    constexpr int kRS = (int)sizeof(RemRec<W>);
    double *gq = reinterpret_cast<double *>(smem);                       // [kGqSlots]: outflow, zero pad slots
    double *psum = reinterpret_cast<double *>(smem + kOffPsum);          // [kVRows]: piece sums by rank
    PrepRow *Pbuf = reinterpret_cast<PrepRow *>(smem + kOffP);           // [2][kNodeTile]
    auto rbuf = [&](int x) { return smem + kOffR + x * tile_rec_buf<W>(); };
    auto ebuf = [&](int x) { return smem + tile_off_e<W>() + x * tile_e_buf<W>(); };
    // E_full, R_full: TMA completion (count 1)
    __shared__ __align__(8) unsigned long long bars[4];
    __shared__ TileScalars sc[2];                    // scalars of the tile in each E buffer
    __shared__ double s_r[kTileBlock / 32], s_l[kTileBlock / 32];
    __shared__ unsigned long long s_c[kTileBlock / 32][2];
    __shared__ bool s_last;
    if (ctrl->done || ctrl->use_pull != kUseTiled) return;
    const double d = ctrl->d;
    const bool gather = ctrl->gather != 0;
    // light records are needed when a previous sweep left pushes, or earlier waves of this one
    const bool recs_on = gather || a.wave > 0;
    const unsigned long long sw = ctrl->sweeps;
    double *__restrict__ Anext = (sw & 1) ? a.A1 : a.A0;
    const double *__restrict__ Aprev = (sw & 1) ? a.A0 : a.A1;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int64_t G = gridDim.x;
    const bool is_rw = tid < kRW;
    auto tid_of = [&](int64_t jt) { return (int64_t)a.wave + (int64_t)a.waves * jt; };   // the wave's jt-th tile
    auto E_full = [&](int x) { return smem_u32(&bars[x]); };
    auto R_full = [&](int x) { return smem_u32(&bars[2 + x]); };
    if (tid == 0) {
        for (int x = 0; x < 2; ++x) {
            mbar_init(E_full(x), 1);
            mbar_init(R_full(x), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < (int)(kGqSlots - kNodeTile)) gq[kNodeTile + tid] = 0.0;   // ELL padding reads these
    __syncthreads();
    double resid = 0.0, leak = 0.0;
    uint32_t nodes = 0;                              // per thread: <= tiles x rounds
    unsigned long long edges = 0;
    unsigned long long *dbg = kProf ? a.dbg + blockIdx.x * kDbg : nullptr;
    if (is_rw) {
        // ------------------------------------------------ round warps
        const int i = tid, wp = tid >> 5;
        auto escal = [&](int64_t jt) {
            const int64_t t = tid_of(jt);
            return TileScalars{a.ltile[t], a.ltile[t + 1], a.lstage[t], 0};
        };
        if (i == 0)
            for (int x = 0; x < 2; ++x)
                if (blockIdx.x + x * G < a.ntw) {
                    sc[x] = escal(blockIdx.x + x * G);
                    issue_edges<W>(a, tid_of(blockIdx.x + x * G), sc[x], ebuf(x), E_full(x));
                }
        long long ls_cyc = 0, b2_cyc = 0, ns_cyc = 0, b1_cyc = 0, rows_w = 0;           // DIT_TILE_TIMING: local sums, wait after them
        int k = 0;
        for (int64_t jt = blockIdx.x; jt < a.ntw; jt += G, ++k) {
            const int x = k & 1;
            const uint32_t ph = (uint32_t)((k >> 1) & 1);
            const int64_t tile = tid_of(jt);
            const int64_t a0 = tile * kNodeTile;
            const int nn = (int)min(kNodeTile, a.n - a0);
            const bool valid = i < nn;
            const int64_t j = a0 + i;
            // scalars of the tile two ahead (loaded now, used after the rounds)
            TileScalars nx{0, 0, 0, 0};
            const bool has_nx = jt + 2 * G < a.ntw;
            if (i == 0 && has_nx) nx = escal(jt + 2 * G);
            long long c0 = kProf ? clock64() : 0;
            bar_sync_n(kBarPFull + x, kTileBlock);
            // f, 1/sum w and the out-degree now; H and wr from P[x] again at the state out
            const PrepRow *prow = Pbuf + x * kNodeTile + i;
            double f = 0.0, pivi = 0.0;
            int32_t pdeg = 0;
            if (valid) {
                f = prow->f;
                pivi = prow->ivi;
                pdeg = prow->deg;
            }
            long long c1 = kProf ? clock64() : 0;
            mbar_wait(E_full(x), ph);
            long long c2 = kProf ? clock64() : 0;
            const TileScalars cur = sc[x];
            unsigned char *E = ebuf(x);
            const uint32_t *vofs_s = reinterpret_cast<const uint32_t *>(E);
            const uint16_t *vf_s = reinterpret_cast<const uint16_t *>(vofs_s + kVofsStride);
            const uint16_t *pl_s = vf_s + kVfStride;
            const int st = cur.st;
            const int64_t cnt = cur.l1 - cur.l0 - st;
            // slot k of the tile: shared memory for k >= st, global below
            const uint16_t *es_sm = reinterpret_cast<const uint16_t *>(E + kMetaBytes) - st;
            const StoreW<W> *ew_sm = reinterpret_cast<const StoreW<W> *>(E + kMetaBytes + cnt * 2) - st;
            const uint16_t *es_gl = a.lsrc + cur.l0;
            const StoreW<W> *ew_gl = kW ? a.lw + cur.l0 : nullptr;
            // the node's pieces (ranks into psum, in edge order): the first four in registers
            const int p0 = valid ? (int)vf_s[i] : 0, np = valid ? (int)vf_s[i + 1] - p0 : 0;
            const int pr0 = np > 0 ? pl_s[p0] : 0, pr1 = np > 1 ? pl_s[p0 + 1] : 0;
            const int pr2 = np > 2 ? pl_s[p0 + 2] : 0, pr3 = np > 3 ? pl_s[p0 + 3] : 0;
            double D = 0.0;
            for (int r = 0; r < a.rounds; ++r) {
                double q = 0.0;
                if (f != 0.0) {                      // invalid threads hold f = 0
                    D += f;                          // Eq. (10)
                    nodes += 1;
                    edges += (unsigned long long)pdeg;
                    q = d * f * pivi;                // d F(i) / sum_k w_{i,k}
                }
                const long long t9 = kProf ? clock64() : 0;
                gq[i] = q;
                bar_sync_n(kBarRW, kRW);
                const long long ta = kProf ? clock64() : 0;
                if (kProf) b1_cyc += ta - t9;
                // Eq. (8) local pushes: this warp's two virtual warps of pieces (longest with shortest)
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    const int vw = h2 ? kVWarps - 1 - wp : wp;
                    const uint32_t o0 = vofs_s[vw];
                    const int K = (int)((vofs_s[vw + 1] - o0) >> 5);
                    if (kProf) rows_w += K;
                    if (K) {
                        double acc;
                        if ((int)o0 >= st) acc = local_sum<W>(es_sm, ew_sm, gq, (int)o0 + lane, K);
                        else acc = local_sum<W>(es_gl, ew_gl, gq, (int)o0 + lane, K);
                        psum[vw * 32 + lane] = acc;
                    }
                }
                const long long tb = kProf ? clock64() : 0;
                bar_sync_n(kBarRW, kRW);
                const long long tc = kProf ? clock64() : 0;
                if (kProf) {
                    ls_cyc += tb - ta;
                    b2_cyc += tc - tb;
                }
                if (np > 0) {                         // the node's pieces, in edge order
                    const double x0 = psum[pr0], x1 = np > 1 ? psum[pr1] : 0.0;
                    const double x2 = np > 2 ? psum[pr2] : 0.0, x3 = np > 3 ? psum[pr3] : 0.0;
                    double acc = 0.0 + x0;
                    if (np > 1) acc += x1;
                    if (np > 2) acc += x2;
                    if (np > 3) acc += x3;
                    for (int p = p0 + 4; p < p0 + np; ++p) acc += psum[pl_s[p]];
                    f = acc;
                } else {
                    f = 0.0;
                }
                if (kProf) {
                    __syncwarp();
                    ns_cyc += clock64() - tc;
                }
            }
            long long c3 = kProf ? clock64() : 0;
            // state out; the remote pushes leave as the outflow A (linearity of Eq. (8))
            if (valid) {
                a.F[j] = f;
                if (D != 0.0) a.H[j] = prow->H + D;
                Anext[j] = d * D * pivi;
                // R13: the pushes still pending carry d D(i) P_{t,i} over the pending
                // out-edges t, i.e. |d D(i)| wr(i) with wr(i) = inv(i) sum_pending w
                resid += fabs(f) + fabs(d * D) * (double)prow->wr;
                if (pdeg == 0) leak += D;             // dangling: the fluid left the system (§3.3)
            }
            if (jt + 2 * G < a.ntw) bar_arrive_n(kBarPEmpty + x, kTileBlock);   // prep syncs it before tile k + 2
            bar_sync_n(kBarRW, kRW);                       // E[x] read by every round warp
            if (i == 0 && has_nx) {
                sc[x] = nx;
                issue_edges<W>(a, tid_of(jt + 2 * G), nx, E, E_full(x));
            }
            if (kProf && i == 0) {
                dbg[st == 0 ? 10 : 12] += c3 - c2;    // rounds of fully / partly staged tiles
                dbg[st == 0 ? 11 : 13] += 1;
                dbg[0] += c1 - c0;                    // waiting for the prepared rows
                dbg[1] += c2 - c1;                    // waiting for the edge bundle
                dbg[2] += c3 - c2;                    // local rounds
                dbg[3] += clock64() - c3;             // state out
                dbg[7] += 1;
            }
        }
        if (kProf && lane == 0) {
            atomicAdd(&dbg[8], (unsigned long long)ls_cyc);
            atomicAdd(&dbg[9], (unsigned long long)b2_cyc);
            atomicAdd(&dbg[14], (unsigned long long)ns_cyc);
            atomicAdd(&dbg[16 + wp], (unsigned long long)ls_cyc);
            atomicAdd(&dbg[32 + wp], (unsigned long long)rows_w);
            atomicAdd(&dbg[15], (unsigned long long)b1_cyc);
        }
    } else {
        // ------------------------------------------------ prep warps
        const int p = tid - kRW;
        auto rscal = [&](int64_t jt, int64_t &r0, int64_t &r1) {
            const int64_t t = tid_of(jt);
            r0 = recs_on ? a.rtile[t] : 0;
            r1 = recs_on ? a.rtile[t + 1] : 0;
        };
        if (p == 0)
            for (int x = 0; x < 2; ++x)
                if (blockIdx.x + x * G < a.ntw) {
                    int64_t r0, r1;
                    rscal(blockIdx.x + x * G, r0, r1);
                    issue_records<W>(a, r0, r1, rbuf(x), R_full(x));
                }
        int k = 0;
        for (int64_t jt = blockIdx.x; jt < a.ntw; jt += G, ++k) {
            const int x = k & 1;
            const uint32_t ph = (uint32_t)((k >> 1) & 1);
            const int64_t tile = tid_of(jt);
            const int64_t a0 = tile * kNodeTile;
            const int nn = (int)min(kNodeTile, a.n - a0);
            long long c0 = kProf ? clock64() : 0;
            // per-node state (independent loads, in flight together): nodes p, p + kPWt
            int64_t r0 = 0, r1 = 0;
            rscal(jt, r0, r1);
            int64_t n0 = 0, n1 = 0;
            const bool has_nx = jt + 2 * G < a.ntw;
            if (p == 0 && has_nx) rscal(jt + 2 * G, n0, n1);
            double Fj[kPN], ivi[kPN], Hj[kPN];
            float wrj[kPN];
            int32_t dg[kPN], hx[kPN];
            int rb[kPN], re[kPN];
#pragma unroll
            for (int u = 0; u < kPN; ++u) {
                const int q = p + u * kPWt;
                const int64_t j = a0 + q;
                Fj[u] = ivi[u] = Hj[u] = 0.0;
                wrj[u] = 0.f;
                dg[u] = 0;
                hx[u] = -1;
                rb[u] = re[u] = 0;
                if (q < nn) {
                    Fj[u] = a.F[j];
                    ivi[u] = a.inv[j];
                    Hj[u] = a.H[j];
                    wrj[u] = a.wr[j];
                    dg[u] = a.deg[j];
                    if (recs_on) {
                        hx[u] = a.hidx[j];
                        rb[u] = (int)a.rrel[j];
                        re[u] = q + 1 < nn ? (int)a.rrel[j + 1] : (int)(r1 - r0);
                    }
                }
            }
            mbar_wait(R_full(x), ph);
            long long c1 = kProf ? clock64() : 0;
            RemRec<W> *recs = reinterpret_cast<RemRec<W> *>(rbuf(x) + (r0 * kRS - ((r0 * kRS) & ~int64_t(15))));
            const int R = (int)(r1 - r0);
            // remote pushes still pending: from the previous sweep, and from this
            // sweep's earlier waves (R15): light records' gathered outflow, in place
#pragma unroll 4
            for (int q = p; q < R; q += kPWt) {
                const RemRec<W> rc = recs[q];
                const bool early = tile_wave(rc.src, a.waves) < a.wave;
                const double v = early ? Anext[rc.src] : (gather ? Aprev[rc.src] : 0.0);
                *reinterpret_cast<double *>(&recs[q]) = v * rec_w(rc);
            }
            double hs[kPN];
#pragma unroll
            for (int u = 0; u < kPN; ++u) hs[u] = hx[u] >= 0 ? a.hsum[hx[u]] : 0.0;
            bar_sync_n(kBarPW, kPWt);
            double sm[kPN];
#pragma unroll
            for (int u = 0; u < kPN; ++u) {
                double acc = 0.0;
                for (int q = rb[u]; q < re[u]; ++q) acc += *reinterpret_cast<const double *>(&recs[q]);
                sm[u] = acc;
            }
            long long c2 = kProf ? clock64() : 0;
            if (k >= 2) bar_sync_n(kBarPEmpty + x, kTileBlock);   // the round warps read P[x] of tile k - 2
            long long c3 = kProf ? clock64() : 0;
#pragma unroll
            for (int u = 0; u < kPN; ++u)
                if (p + u * kPWt < nn)
                    Pbuf[x * kNodeTile + p + u * kPWt] = PrepRow{Fj[u] + sm[u] + hs[u], ivi[u], Hj[u], wrj[u], dg[u]};
            bar_arrive_n(kBarPFull + x, kTileBlock);
            bar_sync_n(kBarPW, kPWt);                      // R[x] read by every prep warp
            if (p == 0 && has_nx) issue_records<W>(a, n0, n1, rbuf(x), R_full(x));
            if (kProf && p == 0) {
                dbg[4] += c1 - c0;                    // node loads + waiting for the records
                dbg[5] += c2 - c1;                    // gathers + sums
                dbg[6] += c3 - c2;                    // waiting for the round warps
            }
        }
    }
    // CTA partials (fixed order) and the last-block end of the sweep
    resid = warp_sum(resid);
    leak = warp_sum(leak);
    const unsigned long long nodes64 = warp_sum((unsigned long long)nodes);
    const unsigned long long edges64 = warp_sum(edges);
    const unsigned w = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s_r[w] = resid;
        s_l[w] = leak;
        s_c[w][0] = nodes64;
        s_c[w][1] = edges64;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double rr = 0.0, ll = 0.0;
        unsigned long long xx = 0, yy = 0;
        for (int q = 0; q < kTileBlock / 32; ++q) {
            rr += s_r[q];
            ll += s_l[q];
            xx += s_c[q][0];
            yy += s_c[q][1];
        }
        a.part[a.wave * 4096 + blockIdx.x] = rr;
        a.part[(a.waves + a.wave) * 4096 + blockIdx.x] = ll;
        if (xx) {
            atomicAdd(&ctrl->diffused_nodes, xx);
            atomicAdd(&ctrl->sel_edges, yy);
        }
        __threadfence();
        const unsigned v = atomicAdd(&ctrl->red_blocks, 1u);
        s_last = (v == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last || threadIdx.x != 0) return;
    __threadfence();
    // last block of the wave: the wave's partials in a fixed order
    volatile double *vp = a.part;
    double r = 0.0, lk = 0.0;
    for (unsigned bb = 0; bb < gridDim.x; ++bb) {
        r += vp[a.wave * 4096 + bb];
        lk += vp[(a.waves + a.wave) * 4096 + bb];
    }
    vp[2 * a.waves * 4096 + 2 * a.wave] = r;
    vp[2 * a.waves * 4096 + 2 * a.wave + 1] = lk;
    ctrl->red_blocks = 0;
    if (a.wave + 1 < a.waves) return;                // the sweep ends with its last wave
    r = 0.0;
    lk = 0.0;
    for (int c = 0; c < a.waves; ++c) {
        r += vp[2 * a.waves * 4096 + 2 * c];
        lk += vp[2 * a.waves * 4096 + 2 * c + 1];
    }
    end_sweep(ctrl, lk);
    ctrl->gather = 1;                                // this sweep's remote pushes are pending in A
    ctrl->n_entries = 0;
    ctrl->sel_edges = 0;
    ctrl->red_blocks = 0;
    if (ctrl->stats_out) {                           // shard: the global values come back through k_control
        ctrl->stats_out[0] = r;
        ctrl->stats_out[1] = 0.0;
        ctrl->stats_out[2] = ctrl->leak;
        ctrl->stats_out[3] = (double)ctrl->last_sel_edges;
        ctrl->stats_is_init = 0;
        return;
    }
    finalize_control(ctrl, r, 0.0, 0, a.m);
}

// The pending remote pushes of the last sweep into F (same arithmetic and
// order as step 1 of k_tile), thread per node.
template <typename W>
__global__ void __launch_bounds__(kThreads) k_tile_flush(TileArgs<W> a, const Ctrl *__restrict__ ctrl) {
    if (!ctrl->gather) return;
    const double *__restrict__ Alast = (ctrl->sweeps & 1) ? a.A0 : a.A1;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < a.n; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = j / kNodeTile;
        const int c = tile_wave(j, a.waves);
        const int64_t base = a.rtile[t];
        const int64_t b = base + a.rrel[j];
        const int64_t e = (j + 1 < a.n && (j + 1) % kNodeTile != 0) ? base + a.rrel[j + 1] : a.rtile[t + 1];
        double s = 0.0;
        for (int64_t k = b; k < e; ++k) {
            // only the pushes not yet taken in: sources of this or a later wave (R15)
            const RemRec<W> r = a.rrec[k];
            const double v = tile_wave(r.src, a.waves) >= c ? Alast[r.src] : 0.0;
            s += v * rec_w(r);
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
    a.vofs = tp.vofs;
    a.vfirst = tp.vfirst;
    a.plist = tp.plist;
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
    a.part = tp.tpart;
    a.n = g.n;
    a.ntile = tp.ntile;
    a.m = g.m;
    a.lstage = tp.lstage;
    a.rounds = rounds;
    a.dbg = nullptr;
    a.wave = 0;
    a.waves = tp.waves;
    a.ntw = tp.ntile;
    return a;
}

// resident CTAs of k_heavy_chunks per SM (its grid is exactly one wave of CTAs)
template <typename W>
static int heavy_ctas_per_sm() {
    static int v = 0;
    if (!v) {
        DI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_heavy_chunks<W>, kThreads, 0));
        if (v < 1) v = 1;
    }
    return v;
}

// the heavy targets' remote inflow hsum of one wave: chunks by ticket, then the fold
template <typename W>
static void launch_heavy_t(di_graph *h, int wave, int force) {
    TilePlan &tp = h->g.tl;
    State &s = h->s;
    if (tp.nh == 0) return;
    const int64_t S = tp.nstripe, g0 = (int64_t)wave * S;
    const int64_t t0 = tp.wave_slot[wave], t1 = tp.wave_slot[wave + 1];
    // one launch per source stripe: the gathered slice of A (kStripeBytes) stays in L2
    for (int64_t sg = 0; sg < S; ++sg) {
        const int64_t a0 = tp.s_chunk[g0 + sg], a1 = tp.s_chunk[g0 + sg + 1];
        if (a1 <= a0) continue;
        const int grid = (int)std::min<int64_t>(a1 - a0, (int64_t)h->num_sms * heavy_ctas_per_sm<W>());
        k_heavy_chunks<W><<<grid, kThreads, 0, h->stream>>>((const RemRec<W> *)tp.hrec, tp.chunk_start, tp.seg_start,
                                                            tp.cfirst, a0, a1, s.A, s.A2, tp.part, wave, tp.waves,
                                                            s.ctrl, force);
        count_launch();
    }

    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((t1 - t0 + kThreads - 1) / kThreads,
                                                                 (int64_t)h->num_sms * 8));
    k_heavy_fold<<<grid, kThreads, 0, h->stream>>>(tp.fold_ptr, tp.fold_h, tp.fold_run, tp.run_seg, tp.part, tp.hsum,
                                                   t0, t1, wave, s.ctrl, force);
    count_launch();
}

template <typename W>
static void launch_tile_kernel_t(di_graph *h, int rounds, int wave) {
    DevGraph &g = h->g;
    State &s = h->s;
    TilePlan &tp = g.tl;
    static bool attr_set = false;                    // once per weight kind, off the sweep path
    if (!attr_set) {
        DI_CUDA(cudaFuncSetAttribute(k_tile<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tile_smem_bytes<W>()));
        DI_CUDA(cudaFuncSetAttribute(k_tile<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     tile_smem_bytes<W>()));
        attr_set = true;
    }
    TileArgs<W> a = tile_args<W>(h, rounds);
    if (getenv("DIT_TILE_TIMING")) {
        if (!g_tile_dbg) {
            DI_CUDA(cudaMalloc(&g_tile_dbg, 4096 * kDbg * sizeof(unsigned long long)));
            DI_CUDA(cudaMemset(g_tile_dbg, 0, 4096 * kDbg * sizeof(unsigned long long)));
        }
        a.dbg = g_tile_dbg;
    }
    a.wave = wave;
    a.ntw = tp.ntile > wave ? (tp.ntile - wave + tp.waves - 1) / tp.waves : 0;
    if (a.ntw == 0) return;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntw, (int64_t)h->num_sms));
    if (a.dbg) k_tile<W, true><<<grid, kTileBlock, tile_smem_bytes<W>(), h->stream>>>(a, s.ctrl);
    else k_tile<W, false><<<grid, kTileBlock, tile_smem_bytes<W>(), h->stream>>>(a, s.ctrl);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

template <typename W>
static void launch_tile_t(di_graph *h, int rounds) {
    const int64_t k = h->s.launched;
    for (int c = 0; c < h->g.tl.waves; ++c) {          // events: [2c] heavy(c) [2c+1] tile(c) [2c+2]
        launch_heavy_t<W>(h, c, 0);
        mark_event(h, k, 2 * c + 1);
        launch_tile_kernel_t<W>(h, rounds, c);
        mark_event(h, k, 2 * c + 2);
    }
}

void launch_tile_sweep(di_graph *h, int rounds) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_tile_t<float>(h, rounds); break;
    case DI_W_F64: launch_tile_t<double>(h, rounds); break;
    default: launch_tile_t<NoW>(h, rounds);
    }
}

// shard sweeps run the two halves separately, the ghost exchange in between
void launch_tile_heavy(di_graph *h, int force, int wave) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_heavy_t<float>(h, wave, force); break;
    case DI_W_F64: launch_heavy_t<double>(h, wave, force); break;
    default: launch_heavy_t<NoW>(h, wave, force);
    }
}

void launch_tile_kernel(di_graph *h, int rounds, int wave) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_tile_kernel_t<float>(h, rounds, wave); break;
    case DI_W_F64: launch_tile_kernel_t<double>(h, rounds, wave); break;
    default: launch_tile_kernel_t<NoW>(h, rounds, wave);
    }
}

int tile_waves(const di_graph *h) { return h->g.tl.waves; }

// ghost slots' inflow (heavy sums of the last sweep's pushes) -> the send buffer
__global__ void k_take_ghost_sums(const int32_t *__restrict__ hidx, const double *__restrict__ hsum, int64_t n,
                                  int64_t ng, double *__restrict__ out, const Ctrl *__restrict__ ctrl, int force) {
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool g = ctrl->gather != 0;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < ng; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = g ? hsum[hidx[n + q]] : 0.0;
}

void launch_take_ghost_sums(di_graph *h, double *out, int force) {
    const int64_t ng = h->g.nt - h->g.n;
    if (ng <= 0) return;
    k_take_ghost_sums<<<grid_for(h, ng), 256, 0, h->stream>>>(h->g.tl.hidx, h->g.tl.hsum, h->g.n, ng, out, h->s.ctrl,
                                                            force);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

template <typename W>
static void launch_flush_t(di_graph *h) {
    for (int c = 0; c < h->g.tl.waves; ++c) launch_heavy_t<W>(h, c, 1);
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

// Debug (not part of include/dit.h): k_tile phase cycles {wait, inflow, rounds,
// state out} summed over CTAs, and the number of (CTA, tile) iterations.
extern "C" int di_debug_tile_timing(double *out8) {
    if (!dit::g_tile_dbg || !out8) return 1;
    std::vector<unsigned long long> v(4096 * dit::kDbg);
    if (cudaMemcpy(v.data(), dit::g_tile_dbg, v.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost))
        return 2;
    for (int q = 0; q < dit::kDbg; ++q) out8[q] = 0;
    for (int bb = 0; bb < 4096; ++bb)
        for (int q = 0; q < dit::kDbg; ++q) out8[q] += (double)v[bb * dit::kDbg + q];
    return 0;
}
