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
// Kernels (B200): k_tile -- persistent, one 736-thread CTA per SM walking the
// tiles of one wave (R15), warp-specialised: 16 round warps (thread i owns
// node i of the tile; the rounds over sliced-ELL slots staged in shared
// memory), 6 prep warps (the next tile's inflow: per-node loads, light-record
// gathers, heavy sums) and one producer warp issuing the TMA bulk copies
// (cp.async.bulk + mbarrier, double-buffered edge bundles and light records);
// named barriers hand the prepared rows from prep to rounds.
// k_heavy_chunks / k_heavy_fold -- per wave: 1024-edge chunks in source-stripe
// order (L2-resident slice of A), then per heavy target its runs in stripe
// order.  Every summation has a fixed order: bitwise reproducible run to run.
#include "dit_tile.cuh"

#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace dit {

// ---------------------------------------------------------------- heavy remote sums
// Heavy targets' remote inflow, per wave, in two launches:
//   k_heavy_chunks -- one launch per wave, CTAs stride statically over its
//     1024-edge chunks in source-stripe order (the gathered slice of the outflow
//     A stays L2-resident; a shared ticket counter was measured 2x slower: 40K same-address
//     atomics per wave serialise at one L2 slice); a CTA stages A(src) w of its
//     chunk in shared memory, then one thread per short segment (target within
//     chunk) / one warp per long one sums it into part;
//   k_heavy_fold -- per heavy target of the wave, its runs (one per source
//     stripe) and their segments summed in stripe / edge order into hsum.
// Every sum has a fixed order whatever CTA takes which chunk: bitwise reproducible.

// the chunks [c0, c1) of one wave (stripe order); CTA per chunk at a time
template <typename W>
__global__ void __launch_bounds__(kHeavyThreads) k_heavy_chunks(const RemRec<W> *__restrict__ hrec,
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
        for (int q = threadIdx.x; q < ns; q += kHeavyThreads) sbnd[q] = (int)(seg_start[sg0 + q] - e0);
        if (threadIdx.x == 0) sbnd[ns] = cnt;
        // all of this thread's records first, then all their gathers (kPer loads in flight each)
        constexpr int kPer = (int)kHeavyChunk / kHeavyThreads;
        RemRec<W> rr[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int k = threadIdx.x + u * kHeavyThreads;
            if (k < cnt) rr[u] = hrec[e0 + k];
        }
        double vv[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            // a source of an earlier wave pushed this sweep; the others in the previous
            // one (still pending); in the flush only the pending pushes are left (R15)
            const int k = threadIdx.x + u * kHeavyThreads;
            vv[u] = 0.0;
            if (k < cnt) {
                const bool early = tile_wave(rr[u].src, waves) < wave;
                if (force ? !early : (early || gather)) vv[u] = (early && !force ? Afresh : Aprev)[rr[u].src];
            }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
            const int k = threadIdx.x + u * kHeavyThreads;
            if (k < cnt) vals[k] = vv[u] * rec_w(rr[u]);
        }
        __syncthreads();
        for (int q0 = (int)(w * 32); q0 < ns; q0 += kHeavyThreads) {
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
    const int32_t *dl_ptr;   // delta in-edges inside the tile (dit_delta.cu, R18) or null
    const uint16_t *dl_src;
    const double *dl_w;
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
#pragma unroll kLsUnroll
    for (; s < Kg; s += kSlotGroup) {
        const int k = o0 + 32 * s + kSlotGroup * lane;
        const uint2 e = *reinterpret_cast<const uint2 *>(es + k);
#ifdef DIT_ABL_NOGATHER
        const double v0 = (double)(e.x & 0xffffu), v1 = (double)(e.x >> 16), v2 = (double)(e.y & 0xffffu), v3 = (double)(e.y >> 16);
#else
        const double v0 = gq[e.x & 0xffffu], v1 = gq[e.x >> 16], v2 = gq[e.y & 0xffffu], v3 = gq[e.y >> 16];
#endif
        if constexpr (kW) {
            if constexpr (sizeof(StoreW<W>) == 4) {
#ifdef DIT_ABL_NOWEIGHT
                const float4 w4 = make_float4(1.f, 1.f, 1.f, 1.f);
#else
                const float4 w4 = *reinterpret_cast<const float4 *>(ew + k);
#endif
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
// arrive, prep and the producer sync), 7 + x = "R[x] read" (prep arrives, the
// producer syncs): a warp waiting at a hardware barrier issues nothing
constexpr int kBarRW = 1, kBarPW = 2, kBarPFull = 3, kBarPEmpty = 5, kBarRFree = 7;

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
#ifndef DIT_NO_EDGE_FENCE
    // order this CTA's earlier generic-proxy reads of the buffer before the async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
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

// Persistent kernel, one kTileBlock-thread CTA per SM, warp-specialised:
//   round warps 0-15 -- thread i owns node i of the current tile: the `rounds`
//     Jacobi rounds over the tile's local in-edges (Eq. (8) pushes, sliced-ELL
//     slots from shared memory), then F, H += D, A = d D inv out;
//   prep warps 16-22 (kPWt threads, <= kPN nodes each) -- meanwhile the NEXT tile's
//     inflow: the remote pushes still
//     pending (heavy sums, light records' gathered outflow) added to F, into P.
// TMA bulk copies bring each tile's edge bundle (round warps) and light records
// (prep warps) into the buffer of its parity; mbarriers hand P between the groups.
template <typename W, bool kProf, bool kDl>
__global__ void __launch_bounds__(kTileBlock, 1) k_tile(TileArgs<W> a, Ctrl *__restrict__ ctrl) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr int kWB = kW ? (int)sizeof(StoreW<W>) : 0;
    constexpr int kRS = (int)sizeof(RemRec<W>);
    double *gq = reinterpret_cast<double *>(smem);                       // [kGqCopies][kGqStride]: outflow, zero pad slots
    double *psum = reinterpret_cast<double *>(smem + kOffPsum);          // [kVRows]: piece sums by rank
    // prepared rows, structure of arrays [2][kNodeTile] each (consecutive threads, consecutive banks)
    double *Pf = reinterpret_cast<double *>(smem + kOffP);
    double *Pivi = Pf + 2 * kNodeTile;
    int32_t *Pdeg = reinterpret_cast<int32_t *>(Pivi + 2 * kNodeTile);
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
    constexpr int kPadSlots = (int)(kGqSlots - kNodeTile);
    if (tid < kPadSlots * kGqCopies)                // ELL padding reads these
        gq[(tid / kPadSlots) * kGqStride + kNodeTile + tid % kPadSlots] = 0.0;
    __syncthreads();
    double resid = 0.0, leak = 0.0;
    uint32_t nodes = 0;                              // per thread: <= tiles x rounds
    unsigned long long edges = 0;
    unsigned long long *dbg = kProf ? a.dbg + blockIdx.x * kDbg : nullptr;
    if (is_rw) {
        // ------------------------------------------------ round warps
        const int i = tid, wp = tid >> 5;
        long long ls_cyc = 0, b2_cyc = 0, ns_cyc = 0, b1_cyc = 0;   // DIT_TILE_TIMING: local sums, wait after them
        long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pn[2] = {0, 0};
        int k = 0;
        for (int64_t jt = blockIdx.x; jt < a.ntw; jt += G, ++k) {
            const int x = k & 1;
            const uint32_t ph = (uint32_t)((k >> 1) & 1);
            const int64_t tile = tid_of(jt);
            const int64_t a0 = tile * kNodeTile;
            const int nn = (int)min(kNodeTile, a.n - a0);
            const bool valid = i < nn;
            const int64_t j = a0 + i;
            long long c0 = kProf ? clock64() : 0;
            bar_sync_n(kBarPFull + x, kRW + kPWt);
            // f, 1/sum w and the out-degree now; H and wr from P[x] again at the state out
            const int pi = x * (int)kNodeTile + i;
            double f = 0.0, pivi = 0.0;
            int32_t pdeg = 0;
            if (valid) {
                f = Pf[pi];
                pivi = Pivi[pi];
                pdeg = Pdeg[pi];
            }
            // delta in-edges inside the tile left by an edge update (R18, rare): pushed in the rounds
            int32_t db = 0, de = 0;
            if (kDl && (pdeg & kDegLocalDelta)) {
                pdeg &= kDegMask;
                db = a.dl_ptr[j];
                de = a.dl_ptr[j + 1];
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
            double D = 0.0, Hj = 0.0;
            float wrj = 0.f;
            for (int r = 0; r < a.rounds; ++r) {
                if (r == a.rounds - 1 && valid) {     // for the state out, in flight during the last round
                    Hj = a.H[j];
                    wrj = a.wr[j];
                }
                double q = 0.0;
                if (f != 0.0) {                      // invalid threads hold f = 0
                    D += f;                          // Eq. (10)
                    nodes += 1;
                    edges += (unsigned long long)pdeg;
                    q = d * f * pivi;                // d F(i) / sum_k w_{i,k}
                }
                const long long t9 = kProf ? clock64() : 0;
#pragma unroll
                for (int c = 0; c < kGqCopies; ++c) gq[c * kGqStride + i] = q;
                bar_sync_n(kBarRW, kRW);
                const long long ta = kProf ? clock64() : 0;
                if (kProf) b1_cyc += ta - t9;
                // Eq. (8) local pushes: the two virtual warps' loads interleave (a
                // shared counter handing out one virtual warp at a time was 20% slower)
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {               // this warp's two: longest with shortest
                    const int vw = h2 ? kVWarps - 1 - wp : wp;
                    const uint32_t o0 = vofs_s[vw];
                    const int K = (int)((vofs_s[vw + 1] - o0) >> 5);
                    if (K) {
                        double acc;
                        if ((int)o0 >= st) acc = local_sum<W>(es_sm, ew_sm, gq, (int)o0 + lane, K);
                        else acc = local_sum<W>(es_gl, ew_gl, gq, (int)o0 + lane, K);
                        psum[vw * 32 + lane] = acc;
                    }
                }
                double dl = 0.0;                      // (this round's gq, before the barrier)
                if constexpr (kDl)
                    for (int32_t u = db; u < de; ++u) dl += gq[a.dl_src[u]] * a.dl_w[u];
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
                    // the rest four at a time: ranks, then values, in flight together
                    for (int p = p0 + 4; p < p0 + np; p += 4) {
                        const int e = p0 + np;
                        const int q1 = p + 1 < e ? pl_s[p + 1] : 0, q2 = p + 2 < e ? pl_s[p + 2] : 0;
                        const int q3 = p + 3 < e ? pl_s[p + 3] : 0;
                        const double y0 = psum[pl_s[p]], y1 = p + 1 < e ? psum[q1] : 0.0;
                        const double y2 = p + 2 < e ? psum[q2] : 0.0, y3 = p + 3 < e ? psum[q3] : 0.0;
                        acc += y0;
                        if (p + 1 < e) acc += y1;
                        if (p + 2 < e) acc += y2;
                        if (p + 3 < e) acc += y3;
                    }
                    f = acc;
                } else {
                    f = 0.0;
                }
                if constexpr (kDl) f += dl;
                if (kProf) {
                    __syncwarp();
                    ns_cyc += clock64() - tc;
                }
            }
            long long c3 = kProf ? clock64() : 0;
            const long long c4 = c3, c5 = c3;
            // state out; the remote pushes leave as the outflow A (linearity of Eq. (8))
            if (valid) {
                a.F[j] = f;
                if (D != 0.0) a.H[j] = Hj + D;
                Anext[j] = d * D * pivi;
                // R13: the pushes still pending carry d D(i) P_{t,i} over the pending
                // out-edges t, i.e. |d D(i)| wr(i) with wr(i) = inv(i) sum_pending w
                resid += fabs(f) + fabs(d * D) * (double)wrj;
                if (pdeg == 0) leak += D;             // dangling: the fluid left the system (§3.3)
            }
            // P[x] and E[x] read by this warp: prep refills them for tile k + 2
            if (jt + 2 * G < a.ntw) bar_arrive_n(kBarPEmpty + x, kTileBlock);
            if (kProf) {                              // thread 0's counters, in registers until the end
                const long long c6 = clock64();
                pc[st == 0 ? 0 : 1] += c3 - c2;       // rounds of fully / partly staged tiles
                pn[st == 0 ? 0 : 1] += 1;
                pc[2] += c1 - c0;                     // waiting for the prepared rows
                pc[3] += c2 - c1;                     // waiting for the edge bundle
                pc[4] += c6 - c3;                     // state out
                pc[5] += c4 - c3;                     // state out: barrier
                pc[6] += c5 - c4;                     // state out: next bundle issued
                pc[7] += c6 - c5;                     // state out: stores
            }
        }
        if (kProf && i == 0) {
            dbg[10] += pc[0];
            dbg[11] += pn[0];
            dbg[12] += pc[1];
            dbg[13] += pn[1];
            dbg[0] += pc[2];
            dbg[1] += pc[3];
            dbg[2] += pc[0] + pc[1];
            dbg[3] += pc[4];
            dbg[32] += pc[5];
            dbg[33] += pc[6];
            dbg[34] += pc[7];
            dbg[7] += pn[0] + pn[1];
        }
        if (kProf && lane == 0) {
            atomicAdd(&dbg[8], (unsigned long long)ls_cyc);
            atomicAdd(&dbg[9], (unsigned long long)b2_cyc);
            atomicAdd(&dbg[14], (unsigned long long)ns_cyc);
            atomicAdd(&dbg[16 + wp], (unsigned long long)ls_cyc);
            atomicAdd(&dbg[15], (unsigned long long)b1_cyc);
        }
    } else if (tid >= kRW + kPWt) {
        // ------------------------------------------------ producer warp: the TMA issue
        // (a bulk copy's issue can stall ~1k cycles: off the round and prep warps)
        auto rscal = [&](int64_t jt, int64_t &r0, int64_t &r1) {
            const int64_t t = tid_of(jt);
            r0 = recs_on ? a.rtile[t] : 0;
            r1 = recs_on ? a.rtile[t + 1] : 0;
        };
        auto escal = [&](int64_t jt) {
            const int64_t t = tid_of(jt);
            return TileScalars{a.ltile[t], a.ltile[t + 1], a.lstage[t], 0};
        };
        if (lane == 0) {
            int64_t r0, r1;
            rscal(blockIdx.x, r0, r1);
            issue_records<W>(a, r0, r1, rbuf(0), R_full(0));
        }
        int k = 0;
        for (int64_t jt = blockIdx.x; jt < a.ntw; jt += G, ++k) {
            const int x = k & 1;
            // the light records of tile k + 1 once prep is done with tile k - 1
            if (jt + G < a.ntw) {
                if (k >= 1) bar_sync_n(kBarRFree + (x ^ 1), kPWt + 32);
                if (lane == 0) {
                    int64_t r0, r1;
                    rscal(jt + G, r0, r1);
                    issue_records<W>(a, r0, r1, rbuf(x ^ 1), R_full(x ^ 1));
                }
            }
            // the edge bundle of tile k once the round warps are done with tile k - 2
            if (k >= 2) bar_sync_n(kBarPEmpty + x, kTileBlock);
            if (lane == 0) {
                sc[x] = escal(jt);
                issue_edges<W>(a, tid_of(jt), sc[x], ebuf(x), E_full(x));
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------ prep warps
        const int p = tid - kRW;
        auto rscal = [&](int64_t jt, int64_t &r0, int64_t &r1) {
            const int64_t t = tid_of(jt);
            r0 = recs_on ? a.rtile[t] : 0;
            r1 = recs_on ? a.rtile[t + 1] : 0;
        };
        int k = 0;
        for (int64_t jt = blockIdx.x; jt < a.ntw; jt += G, ++k) {
            const int x = k & 1;
            const uint32_t ph = (uint32_t)((k >> 1) & 1);
            const int64_t tile = tid_of(jt);
            const int64_t a0 = tile * kNodeTile;
            const int nn = (int)min(kNodeTile, a.n - a0);
            long long c0 = kProf ? clock64() : 0;
            int64_t r0 = 0, r1 = 0;
            rscal(jt, r0, r1);
            // per-node state (independent loads, in flight together): nodes p, p + kPWt, ..
            double Fj[kPN], ivi[kPN];
            int32_t dg[kPN], hx[kPN];
            int rb[kPN], re[kPN];
#pragma unroll
            for (int u = 0; u < kPN; ++u) {
                const int q = p + u * kPWt;
                const int64_t j = a0 + q;
                Fj[u] = ivi[u] = 0.0;
                dg[u] = 0;
                hx[u] = -1;
                rb[u] = re[u] = 0;
                if (q < nn) {
                    Fj[u] = a.F[j];
                    ivi[u] = a.inv[j];
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
#ifdef DIT_ABL_NOPREP
            const int R = 0;
#else
            const int R = (int)(r1 - r0);
#endif
            // remote pushes still pending: from the previous sweep, and from this
            // sweep's earlier waves (R15): light records' gathered outflow, in place
            // in batches of kRecUnroll records per thread, every gather of a batch
            // issued (predicated) before the first product is stored: a loop with a
            // run-time trip count of ~4 ran in the compiler's remainder loop, one
            // dependent HBM gather after another
            for (int q0 = p; q0 < R; q0 += kRecUnroll * kPWt) {
                RemRec<W> rc[kRecUnroll];
                double v[kRecUnroll];
#pragma unroll
                for (int u = 0; u < kRecUnroll; ++u) {
                    const int q = q0 + u * kPWt;
                    if (q < R) rc[u] = recs[q];
                }
#pragma unroll
                for (int u = 0; u < kRecUnroll; ++u) {
                    const int q = q0 + u * kPWt;
                    v[u] = 0.0;
                    if (q < R) {
                        const bool early = tile_wave(rc[u].src, a.waves) < a.wave;
                        if (early || gather) v[u] = (early ? Anext : Aprev)[rc[u].src];
                    }
                }
#pragma unroll
                for (int u = 0; u < kRecUnroll; ++u) {
                    const int q = q0 + u * kPWt;
                    if (q < R) *reinterpret_cast<double *>(&recs[q]) = v[u] * rec_w(rc[u]);
                }
            }
            double hs[kPN];
#pragma unroll
            for (int u = 0; u < kPN; ++u) hs[u] = hx[u] >= 0 ? a.hsum[hx[u]] : 0.0;
            const long long c1g = kProf ? clock64() : 0;
            bar_sync_n(kBarPW, kPWt);
            const long long c1b = kProf ? clock64() : 0;
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
                if (p + u * kPWt < nn) {
                    const int q = x * (int)kNodeTile + p + u * kPWt;
                    Pf[q] = Fj[u] + sm[u] + hs[u];
                    Pivi[q] = ivi[u];
                    Pdeg[q] = dg[u];
                }
            bar_arrive_n(kBarPFull + x, kRW + kPWt);
            if (jt + 2 * G < a.ntw) bar_arrive_n(kBarRFree + x, kPWt + 32);   // R[x] read: the producer refills it
            if (kProf && p == 0) {
                dbg[4] += c1 - c0;                    // node loads + waiting for the records
                dbg[5] += c2 - c1;                    // gathers + sums
                dbg[35] += c1g - c1;                  // gathers (this thread)
                dbg[36] += c1b - c1g;                 // waiting for the other prep warps
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
    a.dl_ptr = tp.nd > 0 ? tp.dl_ptr : nullptr;
    a.dl_src = tp.dl_src;
    a.dl_w = tp.dl_w;
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
        DI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_heavy_chunks<W>, kHeavyThreads, 0));
        if (v < 1) v = 1;
    }
    return v;
}

// the heavy targets' remote inflow hsum of one wave: chunks by ticket, then the fold
template <typename W>
static void launch_heavy_t(di_graph *h, int wave, int force, int group = -1) {
    TilePlan &tp = h->g.tl;
    State &s = h->s;
    if (tp.nh == 0) return;
    if (group < 0) group = wave;                     // the ghost group gathers with wave 0's rule
    const int64_t S = tp.nstripe, g0 = (int64_t)group * S;
    const int64_t t0 = tp.wave_slot[group], t1 = tp.wave_slot[group + 1];
    // one launch over the wave's stripes in stripe order: the CTAs stride over the
    // chunks statically and advance together, so the gathered slice of A
    // (kStripeBytes) of the stripe being worked on stays L2-resident (one launch
    // per stripe was 4% slower at configs[2]: 8 launch tails per wave)
    const int64_t a0 = tp.s_chunk[g0], a1 = tp.s_chunk[g0 + S];
    if (a1 > a0) {
        const int grid = (int)std::min<int64_t>(a1 - a0, (int64_t)h->num_sms * heavy_ctas_per_sm<W>());
        k_heavy_chunks<W><<<grid, kHeavyThreads, 0, h->stream>>>((const RemRec<W> *)tp.hrec, tp.chunk_start, tp.seg_start,
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
        for (auto f : {k_tile<W, false, false>, k_tile<W, true, false>, k_tile<W, false, true>, k_tile<W, true, true>})
            DI_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_smem_bytes<W>()));
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
    // the variant with in-round delta in-edges only after an edge update left some (R18)
    auto kern = a.dl_ptr ? (a.dbg ? k_tile<W, true, true> : k_tile<W, false, true>)
                         : (a.dbg ? k_tile<W, true, false> : k_tile<W, false, false>);
    kern<<<grid, kTileBlock, tile_smem_bytes<W>(), h->stream>>>(a, s.ctrl);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

template <typename W>
static void launch_tile_t(di_graph *h, int rounds) {
    const int64_t k = h->s.launched;
    for (int c = 0; c < h->g.tl.waves; ++c) {          // events: [2c] heavy(c) [2c+1] tile(c) [2c+2]
        launch_heavy_t<W>(h, c, 0);
        launch_delta(h, c, 0);
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
void launch_tile_heavy(di_graph *h, int force, int wave, int group) {
    if (h->g.tl.ntile == 0) return;
    switch (h->g.w_kind) {
    case DI_W_F32: launch_heavy_t<float>(h, wave, force, group); break;
    case DI_W_F64: launch_heavy_t<double>(h, wave, force, group); break;
    default: launch_heavy_t<NoW>(h, wave, force, group);
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
    for (int c = 0; c < h->g.tl.waves; ++c) {
        launch_heavy_t<W>(h, c, 1);
        launch_delta(h, c, 1);
    }
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
