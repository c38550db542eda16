// dit_delta.cu -- Theorem 4 edge updates without a tile-plan rebuild (R18).
//
// PAPER §3.5 (Theorem 4): after P -> P' the corrective fluid d (P' - P) H makes
// D-Iteration converge to the new fixed point from the old H; the update itself
// (dit_graph.cu: new CSR, new scales inv', withdraw / inject over the changed
// columns) is exact.  The sweep then needs the pushes of P' = inv' W'.  The
// tile plan holds the raw weights W of the graph it was built from and k_tile
// multiplies them by the CURRENT inv, so P' is reached by keeping the plan and
// applying W' - W to it (Eq. (8) is linear in the pushed weight):
//  - an edge inside one tile (80% of the added edges of a web graph) patches the
//    plan's sliced-ELL slots of its target: a removal turns its slot into
//    padding, an addition takes a padding slot (k_patch_ell), so it is pushed
//    in every local round like any plan-local edge (kept as a delta entry it
//    would move one hop per sweep: a two-node cycle of added edges then decays
//    only by d per sweep -- measured 29 instead of 18 sweeps at 5M nodes);
//  - the others (across tiles, or no padding slot left) become "delta" in-edges,
//    +w added / -w removed, handled like remote edges: per target wave, before
//    the wave's k_tile, F(t) += sum A(s) w over t's entries (A = d D inv of the
//    sources, this sweep's for sources of earlier waves, the previous sweep's
//    otherwise: the heavy gather's rule, R15); the final flush takes the
//    pending ones.  The stop estimate (R13) counts them as pending: wr'(i) =
//    inv'(i) x (plan-time pending out-weight + sum |w| of i's pending entries).
// Every sum has a fixed order (entries sorted by (wave, target, source), input
// order within): bitwise reproducible.
#include "dit_tile.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace dit {

namespace {

// pending out-weight of node i in the plan built from this CSR (the predicate of
// k_remote_share: leaves the tile and a later wave does not take it in this sweep)
template <typename Wt>
__global__ void k_pending_w(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                            const Wt *__restrict__ w, int64_t n, int waves, double *__restrict__ rw0) {
    const unsigned lane = lane_id();
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        if (i < n) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        if (i < n && e - b <= 32) {
            const int wi = tile_wave(i, waves);
            double s = 0.0;
            for (int64_t q = b; q < e; ++q) {
                const int64_t t = col[q];
                if ((t >> 9) != (i >> 9) && tile_wave(t, waves) <= wi) s += w ? (double)w[q] : 1.0;
            }
            rw0[i] = s;
        }
        for (unsigned big = __ballot_sync(0xffffffffu, i < n && e - b > 32); big; big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int64_t il = __shfl_sync(0xffffffffu, i, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            const int wi = tile_wave(il, waves);
            double s = 0.0;
            for (int64_t q = bl + lane; q < el; q += 32) {
                const int64_t t = col[q];
                if ((t >> 9) != (il >> 9) && tile_wave(t, waves) <= wi) s += w ? (double)w[q] : 1.0;
            }
            s = warp_sum(s);
            if (lane == 0) rw0[il] = s;
        }
    }
}

// removed CSR entries per changed row (old CSR, before the swap): a thread per
// row of <= 32 entries, a warp per longer one (ballot prefix: row order kept)
__global__ void k_del_count(const int64_t *__restrict__ row_ptr, const unsigned char *__restrict__ del,
                            const unsigned char *__restrict__ chg, int64_t n, int64_t *__restrict__ cnt) {
    const unsigned lane = lane_id();
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        const bool c = i < n && chg[i];
        if (c) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        if (i < n && e - b <= 32) {
            int64_t k = 0;
            for (int64_t q = b; q < e; ++q) k += del[q];
            cnt[i] = k;
        }
        for (unsigned big = __ballot_sync(0xffffffffu, e - b > 32); big; big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int64_t il = __shfl_sync(0xffffffffu, i, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            int64_t k = 0;
            for (int64_t q = bl + lane; q < el; q += 32) k += del[q];
            k = warp_sum(k);
            if (lane == 0) cnt[il] = k;
        }
    }
}

template <typename Wt>
__global__ void k_del_emit(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                           const Wt *__restrict__ w, const unsigned char *__restrict__ del,
                           const unsigned char *__restrict__ chg, const int64_t *__restrict__ pos, int64_t n,
                           int32_t *__restrict__ es, int32_t *__restrict__ et, double *__restrict__ ew) {
    const unsigned lane = lane_id();
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        if (i < n && chg[i]) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        if (i < n && e - b <= 32 && e > b) {
            int64_t p = pos[i];
            for (int64_t q = b; q < e; ++q)
                if (del[q]) {
                    es[p] = (int32_t)i;
                    et[p] = col[q];
                    ew[p] = -(w ? (double)w[q] : 1.0);
                    ++p;
                }
        }
        for (unsigned big = __ballot_sync(0xffffffffu, e - b > 32); big; big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int64_t il = __shfl_sync(0xffffffffu, i, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            int64_t p = pos[il];
            for (int64_t q0 = bl; q0 < el; q0 += 32) {
                const int64_t q = q0 + lane;
                const bool d = q < el && del[q];
                const unsigned m = __ballot_sync(0xffffffffu, d);
                if (d) {
                    const int64_t at = p + __popc(m & ((1u << lane) - 1u));
                    es[at] = (int32_t)il;
                    et[at] = col[q];
                    ew[at] = -(w ? (double)w[q] : 1.0);
                }
                p += __popc(m);
            }
        }
    }
}

__global__ void k_add_emit(const int32_t *__restrict__ as, const int32_t *__restrict__ ad,
                           const double *__restrict__ aw, int64_t cnt, int32_t *__restrict__ es,
                           int32_t *__restrict__ et, double *__restrict__ ew) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        es[q] = as[q];
        et[q] = ad[q];
        ew[q] = aw ? aw[q] : 1.0;
    }
}

// sort keys over the current permutation: 0 source, 1 target, 2 wave of the target
__global__ void k_delta_keys(const int32_t *__restrict__ es, const int32_t *__restrict__ et,
                             const uint32_t *__restrict__ perm, int64_t cnt, int what, int waves,
                             uint32_t *__restrict__ key) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = perm[q];
        key[q] = what == 0 ? (uint32_t)es[r] : (what == 1 ? (uint32_t)et[r] : (uint32_t)tile_wave(et[r], waves));
    }
}

__global__ void k_delta_gather_perm(const int32_t *__restrict__ es, const int32_t *__restrict__ et,
                                    const double *__restrict__ ew, const uint32_t *__restrict__ perm, int64_t cnt,
                                    int32_t *__restrict__ os, int32_t *__restrict__ ot, double *__restrict__ ow) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r = perm[q];
        os[q] = es[r];
        ot[q] = et[r];
        ow[q] = ew[r];
    }
}

// changed nodes: plan degree from the new CSR; pending share from the plan-time
// pending weight plus |w| of the node's pending delta entries (sorted by source)
__global__ void k_delta_wr(const int64_t *__restrict__ row_ptr, const unsigned char *__restrict__ chg,
                           const double *__restrict__ inv, const double *__restrict__ rw0,
                           const int32_t *__restrict__ ss, const int32_t *__restrict__ st,
                           const double *__restrict__ sw, int64_t cnt, int64_t n, int waves,
                           float *__restrict__ wr, int32_t *__restrict__ deg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!chg[i]) continue;
        int64_t lo = 0, hi = cnt;                    // first entry with source >= i
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ss[mid] < i) lo = mid + 1;
            else hi = mid;
        }
        const int wi = tile_wave(i, waves);
        double a = 0.0;
        for (int64_t q = lo; q < cnt && ss[q] == i; ++q)   // entries inside the tile: pushed in the rounds
            if ((st[q] >> 9) != (i >> 9) && tile_wave(st[q], waves) <= wi) a += fabs(sw[q]);
        wr[i] = (float)(inv[i] * (rw0[i] + a));
        deg[i] = (int32_t)(row_ptr[i + 1] - row_ptr[i]) | (deg[i] & kDegLocalDelta);
    }
}

// first entry of each target wave in the (wave, target, source)-sorted list
__global__ void k_delta_waves(const int32_t *__restrict__ dt, int64_t cnt, int waves, int64_t *__restrict__ first) {
    const int c = (int)threadIdx.x;
    if (c > waves) return;
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (tile_wave(dt[mid], waves) < c) lo = mid + 1;
        else hi = mid;
    }
    first[c] = lo;
}

// the delta pushes of one wave's entries (force: the flush, pending ones only):
// every entry's A(s) w first (all gathers independent), then per target segment
__global__ void k_delta_vals(const int32_t *__restrict__ ds, const int32_t *__restrict__ dt,
                             const double *__restrict__ dw, int64_t q0, int64_t q1, const double *__restrict__ A0,
                             const double *__restrict__ A1, double *__restrict__ v, int wave, int waves,
                             const Ctrl *__restrict__ ctrl, int force) {
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool gather = ctrl->gather != 0;
    if (force ? !gather : (!gather && wave == 0)) return;
    const double *__restrict__ Aprev = (ctrl->sweeps & 1) ? A0 : A1;
    const double *__restrict__ Afresh = (ctrl->sweeps & 1) ? A1 : A0;
    for (int64_t q = q0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < q1;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = ds[q];
        const bool early = tile_wave(s, waves) < wave;
        // entries inside one tile are pushed within k_tile's rounds (dl list), not here
        const bool local = (s >> 9) == (dt[q] >> 9);
        v[q] = (!local && (force ? !early : (early || gather))) ? (early && !force ? Afresh : Aprev)[s] * dw[q] : 0.0;
    }
}

constexpr int64_t kBigSeg = 4096;               // longer target segments: a block each

// F(t) += the sum of t's entries: a thread per segment of <= 32 entries (in
// order), a warp per longer one (four lane-strided partial sums, butterfly),
// k_delta_big for segments of more than kBigSeg: every order fixed
__global__ void k_delta_seg(const int64_t *__restrict__ seg, const int32_t *__restrict__ dt,
                            const double *__restrict__ v, int64_t s0, int64_t s1, double *__restrict__ F, int wave,
                            const Ctrl *__restrict__ ctrl, int force) {
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool gather = ctrl->gather != 0;
    if (force ? !gather : (!gather && wave == 0)) return;
    const unsigned lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = s0 + gw * 32; base < s1; base += nw * 32) {
        const int64_t k = base + lane;
        int64_t b = 0, e = 0;
        if (k < s1) {
            b = seg[k];
            e = seg[k + 1];
        }
        if (k < s1 && e - b <= 32) {
            double acc = 0.0;
            for (int64_t q = b; q < e; ++q) acc += v[q];
            const int32_t t = dt[b];
            F[t] = F[t] + acc;
        }
        for (unsigned big = __ballot_sync(0xffffffffu, k < s1 && e - b > 32 && e - b <= kBigSeg); big;
             big &= big - 1) {
            const int l = __ffs(big) - 1;
            const int64_t bb = __shfl_sync(0xffffffffu, b, l), be = __shfl_sync(0xffffffffu, e, l);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
            int64_t q = bb + lane;
            for (; q + 96 < be; q += 128) {
                a0 += v[q];
                a1 += v[q + 32];
                a2 += v[q + 64];
                a3 += v[q + 96];
            }
            for (; q < be; q += 32) a0 += v[q];
            const double acc = warp_sum((a0 + a1) + (a2 + a3));
            if (lane == 0) F[dt[bb]] = F[dt[bb]] + acc;
        }
    }
}

// one 1024-thread block per segment of more than kBigSeg entries (hub targets
// of the added edges): eight partial sums per thread, then a fixed-order tree
__global__ void __launch_bounds__(1024) k_delta_big(const int64_t *__restrict__ seg, const int64_t *__restrict__ big,
                                                    int64_t b0, const int32_t *__restrict__ dt,
                                                    const double *__restrict__ v, double *__restrict__ F, int wave,
                                                    const Ctrl *__restrict__ ctrl, int force) {
    if (!force && (ctrl->done || ctrl->use_pull != kUseTiled)) return;
    const bool gather = ctrl->gather != 0;
    if (force ? !gather : (!gather && wave == 0)) return;
    __shared__ double ws[32];
    const int64_t sg = big[b0 + blockIdx.x], bb = seg[sg], be = seg[sg + 1];
    double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int64_t q = bb + threadIdx.x;
    for (; q + 7 * 1024 < be; q += 8 * 1024) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += v[q + u * 1024];
    }
    for (; q < be; q += 1024) a[0] += v[q];
    const double w = warp_sum(((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7])));
    if (lane_id() == 0) ws[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x < 32) {
        const double x = warp_sum(ws[threadIdx.x]);
        if (threadIdx.x == 0) F[dt[bb]] = F[dt[bb]] + x;
    }
}

__global__ void k_delta_bigflag(const int64_t *__restrict__ seg, int64_t nseg, int64_t *__restrict__ flag) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nseg; k += (int64_t)gridDim.x * blockDim.x)
        flag[k] = seg[k + 1] - seg[k] > kBigSeg ? 1 : 0;
}

__global__ void k_delta_bigput(const int64_t *__restrict__ seg, int64_t nseg, const int64_t *__restrict__ pos,
                               int64_t *__restrict__ big) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nseg; k += (int64_t)gridDim.x * blockDim.x)
        if (seg[k + 1] - seg[k] > kBigSeg) big[pos[k]] = k;
}

// (target, source) order: one warp per target with new entries inside its
// tile patches the target's sliced-ELL slots (dit_tile.cuh layout): a removal
// (-w) turns one slot {source, w} into padding, an addition (+w) takes a
// padding slot (source = its index in the tile, gq copy 0).  The warp walks the
// target's pieces 32 slots at a time; each entry in order takes the lowest
// matching slot (ballot).  keep[r] = 0 for an entry so placed; the rest stay
// delta entries (remote pushes).
template <typename W>
__global__ void k_patch_ell(const int32_t *__restrict__ ds, const int32_t *__restrict__ dt,
                            const double *__restrict__ dw, const uint32_t *__restrict__ perm, int64_t cnt,
                            int64_t nold, const int64_t *__restrict__ ltile, const uint32_t *__restrict__ vofs,
                            const uint16_t *__restrict__ vfirst, const uint16_t *__restrict__ plist,
                            uint16_t *__restrict__ lsrc, StoreW<W> *__restrict__ lw, unsigned char *keep) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    const int lane = (int)lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t q = gw; q < cnt; q += nw) {
        if (q > 0 && dt[q - 1] == dt[q]) continue;       // warp-uniform: the warp of the run's first entry
        const int32_t t = dt[q];
        const int64_t tile = t >> 9;
        // the run's entries with a source in t's tile: a contiguous range of the
        // (target, source) order, found by binary search (hub runs are long)
        auto lower = [&](int64_t lo, int32_t sv) {
            int64_t hi = cnt;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (dt[mid] < t || (dt[mid] == t && ds[mid] < sv)) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
        // most runs are short: their first 32 entries in one coalesced load decide
        const int64_t r0 = q + lane;
        const bool in = r0 < cnt && dt[r0] == t;
        const int32_t sv = in ? ds[r0] : 0;
        const unsigned m_in = __ballot_sync(0xffffffffu, in);
        const unsigned m_lo = __ballot_sync(0xffffffffu, in && sv < (int32_t)(tile << 9));
        const unsigned m_hi = __ballot_sync(0xffffffffu, in && sv < (int32_t)((tile + 1) << 9));
        int64_t lo, qe;
        if (m_in != 0xffffffffu) {                       // the run ends inside the first 32
            lo = q + __popc(m_lo);
            qe = q + __popc(m_hi);
        } else {
            lo = lower(q, (int32_t)(tile << 9));
            qe = lower(lo, (int32_t)((tile + 1) << 9));
        }
        if (qe <= lo) continue;
        bool any = false;                                // this run's new entries inside the tile
        for (int64_t r = lo + lane; r < qe; r += 32) {
            const bool mine = perm[r] >= nold;
            if (mine) keep[r] = 2;                       // 2: still to place
            any |= mine;
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        __syncwarp();
        const int i = t & 511;
        const int p0 = vfirst[tile * kVfStride + i], p1 = vfirst[tile * kVfStride + i + 1];
        const int64_t base = ltile[tile];
        for (int pass = 0; pass < 2; ++pass)             // removals first: their slots become free padding
        for (int p = p0; p < p1; ++p) {                  // the target's pieces, their slots
            const int rk = plist[tile * kVRows + p];
            const int vw = rk >> 5, pl = rk & 31;
            const int64_t o = base + vofs[tile * kVofsStride + vw];
            const int64_t K = (vofs[tile * kVofsStride + vw + 1] - vofs[tile * kVofsStride + vw]) >> 5;
            for (int64_t s0 = 0; s0 < K; s0 += 32) {
                const int64_t sl_ = s0 + lane;
                const bool valid = sl_ < K;
                const int64_t k = valid ? o + ell_slot(sl_, pl, K) : 0;
                int src = valid ? lsrc[k] % kGqStride : -1;
                double wv = 0.0;
                if constexpr (kW) wv = valid ? (double)lw[k] : 0.0;
                for (int64_t r = lo; r < qe; ++r) {
                    if (keep[r] != 2) continue;          // warp-uniform (written by lane 0 below)
                    const int sr = ds[r] & 511;
                    const double w = dw[r];
                    if ((w < 0.0) != (pass == 0)) continue;
                    const bool match = valid && (w < 0.0 ? (src == sr && (!kW || wv == -w)) : src >= (int)kNodeTile);
                    const unsigned m = __ballot_sync(0xffffffffu, match);
                    if (m) {
                        if (lane == __ffs(m) - 1) {
                            src = w < 0.0 ? (int)kNodeTile : sr;
                            wv = w < 0.0 ? 0.0 : w;
                            lsrc[k] = (uint16_t)src;     // padding reads a zero gq slot
                            if constexpr (kW) lw[k] = (StoreW<W>)wv;
                        }
                        if (lane == 0) keep[r] = 0;
                        __syncwarp();
                    }
                }
            }
        }
        for (int64_t r = lo + lane; r < qe; r += 32)
            if (keep[r] == 2) keep[r] = 1;              // no slot: stays a delta entry
    }
}

// kept entries inside one tile (no padding slot for them): pushed in k_tile's
// rounds through the per-node list dl_ptr[t] .. dl_ptr[t+1] {source - tile base, w}
__global__ void k_delta_localflag(const int32_t *__restrict__ ds, const int32_t *__restrict__ dt, int64_t cnt,
                                  int64_t *__restrict__ flag) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        flag[q] = (ds[q] >> 9) == (dt[q] >> 9) ? 1 : 0;
}

__global__ void k_delta_localput(const int32_t *__restrict__ ds, const int32_t *__restrict__ dt,
                                 const double *__restrict__ dw, int64_t cnt, const int64_t *__restrict__ pos,
                                 uint16_t *__restrict__ ls, int32_t *__restrict__ lt, double *__restrict__ lw) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        if ((ds[q] >> 9) == (dt[q] >> 9)) {
            const int64_t p = pos[q];
            ls[p] = (uint16_t)(ds[q] & 511);
            lt[p] = dt[q];
            lw[p] = dw[q];
        }
}

__global__ void k_delta_localcnt(const int32_t *__restrict__ lt, int64_t cnt, int64_t *__restrict__ c) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x) {
        if (q > 0 && lt[q - 1] == lt[q]) continue;
        int64_t r = q;
        while (r < cnt && lt[r] == lt[q]) ++r;
        c[lt[q]] = r - q;
    }
}

// dl_ptr from the per-node counts' scan; the plan degree's bit 30 flags a node with such entries
__global__ void k_delta_localptr(const int64_t *__restrict__ cs, const int64_t *__restrict__ c, int64_t n,
                                 int32_t *__restrict__ ptr, int32_t *__restrict__ deg) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= n; q += (int64_t)gridDim.x * blockDim.x) {
        ptr[q] = (int32_t)cs[q];
        if (q < n) deg[q] = (deg[q] & kDegMask) | (c[q] > 0 ? kDegLocalDelta : 0);
    }
}

__global__ void k_flag_u8(const unsigned char *__restrict__ keep, int64_t cnt, int64_t *__restrict__ flag) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        flag[q] = keep[q];
}

__global__ void k_compact(const int32_t *__restrict__ ds, const int32_t *__restrict__ dt,
                          const double *__restrict__ dw, const unsigned char *__restrict__ keep,
                          const int64_t *__restrict__ pos, int64_t cnt, int32_t *__restrict__ os,
                          int32_t *__restrict__ ot, double *__restrict__ ow) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        if (keep[q]) {
            const int64_t p = pos[q];
            os[p] = ds[q];
            ot[p] = dt[q];
            ow[p] = dw[q];
        }
}

// segment starts: flag[q] = 1 where a target's run begins
__global__ void k_delta_flags(const int32_t *__restrict__ dt, int64_t cnt, int64_t *__restrict__ flag) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        flag[q] = (q == 0 || dt[q - 1] != dt[q]) ? 1 : 0;
}

__global__ void k_delta_starts(const int32_t *__restrict__ dt, int64_t cnt, const int64_t *__restrict__ pos,
                               int64_t *__restrict__ seg) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        if (q == 0 || dt[q - 1] != dt[q]) seg[pos[q]] = q;
    if (blockIdx.x == 0 && threadIdx.x == 0) seg[pos[cnt]] = cnt;
}

__global__ void k_iota(uint32_t *__restrict__ v, int64_t cnt) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        v[q] = (uint32_t)q;
}

template <typename T>
T *dalloc(int64_t count, cudaStream_t st) {
    T *p = nullptr;
    DI_CUDA(cudaMallocAsync(&p, (count > 0 ? count : 1) * sizeof(T), st));
    return p;
}

}  // namespace

bool delta_enabled(const di_graph *h) {
    return h->g.tl.built && !h->g.shard && h->g.tl.ntile > 0 && !getenv("DIT_NO_DELTA");
}

// Before the CSR swap (old CSR resident): the plan-time pending weights (first
// update since the plan build) and the removed entries (-w), in row order.
void delta_collect_removed(di_graph *h, const unsigned char *del, const unsigned char *chg, DeltaBatch &out,
                           bool plan) {
    DevGraph &g = h->g;
    TilePlan &tp = g.tl;
    cudaStream_t st = h->stream;
    const int64_t n = g.n;
    if (plan && !tp.rw0) {
        tp.rw0 = dalloc<double>(n, st);
        if (g.w_kind == DI_W_F64)
            k_pending_w<double><<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, g.col, (const double *)g.w, n, tp.waves,
                                                                 tp.rw0);
        else
            k_pending_w<float><<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, g.col, (const float *)g.w, n, tp.waves,
                                                                tp.rw0);
        count_launch();
    }
    int64_t *cnt = dalloc<int64_t>(n, st), *pos = dalloc<int64_t>(n + 1, st);
    k_del_count<<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, del, chg, n, cnt);
    count_launch();
    exclusive_scan_i64(cnt, pos, n, st);
    int64_t nrem = 0;
    DI_CUDA(cudaMemcpyAsync(&nrem, pos + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    out.nrem = nrem;
    out.s = dalloc<int32_t>(nrem, st);
    out.t = dalloc<int32_t>(nrem, st);
    out.w = dalloc<double>(nrem, st);
    if (nrem > 0) {
        if (g.w_kind == DI_W_F64)
            k_del_emit<double><<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, g.col, (const double *)g.w, del, chg, pos, n,
                                                                out.s, out.t, out.w);
        else
            k_del_emit<float><<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, g.col, (const float *)g.w, del, chg, pos, n,
                                                               out.s, out.t, out.w);
        count_launch();
    }
    DI_CUDA(cudaFreeAsync(cnt, st));
    DI_CUDA(cudaFreeAsync(pos, st));
    DI_CUDA(cudaGetLastError());
}

void delta_batch_free(DeltaBatch &b, cudaStream_t st) {
    for (void *p : {(void *)b.s, (void *)b.t, (void *)b.w})
        if (p) cudaFreeAsync(p, st);
    b = DeltaBatch();
}

// After the CSR swap and the new scales: the plan's old entries + this update's
// removed (-w) and added (+w) ones.  (1) in (target, source) order, the new
// entries inside one tile patch the plan's sliced-ELL slots of their target
// (k_patch_ell: a removal turns a matching slot into padding, an addition takes
// a padding slot), (2) the rest -- across tiles, or no slot found -- sorted by
// source for the pending shares and degrees of the changed nodes, then by
// (wave, target, source) for the per-wave gathers.
template <typename SW>
static void patch_ell(di_graph *h, const int32_t *ss, const int32_t *stg, const double *sw, const uint32_t *perm,
                      int64_t N, int64_t nold, unsigned char *keep) {
    TilePlan &tp = h->g.tl;
    DI_CUDA(cudaMemsetAsync(keep, 1, N > 0 ? N : 1, h->stream));
    k_patch_ell<SW><<<grid_for(h, N), 256, 0, h->stream>>>(ss, stg, sw, perm, N, nold, tp.ltile, tp.vofs, tp.vfirst,
                                                          tp.plist, tp.lsrc, (StoreW<SW> *)tp.lw, keep);
    count_launch();
}

void delta_commit(di_graph *h, DeltaBatch &rem, const int32_t *as, const int32_t *ad, const double *aw, int64_t nadd,
                  const unsigned char *chg) {
    DevGraph &g = h->g;
    TilePlan &tp = g.tl;
    cudaStream_t st = h->stream;
    const int64_t n = g.n, nold = tp.nd, N = nold + rem.nrem + nadd;
    if (N >= (int64_t)1 << 31) {
        set_error("di_update_edges: more than 2^31 pending delta edges");
        throw Fail{DI_ERR_INVALID};
    }
    std::vector<void *> tmp;
    auto track = [&](void *p) { tmp.push_back(p); return p; };
    auto sync_read = [&](const int64_t *p) {
        int64_t v = 0;
        DI_CUDA(cudaMemcpyAsync(&v, p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        return v;
    };
    int bn = 1;
    while (bn < 32 && ((int64_t)1 << bn) < n + 1) ++bn;
    int bw = 1;
    while (((int64_t)1 << bw) < tp.waves + 1) ++bw;
    try {
        int32_t *es = (int32_t *)track(dalloc<int32_t>(N, st)), *et = (int32_t *)track(dalloc<int32_t>(N, st));
        double *ew = (double *)track(dalloc<double>(N, st));
        int32_t *ss = (int32_t *)track(dalloc<int32_t>(N, st)), *stg = (int32_t *)track(dalloc<int32_t>(N, st));
        double *sw = (double *)track(dalloc<double>(N, st));
        uint32_t *k0 = (uint32_t *)track(dalloc<uint32_t>(N, st)), *k1 = (uint32_t *)track(dalloc<uint32_t>(N, st));
        uint32_t *v0 = (uint32_t *)track(dalloc<uint32_t>(N, st)), *v1 = (uint32_t *)track(dalloc<uint32_t>(N, st));
        int64_t *flag = (int64_t *)track(dalloc<int64_t>(N, st)), *pos = (int64_t *)track(dalloc<int64_t>(N + 1, st));
        unsigned char *keep = (unsigned char *)track(dalloc<unsigned char>(N, st));
        int64_t *wf = (int64_t *)track(dalloc<int64_t>(tp.waves + 1, st));
        // entries in a deterministic order: the plan's, the removed (row order), the added (input order)
        if (nold > 0) {
            DI_CUDA(cudaMemcpyAsync(es, tp.dsrc, nold * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(et, tp.dtgt, nold * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(ew, tp.dw, nold * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        if (rem.nrem > 0) {
            DI_CUDA(cudaMemcpyAsync(es + nold, rem.s, rem.nrem * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(et + nold, rem.t, rem.nrem * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(ew + nold, rem.w, rem.nrem * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        if (nadd > 0) {
            k_add_emit<<<grid_for(h, nadd), 256, 0, st>>>(as, ad, aw, nadd, es + nold + rem.nrem, et + nold + rem.nrem,
                                                          ew + nold + rem.nrem);
            count_launch();
        }
        // stable LSD sorts of a permutation (dit_pull.cu radix) by `what` (0 source,
        // 1 target, 2 target wave) of the entries (xs, xt)
        auto sort_perm = [&](const int32_t *xs, const int32_t *xt, int64_t cnt, std::initializer_list<int> whats) {
            k_iota<<<grid_for(h, cnt), 256, 0, st>>>(v0, cnt);
            count_launch();
            uint32_t *perm = v0, *pother = v1;
            for (int what : whats) {
                k_delta_keys<<<grid_for(h, cnt), 256, 0, st>>>(xs, xt, perm, cnt, what, tp.waves, k0);
                count_launch();
                const auto r = radix_sort_u32(k0, perm, k1, pother, cnt, what == 2 ? bw : bn, st);
                if (r.second != perm) {
                    pother = perm;
                    perm = r.second;
                }
            }
            return perm;
        };
        phase_mark(st, "delta: entries");
        // (1) (target, source) order; the new entries inside a tile patch the ELL
        uint32_t *perm = sort_perm(es, et, N, {0, 1});
        k_delta_gather_perm<<<grid_for(h, N), 256, 0, st>>>(es, et, ew, perm, N, ss, stg, sw);
        count_launch();
        phase_mark(st, "delta: sort (target, source)");
        switch (g.w_kind) {
        case DI_W_F32: patch_ell<float>(h, ss, stg, sw, perm, N, nold, keep); break;
        case DI_W_F64: patch_ell<double>(h, ss, stg, sw, perm, N, nold, keep); break;
        default: patch_ell<NoW>(h, ss, stg, sw, perm, N, nold, keep);
        }
        phase_mark(st, "delta: patch ELL");
        // (2) the kept entries, compacted in (target, source) order
        k_flag_u8<<<grid_for(h, N), 256, 0, st>>>(keep, N, flag);
        count_launch();
        exclusive_scan_i64(flag, pos, N, st);
        const int64_t M = sync_read(pos + N);
        k_compact<<<grid_for(h, N), 256, 0, st>>>(ss, stg, sw, keep, pos, N, es, et, ew);
        count_launch();
        // kept entries inside one tile, (target, source) order: the in-round list
        k_delta_localflag<<<grid_for(h, M), 256, 0, st>>>(es, et, M, flag);
        count_launch();
        exclusive_scan_i64(flag, pos, M, st);
        const int64_t nl = sync_read(pos + M);
        if (getenv("DIT_BUILD_TIMING"))
            fprintf(stderr, "[dit] delta entries %lld -> kept %lld (inside a tile, in-round: %lld)\n", (long long)N,
                    (long long)M, (long long)nl);
        uint16_t *lsrc = dalloc<uint16_t>(nl, st);
        double *lwt = dalloc<double>(nl, st);
        int32_t *lptr = dalloc<int32_t>(n + 1, st);
        track(lsrc), track(lwt), track(lptr);
        {
            int32_t *ltg = (int32_t *)track(dalloc<int32_t>(nl, st));
            int64_t *lc = (int64_t *)track(dalloc<int64_t>(n, st)), *lcp = (int64_t *)track(dalloc<int64_t>(n + 1, st));
            k_delta_localput<<<grid_for(h, M), 256, 0, st>>>(es, et, ew, M, pos, lsrc, ltg, lwt);
            DI_CUDA(cudaMemsetAsync(lc, 0, (n > 0 ? n : 1) * sizeof(int64_t), st));
            k_delta_localcnt<<<grid_for(h, nl), 256, 0, st>>>(ltg, nl, lc);
            exclusive_scan_i64(lc, lcp, n, st);
            k_delta_localptr<<<grid_for(h, n + 1), 256, 0, st>>>(lcp, lc, n, lptr, tp.deg);
            count_launch(3);
        }
        // by source: the changed nodes' pending shares and degrees
        perm = sort_perm(es, et, M, {0});
        k_delta_gather_perm<<<grid_for(h, M), 256, 0, st>>>(es, et, ew, perm, M, ss, stg, sw);
        count_launch();
        k_delta_wr<<<grid_for(h, n), 256, 0, st>>>(g.row_ptr, chg, g.inv, tp.rw0, ss, stg, sw, M, n, tp.waves, tp.wr,
                                                    tp.deg);
        count_launch();
        phase_mark(st, "delta: compact, wr");
        // by (wave, target, source): the per-wave gather list
        int32_t *ns = dalloc<int32_t>(M, st), *nt = dalloc<int32_t>(M, st);
        double *nw = dalloc<double>(M, st);
        track(ns), track(nt), track(nw);
        perm = sort_perm(ss, stg, M, {1, 2});
        k_delta_gather_perm<<<grid_for(h, M), 256, 0, st>>>(ss, stg, sw, perm, M, ns, nt, nw);
        count_launch();
        k_delta_waves<<<1, (tp.waves + 32) & ~31, 0, st>>>(nt, M, tp.waves, wf);
        count_launch();
        phase_mark(st, "delta: sort (wave, target)");
        // target segments (runs of equal target): starts, and the first segment of each wave
        k_delta_flags<<<grid_for(h, M), 256, 0, st>>>(nt, M, flag);
        count_launch();
        exclusive_scan_i64(flag, pos, M, st);
        const int64_t nseg = sync_read(pos + M);
        std::vector<int64_t> first(tp.waves + 1);
        DI_CUDA(cudaMemcpyAsync(first.data(), wf, (tp.waves + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        int64_t *seg = dalloc<int64_t>(nseg + 1, st);
        double *vals = dalloc<double>(M, st);
        track(seg), track(vals);
        k_delta_starts<<<grid_for(h, M), 256, 0, st>>>(nt, M, pos, seg);
        count_launch();
        DI_CUDA(cudaStreamSynchronize(st));
        std::vector<int64_t> sfirst(tp.waves + 1);
        for (int c = 0; c <= tp.waves; ++c) {        // a wave's entries start a segment
            if (first[c] < M) DI_CUDA(cudaMemcpyAsync(&sfirst[c], pos + first[c], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            else sfirst[c] = nseg;
        }
        // segments of more than kBigSeg entries (ascending, hence grouped by wave)
        int64_t *bf = (int64_t *)track(dalloc<int64_t>(nseg, st)), *bp = (int64_t *)track(dalloc<int64_t>(nseg + 1, st));
        k_delta_bigflag<<<grid_for(h, nseg), 256, 0, st>>>(seg, nseg, bf);
        exclusive_scan_i64(bf, bp, nseg, st);
        const int64_t nbig = sync_read(bp + nseg);
        int64_t *big = dalloc<int64_t>(nbig, st);
        track(big);
        k_delta_bigput<<<grid_for(h, nseg), 256, 0, st>>>(seg, nseg, bp, big);
        count_launch(2);
        std::vector<int64_t> bigh(nbig), bfirst(tp.waves + 1, 0);
        if (nbig) DI_CUDA(cudaMemcpyAsync(bigh.data(), big, nbig * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        DI_CUDA(cudaGetLastError());
        for (int c = 0; c <= tp.waves; ++c)
            bfirst[c] = std::lower_bound(bigh.begin(), bigh.end(), sfirst[c]) - bigh.begin();
        phase_mark(st, "delta: segments");
        // install (the new arrays are no longer temporaries)
        for (void *p : {(void *)tp.dsrc, (void *)tp.dtgt, (void *)tp.dw, (void *)tp.dseg, (void *)tp.dval,
                        (void *)tp.dbig, (void *)tp.dl_ptr, (void *)tp.dl_src, (void *)tp.dl_w})
            if (p) cudaFreeAsync(p, st);
        tp.dl_ptr = nl > 0 ? lptr : nullptr;
        tp.dl_src = lsrc;
        tp.dl_w = lwt;
        if (nl == 0) cudaFreeAsync(lptr, st);
        tp.dsrc = ns;
        tp.dtgt = nt;
        tp.dw = nw;
        tp.dseg = seg;
        tp.dval = vals;
        tp.dbig = big;
        tp.nd = M;
        tp.dwave = first;
        tp.dsegw = sfirst;
        tp.dbigw = bfirst;
        tmp.erase(std::remove_if(tmp.begin(), tmp.end(),
                                 [&](void *p) {
                                     return p == ns || p == nt || p == nw || p == seg || p == vals || p == big ||
                                            p == lsrc || p == lwt || p == lptr;
                                 }),
                  tmp.end());
        for (void *p : tmp) cudaFreeAsync(p, st);
        tmp.clear();
    } catch (...) {
        for (void *p : tmp) cudaFreeAsync(p, st);
        throw;
    }
}

void launch_delta(di_graph *h, int wave, int force) {
    TilePlan &tp = h->g.tl;
    if (tp.nd == 0) return;
    const int64_t q0 = tp.dwave[wave], q1 = tp.dwave[wave + 1];
    if (q1 <= q0) return;
    k_delta_vals<<<grid_for(h, q1 - q0), 256, 0, h->stream>>>(tp.dsrc, tp.dtgt, tp.dw, q0, q1, h->s.A, h->s.A2,
                                                             tp.dval, wave, tp.waves, h->s.ctrl, force);
    const int64_t s0 = tp.dsegw[wave], s1 = tp.dsegw[wave + 1];
    k_delta_seg<<<grid_for(h, s1 - s0), 256, 0, h->stream>>>(tp.dseg, tp.dtgt, tp.dval, s0, s1, h->s.F, wave,
                                                            h->s.ctrl, force);
    count_launch(2);
    const int64_t b0 = tp.dbigw[wave], b1 = tp.dbigw[wave + 1];
    if (b1 > b0) {
        k_delta_big<<<(unsigned)(b1 - b0), 1024, 0, h->stream>>>(tp.dseg, tp.dbig, b0, tp.dtgt, tp.dval, h->s.F, wave,
                                                               h->s.ctrl, force);
        count_launch();
    }
    DI_CUDA(cudaGetLastError());
}

}  // namespace dit

// Debug (not part of include/dit.h): delta entries the tile plan carries (-1: no handle)
extern "C" long long di_debug_delta_entries(const di_graph *h) { return h ? (long long)h->g.tl.nd : -1; }
