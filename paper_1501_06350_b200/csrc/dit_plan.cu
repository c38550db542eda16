// dit_plan.cu -- the tile plan of the tile-local schedule (R12, §4, §5).
#include "dit_tile.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cstdlib>
#include <vector>

namespace dit {

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
// run and segment flags packed in one word (run << 32 | segment): one scan gives
// both ids (the segment count stays below 2^32, so the low field never carries)
__global__ void k_heavy_flags(const uint32_t *__restrict__ st, const uint32_t *__restrict__ hh, int64_t mh,
                              const int64_t *__restrict__ sbeg, int64_t *__restrict__ flags) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = st[p];
        const bool run = p == 0 || st[p - 1] != s || hh[p - 1] != hh[p];
        const bool chk = (p - sbeg[s]) % kHeavyChunk == 0;
        flags[p] = ((int64_t)run << 32) | (int64_t)(run || chk);
    }
}

// chunk c of stripe group s starts at sbeg[s] + (c - s_chunk[s]) kHeavyChunk (closed form)
__global__ void k_heavy_index(const int64_t *__restrict__ flags, const int64_t *__restrict__ ids,
                              const int64_t *__restrict__ sbeg, const int64_t *__restrict__ schunk,
                              const uint32_t *__restrict__ hh, const uint32_t *__restrict__ st, int64_t mh,
                              int64_t nstripe, int64_t nh, int64_t *__restrict__ seg_start,
                              int64_t *__restrict__ chunk_start, int64_t *__restrict__ cfirst,
                              int32_t *__restrict__ run_h, int64_t *__restrict__ run_seg,
                              uint32_t *__restrict__ rkey, uint32_t *__restrict__ rval) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = flags[p], id = ids[p];
        const int64_t segid = id & 0xffffffffLL;
        const uint32_t s = st[p];
        if (f & 1) seg_start[segid] = p;
        if ((p - sbeg[s]) % kHeavyChunk == 0) {
            const int64_t c = schunk[s] + (p - sbeg[s]) / kHeavyChunk;
            chunk_start[c] = p;
            cfirst[c] = segid;
        }
        if (f >> 32) {
            const int64_t r = id >> 32;
            run_h[r] = (int32_t)hh[p];
            run_seg[r] = segid;
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
                               int64_t i0, int64_t i1, int waves, float *__restrict__ wr) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    const int lane = lane_id();
    // leaves the tile and is still pending after the sweep (a later wave takes its
    // pushes in during the sweep, R15); ghost targets always pending
    auto pending = [&](int64_t i, int64_t e) {
        const int64_t t = col[e];
        return t >= n || (t / kNodeTile != i / kNodeTile && tile_wave(t, waves) <= tile_wave(i, waves));
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = i0 + (int64_t)blockIdx.x * blockDim.x; base < i1; base += stride) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        if (i < i1) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        const bool big = e - b > 32;
        if (i < i1 && !big) {
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

// Copies in shared memory: k_tile writes kGqCopies copies of the
// outflow gq, copy c shifted by c bank pairs.  A 64-bit shared load is served per half-warp, one wavefront per
// address sharing a bank pair (equal addresses broadcast), so per load and
// half-warp the plan gives the distinct addresses distinct bank pairs where it
// can (address v can use the pairs v, v+1, .., v+C-1 mod 16) and
// encodes the copy in the index (c * stride + v).  Only the shared-memory
// address of each read changes: values and summation order do not.
//
// match_copies (one thread per half-warp row): v[16] >= 0 an address, -2 a
// padding slot.  A maximum matching of the distinct addresses to bank pairs by
// augmenting paths (Kuhn), the state packed four bits per entry in registers
// (bank of each lane, the holder of each pair, the DFS stack); a lane left
// unmatched keeps copy 0.  Returns the copies packed four bits per lane and the
// zero slot's pair for the padding.
__device__ __forceinline__ uint64_t get4(uint64_t w, int k) { return (w >> (4 * k)) & 15u; }
__device__ __forceinline__ uint64_t set4(uint64_t w, int k, uint64_t x) {
    return (w & ~(15ull << (4 * k))) | (x << (4 * k));
}
__device__ __forceinline__ uint64_t match_copies(const int (&v)[16], int C, int &pad_bank) {
    uint64_t B = 0;                                   // bank pair of each lane's address
    unsigned lead = 0;                                // lanes with an address (equal ones matched apart:
#pragma unroll                                        // a pair each, rare, no conflict either way)
    for (int l = 0; l < 16; ++l) {
        B |= (uint64_t)(v[l] & 15) << (4 * l);
        if (v[l] >= 0) lead |= 1u << l;
    }
    uint64_t MR = 0, CP = 0;                          // holder of each pair, copy of each leader
    unsigned valid = 0;                               // pairs held
    for (unsigned U = lead; U; U &= U - 1) {
        uint64_t SU = (uint64_t)(__ffs(U) - 1), SC = 0, SB = 0;   // DFS stack: lane, next option, pair
        int top = 0;
        unsigned vis = 0;
        while (top >= 0) {
            const int x = (int)get4(SU, top), c = (int)get4(SC, top);
            if (c >= C) {
                --top;
                continue;
            }
            SC += 1ull << (4 * top);
            const int b = ((int)get4(B, x) + c) & 15;
            if ((vis >> b) & 1u) continue;
            vis |= 1u << b;
            SB = set4(SB, top, (uint64_t)b);
            if (!((valid >> b) & 1u)) {               // augment: level k takes pair SB[k]
                for (int k = top; k >= 0; --k) {
                    const int bk = (int)get4(SB, k), xk = (int)get4(SU, k);
                    MR = set4(MR, bk, (uint64_t)xk);
                    valid |= 1u << bk;
                    CP = set4(CP, xk, (uint64_t)((bk - (int)get4(B, xk)) & 15));
                }
                break;
            }
            ++top;                                    // re-route the pair's holder
            SU = set4(SU, top, get4(MR, b));
            SC = set4(SC, top, 0);
        }
    }
    const unsigned fr = ~valid & 0xffffu;
    pad_bank = fr ? __ffs(fr) - 1 : 0;
    return CP;
}

// Two copies (pairs b, b+1 for an address in pair b): the options are arcs of
// two consecutive pairs on the 16-cycle, so a sweep over the pairs assigning
// each pair to the waiting address with the earliest deadline (the one carried
// over from the previous pair first) is a maximum matching; the sweep starts
// after a pair no address starts at (no carry into it).  Addresses left over
// take the less loaded of their two pairs.  O(16) per row.
__device__ __forceinline__ uint64_t match_copies2(const int (&v)[16], int &pad_bank) {
    uint32_t c2 = 0;                                  // min(addresses starting at pair b, 2), two bits each
    uint64_t rk = 0, seen = 0;                        // rank of each lane among its pair's addresses
    uint64_t ldr = 0;                                 // lowest lane with the same address (equal ones share)
    unsigned lead = 0;
#pragma unroll
    for (int l = 0; l < 16; ++l) {
        int d = l;
#pragma unroll
        for (int k = l - 1; k >= 0; --k)
            if (v[k] == v[l]) d = k;
        ldr |= (uint64_t)d << (4 * l);
        if (v[l] >= 0 && d == l) lead |= 1u << l;
    }
#pragma unroll
    for (int l = 0; l < 16; ++l)
        if ((lead >> l) & 1u) {
            const int b = v[l] & 15;
            const uint32_t n = (seen >> (4 * b)) & 15u;
            rk |= (uint64_t)n << (4 * l);
            seen += 1ull << (4 * b);
            if (((c2 >> (2 * b)) & 3u) < 2u) c2 += 1u << (2 * b);
        }
    int s0 = 0;                                       // a pair with no address starting just before it
#pragma unroll
    for (int b = 15; b >= 0; --b)
        if (((c2 >> (2 * ((b + 15) & 15))) & 3u) == 0u) s0 = b;
    uint32_t stay = 0, shift = 0;                     // pair b kept by one of its addresses / pair b+1 taken by one
    uint32_t carry = 0;
    for (int k = 0; k < 16; ++k) {
        const int b = (s0 + k) & 15;
        const uint32_t n = (c2 >> (2 * b)) & 3u;
        uint32_t cn;
        if (carry) {
            cn = n >= 1u;
        } else {
            if (n >= 1u) stay |= 1u << b;
            cn = n >= 2u;
        }
        if (cn && !(k == 15 && ((stay >> s0) & 1u))) shift |= 1u << b;
        carry = cn;
    }
    const uint32_t used = stay | ((shift << 1) | (shift >> 15));
    uint64_t ld = 0;                                  // addresses per pair, four bits each
#pragma unroll
    for (int b = 0; b < 16; ++b) ld |= (uint64_t)((used >> b) & 1u) << (4 * b);
    uint64_t cp = 0;
#pragma unroll
    for (int l = 0; l < 16; ++l)
        if ((lead >> l) & 1u) {
            const int b = v[l] & 15, b1 = (b + 1) & 15;
            const uint32_t r = (uint32_t)((rk >> (4 * l)) & 15u), st = (stay >> b) & 1u;
            if (((shift >> b) & 1u) && r == st) {
                cp |= 1ull << (4 * l);
            } else if (!(st && r == 0)) {             // unmatched: the less loaded of its two pairs
                if (get4(ld, b1) < get4(ld, b)) {
                    cp |= 1ull << (4 * l);
                    ld += 1ull << (4 * b1);
                } else {
                    ld += 1ull << (4 * b);
                }
            }
        }
    int bp = 0;                                       // the padding: the least loaded pair
#pragma unroll
    for (int b = 1; b < 16; ++b)
        if (get4(ld, b) < get4(ld, bp)) bp = b;
    pad_bank = bp;
    uint64_t out = 0;                                 // equal addresses: the first one's copy
#pragma unroll
    for (int l = 0; l < 16; ++l) out |= get4(cp, (int)get4(ldr, l)) << (4 * l);
    return out;
}

// gq copies of the local slots: one thread per (tile, virtual warp, half-warp), per slot row
__global__ void __launch_bounds__(128) k_ell_copies(const int64_t *__restrict__ ltile,
                                                           const uint32_t *__restrict__ vofs, int64_t t0, int64_t t1,
                                                           uint16_t *__restrict__ lsrc) {
    const int64_t nitem = (t1 - t0) * kVWarps * 2;
    for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < nitem;
         item += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = t0 + item / (kVWarps * 2);
        const int vw = (int)((item / 2) % kVWarps), half = (int)(item & 1);
        const uint32_t o0 = vofs[tile * kVofsStride + vw];
        const int K = (int)((vofs[tile * kVofsStride + vw + 1] - o0) >> 5);
        const int64_t base = ltile[tile] + o0;
        for (int s = 0; s < K; ++s) {
            int v[16];
#pragma unroll
            for (int l = 0; l < 16; ++l) {
                const int x = lsrc[base + ell_slot(s, 16 * half + l, K)];
                v[l] = x >= (int)kNodeTile ? -2 : x;
            }
            int bp;
            const uint64_t cp = kGqCopies == 2 ? match_copies2(v, bp) : match_copies(v, kGqCopies, bp);
#pragma unroll
            for (int l = 0; l < 16; ++l)
                lsrc[base + ell_slot(s, 16 * half + l, K)] =
                    (uint16_t)(v[l] >= 0 ? (int)get4(cp, l) * kGqStride + v[l] : (int)kNodeTile + bp);
        }
    }
}

__global__ void k_tile_max_edges(const int64_t *__restrict__ ltile, int64_t ntile, unsigned long long *__restrict__ mx) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntile; t += (int64_t)gridDim.x * blockDim.x)
        atomicMax(mx, (unsigned long long)(ltile[t + 1] - ltile[t]));
}

void free_tiles(TilePlan &t, cudaStream_t st) {
    for (void *p : {(void *)t.rrel, (void *)t.hidx, (void *)t.wr, (void *)t.deg, (void *)t.ltile, (void *)t.rtile,
                    (void *)t.vofs, (void *)t.lstage, (void *)t.vfirst, (void *)t.plist, (void *)t.lsrc, t.lw, t.rrec, t.hrec, (void *)t.chunk_start,
                    (void *)t.seg_start, (void *)t.cfirst, (void *)t.run_h, (void *)t.run_seg, (void *)t.part,
                    (void *)t.hsum, (void *)t.tpart, (void *)t.fold_ptr, (void *)t.fold_h, (void *)t.fold_run,
                    (void *)t.dsrc, (void *)t.dtgt, (void *)t.dw, (void *)t.rw0, (void *)t.dseg, (void *)t.dval, (void *)t.dbig,
                    (void *)t.dl_ptr, (void *)t.dl_src, (void *)t.dl_w})
        if (p) cudaFreeAsync(p, st);
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

// per-stripe edge counts of the sorted stripe keys
__global__ void k_stripe_count(const uint32_t *__restrict__ st, int64_t mh, unsigned long long *__restrict__ cnt) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < mh; p += (int64_t)gridDim.x * blockDim.x)
        if (p == mh - 1 || st[p + 1] != st[p]) atomicAdd(&cnt[st[p]], (unsigned long long)(p + 1));
}

// ---------------------------------------------------------------- direct plan build
// The plan is built from the CSR by source, one chunk of whole tiles at a time
// (so that create can overlap it with the upload): no transpose.
//   phase 1 (col of the chunk):   k_plan_count -- per tile: local in-degree of
//     every target, local / remote out-degree of every source, the sliced-ELL
//     layout; scans give the tiles' ELL bases and the sources' remote offsets;
//   phase 2 (weights of the chunk): k_plan_place -- local edges (source order)
//     into a chunk staging list keyed by target, remote edges into the remote
//     list; a stable radix sort of the staging by target; k_plan_ell -- every
//     target's local in-edges (ascending source) into its ELL pieces;
//   phase 3 (all chunks done): the remote list sorted by target (stable:
//     ascending source), light / heavy split, records, heavy index.
// Every position comes from a scan or a stable sort: the plan is the same bits
// whatever the chunking.

#ifndef DIT_CAP_ROUND
#define DIT_CAP_ROUND 8
#endif
constexpr int64_t kCapRound = DIT_CAP_ROUND;

// sliced-ELL layout of tile t from the local in-degrees (thread k = node k of the tile)
__device__ void tile_layout(int64_t t, int k, int64_t dk, int eb, int64_t stage_cap, uint32_t *__restrict__ vofs,
                            uint16_t *__restrict__ vfirst, uint16_t *__restrict__ plist, int32_t *__restrict__ vcap,
                            int64_t *__restrict__ pcnt, int32_t *__restrict__ lstage) {
    __shared__ int32_t len_s[kVRows], lenr_s[kVRows];
    __shared__ uint16_t vf_s[kNodeTile + 1], rank_s[kVRows];
    __shared__ int s_V;
    __shared__ int64_t s_red[kNodeTile / 32 + 1];
    __shared__ int s_scan[kNodeTile / 32 + 1];
    // cap: at most kVRows pieces (E / cap + nonzero rows <= kVRows); block sums
    const int64_t E = block_sum_512(dk, s_red), nz = block_sum_512((int64_t)(dk > 0), s_red);
    int64_t cap = nz ? std::max<int64_t>(1, (E + (kVRows - nz) - 1) / (kVRows - nz)) : 1;
    cap = (cap + kCapRound - 1) / kCapRound * kCapRound;   // full pieces: whole slot groups
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
    for (int p = k; p < V; p += kTileThreads) {       // rank: longest first, ties by piece order
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

// phase 1: CTA per tile of [t0, t1); thread k = source / target node k of the tile
// (rows of more than 32 edges walked by the whole warp)
__global__ void __launch_bounds__(kTileThreads) k_plan_count(const int64_t *__restrict__ row_ptr,
                                                              const int32_t *__restrict__ col, int64_t n, int64_t t0,
                                                              int eb, int64_t stage_cap, int64_t *__restrict__ lc,
                                                              int64_t *__restrict__ lsc, int64_t *__restrict__ rsc,
                                                              uint32_t *__restrict__ vofs,
                                                              uint16_t *__restrict__ vfirst,
                                                              uint16_t *__restrict__ plist, int32_t *__restrict__ vcap,
                                                              int64_t *__restrict__ pcnt, int32_t *__restrict__ lstage) {
    __shared__ int cnt_s[kNodeTile];
    const int k = threadIdx.x, lane = (int)lane_id();
    const int64_t t = t0 + blockIdx.x;
    const int64_t a0 = t * kNodeTile;
    const int nn = (int)min(kNodeTile, n - a0);
    cnt_s[k] = 0;
    __syncthreads();
    const int64_t i = a0 + k;
    int64_t b = 0, e = 0;
    if (k < nn) {
        b = row_ptr[i];
        e = row_ptr[i + 1];
    }
    const bool big = e - b > 32;
    int64_t nl = 0, nr = 0;
    if (k < nn && !big)
        for (int64_t q = b; q < e; ++q) {
            const int64_t c = col[q];
            if (c >= a0 && c < a0 + nn) {
                atomicAdd(&cnt_s[c - a0], 1);
                ++nl;
            } else {
                ++nr;
            }
        }
    unsigned bm = __ballot_sync(0xffffffffu, k < nn && big);
    while (bm) {
        const int l = __ffs(bm) - 1;
        bm &= bm - 1;
        const int64_t bl = __shfl_sync(0xffffffffu, b, l), el = __shfl_sync(0xffffffffu, e, l);
        int64_t ml = 0, mr = 0;
        for (int64_t q = bl + lane; q < el; q += 32) {
            const int64_t c = col[q];
            if (c >= a0 && c < a0 + nn) {
                atomicAdd(&cnt_s[c - a0], 1);
                ++ml;
            } else {
                ++mr;
            }
        }
        ml = warp_sum(ml);
        mr = warp_sum(mr);
        if (lane == l) {
            nl = ml;
            nr = mr;
        }
    }
    if (k < nn) {
        lsc[i] = nl;
        rsc[i] = nr;
    }
    __syncthreads();
    const int64_t dk = k < nn ? cnt_s[k] : 0;
    if (k < nn) lc[i] = dk;
    tile_layout(t, k, dk, eb, stage_cap, vofs, vfirst, plist, vcap, pcnt, lstage);
}

// out[q] = base + in[q] for q in [0, cnt], base read from *base_ptr first (out may alias base_ptr)
__global__ void k_add_base(const int64_t *__restrict__ in, int64_t cnt, const int64_t *base_ptr, int64_t *out) {
    const int64_t base = *base_ptr;
    __syncthreads();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= cnt; q += (int64_t)gridDim.x * blockDim.x)
        out[q] = base + in[q];
}

// packed edge payload: source in the high word, the f32 weight bits (or, for f64
// weights, an index into a side array) in the low word
template <typename W>
__device__ __forceinline__ uint64_t pack_edge(int64_t src, const StoreW<W> *w, int64_t e, int64_t alt) {
    uint32_t lo = 0;
    if constexpr (std::is_same<W, float>::value) lo = __float_as_uint(w[e]);
    else if constexpr (std::is_same<W, double>::value) lo = (uint32_t)alt;
    return ((uint64_t)(uint32_t)src << 32) | lo;
}

// phase 2: thread per source of [i0, i1) (long rows by the warp): local edges in
// source-major order into the chunk staging (key = target - i0), remote edges
// into the remote list at the source's global offset (key = target)
template <typename W>
__global__ void k_plan_place(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                             const StoreW<W> *__restrict__ w, int64_t n, int64_t i0, int64_t i1, int64_t e0,
                             const int64_t *__restrict__ lsp, const int64_t *__restrict__ rsp,
                             uint32_t *__restrict__ skey, uint64_t *__restrict__ sval, uint32_t *__restrict__ rkey,
                             uint64_t *__restrict__ rval, double *__restrict__ rw64) {
    const int lane = lane_id();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = i0 + (int64_t)blockIdx.x * blockDim.x; base < i1; base += stride) {
        const int64_t i = base + threadIdx.x;
        int64_t b = 0, e = 0;
        if (i < i1) {
            b = row_ptr[i];
            e = row_ptr[i + 1];
        }
        const bool big = e - b > 32;
        if (i < i1 && !big) {
            const int64_t a0 = (i / kNodeTile) * kNodeTile, z = min(n, a0 + kNodeTile);
            int64_t pl = lsp[i - i0], pr = rsp[i - i0];
            for (int64_t q = b; q < e; ++q) {
                const int64_t c = col[q];
                if (c >= a0 && c < z) {
                    skey[pl] = (uint32_t)(c - i0);
                    sval[pl] = pack_edge<W>(i - a0, w, q, q - e0);
                    ++pl;
                } else {
                    rkey[pr] = (uint32_t)c;
                    rval[pr] = pack_edge<W>(i, w, q, pr);
                    if constexpr (std::is_same<W, double>::value) rw64[pr] = w[q];
                    ++pr;
                }
            }
        }
        unsigned bm = __ballot_sync(0xffffffffu, i < i1 && big);
        while (bm) {
            const int l = __ffs(bm) - 1;
            bm &= bm - 1;
            const int64_t il = __shfl_sync(0xffffffffu, i, l), bl = __shfl_sync(0xffffffffu, b, l),
                          el = __shfl_sync(0xffffffffu, e, l);
            const int64_t a0 = (il / kNodeTile) * kNodeTile, z = min(n, a0 + kNodeTile);
            int64_t pl = lsp[il - i0], pr = rsp[il - i0];
            for (int64_t q0 = bl; q0 < el; q0 += 32) {
                const int64_t q = q0 + lane;
                const bool ok = q < el;
                const int64_t c = ok ? col[q] : 0;
                const bool loc = ok && c >= a0 && c < z;
                const unsigned ml = __ballot_sync(0xffffffffu, loc), mr = __ballot_sync(0xffffffffu, ok && !loc);
                const unsigned lt = (1u << lane) - 1u;
                if (loc) {
                    const int64_t p = pl + __popc(ml & lt);
                    skey[p] = (uint32_t)(c - i0);
                    sval[p] = pack_edge<W>(il - a0, w, q, q - e0);
                } else if (ok) {
                    const int64_t p = pr + __popc(mr & lt);
                    rkey[p] = (uint32_t)c;
                    rval[p] = pack_edge<W>(il, w, q, p);
                    if constexpr (std::is_same<W, double>::value) rw64[p] = w[q];
                }
                pl += __popc(ml);
                pr += __popc(mr);
            }
        }
    }
}

// phase 2: thread per target of [i0, i1): its local in-edges (sorted staging,
// ascending source) into the slots of its pieces
template <typename W>
__global__ void k_plan_ell(int64_t i0, int64_t i1, const uint64_t *__restrict__ sval, const int64_t *__restrict__ lst,
                           const int64_t *__restrict__ lc, const int64_t *__restrict__ ltile,
                           const uint32_t *__restrict__ vofs, const uint16_t *__restrict__ vfirst,
                           const uint16_t *__restrict__ plist, const int32_t *__restrict__ vcap,
                           const StoreW<W> *__restrict__ w, int64_t e0, uint16_t *__restrict__ lsrc,
                           StoreW<W> *__restrict__ lw) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    for (int64_t j = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < i1; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cnt = lc[j];
        if (cnt == 0) continue;
        const int64_t tile = j / kNodeTile;
        const int tl = (int)(j - tile * kNodeTile);
        const int64_t cap = vcap[tile], base = ltile[tile], s0 = lst[j - i0];
        const int pf = vfirst[tile * kVfStride + tl];
        for (int64_t q = 0; q < cnt; ++q) {
            const uint64_t v = sval[s0 + q];
            const int r = plist[tile * kVRows + pf + (int)(q / cap)];
            const uint32_t o0 = vofs[tile * kVofsStride + r / 32], o1 = vofs[tile * kVofsStride + r / 32 + 1];
            const int64_t o = base + o0 + ell_slot(q % cap, r % 32, (o1 - o0) / 32);
            lsrc[o] = (uint16_t)(v >> 32);
            if constexpr (std::is_same<W, float>::value) lw[o] = __uint_as_float((uint32_t)v);
            else if constexpr (std::is_same<W, double>::value) lw[o] = w[e0 + (int64_t)(uint32_t)v];
            (void)kW;
        }
    }
}

// remote in-degree of every target from the sorted remote keys
__global__ void k_plan_rcount(const uint32_t *__restrict__ sk, int64_t R, int64_t *__restrict__ rc) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < R; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = sk[p];
        if (p == 0 || sk[p - 1] != k) atomicAdd((unsigned long long *)&rc[k], (unsigned long long)(-p));
        if (p == R - 1 || sk[p + 1] != k) atomicAdd((unsigned long long *)&rc[k], (unsigned long long)(p + 1));
    }
}

// every sorted remote edge to its class: light record of its tile or heavy edge
// keyed by (wave of the target, stripe of the source)
template <typename W>
__global__ void k_split_remote(const uint32_t *__restrict__ sk, const uint64_t *__restrict__ sv, int64_t R,
                               const int64_t *__restrict__ rs, const double *__restrict__ rw64, int64_t n,
                               const int64_t *__restrict__ rptr, const int64_t *__restrict__ hptr,
                               const int32_t *__restrict__ hidx, int64_t stripe_nodes, int64_t nstripe, int waves,
                               RemRec<W> *__restrict__ rrec, RemRec<W> *__restrict__ htmp, uint32_t *__restrict__ hkey,
                               uint32_t *__restrict__ hval, uint32_t *__restrict__ hof) {
    constexpr bool kW = !std::is_same<W, NoW>::value;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < R; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = sk[p];
        const uint64_t v = sv[p];
        const int64_t rank = p - rs[t];
        RemRec<W> r{};
        r.src = (int32_t)(v >> 32);
        if constexpr (std::is_same<W, float>::value) r.w = __uint_as_float((uint32_t)v);
        else if constexpr (std::is_same<W, double>::value) r.w = rw64[(uint32_t)v];
        else r.w = 1.0f;
        (void)kW;
        const int32_t hx = hidx[t];
        if (hx >= 0) {
            const int64_t o = hptr[t] + rank;
            htmp[o] = r;
            // heavy group: the target's wave; a shard's ghost slots form one more group (waves),
            // gathered first in a sweep so that the exchange overlaps the local heavy gather
            hkey[o] = (uint32_t)((t < n ? tile_wave(t, waves) : waves) * nstripe + r.src / stripe_nodes);
            hval[o] = (uint32_t)o;
            hof[o] = (uint32_t)hx;
        } else {
            rrec[rptr[t] + rank] = r;
        }
    }
}

// Stable sort of (u32 key, u64 payload) pairs on the low `bits` key bits: the
// toolkit's onesweep radix sort (graph-builder plumbing, 2-4x faster than ours
// here) under 2^31 items, else -- or with DIT_OWN_RADIX -- our LSD radix sort.
static std::pair<uint32_t *, uint64_t *> sort_pairs(di_graph *h, uint32_t *k0, uint64_t *v0, uint32_t *k1,
                                                    uint64_t *v1, int64_t count, int bits) {
    cudaStream_t st = h->stream;
    if (count <= 0) return {k0, v0};
    if (count >= (int64_t)0x7fffffff || getenv("DIT_OWN_RADIX")) return radix_sort_u32_u64(k0, v0, k1, v1, count, bits, st);
    cub::DoubleBuffer<uint32_t> kb(k0, k1);
    cub::DoubleBuffer<unsigned long long> vb((unsigned long long *)v0, (unsigned long long *)v1);
    size_t tb = 0;
    DI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)count, 0, bits, st));
    std::lock_guard<std::mutex> lock(scratch_mutex(h->device));
    DI_CUDA(cub::DeviceRadixSort::SortPairs(cub_scratch(h->device, tb), tb, kb, vb, (int)count, 0, bits, st));
    DI_CUDA(cudaStreamSynchronize(st));              // the cached scratch is free for the next build
    return {kb.Current(), (uint64_t *)vb.Current()};
}

// row offset of every tile's first node (and of n)
__global__ void k_tile_rowptr(const int64_t *__restrict__ row_ptr, int64_t n, int64_t ntile, int64_t *__restrict__ out) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= ntile; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = row_ptr[min(n, t * kNodeTile)];
}

static int64_t grid_cap(di_graph *h, int64_t count, int per_block = 256) {
    return std::max<int64_t>(1, std::min<int64_t>((count + per_block - 1) / per_block, (int64_t)h->num_sms * 16));
}

// A second stream for plan work nothing else in the build reads (the shared-memory
// copies of each chunk's ELL): it runs beside the next chunks and the remote
// phase.  join() orders the main stream after it (before anything frees or
// reads those arrays); the destructor joins too (error paths).
struct SideStream {
    cudaStream_t main, s = nullptr;
    std::vector<cudaEvent_t> evs;
    explicit SideStream(cudaStream_t m) : main(m) {}
    cudaEvent_t mark(cudaStream_t on) {
        cudaEvent_t e = nullptr;
        DI_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        evs.push_back(e);
        DI_CUDA(cudaEventRecord(e, on));
        return e;
    }
    cudaStream_t after_main() {                      // ordered after the main stream's work so far
        if (!s) DI_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        DI_CUDA(cudaStreamWaitEvent(s, mark(main), 0));
        return s;
    }
    void join() {
        if (!s) return;
        cudaStream_t x = s;
        s = nullptr;
        DI_CUDA(cudaStreamWaitEvent(main, mark(x), 0));
        DI_CUDA(cudaStreamDestroy(x));               // released once its work completes
    }
    ~SideStream() {
        if (s) {
            cudaEvent_t e = nullptr;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess) {
                cudaEventRecord(e, s);
                cudaStreamWaitEvent(main, e, 0);
                evs.push_back(e);
            }
            cudaStreamDestroy(s);
        }
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
    }
};

template <typename W>
static void build_tiles_t(di_graph *h, const PlanFeed *feed, const int *bad) {
    DevGraph &g = h->g;
    TilePlan &tp = g.tl;
    cudaStream_t st = h->stream;
    const int64_t n = g.n, m = g.m;
    using SW = StoreW<W>;
    constexpr bool kW = !std::is_same<W, NoW>::value;
    constexpr bool k64 = std::is_same<W, double>::value;
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
    tp.groups = tp.waves + (g.nt > n ? 1 : 0);       // + the ghost slots' group on a shard
    const int64_t S = tp.groups * nS;                // heavy groups (group, stripe)
    if (nt >= (int64_t)0xffffffffLL || m >= ((int64_t)1 << 40)) {
        set_error("tiled plan: graph too large for one handle (fluid slots >= 2^32)");
        throw Fail{DI_ERR_INVALID};
    }
    // chunks of whole tiles (the feed's, else about kPlanChunkEdgesLazy edges each)
    std::vector<int64_t> ctile, cedge;               // chunks: tile ranges and their first edges
    if (feed) {
        ctile = feed->tile_lo;
        cedge = feed->edge_lo;
    } else {
        std::vector<int64_t> rp(tp.ntile + 1);
        // tile starts' row offsets (host) to cut the chunks
        int64_t *d = nullptr;
        DI_CUDA(cudaMallocAsync(&d, (tp.ntile + 1) * sizeof(int64_t), st));
        k_tile_rowptr<<<(int)grid_cap(h, tp.ntile + 1), 256, 0, st>>>(g.row_ptr, n, tp.ntile, d);
        count_launch();
        DI_CUDA(cudaMemcpyAsync(rp.data(), d, (tp.ntile + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        DI_CUDA(cudaFreeAsync(d, st));
        ctile.push_back(0);
        for (int64_t t = 1; t <= tp.ntile; ++t)
            if (t == tp.ntile || rp[t] - rp[ctile.back()] >= kPlanChunkEdgesLazy) ctile.push_back(t);
        for (int64_t t : ctile) cedge.push_back(rp[t]);
    }
    const int nch = (int)ctile.size() - 1;
    auto node_of = [&](int64_t t) { return std::min(n, t * kNodeTile); };
    // ---- per-node / per-tile arrays
    int64_t *lc, *lsc, *rsc, *lsp, *lst, *rsp, *pcnt;
    for (int64_t **p : {&lc, &lsc, &rsc, &lsp, &lst, &rsp}) DI_CUDA(cudaMallocAsync(p, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemsetAsync(lc, 0, (nt + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemsetAsync(rsp, 0, sizeof(int64_t), st));
    int32_t *vcap;
    DI_CUDA(cudaMallocAsync(&vcap, (tp.ntile + 1) * sizeof(int32_t), st));
    DI_CUDA(cudaMallocAsync(&pcnt, (tp.ntile + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&tp.vofs, tp.ntile * kVofsStride * sizeof(uint32_t), st));
    DI_CUDA(cudaMallocAsync(&tp.vfirst, tp.ntile * kVfStride * sizeof(uint16_t), st));
    DI_CUDA(cudaMallocAsync(&tp.plist, tp.ntile * kVRows * sizeof(uint16_t), st));
    DI_CUDA(cudaMallocAsync(&tp.ltile, (tp.ntile + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&tp.lstage, (tp.ntile + 1) * sizeof(int32_t), st));
    DI_CUDA(cudaMemsetAsync(tp.ltile, 0, sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&tp.wr, n * sizeof(float) + 16, st));
    int64_t *tmp;
    DI_CUDA(cudaMallocAsync(&tmp, (nt + 1) * sizeof(int64_t), st));
    const int eb = (int)(2 + (kW ? sizeof(SW) : 0));
    const int64_t stage_cap = (int64_t)(tile_e_buf<W>() - kMetaBytes);
    // ---- phase 1: counts and layout, chunk by chunk as the targets arrive
    for (int c = 0; c < nch; ++c) {
        const int64_t t0 = ctile[c], t1 = ctile[c + 1], i0 = node_of(t0), i1 = node_of(t1);
        if (feed) {
            DI_CUDA(cudaStreamWaitEvent(st, feed->col_ready[c], 0));
            if (feed->on_col) feed->on_col(c);
        }
        k_plan_count<<<(unsigned)(t1 - t0), kTileThreads, 0, st>>>(g.row_ptr, g.col, n, t0, eb, stage_cap, lc, lsc,
                                                                    rsc, tp.vofs, tp.vfirst, tp.plist, vcap, pcnt,
                                                                    tp.lstage);
        count_launch();
        // tiles' ELL bases and sources' remote offsets continue the previous chunk's
        exclusive_scan_i64(pcnt + t0, tmp, t1 - t0, st);
        k_add_base<<<(int)grid_cap(h, t1 - t0 + 1), 256, 0, st>>>(tmp, t1 - t0, tp.ltile + t0, tp.ltile + t0);
        exclusive_scan_i64(rsc + i0, tmp, i1 - i0, st);
        k_add_base<<<(int)grid_cap(h, i1 - i0 + 1), 256, 0, st>>>(tmp, i1 - i0, rsp + i0, rsp + i0);
        count_launch(2);
    }
    phase_mark(st, "tiles: counts + layout");
    tp.mpad = read_i64(tp.ltile + tp.ntile, st);
    const int64_t R = read_i64(rsp + n, st);         // remote edges
    if (R >= (int64_t)0x7fffffff) {
        set_error("tiled plan: more than 2^31 remote edges in one graph handle");
        throw Fail{DI_ERR_INVALID};
    }
    // +16 B: aligned TMA supersets may read up to 15 bytes past the end
    DI_CUDA(cudaMallocAsync(&tp.lsrc, tp.mpad * sizeof(uint16_t) + 16, st));
    if (kW) DI_CUDA(cudaMallocAsync(&tp.lw, tp.mpad * sizeof(SW) + 16, st));
    if (tp.mpad > 0) {
        k_fill_pad<W><<<(int)grid_cap(h, tp.mpad), 256, 0, st>>>(tp.lsrc, (SW *)tp.lw, tp.mpad);
        count_launch();
    }
    const int64_t R1 = R > 0 ? R : 1;
    uint32_t *rk0, *rk1;
    uint64_t *rv0, *rv1;
    double *rw64 = nullptr;
    DI_CUDA(cudaMallocAsync(&rk0, R1 * 4, st));
    DI_CUDA(cudaMallocAsync(&rk1, R1 * 4, st));
    DI_CUDA(cudaMallocAsync(&rv0, R1 * 8, st));
    DI_CUDA(cudaMallocAsync(&rv1, R1 * 8, st));
    if (k64) DI_CUDA(cudaMallocAsync(&rw64, R1 * 8, st));
    // chunk staging (the largest chunk's local edges)
    int64_t cmax = 1;
    {
        std::vector<int64_t> lsum(nch + 1, 0);
        for (int c = 0; c < nch; ++c) {
            const int64_t i0 = node_of(ctile[c]), i1 = node_of(ctile[c + 1]);
            exclusive_scan_i64(lsc + i0, tmp, i1 - i0, st);
            lsum[c] = read_i64(tmp + (i1 - i0), st);
            cmax = std::max(cmax, lsum[c]);
        }
    }
    uint32_t *sk0, *sk1;
    uint64_t *sv0, *sv1;
    DI_CUDA(cudaMallocAsync(&sk0, cmax * 4, st));
    DI_CUDA(cudaMallocAsync(&sk1, cmax * 4, st));
    DI_CUDA(cudaMallocAsync(&sv0, cmax * 8, st));
    DI_CUDA(cudaMallocAsync(&sv1, cmax * 8, st));
    phase_mark(st, "tiles: allocate");
    // ---- phase 2: local edges into the ELL, remote edges into the remote list
    const bool bank_order = getenv("DIT_BANK_ORDER") != nullptr;
    SideStream side(st);
    for (int c = 0; c < nch; ++c) {
        const int64_t i0 = node_of(ctile[c]), i1 = node_of(ctile[c + 1]);
        if (feed) {
            if (c < (int)feed->w_ready.size()) DI_CUDA(cudaStreamWaitEvent(st, feed->w_ready[c], 0));
            if (feed->on_w) feed->on_w(c);
        }
        const int64_t e0 = cedge[c];
        if (k64 && cedge[c + 1] - e0 >= (int64_t)0xffffffffLL) {
            set_error("tiled plan: a plan chunk of 2^32 edges or more (f64 weights)");
            throw Fail{DI_ERR_INVALID};
        }
        exclusive_scan_i64(lsc + i0, lsp + i0, i1 - i0, st);   // chunk-relative staging offsets
        exclusive_scan_i64(lc + i0, lst + i0, i1 - i0, st);    // targets' starts in the sorted staging
        const int64_t cl = read_i64(lsp + i1, st);
        k_plan_place<W><<<(int)grid_cap(h, i1 - i0), 256, 0, st>>>(g.row_ptr, g.col, (const SW *)g.w, n, i0, i1, e0,
                                                                   lsp + i0, rsp + i0, sk0, sv0, rk0, rv0, rw64);
        k_remote_share<W><<<(int)grid_cap(h, i1 - i0), 256, 0, st>>>(g.row_ptr, g.col, (const SW *)g.w, g.inv, n, i0,
                                                                     i1, tp.waves, tp.wr);
        count_launch(2);
        auto sorted = sort_pairs(h, sk0, sv0, sk1, sv1, cl, bits_for(i1 - i0 + 1));
        k_plan_ell<W><<<(int)grid_cap(h, i1 - i0), 256, 0, st>>>(i0, i1, sorted.second, lst + i0, lc, tp.ltile,
                                                                 tp.vofs, tp.vfirst, tp.plist, vcap, (const SW *)g.w,
                                                                 e0, tp.lsrc, (SW *)tp.lw);
        count_launch();
        // k_plan_ell has placed the chunk's slots: their gq copies beside the next chunks
        if (kGqCopies > 1 && !bank_order && ctile[c + 1] > ctile[c]) {
            k_ell_copies<<<(int)grid_cap(h, (ctile[c + 1] - ctile[c]) * kVWarps * 2, 128), 128, 0, side.after_main()>>>(
                tp.ltile, tp.vofs, ctile[c], ctile[c + 1], tp.lsrc);
            count_launch();
        }
    }
    phase_mark(st, "tiles: local edges");
    if (tp.mpad > 0 && bank_order) {                 // opt-in: ~1% faster rounds for ~55 ms of build (configs[2])
        k_ell_balance<W><<<(int)std::min<int64_t>(tp.ntile * kVWarps / kBalWarps + 1, (int64_t)h->num_sms * 16),
                           kBalWarps * 32, 0, st>>>(tp.ltile, tp.vofs, tp.ntile, tp.lsrc, (SW *)tp.lw);
        k_ell_copies<<<(int)grid_cap(h, tp.ntile * kVWarps * 2, 128), 128, 0, st>>>(tp.ltile, tp.vofs, 0, tp.ntile,
                                                                              tp.lsrc);
        count_launch(2);
    }
    for (void *p : {(void *)sk0, (void *)sk1, (void *)sv0, (void *)sv1, (void *)lsc, (void *)lsp, (void *)lst})
        DI_CUDA(cudaFreeAsync(p, st));
    if (bad) {                                       // invalid input: stop before the remote keys are used
        int fl = 0;
        DI_CUDA(cudaMemcpyAsync(&fl, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        DI_CUDA(cudaStreamSynchronize(st));
        if (fl) {
            for (void *p : {(void *)rk0, (void *)rk1, (void *)rv0, (void *)rv1, (void *)rw64, (void *)lc, (void *)rsc,
                            (void *)rsp, (void *)pcnt, (void *)tmp, (void *)vcap})
                cudaFreeAsync(p, st);
            side.join();
            free_tiles(tp, st);
            return;                                  // the caller reports the error
        }
    }
    // ---- phase 3: remote edges by target (stable: ascending source), classes
    auto rsorted = sort_pairs(h, rk0, rv0, rk1, rv1, R, bits_for(nt + 1));
    int64_t *rc = rsc;                               // reused: remote in-degree per target
    DI_CUDA(cudaMemsetAsync(rc, 0, (nt + 1) * sizeof(int64_t), st));
    if (R > 0) {
        k_plan_rcount<<<(int)grid_cap(h, R), 256, 0, st>>>(rsorted.first, R, rc);
        count_launch();
    }
    int64_t *rstart = lc;                            // lc no longer needed: targets' starts in the sorted list
    exclusive_scan_i64(rc, rstart, nt, st);
    phase_mark(st, "tiles: remote sort");
    int64_t *lrc, *hc, *hflag, *rptr, *hptr, *hpos;
    for (int64_t **p : {&lrc, &hc, &hflag, &rptr, &hptr, &hpos})
        DI_CUDA(cudaMallocAsync(p, (nt + 1) * sizeof(int64_t), st));
    k_classify<<<(int)grid_cap(h, tp.ntile), 256, 0, st>>>(rc, n, tp.ntile, lrc, hc, hflag);
    count_launch();
    if (nt > n) {
        k_classify_ghosts<<<(int)grid_cap(h, nt - n), 256, 0, st>>>(rc, n, nt, lrc, hc, hflag);
        count_launch();
    }
    exclusive_scan_i64(lrc, rptr, nt, st);
    exclusive_scan_i64(hc, hptr, nt, st);
    exclusive_scan_i64(hflag, hpos, nt, st);
    tp.mlight = read_i64(rptr + nt, st);
    tp.mh = read_i64(hptr + nt, st);
    tp.nh = read_i64(hpos + nt, st);
    tp.mloc = g.m - tp.mlight - tp.mh;
    if (tp.mh >= (int64_t)0xffffffffLL) {
        set_error("tiled plan: too many heavy remote edges for one graph handle");
        throw Fail{DI_ERR_INVALID};
    }
    // ---- per-node arrays, tile bases
    DI_CUDA(cudaMallocAsync(&tp.rrel, n * sizeof(uint32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.hidx, nt * sizeof(int32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.deg, n * sizeof(int32_t) + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.rtile, (tp.ntile + 1) * sizeof(int64_t), st));
    k_tile_rel<<<(int)grid_cap(h, nt + 1), 256, 0, st>>>(rptr, hpos, hflag, g.row_ptr, n, nt, tp.ntile, tp.rrel,
                                                         tp.hidx, tp.deg, tp.rtile);
    count_launch();
    phase_mark(st, "tiles: classes + node arrays");
    // ---- remote edges to their classes
    DI_CUDA(cudaMallocAsync(&tp.rrec, tp.mlight * rs + 16, st));
    DI_CUDA(cudaMallocAsync(&tp.hrec, tp.mh * rs + 16, st));
    const int64_t mh1 = tp.mh > 0 ? tp.mh : 1;
    RemRec<W> *htmp;
    uint32_t *k0, *v0, *k1, *v1, *hof, *hh;
    DI_CUDA(cudaMallocAsync(&htmp, mh1 * rs, st));
    for (uint32_t **p : {&k0, &v0, &k1, &v1, &hof, &hh}) DI_CUDA(cudaMallocAsync(p, mh1 * sizeof(uint32_t), st));
    if (R > 0) {
        k_split_remote<W><<<(int)grid_cap(h, R), 256, 0, st>>>(rsorted.first, rsorted.second, R, rstart, rw64, n,
                                                               rptr, hptr, tp.hidx, tp.stripe_nodes, nS, tp.waves,
                                                               (RemRec<W> *)tp.rrec, htmp, k0, v0, hof);
        count_launch();
    }
    for (void *p : {(void *)rk0, (void *)rk1, (void *)rv0, (void *)rv1, (void *)rw64}) DI_CUDA(cudaFreeAsync(p, st));
    phase_mark(st, "tiles: split remote");
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
        int64_t *hfl, *hid, *schunk_d;
        for (int64_t **p : {&hfl, &hid}) DI_CUDA(cudaMallocAsync(p, (tp.mh + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&schunk_d, (S + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMemcpyAsync(schunk_d, tp.s_chunk.data(), (S + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        k_heavy_flags<<<grid_for(h, tp.mh), 256, 0, st>>>(skey, hh, tp.mh, sbeg_d, hfl);
        count_launch();
        exclusive_scan_i64(hfl, hid, tp.mh, st);
        phase_mark(st, "heavy: flags + scans");
        {
            const int64_t tot = read_i64(hid + tp.mh, st);
            tp.nrun = tot >> 32;
            tp.nseg = tot & 0xffffffffLL;
        }
        DI_CUDA(cudaMallocAsync(&tp.seg_start, (tp.nseg + 1) * sizeof(int64_t) + 16, st));   // +16: TMA supersets
        DI_CUDA(cudaMallocAsync(&tp.chunk_start, (tp.nchunk + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.cfirst, (tp.nchunk + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.run_h, tp.nrun * sizeof(int32_t), st));
        DI_CUDA(cudaMallocAsync(&tp.run_seg, (tp.nrun + 1) * sizeof(int64_t), st));
        DI_CUDA(cudaMallocAsync(&tp.part, tp.nseg * sizeof(double), st));
        uint32_t *rk0, *rv0, *rk1, *rv1;
        for (uint32_t **p : {&rk0, &rv0, &rk1, &rv1}) DI_CUDA(cudaMallocAsync(p, tp.nrun * sizeof(uint32_t), st));
        k_heavy_index<<<grid_for(h, tp.mh), 256, 0, st>>>(hfl, hid, sbeg_d, schunk_d, hh, skey, tp.mh, nS,
                                                          tp.nh, tp.seg_start, tp.chunk_start, tp.cfirst, tp.run_h,
                                                          tp.run_seg, rk0, rv0);
        count_launch();
        if ((int64_t)tp.groups * tp.nh >= (int64_t)0xffffffffLL) {
            set_error("tiled plan: too many heavy targets for one graph handle");
            throw Fail{DI_ERR_INVALID};
        }
        // the heavy targets of each group, each with its runs in stripe order (k_heavy_fold)
        {
            auto fs = radix_sort_u32(rk0, rv0, rk1, rv1, tp.nrun, bits_for((int64_t)tp.groups * tp.nh + 1), st);
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
            DI_CUDA(cudaMallocAsync(&wf, (tp.groups + 1) * sizeof(unsigned long long), st));
            k_fill_u64<<<1, 64, 0, st>>>(wf, tp.groups + 1, (unsigned long long)nslot);
            k_fold_index<<<grid_for(h, tp.nrun), 256, 0, st>>>(fs.first, ff, fslot, tp.nrun, tp.nh, tp.fold_ptr,
                                                               tp.fold_h, wf);
            count_launch(3);
            DI_CUDA(cudaMemcpyAsync(tp.fold_run, fs.second, tp.nrun * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
            DI_CUDA(cudaMemcpyAsync(tp.fold_ptr + nslot, &tp.nrun, sizeof(int64_t), cudaMemcpyHostToDevice, st));
            std::vector<unsigned long long> w(tp.groups + 1);
            DI_CUDA(cudaMemcpyAsync(w.data(), wf, (tp.groups + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                    st));
            DI_CUDA(cudaStreamSynchronize(st));
            tp.wave_slot.assign(tp.groups + 1, nslot);
            for (int c = tp.groups - 1; c >= 0; --c) tp.wave_slot[c] = std::min<int64_t>((int64_t)w[c], tp.wave_slot[c + 1]);
            for (void *p : {(void *)ff, (void *)fslot, (void *)wf, (void *)rk0, (void *)rv0, (void *)rk1, (void *)rv1})
                DI_CUDA(cudaFreeAsync(p, st));
        }
        DI_CUDA(cudaMemcpyAsync(tp.seg_start + tp.nseg, &tp.mh, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.chunk_start + tp.nchunk, &tp.mh, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.cfirst + tp.nchunk, &tp.nseg, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DI_CUDA(cudaMemcpyAsync(tp.run_seg + tp.nrun, &tp.nseg, sizeof(int64_t), cudaMemcpyHostToDevice, st));
        phase_mark(st, "heavy: index");
        for (int64_t *p : {hfl, hid, schunk_d, sbeg_d}) DI_CUDA(cudaFreeAsync(p, st));
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
    for (int64_t *p : {lc, rsc, lrc, hc, hflag, rptr, hptr, hpos, pcnt, rsp, tmp}) DI_CUDA(cudaFreeAsync(p, st));
    for (uint32_t *p : {k0, v0, k1, v1, hof, hh}) DI_CUDA(cudaFreeAsync(p, st));
    DI_CUDA(cudaFreeAsync(htmp, st));
    DI_CUDA(cudaFreeAsync(vcap, st));
    DI_CUDA(cudaFreeAsync(mx, st));
    side.join();
    DI_CUDA(cudaStreamSynchronize(st));
    DI_CUDA(cudaGetLastError());
    tp.max_tile_edges = (int64_t)mxh;
    tp.built = true;
    phase_mark(st, "tiles: free + done");
}

void build_tiles(di_graph *h, const PlanFeed *feed, const int *bad) {
    DevGraph &g = h->g;
    if (g.tl.built || g.n == 0) return;
    switch (g.w_kind) {
    case DI_W_F32: build_tiles_t<float>(h, feed, bad); break;
    case DI_W_F64: build_tiles_t<double>(h, feed, bad); break;
    default: build_tiles_t<NoW>(h, feed, bad);
    }
}
}  // namespace dit
