// dit_tile.cuh -- shared definitions of the tile-local schedule (R12, §5):
// tile geometry, record layouts, k_tile's shared-memory layout, TMA / mbarrier
// helpers.  Used by the plan builder (dit_plan.cu) and the sweep (dit_tile.cu).
#pragma once

#include "dit_internal.cuh"

#include <type_traits>

namespace dit {

constexpr int kTileThreads = (int)kNodeTile;     // build kernels: thread i owns node i of the tile
// k_tile: one CTA per SM of 23 warps: 16 round warps (thread i owns node i), 6
// prep warps (the next tile's inflow, up to 3 nodes per thread) and a producer
// warp issuing the TMA bulk copies
constexpr int kRW = (int)kNodeTile;
#ifndef DIT_LS_UNROLL
#define DIT_LS_UNROLL 2
#endif
constexpr int kLsUnroll = DIT_LS_UNROLL;          // k_tile: slot groups per unrolled local-sum step
#ifndef DIT_REC_UNROLL
#define DIT_REC_UNROLL 2
#endif
constexpr int kRecUnroll = DIT_REC_UNROLL;        // k_tile prep: light-record gathers in flight per thread
#ifndef DIT_PREP_WARPS
#define DIT_PREP_WARPS 6
#endif
constexpr int kPWt = 32 * DIT_PREP_WARPS;        // prep threads
constexpr int kPN = ((int)kNodeTile + kPWt - 1) / kPWt;   // nodes per prep thread (at most)
constexpr int kTileBlock = kRW + kPWt + 32;      // + the producer warp (TMA issue)
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kVRows = 2 * (int)kNodeTile;       // local-edge pieces per tile (at most)
constexpr int kVWarps = kVRows / 32;             // virtual warps: round warp w runs w and kVWarps-1-w
constexpr int kVofsStride = 36;                  // u32 per tile (kVWarps + 1, padded to 16 B)
constexpr int kVfStride = 520;                   // u16 per tile (kNodeTile + 1, padded to 16 B)
constexpr int kMetaBytes = kVofsStride * 4 + kVfStride * 2 + kVRows * 2;   // per-tile layout, TMA-staged
constexpr int64_t kGqSlots = kNodeTile + 16;     // outflow per node + one zero slot per bank pair (ELL padding)
// k_tile keeps kGqCopies copies of gq, copy c at c * kGqStride: slot j of copy c sits
// in bank pair (j + c) mod 16, and the plan picks per slot the copy that the
// half-warp's other reads leave free (k_ell_copies; lsrc holds c * kGqStride + j)
#ifndef DIT_GQ_COPIES
#define DIT_GQ_COPIES 2
#endif
constexpr int kGqCopies = DIT_GQ_COPIES;
constexpr int kGqStride = (int)kGqSlots + 1;
static_assert(kGqCopies >= 1 && kGqCopies <= 16 && kGqStride % 16 == 1, "gq copies shift by one bank pair");
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
// prepared row of a node (structure of arrays [2][kNodeTile] each): the
// inflow-completed fluid f and 1/sum w (double), the out-degree (int32).  H and
// the pending share wr are read by the round warps themselves at the state out.
constexpr int kPrepBytes = 8 + 8 + 4;
constexpr int kOffPsum = (kGqCopies * kGqStride * 8 + 127) & ~127;
constexpr int kOffP = kOffPsum + kVRows * 8;
constexpr int kOffR = kOffP + 2 * (int)kNodeTile * kPrepBytes;
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
#define DIT_TILE_WAVES DI_TILE_WAVES   // include/dit.h
#endif
constexpr int kTileWaves = DIT_TILE_WAVES;      // tile waves per sweep (R15), single GPU
// node ids are < 2^31 (int32 columns): 32-bit arithmetic
static_assert(kNodeTile == 512, "tile_wave shifts by 9");
__device__ __forceinline__ int tile_wave(int64_t node, int waves) {
    return (int)((uint32_t)(node >> 9) % (uint32_t)waves);
}

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

}  // namespace dit
