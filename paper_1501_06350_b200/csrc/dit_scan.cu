// dit_scan.cu -- device-wide exclusive prefix sum of int64 (graph builder plumbing:
// CSR offsets of the transpose and of an updated graph).  Three phases:
// tile sums -> one-block scan of the tile sums -> tile-local scan + offset.
#include "dit_internal.cuh"

#include <chrono>
#include <string>
#include <vector>
#include <cstdio>
#include <cstdlib>

namespace dit {

constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;   // 2048 items per block

__device__ __forceinline__ long long block_excl_scan(long long v, long long *total) {
    __shared__ long long s_w[kWarps];
    const unsigned lane = lane_id(), w = threadIdx.x >> 5;
    long long incl = warp_incl_scan(v);
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
        long long x = lane < (unsigned)kWarps ? s_w[lane] : 0;
        long long xi = warp_incl_scan(x);
        if (lane < (unsigned)kWarps) s_w[lane] = xi - x;
        if (lane == (unsigned)kWarps - 1 && total) *total = xi;
    }
    __syncthreads();
    const long long r = s_w[w] + incl - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kThreads) k_tile_sums(const int64_t *__restrict__ in, int64_t count,
                                                        int64_t *__restrict__ tile_sum) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
        if (base + k < count) s += in[base + k];
    __shared__ long long tot;
    block_excl_scan(s, &tot);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = tot;
}

// single block: exclusive scan of the tile sums in place
__global__ void __launch_bounds__(kThreads) k_scan_tiles(int64_t *__restrict__ ts, int64_t ntiles) {
    __shared__ long long carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < ntiles; b += kThreads) {
        const int64_t i = b + threadIdx.x;
        const long long v = i < ntiles ? ts[i] : 0;
        __shared__ long long tot;
        const long long ex = block_excl_scan(v, &tot);
        __syncthreads();
        if (i < ntiles) ts[i] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) k_scan_apply(const int64_t *__restrict__ in, int64_t count,
                                                         const int64_t *__restrict__ ts, int64_t *__restrict__ out) {
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    long long v[kScanItems];
    long long s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < count ? in[base + k] : 0;
        s += v[k];
    }
    long long ex = block_excl_scan(s, nullptr) + ts[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < count) out[base + k] = ex;
        ex += v[k];
    }
}

// out[0..count] = exclusive scan of in[0..count-1], out[count] = total.
// `out` must hold count+1 entries and must not alias `in`.
void exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t count, cudaStream_t st) {
    const int64_t ntiles = (count + kScanTile - 1) / kScanTile;
    int64_t *ts = nullptr;
    DI_CUDA(cudaMallocAsync(&ts, (ntiles + 1) * sizeof(int64_t), st));
    if (ntiles > 0) {
        k_tile_sums<<<(unsigned)ntiles, kThreads, 0, st>>>(in, count, ts);
        count_launch();
    } else {
        DI_CUDA(cudaMemsetAsync(ts, 0, sizeof(int64_t), st));
    }
    // ts[ntiles] must hold the grand total: scan ntiles+1 entries with a zero tail
    DI_CUDA(cudaMemsetAsync(ts + ntiles, 0, sizeof(int64_t), st));
    k_scan_tiles<<<1, kThreads, 0, st>>>(ts, ntiles + 1);
    count_launch();
    if (ntiles > 0) {
        k_scan_apply<<<(unsigned)ntiles, kThreads, 0, st>>>(in, count, ts, out);
        count_launch();
    }
    DI_CUDA(cudaMemcpyAsync(out + count, ts + ntiles, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    DI_CUDA(cudaFreeAsync(ts, st));
    DI_CUDA(cudaGetLastError());
}

// DIT_BUILD_TIMING=1: print the time since the previous mark (stream synchronised);
// =2: CUDA events only (no synchronisation), printed at the plan's "done" mark
void phase_mark(cudaStream_t st, const char *name) {
    static const char *env = getenv("DIT_BUILD_TIMING");
    static const bool on = env != nullptr;
    if (!on) return;
    if (env[0] == '2') {
        static std::vector<std::pair<cudaEvent_t, std::string>> marks;
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, st);
        marks.emplace_back(ev, name);
        if (std::string(name).find("done") != std::string::npos) {
            cudaEventSynchronize(ev);
            for (size_t i = 1; i < marks.size(); ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, marks[i - 1].first, marks[i].first);
                fprintf(stderr, "[dit] ev %-25s %9.2f ms\n", marks[i].second.c_str(), ms);
            }
            for (auto &m : marks) cudaEventDestroy(m.first);
            marks.clear();
        }
        return;
    }
    static auto last = std::chrono::steady_clock::now();
    if (env[0] == '3') {                             // host clock only, no synchronisation
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[dit] host %-24s %9.2f ms\n", name, std::chrono::duration<double, std::milli>(now - last).count());
        last = now;
        return;
    }
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[dit] %-28s %9.2f ms\n", name, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

}  // namespace dit
