// mb_rounds.cu -- microbenchmark (not part of libdit): the cost of one tile's
// local diffusion rounds (dit_tile.cu step 2) when the tile's sliced-ELL
// edges sit in SHARED memory, per SM, for a few launch shapes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_rounds scripts/mb_rounds.cu && ./mb_rounds
//
// One persistent CTA per SM runs `tiles` tiles of 512 nodes with K slots per
// lane in each of 32 virtual warps (32 x 32 x K local edges), 4 rounds each
// (gq write, barrier, piece sums, barrier, node sums).  Sources are random in
// [0, 512) (bank conflicts as in the real tiles) or spread (conflict-free).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

constexpr int kNode = 512, kVW = 32;

__device__ __forceinline__ double f2d_int(float w) {
    const uint32_t u = __float_as_uint(w);
    const uint32_t hi = (u & 0x80000000u) | (((u >> 3) & 0x0fffffffu) + (896u << 20));
    const uint32_t lo = u << 29;
    return __hiloint2double((int)hi, (int)lo);
}

template <int kWarps, bool kIntConv>
__global__ void __launch_bounds__(kWarps * 32, 1) k_rounds(const uint16_t *__restrict__ gsrc, const float *__restrict__ gw,
                                                          int K, int tiles, int rounds, double *__restrict__ out,
                                                          unsigned long long *__restrict__ cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int S = kVW * 32 * K;
    uint16_t *es = reinterpret_cast<uint16_t *>(sm);
    float *ew = reinterpret_cast<float *>(sm + ((S * 2 + 15) & ~15));
    double *gq = reinterpret_cast<double *>(sm + ((S * 2 + 15) & ~15) + S * 4);
    double *psum = gq + kNode + 2;
    const int i = threadIdx.x, lane = i & 31, wp = i >> 5;
    for (int q = i; q < S; q += blockDim.x) {
        es[q] = gsrc[q];
        ew[q] = gw[q];
    }
    if (i == 0) gq[kNode] = gq[kNode + 1] = 0.0;
    __syncthreads();
    double acc_out = 0.0;
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
        double f = (i < kNode) ? 1.0 + 1e-3 * (i + t) : 0.0;
        for (int r = 0; r < rounds; ++r) {
            if (i < kNode) gq[i] = 0.85 * f * 0.1;
            __syncthreads();
            constexpr int kPer = kVW / kWarps;
#pragma unroll
            for (int h = 0; h < kPer; ++h) {
                const int vw = kPer == 1 ? wp : (kPer == 2 ? (h ? kVW - 1 - wp : wp) : wp + h * kWarps);
                const int o0 = vw * 32 * K;
                double acc = 0.0;
                for (int s = 0; s < K; s += 4) {
                    const int k = o0 + 32 * s + 4 * lane;
                    const uint2 e = *reinterpret_cast<const uint2 *>(es + k);
                    const float4 w4 = *reinterpret_cast<const float4 *>(ew + k);
                    const double v0 = gq[e.x & 0xffffu], v1 = gq[e.x >> 16], v2 = gq[e.y & 0xffffu], v3 = gq[e.y >> 16];
                    if constexpr (kIntConv) {
                        acc = fma(v0, f2d_int(w4.x), acc);
                        acc = fma(v1, f2d_int(w4.y), acc);
                        acc = fma(v2, f2d_int(w4.z), acc);
                        acc = fma(v3, f2d_int(w4.w), acc);
                    } else {
                        acc = fma(v0, (double)w4.x, acc);
                        acc = fma(v1, (double)w4.y, acc);
                        acc = fma(v2, (double)w4.z, acc);
                        acc = fma(v3, (double)w4.w, acc);
                    }
                }
                psum[vw * 32 + lane] = acc;
            }
            __syncthreads();
            if (i < kNode) f = psum[i] + psum[(i * 7 + 3) & 1023];
            if (kWarps * 32 < kNode) {                // fewer threads than nodes: the second node of each thread
                const int i2 = i + kWarps * 32;
                if (i2 < kNode) gq[i2] = 0.85 * f * 0.1;
            }
        }
        acc_out += f;
    }
    const long long t1 = clock64();
    if (i == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    out[blockIdx.x * blockDim.x + i] = acc_out;
}

template <int kWarps, bool kIntConv>
void run(const char *name, const uint16_t *dsrc, const float *dw, int K, int tiles, int rounds, double *dout,
         unsigned long long *dcyc, int nsm, int ctas_per_sm = 1) {
    const int S = kVW * 32 * K;
    const size_t smem = ((S * 2 + 15) & ~15) + (size_t)S * 4 + (kNode + 2) * 8 + 1024 * 8;
    cudaFuncSetAttribute(k_rounds<kWarps, kIntConv>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    nsm *= ctas_per_sm;
    k_rounds<kWarps, kIntConv><<<nsm, kWarps * 32, smem>>>(dsrc, dw, K, 2, rounds, dout, dcyc);   // warm
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rounds<kWarps, kIntConv><<<nsm, kWarps * 32, smem>>>(dsrc, dw, K, tiles, rounds, dout, dcyc);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        exit(1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<unsigned long long> c(nsm);
    cudaMemcpy(c.data(), dcyc, nsm * 8, cudaMemcpyDeviceToHost);
    double cm = 0;
    for (auto x : c) cm += (double)x;
    cm /= nsm;
    const double edges = (double)S * rounds * tiles;
    printf("%-40s K=%2d smem=%6zu  %8.1f cycles/tile (%6.1f /round)  %.3f edges/cycle/SM  %.3f ms\n", name, K, smem,
           cm / tiles / ctas_per_sm, cm / tiles / rounds / ctas_per_sm, edges * ctas_per_sm / cm, ms);
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int Kmax = 12, tiles = 400, rounds = 4;
    const int S = kVW * 32 * Kmax;
    std::vector<uint16_t> src_r(S), src_c(S), src_h(S), src_b(S);
    std::vector<float> w(S);
    srand(1);
    for (int q = 0; q < S; ++q) {
        src_r[q] = (uint16_t)(rand() % kNode);
        w[q] = 0.5f + (rand() % 1000) * 1.5e-3f;
    }
    // slot of (virtual warp vw, lane, slot s) in the grouped layout (runs of 4 per lane)
    auto pos = [&](int vw, int lane, int s, int K) { return vw * 32 * K + 32 * 4 * (s / 4) + 4 * lane + (s % 4); };
    for (int vw = 0; vw < kVW; ++vw)
        for (int lane = 0; lane < 32; ++lane)
            for (int s = 0; s < Kmax; ++s) {
                const int q = pos(vw, lane, s, Kmax);
                src_c[q] = (uint16_t)((lane % 16) + 16 * (rand() % 32));   // distinct bank pair within each half-warp
                src_b[q] = (uint16_t)((lane / 2) + 16 * (rand() % 32));    // each bank pair twice per warp
            }
    // heuristic: each lane's slots ordered by (src - lane) mod 16 (random sources)
    auto heur = [&](int K) {
        for (int vw = 0; vw < kVW; ++vw)
            for (int lane = 0; lane < 32; ++lane) {
                std::vector<int> v(K);
                for (int s = 0; s < K; ++s) v[s] = src_r[pos(vw, lane, s, K)];
                std::sort(v.begin(), v.end(), [&](int a, int b) { return ((a - lane) & 15) < ((b - lane) & 15); });
                for (int s = 0; s < K; ++s) src_h[pos(vw, lane, s, K)] = (uint16_t)v[s];
            }
    };
    uint16_t *dr, *dc;
    float *dw;
    double *dout;
    unsigned long long *dcyc;
    cudaMalloc(&dr, S * 2);
    cudaMalloc(&dc, S * 2);
    cudaMalloc(&dw, S * 4);
    cudaMalloc(&dout, (size_t)nsm * 3 * 1024 * 8);
    cudaMalloc(&dcyc, nsm * 3 * 8);
    cudaMemcpy(dr, src_r.data(), S * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, src_c.data(), S * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), S * 4, cudaMemcpyHostToDevice);
    uint16_t *dh, *db;
    cudaMalloc(&dh, S * 2);
    cudaMalloc(&db, S * 2);
    cudaMemcpy(db, src_b.data(), S * 2, cudaMemcpyHostToDevice);
    for (int K : {8}) {
        run<16, false>("1 CTA x 16 warps, random", dr, dw, K, tiles, rounds, dout, dcyc, nsm, 1);
        run<8, false>("2 CTAs x 8 warps, random", dr, dw, K, tiles, rounds, dout, dcyc, nsm, 2);
        run<8, false>("1 CTA x 8 warps, random", dr, dw, K, tiles, rounds, dout, dcyc, nsm, 1);
        run<16, false>("2 CTAs x 16 warps, random", dr, dw, K, tiles, rounds, dout, dcyc, nsm, 2);
        run<8, false>("3 CTAs x 8 warps, random", dr, dw, K, tiles, rounds, dout, dcyc, nsm, 3);
        run<16, false>("1 CTA x 16 warps, half-warp distinct", dc, dw, K, tiles, rounds, dout, dcyc, nsm, 1);
        run<8, false>("2 CTAs x 8 warps, half-warp distinct", dc, dw, K, tiles, rounds, dout, dcyc, nsm, 2);
    }
    return 0;
}
