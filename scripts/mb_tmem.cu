// mb_tmem.cu -- microbenchmark (not part of libdit): where should a tile's
// local edges {source u16, weight f32} live during the 4 local rounds of
// k_tile?  Same shape as mb_rounds.cu (one CTA of 16 warps per SM, 32 virtual
// warps of K slots per lane, two per warp, gq gathered from shared memory):
//   smem -- sources and weights read from shared memory every round (k_tile now)
//   regs -- read from shared memory once per tile into registers (upper bound)
//   tmem -- read from shared memory once per tile, tcgen05.st into tensor
//           memory, tcgen05.ld back every round (shared-memory pipe left to gq)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_tmem scripts/mb_tmem.cu && ./scripts/mb_tmem
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int kNode = 512, kVW = 32, K = 8;   // K slots per lane per virtual warp
constexpr int S = kVW * 32 * K;

__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
}
__device__ __forceinline__ void tm_st4(uint32_t a, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mode 0 smem, 1 regs, 2 tmem
template <int kMode>
__global__ void __launch_bounds__(512, 1) k_rounds(const uint16_t *__restrict__ gsrc, const float *__restrict__ gw,
                                                  int tiles, int rounds, double *__restrict__ out,
                                                  unsigned long long *__restrict__ cyc) {
    extern __shared__ __align__(16) unsigned char sm[];
    uint16_t *es = reinterpret_cast<uint16_t *>(sm);
    float *ew = reinterpret_cast<float *>(sm + S * 2);
    double *gq = reinterpret_cast<double *>(sm + S * 6);
    double *psum = gq + kNode + 2;
    __shared__ uint32_t s_taddr;
    const int i = threadIdx.x, lane = i & 31, wp = i >> 5;
    for (int q = i; q < S; q += blockDim.x) {
        es[q] = gsrc[q];
        ew[q] = gw[q];
    }
    if (i == 0) gq[kNode] = gq[kNode + 1] = 0.0;
    if constexpr (kMode == 2) {
        if (wp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(&s_taddr))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    uint32_t tbase = 0;
    if constexpr (kMode == 2) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // warp w: lanes 32 (w % 4) .., columns 24 (w / 4) ..: per virtual warp 4 source words + 8 weights
        tbase = s_taddr + ((uint32_t)(32 * (wp & 3)) << 16) + (uint32_t)(24 * (wp >> 2));
    }
    double acc_out = 0.0;
    const long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
        double f = 1.0 + 1e-3 * (i + t);
        uint32_t rs[2][4], rw[2][8];
        if constexpr (kMode != 0) {                  // once per tile: this thread's slots
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int vw = h ? kVW - 1 - wp : wp;
                const int o0 = vw * 32 * K;
#pragma unroll
                for (int g = 0; g < K / 4; ++g) {
                    const int k = o0 + 32 * 4 * g + 4 * lane;
                    const uint2 e = *reinterpret_cast<const uint2 *>(es + k);
                    const uint4 w4 = *reinterpret_cast<const uint4 *>(ew + k);
                    rs[h][2 * g] = e.x;
                    rs[h][2 * g + 1] = e.y;
                    rw[h][4 * g] = w4.x;
                    rw[h][4 * g + 1] = w4.y;
                    rw[h][4 * g + 2] = w4.z;
                    rw[h][4 * g + 3] = w4.w;
                }
            }
            if constexpr (kMode == 2) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    tm_st4(tbase + 12 * h, rs[h]);
                    tm_st8(tbase + 12 * h + 4, rw[h]);
                }
                tm_wait_st();
            }
        }
        for (int r = 0; r < rounds; ++r) {
            gq[i] = 0.85 * f * 0.1;
            __syncthreads();
            if constexpr (kMode == 2) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    tm_ld4(tbase + 12 * h, rs[h]);
                    tm_ld8(tbase + 12 * h + 4, rw[h]);
                }
                tm_wait_ld();
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int vw = h ? kVW - 1 - wp : wp;
                const int o0 = vw * 32 * K;
                double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                for (int g = 0; g < K / 4; ++g) {
                    uint32_t ex, ey;
                    float w0, w1, w2, w3;
                    if constexpr (kMode == 0) {
                        const int k = o0 + 32 * 4 * g + 4 * lane;
                        const uint2 e = *reinterpret_cast<const uint2 *>(es + k);
                        const float4 w4 = *reinterpret_cast<const float4 *>(ew + k);
                        ex = e.x, ey = e.y, w0 = w4.x, w1 = w4.y, w2 = w4.z, w3 = w4.w;
                    } else {
                        ex = rs[h][2 * g], ey = rs[h][2 * g + 1];
                        w0 = __uint_as_float(rw[h][4 * g]), w1 = __uint_as_float(rw[h][4 * g + 1]);
                        w2 = __uint_as_float(rw[h][4 * g + 2]), w3 = __uint_as_float(rw[h][4 * g + 3]);
                    }
                    const double v0 = gq[ex & 0xffffu], v1 = gq[ex >> 16], v2 = gq[ey & 0xffffu], v3 = gq[ey >> 16];
                    a0 = fma(v0, (double)w0, a0);
                    a1 = fma(v1, (double)w1, a1);
                    a2 = fma(v2, (double)w2, a2);
                    a3 = fma(v3, (double)w3, a3);
                }
                psum[vw * 32 + lane] = (a0 + a1) + (a2 + a3);
            }
            __syncthreads();
            f = psum[i] + psum[(i * 7 + 3) & 1023];
        }
        acc_out += f;
    }
    const long long t1 = clock64();
    if (i == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    out[blockIdx.x * blockDim.x + i] = acc_out;
    if constexpr (kMode == 2) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (wp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(s_taddr) : "memory");
    }
}

template <int kMode>
double run(const char *name, const uint16_t *dsrc, const float *dw, int tiles, int rounds, double *dout,
           unsigned long long *dcyc, int nsm) {
    const size_t smem = (size_t)S * 6 + (kNode + 2) * 8 + 1024 * 8;
    cudaFuncSetAttribute(k_rounds<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_rounds<kMode><<<nsm, 512, smem>>>(dsrc, dw, 2, rounds, dout, dcyc);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rounds<kMode><<<nsm, 512, smem>>>(dsrc, dw, tiles, rounds, dout, dcyc);
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
    std::vector<double> o(nsm * 512);
    cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
    double cs = 0;
    for (double x : o) cs += x;
    printf("%-6s %8.1f cycles/tile (%6.1f /round)  %.3f edges/cycle/SM  %.3f ms  checksum %.10e\n", name, cm / tiles,
           cm / tiles / rounds, (double)S * rounds * tiles / cm, ms, cs);
    return cs;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = 400, rounds = 4;
    std::vector<uint16_t> src(S);
    std::vector<float> w(S);
    srand(1);
    for (int q = 0; q < S; ++q) {
        src[q] = (uint16_t)(rand() % kNode);
        w[q] = 0.5f + (rand() % 1000) * 1.5e-3f;
    }
    uint16_t *ds;
    float *dw;
    double *dout;
    unsigned long long *dcyc;
    cudaMalloc(&ds, S * 2);
    cudaMalloc(&dw, S * 4);
    cudaMalloc(&dout, (size_t)nsm * 512 * 8);
    cudaMalloc(&dcyc, nsm * 8);
    cudaMemcpy(ds, src.data(), S * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, w.data(), S * 4, cudaMemcpyHostToDevice);
    const double c0 = run<0>("smem", ds, dw, tiles, rounds, dout, dcyc, nsm);
    const double c1 = run<1>("regs", ds, dw, tiles, rounds, dout, dcyc, nsm);
    const double c2 = run<2>("tmem", ds, dw, tiles, rounds, dout, dcyc, nsm);
    printf("checksums equal: %d %d\n", c0 == c1, c0 == c2);
    return 0;
}
