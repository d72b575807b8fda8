// int_peak.cu — measured integer warp-issue peak of this B200 (the roofline
// denominator of the issue-bound K1; MEASURED_PEAKS.json has only HBM and
// bf16 numbers).
//
// Each kernel runs independent chains (8 per thread, so dependent-issue
// latency is hidden) of one integer instruction class for a fixed number of
// iterations; lane-ops/s = threads * chains * iterations * ops / time.  The
// SASS of each loop body was checked with cuobjdump -sass: k_iadd3 2 adds
// per chain-iteration (134 IADD3 + 129 IMAD per 16x8 body: ptxas spreads
// integer adds over the ALU and FMA pipes), k_lop3 1 LOP3, k_add64
// IADD3 + IADD3.X per u64 add, k_ffma 1 FFMA; loop overhead < 3% of the
// body, not counted.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak scripts/int_peak.cu
//   ./int_peak > profiles/round2_int_peak.json
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int kChains = 8;
constexpr int kIters = 4096;

// One instruction per chain per iteration, written as volatile PTX so the
// compiler cannot fold the chains (plain C++ lets it collapse the loop).
#define CHAIN_KERNEL(NAME, T, REG, INIT, BODY)                                  \
    __global__ void NAME(T *out, T seed) {                                       \
        T a[kChains];                                                            \
        _Pragma("unroll") for (int c = 0; c < kChains; ++c) a[c] = INIT;         \
        const T b = seed + static_cast<T>(blockIdx.x), d = seed * static_cast<T>(3); \
        _Pragma("unroll 16") for (int i = 0; i < kIters; ++i) {                  \
            _Pragma("unroll") for (int c = 0; c < kChains; ++c) {                \
                asm volatile(BODY : "+" REG(a[c]) : REG(b), REG(d));             \
            }                                                                    \
        }                                                                        \
        T r = a[0];                                                              \
        _Pragma("unroll") for (int c = 1; c < kChains; ++c) r += a[c];           \
        if (r == static_cast<T>(12345)) out[0] = r;                              \
    }

CHAIN_KERNEL(k_iadd3, uint32_t, "r", seed * (threadIdx.x + c + 1), "add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;")
CHAIN_KERNEL(k_lop3, uint32_t, "r", seed * (threadIdx.x + c + 1), "lop3.b32 %0, %0, %1, %2, 0x96;")
CHAIN_KERNEL(k_add64, uint64_t, "l", seed * (threadIdx.x + c + 1), "add.u64 %0, %0, %1;")
CHAIN_KERNEL(k_ffma, float, "f", seed * (threadIdx.x + c + 1), "fma.rn.f32 %0, %0, %1, %2;")

template <class K, class T>
double run(K kern, T *buf, T seed, int grid, int block, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<grid, block>>>(buf, seed);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(a);
        kern<<<grid, block>>>(buf, seed);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best * 1e-3;
}

int main() {
    cudaDeviceProp p{};
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const int block = 512, grid = p.multiProcessorCount * 4;  // 64 warps per SM
    const double lanes = static_cast<double>(grid) * block * kChains * kIters;
    void *buf = nullptr;
    cudaMalloc(&buf, 64);
    const double t_iadd = run(k_iadd3, static_cast<uint32_t *>(buf), 7u, grid, block, 5);
    const double t_lop = run(k_lop3, static_cast<uint32_t *>(buf), 7u, grid, block, 5);
    const double t_add64 = run(k_add64, static_cast<uint64_t *>(buf), uint64_t{7}, grid, block, 5);
    const double t_ffma = run(k_ffma, static_cast<float *>(buf), 1.0001f, grid, block, 5);
    const double nominal = static_cast<double>(p.multiProcessorCount) * 128.0 * clk_khz * 1e3;
    std::printf("{\"gpu\": \"%s\", \"sms\": %d, \"sm_clock_max_mhz\": %.0f,\n", p.name, p.multiProcessorCount,
                clk_khz / 1e3);
    std::printf(" \"nominal_lane_ops_per_s\": %.4e,\n", nominal);
    std::printf(" \"int_add_lane_ops_per_s\": %.4e,  \"int_add_note\": \"2 adds per chain-iteration; ptxas "
                "issues them as IADD3 (ALU pipe) and IMAD (FMA pipe) about half and half\",\n",
                2.0 * lanes / t_iadd);
    std::printf(" \"lop3_lane_ops_per_s\": %.4e,\n", lanes / t_lop);
    std::printf(" \"add64_lane_ops_per_s\": %.4e,  \"add64_note\": \"one u64 add = IADD3 + IADD3.X; counted as 2 lane-ops\",\n",
                2.0 * lanes / t_add64);
    std::printf(" \"ffma_lane_ops_per_s\": %.4e,\n", lanes / t_ffma);
    std::printf(" \"block\": %d, \"grid\": %d, \"chains_per_thread\": %d, \"iterations\": %d}\n", block, grid, kChains,
                kIters);
    cudaFree(buf);
    return 0;
}
