// Micro-benchmark: HBM -> smem streaming rate of the copy shapes a dense-layer kernel can
// use for its weight operand, with no compute behind them (a consumer thread frees each
// ring stage as soon as it lands). Answers whether the 2D TMA tiles of 128 rows x 128 B
// that the UMMA SWIZZLE_128B K-major operand needs (one 128-byte row segment per W row)
// stream as fast as contiguous bulk copies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe profiles/tma_probe.cu -lcuda && /tmp/tma_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done)
                     : "r"(sa(b)), "r"(parity)
                     : "memory");
}

// MODE 0: 2D TMA boxes {inner = 32 floats (128 B), rows} of a [rows_total x cols] fp32 matrix, CTA
//         (q, mtile) walks K atoms like mma_ring_kernel (BOXES boxes per stage stacked in rows)
// MODE 1: cp.async.bulk of 16 KB contiguous per stage (the same bytes, pre-tiled in HBM)
template <int MODE>
__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap tmap, const float* src, int cols,
                                                    int atoms_per_cta, int stages, int box_rows, unsigned long long* sink) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    constexpr int kStage = 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * kStage);
    uint64_t* empty = full + stages;
    const int q = blockIdx.x, mt = blockIdx.y;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            bar_init(full + s, 1);
            bar_init(empty + s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < atoms_per_cta; ++i) {
            const int s = i % stages;
            if (i >= stages) bar_wait(empty + s, ((i / stages) - 1) & 1);
            bar_expect(full + s, kStage);
            unsigned char* dst = base + s * kStage;
            const int atom = q * atoms_per_cta + i;
            if (MODE == 0) {
                for (int r = 0; r < 128; r += box_rows)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                            sa(dst + r * 128)),
                        "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(atom * 32), "r"(mt * 128 + r), "r"(sa(full + s))
                        : "memory");
            } else {
                const size_t tile = (static_cast<size_t>(mt) * (cols / 32) + atom) * kStage;
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                    "l"(reinterpret_cast<const unsigned char*>(src) + tile), "r"(kStage), "r"(sa(full + s))
                    : "memory");
            }
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (int i = 0; i < atoms_per_cta; ++i) {
            const int s = i % stages;
            bar_wait(full + s, (i / stages) & 1);
            acc += *reinterpret_cast<const unsigned*>(base + s * kStage + (i & 127) * 4);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
        }
        sink[blockIdx.y * gridDim.x + blockIdx.x] = acc;
    }
}

__global__ void ldg_kernel(const float4* src, size_t n, float* out) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const float4 v = __ldcs(src + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main(int argc, char** argv) {
    const int rows = argc > 1 ? std::atoi(argv[1]) : 4096, cols = 4096;  // 4096: a config-5 layer, fp32: 64 MB
    const size_t bytes = static_cast<size_t>(rows) * cols * 4;
    float* w;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 0, bytes);
    unsigned char* flush;
    cudaMalloc(&flush, 512u << 20);
    unsigned long long* sink;
    cudaMalloc(&sink, 1 << 20);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &qr);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int mtiles = rows / 128, katoms = cols / 32;
    std::printf("shape            ctas/SM stages  splits  us      TB/s\n");
    for (int mode = 0; mode < 2; ++mode)
        for (int box_rows : {128, 32, 256})
            for (int per_sm : {1, 2})
                for (int stages : {3, 6, 12}) {
                    if (mode == 1 && box_rows != 128) continue;
                    if (box_rows == 256) continue;  // box <= 256 rows but the stage is 128 rows
                    const size_t smem = 1024 + static_cast<size_t>(stages) * 16384 + stages * 16 + 64;
                    if (smem * per_sm > 225 * 1024) continue;
                    const int S = std::min(per_sm * 148 / mtiles, katoms);
                    const int apc = (katoms + S - 1) / S;
                    const int Sx = (katoms + apc - 1) / apc;
                    CUtensorMap tm{};
                    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
                    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
                    const cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
                    const cuuint32_t es[2] = {1, 1};
                    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                    auto fn = mode == 0 ? stream_kernel<0> : stream_kernel<1>;
                    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
                    float best = 1e9f;
                    for (int rep = 0; rep < 5; ++rep) {
                        cudaMemset(flush, rep, 512u << 20);  // W cold
                        cudaEventRecord(a);
                        fn<<<dim3(Sx, mtiles), 64, smem>>>(tm, w, cols, apc, stages, box_rows, sink);
                        cudaEventRecord(b);
                        cudaEventSynchronize(b);
                        float ms;
                        cudaEventElapsedTime(&ms, a, b);
                        if (rep > 0 && ms < best) best = ms;
                    }
                    const cudaError_t e = cudaGetLastError();
                    std::printf("%-16s %7d %6d %7d %7.2f %6.2f %s\n",
                                mode == 0 ? (box_rows == 128 ? "tma2d 128x128B" : "tma2d 4x(32x128B)") : "bulk 16KB",
                                per_sm, stages, Sx, best * 1e3, bytes / (best * 1e-3) / 1e12,
                                e == cudaSuccess ? "" : cudaGetErrorString(e));
                }
    for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, 512u << 20);
            cudaEventRecord(a);
            ldg_kernel<<<blocks, 512>>>(reinterpret_cast<const float4*>(w), bytes / 16, reinterpret_cast<float*>(sink));
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms < best) best = ms;
        }
        std::printf("ldg float4 grid=%d          %7.2f %6.2f\n", blocks, best * 1e3, bytes / (best * 1e-3) / 1e12);
    }
    return 0;
}
