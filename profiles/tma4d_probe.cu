// Which 4D TMA tensor-map variants are legal on sm_100a for the conv B operand
// ([B][C][H][W] fp32, box {w, rows, 32 channels, images})? Loads one box per variant
// (including negative / out-of-range start coordinates) and checks the smem image.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tma4d profiles/tma4d_probe.cu -lcuda && /tmp/tma4d
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void load4d(const __grid_constant__ CUtensorMap m, int c0, int c1, int c2, int c3, float* out, int n) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(n * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                sa(base)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(&bar))
            : "memory");
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(sa(&bar))
                         : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = reinterpret_cast<const float*>(base)[i];
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? std::atoi(argv[1]) : -1;
    const int W = 32, H = 32, C = 64, B = 2;
    std::vector<float> h(static_cast<size_t>(W) * H * C * B);
    for (size_t i = 0; i < h.size(); ++i) h[i] = static_cast<float>(i);
    float *x, *out;
    cudaMalloc(&x, h.size() * 4);
    cudaMemcpy(x, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 1 << 20);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    struct V {
        const char* name;
        CUtensorMapSwizzle sw;
        cuuint32_t box[4];
        int c[4];
    } vs[] = {
        {"sw128 {32,1,32,1} at (0,0,0,0)", CU_TENSOR_MAP_SWIZZLE_128B, {32, 1, 32, 1}, {0, 0, 0, 0}},
        {"sw128_32B {32,1,32,1} at (0,0,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {0, 0, 0, 0}},
        {"none {32,1,32,1} at (0,0,0,0)", CU_TENSOR_MAP_SWIZZLE_NONE, {32, 1, 32, 1}, {0, 0, 0, 0}},
        {"sw128_32B {32,1,32,1} at (-1,-1,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {-1, -1, 0, 0}},
        {"sw128_32B {16,2,32,1} at (1,0,32,1)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {16, 2, 32, 1}, {1, 0, 32, 1}},
        {"sw128 {32,1,32,1} at (-1,-1,0,0)", CU_TENSOR_MAP_SWIZZLE_128B, {32, 1, 32, 1}, {-1, -1, 0, 0}},
        {"none {32,1,32,1} at (-1,-1,0,0)", CU_TENSOR_MAP_SWIZZLE_NONE, {32, 1, 32, 1}, {-1, -1, 0, 0}},
        {"sw128_32B {32,1,32,1} at (1,31,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {1, 31, 0, 0}},
        {"sw128_32B {32,1,32,1} at (0,-1,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {0, -1, 0, 0}},
        {"sw128_32B {32,1,32,1} at (-1,0,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {-1, 0, 0, 0}},
        {"sw128_32B {32,1,32,1} at (1,32,0,0)", CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, {32, 1, 32, 1}, {1, 32, 0, 0}},
    };
    int idx = -1;
    for (const V& v : vs) {
        if (only >= 0 && ++idx != only) continue;
        CUtensorMap m;
        const cuuint64_t dims[4] = {W, H, C, B};
        const cuuint64_t strides[3] = {W * 4ull, H * W * 4ull, static_cast<cuuint64_t>(C) * H * W * 4};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, strides, v.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         v.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int n = v.box[0] * v.box[1] * v.box[2] * v.box[3];
        if (r != CUDA_SUCCESS) {
            std::printf("%-40s encode error %d\n", v.name, static_cast<int>(r));
            continue;
        }
        cudaMemset(out, 0xff, n * 4);
        load4d<<<1, 128, 8192 + 1024>>>(m, v.c[0], v.c[1], v.c[2], v.c[3], out, n);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> o(n);
        cudaMemcpy(o.data(), out, n * 4, cudaMemcpyDeviceToHost);
        std::printf("%-40s %s  first: %g %g %g %g | [32]: %g %g | [128]: %g\n", v.name, cudaGetErrorString(e), o[0], o[1],
                    o[2], o[3], o[32], o[33], o[128]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
