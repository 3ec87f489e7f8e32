// Probe: resource attributes of update_group_kernel and a trial launch at its smem size.
#include "../../paper_2503_12053_b200/csrc/kernels.cu"
int main() {
    using namespace fb200;
    const void* f = group_func<16>();
    cudaFuncAttributes at{};
    cudaError_t e = cudaFuncGetAttributes(&at, f);
    printf("attr %s regs %d static %zu maxThreads %d maxDyn %d local %zu\n", cudaGetErrorString(e), at.numRegs,
           at.sharedSizeBytes, at.maxThreadsPerBlock, at.maxDynamicSharedSizeBytes, at.localSizeBytes);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    printf("optin %d kGrpSmem %zu threads %d\n", optin, kGrpSmem, kGrpThreads);
    GroupArgs a{};
    a.n_tiles = 0; a.n_wtiles = 0; a.G = 1; a.n0 = 1; a.B = 1;
    void* args[] = {&a};
    e = cudaLaunchKernel(f, dim3(1), dim3(kGrpThreads), args, kGrpSmem, 0);
    printf("launch %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync %s\n", cudaGetErrorString(e));
    return 0;
}
