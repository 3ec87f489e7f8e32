// Micro-benchmark: per-node cost of a serial CUDA graph of trivial kernels on
// B200 as a function of the kernel-parameter size and grid size, and the cost
// of one dependent global-memory round trip. Guides how small the trainer's
// graph nodes can usefully get.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/graph_floor profiles/graph_floor.cu && /tmp/graph_floor
#include <cstdio>
#include <vector>

#include <cuda_runtime.h>

template <int BYTES>
struct Params {
    unsigned char pad[BYTES];
};

template <int BYTES>
__global__ void touch(Params<BYTES> p, float* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += p.pad[BYTES - 1];
}

__global__ void chase(const int* next, int hops, int* out) {
    int i = 0;
    for (int h = 0; h < hops; ++h) i = next[i];
    if (threadIdx.x == 0) out[blockIdx.x] = i;
}

template <int BYTES>
float serial_graph_us(int nodes, int grid, float* buf) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    Params<BYTES> p{};
    cudaGraphNode_t prev = nullptr;
    for (int i = 0; i < nodes; ++i) {
        void* args[] = {&p, &buf};
        cudaKernelNodeParams kp{};
        kp.func = (void*)touch<BYTES>;
        kp.gridDim = dim3(grid);
        kp.blockDim = dim3(256);
        kp.kernelParams = args;
        cudaGraphNode_t n;
        cudaGraphAddKernelNode(&n, g, prev ? &prev : nullptr, prev ? 1 : 0, &kp);
        prev = n;
    }
    cudaGraphExec_t e;
    cudaGraphInstantiate(&e, g, 0);
    cudaGraphLaunch(e, s);
    cudaStreamSynchronize(s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int r = 0; r < 5; ++r) cudaGraphLaunch(e, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(e);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
    return 1e3f * ms / (5.f * nodes);
}

int main() {
    float* buf;
    cudaMalloc(&buf, 1024);
    cudaMemset(buf, 0, 1024);
    printf("serial graph, us per node (256 threads/CTA)\n");
    printf("%10s %8s %8s %8s %8s\n", "param_B", "grid1", "grid148", "grid1024", "grid4096");
#define ROW(BYTES)                                                                                        \
    printf("%10d %8.2f %8.2f %8.2f %8.2f\n", BYTES, serial_graph_us<BYTES>(500, 1, buf),                 \
           serial_graph_us<BYTES>(500, 148, buf), serial_graph_us<BYTES>(500, 1024, buf),                 \
           serial_graph_us<BYTES>(500, 4096, buf));
    ROW(16) ROW(512) ROW(1024) ROW(2048) ROW(4096)
    // dependent round trips: L2-resident pointer chase
    const int n = 1 << 20;
    std::vector<int> h(n);
    for (int i = 0; i < n; ++i) h[i] = (int)((i * 7919LL + 104729) % n);
    int *d, *o;
    cudaMalloc(&d, n * sizeof(int));
    cudaMalloc(&o, 4096);
    cudaMemcpy(d, h.data(), n * sizeof(int), cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int hops : {1, 64}) {
        chase<<<1, 32>>>(d, hops, o);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) chase<<<1, 32>>>(d, hops, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("pointer chase %3d hops: %.2f us per kernel\n", hops, 1e3f * ms / 20);
    }
    return 0;
}
