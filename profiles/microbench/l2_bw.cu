// L2 bandwidth and launch-overhead probes for sm_100a (B200): the numbers the reference's machine
// profile schema asks for (data/profiles/*.json: l2_read_bw, l2_write_bw, dram_bw, launch_overhead)
// and that MEASURED_PEAKS.json does not hold.  Read / write / copy sweeps over a buffer that stays
// L2-resident (32 MB) and one that does not (2 GB), 256-bit accesses, grid = 148 x 8 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ p, size_t n, uint32_t* sink, int passes) {
    uint32_t acc = 0;
    for (int r = 0; r < passes; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcg(p + i);          // .cg: served by the L2, not by the SM-local L1
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void wr(uint4* __restrict__ p, size_t n, uint32_t s, int passes) {
    for (int r = 0; r < passes; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(s, s + 1, s + 2, (uint32_t)i);
}
__global__ void cp(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n, int passes) {
    for (int r = 0; r < passes; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = __ldcg(a + i);
}
__global__ void empty_kernel() {}

template <class F>
static double time_ms(F launch, int reps) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
    const int grid = prop.multiProcessorCount * 8, block = 256;
    uint32_t* sink; cudaMalloc(&sink, 4);
    const size_t sizes[2] = {size_t(32) << 20, size_t(2) << 30};
    for (size_t bytes : sizes) {
        uint4 *a, *b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
        cudaMemset(a, 1, bytes); cudaMemset(b, 2, bytes);
        const size_t n = bytes / 16;
        const int reps = 10, passes = bytes > (size_t(1) << 30) ? 1 : 64;   // many sweeps per launch when resident
        double r = time_ms([&] { rd<<<grid, block>>>(a, n, sink, passes); }, reps);
        double w = time_ms([&] { wr<<<grid, block>>>(a, n, 7u, passes); }, reps);
        double c = time_ms([&] { cp<<<grid, block>>>(a, b, n / 2, passes); }, reps);   // half the buffer each way
        printf("%6zu MB  read %8.1f GB/s  write %8.1f GB/s  copy(r+w) %8.1f GB/s\n", bytes >> 20,
               bytes * passes / r / 1e6, bytes * passes / w / 1e6, bytes * passes / c / 1e6);
        cudaFree(a); cudaFree(b);
    }
    // launch overhead: a chain of empty kernels, eagerly and as one graph
    cudaStream_t st; cudaStreamCreate(&st);
    const int chain = 1000;
    double eager = time_ms([&] { for (int i = 0; i < chain; ++i) empty_kernel<<<1, 32, 0, st>>>(); cudaStreamSynchronize(st); }, 3);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < chain; ++i) empty_kernel<<<1, 32, 0, st>>>();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    double graph = time_ms([&] { cudaGraphLaunch(ge, st); cudaStreamSynchronize(st); }, 10);
    printf("dependent empty kernels: eager %.2f us each, in a graph %.2f us each\n", eager * 1e3 / chain, graph * 1e3 / chain);
    return 0;
}
