// FP64 tensor-core (DMMA, mma.sync m8n8k4 / m16n8k8) throughput on sm_100a, against DFMA:
// decides whether a split-integer BConv contraction on the FP64 MMA path can beat the
// integer pipe (IMAD.WIDE at ~22 thread-ops/clk/SM).  Result = FMA / clk / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 2048
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1688(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int OP, int CH>
__global__ void probe(double* out) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 + threadIdx.x * 1e-9;
    double a4[4] = {a, a + 1, a + 2, a + 3}, b2[2] = {b, b + 1};
    double c2[CH][2], c4[CH][4];
#pragma unroll
    for (int i = 0; i < CH; ++i) { c2[i][0] = c2[i][1] = 0; c4[i][0] = c4[i][1] = c4[i][2] = c4[i][3] = 0; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (OP == 0) dmma884(c2[i], a, b);
            if (OP == 1) dmma1688(c4[i], a4, b2);
            if (OP == 2) { c2[i][0] = fma(a, b, c2[i][0]); c2[i][1] = fma(a, b, c2[i][1]); }
        }
    }
    double acc = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) acc += c2[i][0] + c2[i][1] + c4[i][0] + c4[i][1] + c4[i][2] + c4[i][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP, int CH>
void run(const char* name, double fma_per_warp_op, int warps_per_sm) {
    int dev; cudaGetDevice(&dev);
    cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    int sms = p.multiProcessorCount;
    int threads = 256, blocks = sms * warps_per_sm * 32 / threads;
    double* out; cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    probe<OP, CH><<<blocks, threads>>>(out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    probe<OP, CH><<<blocks, threads>>>(out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double warps = (double)blocks * threads / 32;
    double total = warps * ITERS * CH * fma_per_warp_op;
    double per_s = total / (ms * 1e-3);
    printf("%-34s warps/SM %2d chains %d  %8.3f ms  %8.2f TFMA/s  %7.1f FMA/clk/SM (at %d MHz)\n", name, warps_per_sm, CH,
           ms, per_s / 1e12, per_s / sms / (clk_khz * 1e3), clk_khz / 1000);
    cudaFree(out);
}

int main() {
    for (int w : {8, 16, 32, 64}) {
        run<0, 4>("DMMA m8n8k4 (256 FMA/warp-op)", 256, w);
        run<0, 8>("DMMA m8n8k4 (256 FMA/warp-op)", 256, w);
        run<1, 4>("DMMA m16n8k8 (1024 FMA/warp-op)", 1024, w);
        run<2, 8>("DFMA x2 (64 FMA/warp-op pair)", 64, w);
    }
    return 0;
}
