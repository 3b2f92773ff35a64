// Integer-pipe throughput probes for sm_100a (B200): which of the instructions the
// NTT / BConv inner loops are built from issue at which rate.  Each kernel runs a long
// unrolled chain of ILP-8 independent ops per thread; result = thread-ops / clk / SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
template <int OP>
__global__ void probe(uint32_t* out, uint32_t a0, uint32_t b0, uint32_t q) {
    uint32_t x[8];
    uint64_t w[8];
    double d[8];
    const double db = 1.0000001 + threadIdx.x * 1e-9, dq = 0.5;
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = a0 + threadIdx.x * 8 + i; w[i] = x[i]; d[i] = (double)x[i]; }
    uint32_t b = b0 + threadIdx.x;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = x[i] * b + q;                       // IMAD (lo)
            if (OP == 1) x[i] = __umulhi(x[i], b) + q;              // IMAD.HI
            if (OP == 2) w[i] = (uint64_t)(uint32_t)w[i] * b + w[i];// IMAD.WIDE with 64-bit accumulate
            if (OP == 3) x[i] = min(x[i], x[i] - q);                // VIADDMNMX
            if (OP == 4) x[i] = x[i] + b + q;                       // IADD3
            if (OP == 5) { uint32_t t = __umulhi(x[i], b); x[i] = x[i] * a0 - t * q; x[i] = min(x[i], x[i] - q); } // Shoup mul
            if (OP == 6) w[i] = w[i] + (((uint64_t)b << 32) | x[i]); // 64-bit add
            if (OP == 7) x[i] = (x[i] ^ b) + q;                     // LOP3 + IADD
            if (OP == 8) { uint64_t t = (uint64_t)x[i] * b; x[i] = (uint32_t)t ^ (uint32_t)(t >> 32); } // IMAD.WIDE no acc + LOP
            if (OP == 9) d[i] = fma(d[i], db, dq);                  // DFMA
            if (OP == 10) { w[i] = __double2ull_rz(d[i]) + w[i]; d[i] += 1.0; }  // F2I.U64.F64 (+DADD)
            if (OP == 11) { d[i] = (double)x[i] + d[i]; x[i] += 3; }             // I2F.F64.U32 (+DADD)
            if (OP == 12) x[i] = x[i] + b * (x[i] >> 3);                         // SHF + IMAD
        }
    }
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += x[i] + (uint32_t)w[i] + (uint32_t)(w[i] >> 32) + (uint32_t)__double2uint_rz(d[i] * 1e-300);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int OP>
void run(const char* name, double ops_per_iter) {
    int dev; cudaGetDevice(&dev);
    cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    int sms = p.multiProcessorCount;
    uint32_t* out; cudaMalloc(&out, sizeof(uint32_t) * sms * 8 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    probe<OP><<<sms * 8, 256>>>(out, 12345u, 678u, 2147352577u);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    probe<OP><<<sms * 8, 256>>>(out, 12345u, 678u, 2147352577u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    double total = (double)sms * 8 * 256 * ITERS * 8 * ops_per_iter;
    double per_s = total / (ms * 1e-3);
    printf("%-28s %8.3f ms  %8.1f Gop/s  %6.1f thread-ops/clk/SM (at %d MHz)\n", name, ms, per_s / 1e9,
           per_s / sms / (clk_khz * 1e3), clk_khz / 1000);
    cudaFree(out);
}

int main() {
    run<0>("IMAD.lo", 1);
    run<1>("IMAD.HI", 1);
    run<2>("IMAD.WIDE (64b acc)", 1);
    run<3>("VIADDMNMX (csub)", 1);
    run<4>("IADD3", 1);
    run<5>("Shoup mul (3 IMAD + csub)", 1);
    run<6>("64-bit add", 1);
    run<7>("LOP3+IADD", 1);
    run<8>("IMAD.WIDE no-acc + LOP3", 1);
    run<9>("DFMA", 1);
    run<10>("F2I.U64.F64 + IADD64 + DADD", 1);
    run<11>("I2F.F64.U32 + DADD + IADD", 1);
    run<12>("SHF + IMAD", 1);
    return 0;
}
