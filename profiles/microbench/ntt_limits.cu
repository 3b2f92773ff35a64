// What bounds the N = 2^16 transform kernels on B200?  Three probes built from the same
// radix-16 Shoup butterfly passes as csrc/ntt.cu:
//   compute : the two register passes + the shared-memory transpose of ntt16_fwd_strided, looped
//             on registers (no global traffic)            -> butterflies / clk / SM vs resident CTAs
//   memory  : the strided kernel's global access pattern only (16 column loads, 16 column stores)
//   full    : load + compute + store, one tile per CTA (the production shape)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ntt_limits ntt_limits.cu -lcuda && ./ntt_limits
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t q) { return min(x, x - q); }
__device__ __forceinline__ uint32_t shoup_mul(uint32_t y, uint32_t w, uint32_t ws, uint32_t q) {
    uint32_t t = __umulhi(y, ws);
    return csub(y * w - t * q, q);
}
__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint32_t v, uint32_t q) {
    const uint32_t xc = csub(x, q);
    x = xc + v;
    y = xc - v + q;
}
template <class MUL>
__device__ __forceinline__ void ct16(uint32_t (&v)[16], uint32_t q, MUL mul) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int half = 8 >> s;
            const int g = b >> (3 - s), j = b & (half - 1);
            const int i0 = g * 2 * half + j;
            ct_bfly(v[i0], v[i0 + half], mul(s, g, v[i0 + half]), q);
        }
    }
}
#define TW_MUL(expr) [&](int s, int gi, uint32_t y) { const uint2 w = (expr); return shoup_mul(y, w.x, w.y, q); }

#ifndef NCOLS
#define NCOLS 16
#endif
constexpr int COLS = NCOLS;          // -DNCOLS=32: 128-byte row segments, 512-thread CTAs (probe<> only)
constexpr int THREADS = 16 * COLS;
constexpr int kN = 65536;

// MODE 0: full, 1: compute only (ITERS tiles on registers), 2: memory only, 3: loads + compute, 4: compute + stores
template <int MODE>
__global__ void __launch_bounds__(THREADS) probe(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q, int iters) {
    __shared__ uint2 s_tw[256];
    __shared__ uint32_t tile[271 * COLS];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    for (int i = tid; i < 256; i += THREADS) s_tw[i] = tw[i];
    const size_t base = (size_t)blockIdx.y * kN + blockIdx.x * COLS + c;
    uint32_t v[16];
    if (MODE == 1 || MODE == 4) {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = tid * 16 + k + blockIdx.x;
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = in[base + (g + 16 * k) * 256];
    }
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        if (MODE != 2) {
            ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));
#pragma unroll
            for (int k = 0; k < 16; ++k) tile[(g + 17 * k) * COLS + c] = v[k];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] = tile[(17 * g + k) * COLS + c];
            ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));
            if (MODE == 1) __syncthreads();
        }
    }
    if (MODE == 1 || MODE == 3) {
        uint32_t acc = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc ^= v[k];
        if (acc == 0x12345u) out[tid] = acc;
    } else {
#pragma unroll
        for (int k = 0; k < 16; ++k) out[base + (16 * g + k) * 256] = csub(v[k], q);
    }
}

// Pipelined variant: a CTA walks T consecutive tiles of one limb; tile i+1 is fetched with
// cp.async (16-byte chunks, no register staging) into the other half of a double buffer while
// tile i is transformed; the twiddles of the limb are staged once.
#if NCOLS == 16
template <int T>
__global__ void __launch_bounds__(256) probe_pipe(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q) {
    __shared__ uint2 s_tw[256];
    // row j of a tile lives at padded row j + (j >> 4): the layout both register passes read and
    // write without bank conflicts, so the landing buffer is also the transpose buffer
    __shared__ __align__(16) uint32_t inbuf[2][272 * COLS];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    for (int i = tid; i < 256; i += 256) s_tw[i] = tw[i];
    const uint32_t* limb = in + (size_t)blockIdx.y * kN;
    auto issue = [&](int t, int buf) {
        const int col0 = (blockIdx.x * T + t) * COLS;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int chunk = tid + 256 * k, row = chunk >> 2, part = chunk & 3;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&inbuf[buf][(row + (row >> 4)) * COLS + part * 4]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(limb + row * 256 + col0 + part * 4));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue(0, 0);
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        if (t + 1 < T) { issue(t + 1, (t + 1) & 1); asm volatile("cp.async.wait_group 1;" ::: "memory"); }
        else asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        uint32_t v[16];
#pragma unroll
        uint32_t* tile = inbuf[t & 1];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = tile[(g + 17 * k) * COLS + c];
        ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));
#pragma unroll
        for (int k = 0; k < 16; ++k) tile[(g + 17 * k) * COLS + c] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = tile[(17 * g + k) * COLS + c];
        ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));
        uint32_t* dst = out + (size_t)blockIdx.y * kN + (blockIdx.x * T + t) * COLS + c;
#pragma unroll
        for (int k = 0; k < 16; ++k) dst[(16 * g + k) * 256] = csub(v[k], q);
    }
}

// Staggered start: in the first wave every other resident CTA of an SM waits `delay_ns` before it
// loads, so that one half of the SM's CTAs computes while the other half loads (without it the
// CTAs of a wave move through load / compute / store in lock-step).
__global__ void __launch_bounds__(256) probe_stagger(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q, int sms, unsigned delay_ns) {
    __shared__ uint2 s_tw[256];
    __shared__ uint32_t tile[271 * COLS];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    for (int i = tid; i < 256; i += 256) s_tw[i] = tw[i];
    const unsigned lin = blockIdx.y * gridDim.x + blockIdx.x;
    if (lin < 8u * sms && ((lin / sms) & 1)) __nanosleep(delay_ns);
    const size_t base = (size_t)blockIdx.y * kN + blockIdx.x * COLS + c;
    uint32_t v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = in[base + (g + 16 * k) * 256];
    __syncthreads();
    ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(g + 17 * k) * COLS + c] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[(17 * g + k) * COLS + c];
    ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) out[base + (16 * g + k) * 256] = csub(v[k], q);
}

template <int T>
void run_pipe(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q, int rows_buf, int sms, int clk_khz) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r : {48, 96, 192, 384}) {
        dim3 grid(256 / COLS / T, r);
        float best = 1e9, ms;
        for (int rep = 0; rep < 5; ++rep) {
            const uint32_t* src = in + (size_t)(rep & 1) * rows_buf * kN * (r <= 192);
            cudaEventRecord(a);
            probe_pipe<T><<<grid, 256>>>(src, out, tw, q);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double bf = (double)r * 32768 * 8;
        printf("pipe T=%d rows=%3d: %7.2f us  %6.0f GB/s (r+w)  %5.2f butterflies/clk/SM (%s)\n", T, r, best * 1e3,
               2.0 * r * kN * 4 / (best * 1e-3) / 1e9, bf / (best * 1e-3) / sms / (clk_khz * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
}

// Co-scheduling probe: a thin persistent HBM-streaming kernel (grid = SMs x ctas_per_sm) next to
// the transform kernel on a second stream.  Do the two proceed concurrently at full speed?
__global__ void __launch_bounds__(256) stream_read(const uint4* src, size_t n16, uint32_t* out) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
        for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x1234567u) out[0] = acc.x;
}

void run_overlap(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q, int sms) {
    const size_t big_bytes = (size_t)2 << 30;
    uint4* big; cudaMalloc(&big, big_bytes); cudaMemset(big, 5, big_bytes);
    cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
    cudaEvent_t a, b, e2; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&e2);
    float ms;
    const int reps = 8;
    dim3 grid(256 / COLS, 192);
    for (int per_sm : {1, 2, 4, 8}) {
        // alone: stream kernel
        cudaDeviceSynchronize();
        cudaEventRecord(a, s1);
        stream_read<<<sms * per_sm, 256, 0, s1>>>(big, big_bytes / 16, out);
        cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        const float t_stream = ms;
        // alone: transforms
        cudaEventRecord(a, s2);
        for (int r = 0; r < reps; ++r) probe<0><<<grid, THREADS, 0, s2>>>(in + (size_t)(r & 1) * 192 * kN, out + 64, tw, q, 1);
        cudaEventRecord(b, s2); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        const float t_ntt = ms;
        // both
        cudaDeviceSynchronize();
        cudaEventRecord(a, s1);
        cudaStreamWaitEvent(s2, a, 0);
        stream_read<<<sms * per_sm, 256, 0, s1>>>(big, big_bytes / 16, out);
        for (int r = 0; r < reps; ++r) probe<0><<<grid, THREADS, 0, s2>>>(in + (size_t)(r & 1) * 192 * kN, out + 64, tw, q, 1);
        cudaEventRecord(e2, s2);
        cudaStreamWaitEvent(s1, e2, 0);
        cudaEventRecord(b, s1); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("co-schedule: stream kernel %d CTA/SM alone %7.1f us (%5.0f GB/s), 8 x NTT(192 rows) alone %7.1f us, together %7.1f us (sum %7.1f, max %7.1f)\n",
               per_sm, t_stream * 1e3, big_bytes / (t_stream * 1e-3) / 1e9, t_ntt * 1e3, ms * 1e3, (t_stream + t_ntt) * 1e3,
               (t_stream > t_ntt ? t_stream : t_ntt) * 1e3);
    }
    cudaFree(big);
}

// TMA variant: the 256 x 16 input tile arrives with ONE cp.async.bulk.tensor.2d (box 16 x 256 of a
// [rows * 256][256] u32 tensor) signalled on an mbarrier, instead of 16 column loads per thread.
// T tiles per CTA, double buffered: tile t + 1 is requested before tile t is transformed.
template <int T>
__global__ void __launch_bounds__(256) probe_tma(const __grid_constant__ CUtensorMap tmap, uint32_t* out, const uint2* tw, uint32_t q) {
    // the landing buffer doubles as the transpose buffer: after the first pass row j is written back at
    // row j ^ ((j >> 4) & 1), which makes both the write (j = g + 16k) and the read (j = 16g + k) conflict-free
    __shared__ __align__(128) uint32_t inbuf[2][256 * COLS];
    __shared__ uint2 s_tw[256];
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    for (int i = tid; i < 256; i += 256) s_tw[i] = tw[i];
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0 + 8));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int t, int buf) {
        if (tid == 0) {
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&inbuf[buf][0]);
            const int c0 = (blockIdx.x * T + t) * COLS, c1 = blockIdx.y * 256;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar0 + 8 * buf), "r"(256 * COLS * 4) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         :: "r"(dst), "l"(&tmap), "r"(c0), "r"(c1), "r"(bar0 + 8 * buf) : "memory");
        }
    };
    issue(0, 0);
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        if (t + 1 < T) issue(t + 1, (t + 1) & 1);
        const uint32_t b = bar0 + 8 * (t & 1), parity = (t >> 1) & 1;
        asm volatile("{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra DONE;\n bra WAIT;\n DONE:\n}" :: "r"(b), "r"(parity) : "memory");
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = inbuf[t & 1][(g + 16 * k) * COLS + c];
        __syncthreads();       // all inputs are in registers before anyone writes back
        ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));
        uint32_t* tile = inbuf[t & 1];
#pragma unroll
        for (int k = 0; k < 16; ++k) tile[((g ^ (k & 1)) + 16 * k) * COLS + c] = v[k];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = tile[(16 * g + (k ^ (g & 1))) * COLS + c];
        ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));
        uint32_t* dst = out + (size_t)blockIdx.y * kN + (blockIdx.x * T + t) * COLS + c;
#pragma unroll
        for (int k = 0; k < 16; ++k) dst[(16 * g + k) * 256] = csub(v[k], q);
        __syncthreads();       // everyone is done with inbuf[t & 1] before it is refilled
    }
}

template <int T>
void run_tma(const uint32_t* in, uint32_t* out, const uint2* tw, uint32_t q, int rows_buf, int sms, int clk_khz) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int r : {24, 48, 96, 192, 384}) {
        float best = 1e9, ms;
        for (int rep = 0; rep < 5; ++rep) {
            const uint32_t* src = in + (size_t)(rep & 1) * rows_buf * kN * (r <= 192);
            CUtensorMap tmap;
            cuuint64_t dims[2] = {256, (cuuint64_t)r * 256};
            cuuint64_t strides[1] = {256 * 4};
            cuuint32_t box[2] = {COLS, 256};
            cuuint32_t estr[2] = {1, 1};
            CUresult rc = cuTensorMapEncodeTiled(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)src, dims, strides, box, estr,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (rc != CUDA_SUCCESS) { printf("cuTensorMapEncodeTiled failed: %d\n", (int)rc); return; }
            dim3 grid(256 / COLS / T, r);
            cudaEventRecord(a);
            probe_tma<T><<<grid, 256>>>(tmap, out, tw, q);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double bf = (double)r * 32768 * 8;
        printf("tma  T=%d rows=%3d: %7.2f us  %6.0f GB/s (r+w)  %5.2f butterflies/clk/SM (%s)\n", T, r, best * 1e3,
               2.0 * r * kN * 4 / (best * 1e-3) / 1e9, bf / (best * 1e-3) / sms / (clk_khz * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
}

#endif  // NCOLS == 16

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const uint32_t q = 2147352577u;
    const int rows = 192;
    uint32_t *in, *out; uint2* tw;
    cudaMalloc(&in, sizeof(uint32_t) * rows * kN * 2);
    cudaMalloc(&out, sizeof(uint32_t) * rows * kN * 2);
    cudaMalloc(&tw, sizeof(uint2) * 256);
    cudaMemset(in, 1, sizeof(uint32_t) * rows * kN * 2);
    cudaMemset(tw, 3, sizeof(uint2) * 256);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms;
    // compute only: grid = sms * ctas_per_sm, pad dynamic smem to cap residency
    for (int per_sm = 1; per_sm <= 8; ++per_sm) {
        const int iters = 256;
        // 19.4 KB static smem per CTA; add dynamic padding so at most per_sm CTAs fit in 227 KB
        size_t pad = per_sm >= 8 ? 0 : (size_t)(227 * 1024 / per_sm) - 21 * 1024;
        if (pad > 200 * 1024) pad = 200 * 1024;
        cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pad);
        dim3 grid(sms * per_sm, 1);
        probe<1><<<grid, THREADS, pad>>>(in, out, tw, q, iters);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        probe<1><<<grid, THREADS, pad>>>(in, out, tw, q, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        const double bf = (double)grid.x * THREADS * 64 * iters;
        printf("compute-only  %d CTA/SM (%2d warps/SM): %7.3f ms  %5.2f butterflies/clk/SM  (%s)\n", per_sm, per_sm * THREADS / 32, ms,
               bf / (ms * 1e-3) / sms / (clk_khz * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
    for (int r : {24, 48, 96, 192, 384}) {
        dim3 grid(256 / COLS, r);
        for (int mode = 0; mode < 3; mode += 2) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                const uint32_t* src = in + (size_t)(rep & 1) * rows * kN * (r <= 192);
                cudaEventRecord(a);
                if (mode == 0) probe<0><<<grid, THREADS>>>(src, out, tw, q, 1);
                else probe<2><<<grid, THREADS>>>(src, out, tw, q, 1);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const double bf = (double)r * 32768 * 8;
            printf("%s rows=%3d: %7.2f us  %6.0f GB/s (r+w)  %5.2f butterflies/clk/SM\n", mode == 0 ? "full  " : "memory", r,
                   best * 1e3, 2.0 * r * kN * 4 / (best * 1e-3) / 1e9, mode == 0 ? bf / (best * 1e-3) / sms / (clk_khz * 1e3) : 0.0);
        }
    }
    for (int mode = 3; mode <= 4; ++mode)
        for (int r : {192, 384}) {
            dim3 grid(256 / COLS, r);
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                const uint32_t* src = in + (size_t)(rep & 1) * rows * kN * (r <= 192);
                cudaEventRecord(a);
                if (mode == 3) probe<3><<<grid, THREADS>>>(src, out, tw, q, 1);
                else probe<4><<<grid, THREADS>>>(src, out, tw, q, 1);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%s rows=%3d: %7.2f us  %5.2f butterflies/clk/SM\n", mode == 3 ? "loads + compute " : "compute + stores", r, best * 1e3,
                   (double)r * 32768 * 8 / (best * 1e-3) / sms / (clk_khz * 1e3));
        }
    for (int per_sm : {2, 3, 4, 6, 8}) {
        size_t pad = per_sm >= 8 ? 0 : (size_t)(227 * 1024 / per_sm) - 21 * 1024;
        cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pad);
        dim3 grid(256 / COLS, 384);
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            probe<0><<<grid, THREADS, pad>>>(in, out, tw, q, 1);
            cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("full rows=384 at most %d CTA/SM: %7.2f us  %5.2f butterflies/clk/SM\n", per_sm, best * 1e3,
               (double)384 * 32768 * 8 / (best * 1e-3) / sms / (clk_khz * 1e3));
    }
#if NCOLS == 16
    run_tma<1>(in, out, tw, q, rows, sms, clk_khz);
    run_tma<2>(in, out, tw, q, rows, sms, clk_khz);
    run_tma<4>(in, out, tw, q, rows, sms, clk_khz);
    run_overlap(in, out, tw, q, sms);
    for (unsigned delay : {0u, 1000u})
        for (int r : {96, 192, 384}) {
            dim3 grid(256 / COLS, r);
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                const uint32_t* src = in + (size_t)(rep & 1) * rows * kN * (r <= 192);
                cudaEventRecord(a);
                probe_stagger<<<grid, 256>>>(src, out, tw, q, sms, delay);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("stagger %4u ns rows=%3d: %7.2f us  %5.2f butterflies/clk/SM\n", delay, r, best * 1e3,
                   (double)r * 32768 * 8 / (best * 1e-3) / sms / (clk_khz * 1e3));
        }
    run_pipe<2>(in, out, tw, q, rows, sms, clk_khz);
    run_pipe<4>(in, out, tw, q, rows, sms, clk_khz);
#endif
    return 0;
}
