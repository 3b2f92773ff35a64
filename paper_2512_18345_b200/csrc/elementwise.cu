// elementwise.cu -- limb-wise add/sub/mul and the ring automorphism.
//
// Reference: rns.py:243-258 (poly_elementwise), rns.py:261-320 (automorphism).
// All three are HBM-bound streaming kernels: 128-bit accesses, one pass.
#include "common.cuh"
#include "internal.h"

namespace ckks {

template <int KIND>
__device__ __forceinline__ uint32_t ew_op(uint32_t a, uint32_t b, const ModSlot& m) {
    if (KIND == 0) return m.q >> 31 ? (uint32_t)(((uint64_t)a + b) % m.q) : add_mod(a, b, m.q);
    if (KIND == 1) return m.q >> 31 ? (uint32_t)(((uint64_t)a + m.q - b) % m.q) : sub_mod(a, b, m.q);
    return mul_mod(a, b, m);
}

template <int KIND>
__global__ void __launch_bounds__(256)
elementwise_vec4(const uint4* a, const uint4* b, uint4* out, const int32_t* __restrict__ row_slot,
                 const ModSlot* __restrict__ slots, size_t cols4) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols4; i += stride) {
        const uint4 x = a[row * cols4 + i], y = b[row * cols4 + i];
        uint4 r;
        r.x = ew_op<KIND>(x.x, y.x, m);
        r.y = ew_op<KIND>(x.y, y.y, m);
        r.z = ew_op<KIND>(x.z, y.z, m);
        r.w = ew_op<KIND>(x.w, y.w, m);
        out[row * cols4 + i] = r;
    }
}

template <int KIND>
__global__ void __launch_bounds__(256)
elementwise_scalar(const uint32_t* a, const uint32_t* b, uint32_t* out,
                   const int32_t* __restrict__ row_slot, const ModSlot* __restrict__ slots,
                   size_t cols) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols; i += stride)
        out[row * cols + i] = ew_op<KIND>(a[row * cols + i], b[row * cols + i], m);
}

int elementwise_launch(const uint32_t* a, const uint32_t* b, uint32_t* out, const int32_t* row_slot,
                       const ModSlot* slots, int rows, size_t cols, int kind, cudaStream_t st) {
    if (rows <= 0 || cols == 0) return CKKS_OK;
    if (rows > 65535) { set_last_error("more than 65535 rows per launch is not supported"); return CKKS_ERR_UNSUPPORTED; }
    const bool vec = (cols % 4 == 0) && (((uintptr_t)a | (uintptr_t)b | (uintptr_t)out) % 16 == 0);
    const size_t work = vec ? cols / 4 : cols;
    unsigned gx = (unsigned)((work + 255) / 256);
    if (gx > 1024) gx = 1024;
    dim3 grid(gx, rows);
    ProfScope ps("elementwise", st);
#define EW_DISPATCH(K)                                                                             \
    if (vec)                                                                                       \
        elementwise_vec4<K><<<grid, 256, 0, st>>>((const uint4*)a, (const uint4*)b, (uint4*)out,   \
                                                  row_slot, slots, work);                          \
    else                                                                                           \
        elementwise_scalar<K><<<grid, 256, 0, st>>>(a, b, out, row_slot, slots, work);
    if (kind == 0) { EW_DISPATCH(0) }
    else if (kind == 1) { EW_DISPATCH(1) }
    else if (kind == 2) { EW_DISPATCH(2) }
    else { set_last_error("unknown element-wise kind %d", kind); return CKKS_ERR_ARG; }
#undef EW_DISPATCH
    CK(cudaGetLastError());
    return CKKS_OK;
}

// Evaluation-domain automorphism: out[:, t] = in[:, j(t)] with
//   j = bitrev(((2*bitrev(t) + 1) * k mod 2N - 1) / 2)            (SURVEY 8a'.4)
// the closed form of the permutation the reference derives by probing its own
// transform (rns.py:268-292).  Within a warp the 32 source columns fall in one
// aligned 128-byte line (only the low five bits of j vary), so the gather is
// as coalesced as the store.
__global__ void __launch_bounds__(256)
automorphism_eval_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t n,
                         uint32_t lg, uint32_t k) {
    const size_t row = blockIdx.y;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const uint32_t u = __brev(t) >> (32 - lg);
        const uint32_t e = ((2 * u + 1) * k) & (2 * n - 1);
        const uint32_t j = __brev((e - 1) >> 1) >> (32 - lg);
        out[row * n + t] = in[row * n + j];
    }
}

int automorphism_eval_launch(const uint32_t* in, uint32_t* out, int rows, uint32_t n, uint32_t k,
                             cudaStream_t st) {
    if (rows <= 0) return CKKS_OK;
    if (rows > 65535) { set_last_error("more than 65535 rows per launch is not supported"); return CKKS_ERR_UNSUPPORTED; }
    if (in == out) { set_last_error("automorphism cannot run in place"); return CKKS_ERR_ARG; }
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    if (lg == 0) {
        CK(cudaMemcpyAsync(out, in, sizeof(uint32_t) * rows, cudaMemcpyDeviceToDevice, st));
        return CKKS_OK;
    }
    unsigned gx = (n + 255) / 256;
    if (gx > 256) gx = 256;
    ProfScope ps("automorphism_eval", st);
    automorphism_eval_kernel<<<dim3(gx, rows), 256, 0, st>>>(in, out, n, lg, k);
    CK(cudaGetLastError());
    return CKKS_OK;
}

// Coefficient-domain automorphism: coefficient i moves to i*k mod 2N, negated
// when it wraps past N (rns.py:261-265, :306-312).  k odd makes it a bijection.
__global__ void __launch_bounds__(256)
automorphism_coeff_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                          const int32_t* __restrict__ row_slot, const ModSlot* __restrict__ slots,
                          uint32_t n, uint32_t k) {
    const size_t row = blockIdx.y;
    const uint32_t q = slots[row_slot[row]].q;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t j = (uint32_t)(((uint64_t)i * k) & (2ull * n - 1));
        uint32_t v = in[row * n + i];
        if (j >= n) v = v ? q - v : 0;
        out[row * n + (j & (n - 1))] = v;
    }
}

int automorphism_coeff_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                              const ModSlot* slots, int rows, uint32_t n, uint32_t k, cudaStream_t st) {
    if (rows <= 0) return CKKS_OK;
    if (rows > 65535) { set_last_error("more than 65535 rows per launch is not supported"); return CKKS_ERR_UNSUPPORTED; }
    if (in == out) { set_last_error("automorphism cannot run in place"); return CKKS_ERR_ARG; }
    unsigned gx = (n + 255) / 256;
    if (gx > 256) gx = 256;
    ProfScope ps("automorphism_coeff", st);
    automorphism_coeff_kernel<<<dim3(gx, rows), 256, 0, st>>>(in, out, row_slot, slots, n, k);
    CK(cudaGetLastError());
    return CKKS_OK;
}

}  // namespace ckks
