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
    ProfScope ps("elementwise", st, 12.0 * rows * cols);
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
    ProfScope ps("automorphism_eval", st, 8.0 * rows * n);
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
    ProfScope ps("automorphism_coeff", st, 8.0 * rows * n);
    automorphism_coeff_kernel<<<dim3(gx, rows), 256, 0, st>>>(in, out, row_slot, slots, n, k);
    CK(cudaGetLastError());
    return CKKS_OK;
}

// Exact centred lift from two limbs to many (bootstrapping ModRaise): for every
// column the value v in (-Q0/2, Q0/2], Q0 = q0*q1, is rebuilt from its two
// residues by Garner's formula and reduced modulo every target modulus.  (The
// non-centred fast conversion of baseconv.py would add Q0 * (0/1 polynomial) to
// the mask, which inflates the integer part EvalMod has to remove.)
__global__ void __launch_bounds__(256)
lift2_centered_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                      const int32_t* __restrict__ row_slot, const ModSlot* __restrict__ slots,
                      int32_t slot0, int32_t slot1, uint32_t q0_inv_mod_q1, int rows, size_t n) {
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const ModSlot m1 = slots[slot1];
    const uint64_t q0 = slots[slot0].q, q1 = m1.q;
    const uint32_t r0 = in[c], r1 = in[n + c];
    const uint32_t d = (uint32_t)(((uint64_t)r1 + q1 - r0 % q1) % q1);
    const uint64_t t = (uint64_t)d * q0_inv_mod_q1 % q1;
    const uint64_t v = r0 + q0 * t;                       // in [0, Q0)
    const uint64_t big = q0 * q1;
    const bool neg = v > big / 2;
    const uint64_t mag = neg ? big - v : v;
    for (int i = blockIdx.y; i < rows; i += gridDim.y) {
        const ModSlot& m = slots[row_slot[i]];
        uint32_t r = reduce64(mag, m);
        if (neg) r = r ? m.q - r : 0;
        out[(size_t)i * n + c] = r;
    }
}

int lift2_centered_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                          const ModSlot* slots, int32_t slot0, int32_t slot1, uint32_t inv,
                          int rows, size_t n, cudaStream_t st) {
    if (rows <= 0 || n == 0) return CKKS_OK;
    ProfScope ps("lift2_centered", st, 4.0 * n * (2 + rows));
    dim3 grid((unsigned)((n + 255) / 256), rows < 16 ? rows : 16);
    lift2_centered_kernel<<<grid, 256, 0, st>>>(in, out, row_slot, slots, slot0, slot1, inv, rows, n);
    CK(cudaGetLastError());
    return CKKS_OK;
}

// acc += x (.) p on both halves of a ciphertext in one pass (the inner loop of
// the BSGS linear transforms): acc, x are [2][rows][n], p is [rows][n].
__global__ void __launch_bounds__(256)
pmult_acc_kernel(const uint4* __restrict__ x, const uint4* __restrict__ p, uint4* acc,
                 const int32_t* __restrict__ row_slot, const ModSlot* __restrict__ slots,
                 int rows, size_t cols4, int first) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    const size_t half = (size_t)rows * cols4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols4; i += stride) {
        const uint4 pv = p[row * cols4 + i];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const size_t at = h * half + row * cols4 + i;
            const uint4 xv = x[at];
            uint4 r;
            r.x = mul_mod(xv.x, pv.x, m); r.y = mul_mod(xv.y, pv.y, m);
            r.z = mul_mod(xv.z, pv.z, m); r.w = mul_mod(xv.w, pv.w, m);
            if (!first) {
                const uint4 a = acc[at];
                r.x = add_mod(r.x, a.x, m.q); r.y = add_mod(r.y, a.y, m.q);
                r.z = add_mod(r.z, a.z, m.q); r.w = add_mod(r.w, a.w, m.q);
            }
            acc[at] = r;
        }
    }
}

int pmult_acc_launch(const uint32_t* x, const uint32_t* p, uint32_t* acc, const int32_t* row_slot,
                     const ModSlot* slots, int rows, size_t cols, int first, cudaStream_t st) {
    if (rows <= 0 || cols == 0) return CKKS_OK;
    if (cols % 4 || rows > 65535) { set_last_error("pmult_acc needs cols % 4 == 0 and <= 65535 rows"); return CKKS_ERR_UNSUPPORTED; }
    ProfScope ps("pmult_acc", st, 4.0 * cols * rows * (first ? 5.0 : 7.0));
    unsigned gx = (unsigned)((cols / 4 + 255) / 256);
    pmult_acc_kernel<<<dim3(gx, rows), 256, 0, st>>>((const uint4*)x, (const uint4*)p, (uint4*)acc,
                                                     row_slot, slots, rows, cols / 4, first);
    CK(cudaGetLastError());
    return CKKS_OK;
}

}  // namespace ckks
