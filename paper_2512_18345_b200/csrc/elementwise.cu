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
    pdl_trigger();
    pdl_wait();
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
        CK(launch_pdl(elementwise_vec4<K>, grid, dim3(256), 0, st, (const uint4*)a, (const uint4*)b, \
                      (uint4*)out, row_slot, slots, work));                                        \
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
    pdl_trigger();
    pdl_wait();
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
    CK(launch_pdl(automorphism_eval_kernel, dim3(gx, rows), dim3(256), 0, st, in, out, n, lg, k));
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

// Fused inner sum of a BSGS linear transform: out = sum_t x_t (.) p_t over up to
// kMaxTerms (rotated ciphertext, plaintext diagonal) pairs in one pass -- every operand
// is read once and the accumulator never leaves registers (products are summed in 64
// bits, four at a time, then reduced).  With p_t == null the term is x_t itself (plain
// sum of ciphertexts, the giant-step accumulation).
__global__ void __launch_bounds__(256)
fused_terms_kernel(FusedTerms terms, uint4* out, const int32_t* __restrict__ row_slot,
                   const ModSlot* __restrict__ slots, int rows, size_t cols4) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    pdl_trigger();
    pdl_wait();
    const size_t half = (size_t)rows * cols4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint64_t pol = l2_evict_first_policy();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols4; i += stride) {
        const size_t at = row * cols4 + i;
        uint64_t sa[4] = {0, 0, 0, 0}, sb[4] = {0, 0, 0, 0};
        uint32_t ra[4] = {0, 0, 0, 0}, rb[4] = {0, 0, 0, 0};
        int pending = 0;
        for (int t = 0; t < terms.count; ++t) {
            const uint4* x = reinterpret_cast<const uint4*>(terms.x[t]);
            const uint4* xh = terms.xb[t] ? reinterpret_cast<const uint4*>(terms.xb[t]) : x + half;
            const uint4 xa = x[at], xb = xh[at];
            if (terms.p[t]) {
                const uint4 pv = ld_stream(reinterpret_cast<const uint4*>(terms.p[t]) + at, pol);
                sa[0] += (uint64_t)xa.x * pv.x; sa[1] += (uint64_t)xa.y * pv.y;
                sa[2] += (uint64_t)xa.z * pv.z; sa[3] += (uint64_t)xa.w * pv.w;
                sb[0] += (uint64_t)xb.x * pv.x; sb[1] += (uint64_t)xb.y * pv.y;
                sb[2] += (uint64_t)xb.z * pv.z; sb[3] += (uint64_t)xb.w * pv.w;
            } else {
                sa[0] += xa.x; sa[1] += xa.y; sa[2] += xa.z; sa[3] += xa.w;
                sb[0] += xb.x; sb[1] += xb.y; sb[2] += xb.z; sb[3] += xb.w;
            }
            if (++pending == 4 || t == terms.count - 1) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    ra[k] = add_mod(ra[k], reduce64(sa[k], m), m.q);
                    rb[k] = add_mod(rb[k], reduce64(sb[k], m), m.q);
                    sa[k] = sb[k] = 0;
                }
                pending = 0;
            }
        }
        out[at] = make_uint4(ra[0], ra[1], ra[2], ra[3]);
        out[half + at] = make_uint4(rb[0], rb[1], rb[2], rb[3]);
    }
}

int fused_terms_launch(const FusedTerms& terms, uint32_t* out, const int32_t* row_slot,
                       const ModSlot* slots, int rows, size_t cols, cudaStream_t st) {
    if (rows <= 0 || cols == 0 || terms.count <= 0) return CKKS_OK;
    if (cols % 4 || rows > 65535 || terms.count > kMaxTerms) {
        set_last_error("fused_terms needs cols %% 4 == 0, <= 65535 rows, <= %d terms", kMaxTerms);
        return CKKS_ERR_UNSUPPORTED;
    }
    ProfScope ps("fused_terms", st, 4.0 * cols * rows * (3.0 * terms.count + 2.0));
    unsigned gx = (unsigned)((cols / 4 + 255) / 256);
    CK(launch_pdl(fused_terms_kernel, dim3(gx, rows), dim3(256), 0, st, terms, (uint4*)out, row_slot, slots, rows, cols / 4));
    CK(cudaGetLastError());
    return CKKS_OK;
}

// All giant-step inner sums of a BSGS linear transform in one pass:
//     out[g] = sum_b x[b] (.) p[g][b]          (absent diagonal: p[g][b] = a.zero, all zeros)
// Every baby-step ciphertext x[b] is read once for all NG outputs instead of once per
// giant step; only the plaintext diagonals (each used exactly once) scale with NG * NB.
// Two columns per thread keep the NG * 2 * 2 64-bit accumulators in registers.
template <int NG>
__global__ void __launch_bounds__(256)
fused_terms_multi_kernel(FusedMulti a, const int32_t* __restrict__ row_slot,
                         const ModSlot* __restrict__ slots, int rows, size_t cols2) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    pdl_trigger();
    pdl_wait();
    const size_t half = (size_t)rows * cols2;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cols2) return;
    const size_t at = row * cols2 + i;
    const uint64_t pol = l2_evict_first_policy();
    // 64-bit accumulators only: after every chunk of four terms a sum is folded to its residue
    // and carried as the seed of the next chunk (4 (q-1)^2 + q < 2^64 for q < 2^31), which
    // leaves the registers to keep a whole chunk of loads in flight
    uint64_t sa[NG][2], sb[NG][2];
#pragma unroll
    for (int g = 0; g < NG; ++g) sa[g][0] = sa[g][1] = sb[g][0] = sb[g][1] = 0;
    for (int b0 = 0; b0 < a.nb; b0 += 4) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int b = b0 + c;
            if (b < a.nb) {
                const uint2* x = reinterpret_cast<const uint2*>(a.x[b]);
                const uint2 xa = x[at], xb = x[half + at];
#pragma unroll
                for (int g = 0; g < NG; ++g) {
                    // absent diagonals point at a zero plaintext (host side): no branch, so the
                    // loads of a chunk are all issued before the first product
                    const uint2 pv = ld_stream2(reinterpret_cast<const uint2*>(a.p[g][b]) + at, pol);
                    sa[g][0] += (uint64_t)xa.x * pv.x; sa[g][1] += (uint64_t)xa.y * pv.y;
                    sb[g][0] += (uint64_t)xb.x * pv.x; sb[g][1] += (uint64_t)xb.y * pv.y;
                }
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                sa[g][k] = m.fast ? reduce64(sa[g][k], m) : sa[g][k] % m.q;
                sb[g][k] = m.fast ? reduce64(sb[g][k], m) : sb[g][k] % m.q;
            }
        }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        uint2* o = reinterpret_cast<uint2*>(a.out[g]);
        o[at] = make_uint2((uint32_t)sa[g][0], (uint32_t)sa[g][1]);
        o[half + at] = make_uint2((uint32_t)sb[g][0], (uint32_t)sb[g][1]);
    }
}

int fused_terms_multi_launch(const FusedMulti& a, const int32_t* row_slot, const ModSlot* slots,
                             int rows, size_t cols, cudaStream_t st) {
    if (rows <= 0 || cols == 0) return CKKS_OK;
    if (cols % 2 || rows > 65535 || a.nb < 1 || a.nb > kMaxTerms || a.ng < 1 || a.ng > kMaxGiants) {
        set_last_error("fused_terms_multi needs even cols, <= 65535 rows, <= %d terms, <= %d outputs", kMaxTerms, kMaxGiants);
        return CKKS_ERR_UNSUPPORTED;
    }
    double limbs = 2.0 * a.nb + 2.0 * a.ng;
    for (int g = 0; g < a.ng; ++g)
        for (int b = 0; b < a.nb; ++b) limbs += a.p[g][b] != a.zero ? 1.0 : 0.0;
    ProfScope ps("fused_terms", st, 4.0 * cols * rows * limbs);
    dim3 grid((unsigned)((cols / 2 + 255) / 256), rows);
    switch (a.ng) {
#define MULTI_CASE(G) case G: CK(launch_pdl(fused_terms_multi_kernel<G>, grid, dim3(256), 0, st, a, row_slot, slots, rows, cols / 2)); break;
        MULTI_CASE(1) MULTI_CASE(2) MULTI_CASE(3) MULTI_CASE(4) MULTI_CASE(5) MULTI_CASE(6) MULTI_CASE(7) MULTI_CASE(8)
#undef MULTI_CASE
    }
    CK(cudaGetLastError());
    return CKKS_OK;
}

// Tensor product of two ciphertexts in one pass (the front of HMult):
// d0 = b1*b2, d1 = a1*b2 + a2*b1, d2 = a1*a2; the four halves are [rows][n] each (separate
// pointers, so level-dropped views need no gathering copy), out is [3][rows][n] (d0, d1, d2).
__global__ void __launch_bounds__(256)
tensor_kernel(const uint4* __restrict__ xa, const uint4* __restrict__ xb, const uint4* __restrict__ ya,
              const uint4* __restrict__ yb, uint4* out, const int32_t* __restrict__ row_slot,
              const ModSlot* __restrict__ slots, int rows, size_t cols4) {
    const size_t row = blockIdx.y;
    const ModSlot m = slots[row_slot[row]];
    pdl_trigger();
    pdl_wait();
    const size_t half = (size_t)rows * cols4;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols4; i += stride) {
        const size_t at = row * cols4 + i;
        const uint4 a1 = xa[at], b1 = xb[at], a2 = ya[at], b2 = yb[at];
        const uint32_t A1[4] = {a1.x, a1.y, a1.z, a1.w}, B1[4] = {b1.x, b1.y, b1.z, b1.w};
        const uint32_t A2[4] = {a2.x, a2.y, a2.z, a2.w}, B2[4] = {b2.x, b2.y, b2.z, b2.w};
        uint32_t d0[4], d1[4], d2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            d0[k] = mul_mod(B1[k], B2[k], m);
            d2[k] = mul_mod(A1[k], A2[k], m);
            d1[k] = reduce64((uint64_t)A1[k] * B2[k] + (uint64_t)A2[k] * B1[k], m);
        }
        out[at] = make_uint4(d0[0], d0[1], d0[2], d0[3]);
        out[half + at] = make_uint4(d1[0], d1[1], d1[2], d1[3]);
        out[2 * half + at] = make_uint4(d2[0], d2[1], d2[2], d2[3]);
    }
}

int tensor_launch(const uint32_t* xa, const uint32_t* xb, const uint32_t* ya, const uint32_t* yb,
                  uint32_t* out, const int32_t* row_slot, const ModSlot* slots, int rows, size_t cols,
                  cudaStream_t st) {
    if (rows <= 0 || cols == 0) return CKKS_OK;
    if (cols % 4 || rows > 65535) { set_last_error("tensor needs cols %% 4 == 0 and <= 65535 rows"); return CKKS_ERR_UNSUPPORTED; }
    ProfScope ps("tensor", st, 4.0 * cols * rows * 7.0);
    unsigned gx = (unsigned)((cols / 4 + 255) / 256);
    CK(launch_pdl(tensor_kernel, dim3(gx, rows), dim3(256), 0, st, (const uint4*)xa, (const uint4*)xb,
                  (const uint4*)ya, (const uint4*)yb, (uint4*)out, row_slot, slots, rows, cols / 4));
    CK(cudaGetLastError());
    return CKKS_OK;
}

}  // namespace ckks
