// common.cuh -- device arithmetic and shared structures of libckks_b200.so.
//
// Word size: residues are u32 in [0, q), q < 2^31 on every fast path (all
// parameter sets of the reference are 31-bit, data/params/*.json).  With
// 2q < 2^32 a value in [0, 2q) fits a register, which is what the lazy Shoup
// butterflies below rely on.  Every kernel canonicalises to [0, q) before a
// store that crosses the C ABI (reference rns.py:4-6).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ckks {

// One registered (q, n, psi): per-modulus constants and twiddle tables in HBM.
// Twiddles are {w, floor(w * 2^32 / q)} pairs (Shoup form) in the slot order
// of the reference tables: fwd[t] = psi^bitrev(t), inv[t] = psi^-bitrev(t)
// (transform.py:43-49, :97-100).
struct ModSlot {
    uint32_t q;
    uint32_t n;            // ring degree the tables were built for (0: none)
    uint32_t qinv;         // q^-1 mod 2^32          (Montgomery, subtractive form)
    uint32_t r1, r1s;      // 2^32 mod q and its Shoup companion
    uint32_t r2, r2s;      // 2^64 mod q and its Shoup companion
    uint32_t n_inv, n_inv_s;      // N^-1 mod q (transform.py:112)
    uint32_t w_last, w_last_s;    // inv[1] * N^-1: twiddle of the last GS stage (:243-246)
    uint32_t fast;         // 1 when 2^30 < q < 2^31 (two-subtraction range tricks valid)
    const uint2* fwd;      // [n]
    const uint2* inv;      // [n]
};

// ---- scalar modular arithmetic ------------------------------------------------

// x in [0, 2q) -> [0, q).  One VIADDMNMX on sm_100a.
__device__ __forceinline__ uint32_t csub(uint32_t x, uint32_t q) {
    return min(x, x - q);
}

// y * w mod q, lazily: result in [0, 2q).  Valid for ANY 32-bit y, w < q,
// ws = floor(w * 2^32 / q), q < 2^31.
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t y, uint32_t w, uint32_t ws, uint32_t q) {
    uint32_t t = __umulhi(y, ws);
    return y * w - t * q;
}

__device__ __forceinline__ uint32_t shoup_mul(uint32_t y, uint32_t w, uint32_t ws, uint32_t q) {
    return csub(shoup_lazy(y, w, ws, q), q);
}

__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t q) {
    return csub(a + b, q);
}

__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t q) {
    uint32_t d = a - b;
    return min(d, d + q);
}

// Montgomery REDC, subtractive form: (hi:lo) * 2^-32 mod q in [0, q).
// Requires hi < q.
__device__ __forceinline__ uint32_t redc(uint32_t lo, uint32_t hi, uint32_t q, uint32_t qinv) {
    uint32_t m = lo * qinv;
    uint32_t u = __umulhi(m, q);
    uint32_t r = hi - u;
    return min(r, r + q);
}

// x mod q for any 64-bit x.  Fast moduli (2^30 < q < 2^31): x = hi * 2^32 + lo, so
// x = hi * (2^32 mod q) + lo (mod q): one lazy Shoup product (valid for any 32-bit hi) and
// conditional subtractions -- 1 IMAD.HI + 2 IMAD on the multiplier pipe.  (Rounds 1-2 used a
// Montgomery REDC followed by a Shoup multiplication by 2^32 mod q to cancel its factor: 2 IMAD.HI
// + 3 IMAD for the same canonical residue.)
__device__ __forceinline__ uint32_t reduce64(uint64_t x, const ModSlot& m) {
    if (m.fast) {
        uint32_t lo = (uint32_t)x;
        const uint32_t hi = (uint32_t)(x >> 32);
        const uint32_t t = shoup_mul(hi, m.r1, m.r1s, m.q);     // hi * 2^32 mod q, canonical
        lo = min(lo, lo - 2u * m.q);                             // lo < 2^32 < 4q
        lo = csub(lo, m.q);
        return csub(t + lo, m.q);
    }
    return (uint32_t)(x % m.q);
}

// a * b mod q for canonical a, b.
__device__ __forceinline__ uint32_t mul_mod(uint32_t a, uint32_t b, const ModSlot& m) {
    return reduce64((uint64_t)a * b, m);
}

// Source column of output column t under the evaluation-domain automorphism X -> X^k
// (closed form of reference rns.py:268-292, SURVEY 8a'.4).
__device__ __forceinline__ uint32_t galois_src(uint32_t t, uint32_t k, uint32_t n, uint32_t lg) {
    const uint32_t u = __brev(t) >> (32 - lg);
    const uint32_t e = ((2 * u + 1) * k) & (2 * n - 1);
    return __brev((e - 1) >> 1) >> (32 - lg);
}

// ---- programmatic dependent launch --------------------------------------------------
// Kernels on the hot path are launched with programmatic stream serialisation
// (internal.h launch_pdl): a kernel may start while its predecessor in the stream is
// still draining.  pdl_trigger() (first statement) lets the NEXT kernel begin launching;
// everything before pdl_wait() may only touch static tables (twiddles, conversion tables,
// switching keys); pdl_wait() returns once the predecessor grid has completed and its
// writes are visible, and must precede the first access to any operand buffer.  Both are
// no-ops for a kernel launched the ordinary way.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---- memory helpers -------------------------------------------------------------

// Streaming loads for data read exactly once per kernel (switching keys, encoded
// plaintext diagonals): no L1 allocation and an L2 evict-first policy, so that the
// ~8 GB a bootstrap streams do not push the working set the next kernel re-reads
// (raised digits, accumulators, twiddles) out of the 126 MB L2.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ uint2 ld_stream2(const uint2* p, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

}  // namespace ckks

// status codes of the C ABI (include/ckks_b200.h)
#define CKKS_OK 0
#define CKKS_ERR_ARG 1
#define CKKS_ERR_CUDA 2
#define CKKS_ERR_UNSUPPORTED 3
#define CKKS_ERR_STATE 4
