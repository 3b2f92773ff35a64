// keyswitch.cu -- the element-wise kernels of hybrid key switching.
//
// Stage 2 (reference keyswitch.py:318-355): acc_a = sum_t d_t (.) evk_t.a and
// acc_b = sum_t d_t (.) evk_t.b over the extended basis.  The key matrix
// (2*beta*(L+alpha) limbs, 125.8 MB at ks48) is streamed from HBM exactly once;
// products are accumulated in 64 bits (four 62-bit products fit) and reduced
// once, so the kernel is purely DRAM-bound.
//
// Stage 3 epilogue (keyswitch.py:412-418, :452): out = (x_Q - conv) * P^-1,
// with the ciphertext b-part folded into the b half in the same pass.
#include <cstdlib>
#include "common.cuh"
#include "internal.h"

namespace ckks {

__device__ __forceinline__ uint64_t mad64(uint32_t a, uint32_t b, uint64_t c) {
    return (uint64_t)a * b + c;
}

// W consecutive words (W = 1, 2, 4) as one access
template <int W>
__device__ __forceinline__ void ldw(const uint32_t* p, uint32_t (&v)[W]) {
    if (W == 4) { const uint4 t = *reinterpret_cast<const uint4*>(p); v[0] = t.x; v[W > 1 ? 1 : 0] = t.y; v[W > 2 ? 2 : 0] = t.z; v[W > 3 ? 3 : 0] = t.w; }
    else if (W == 2) { const uint2 t = *reinterpret_cast<const uint2*>(p); v[0] = t.x; v[W > 1 ? 1 : 0] = t.y; }
    else v[0] = p[0];
}
template <int W>
__device__ __forceinline__ void ldw_stream(const uint32_t* p, uint64_t pol, uint32_t (&v)[W]) {
    if (W == 4) { const uint4 t = ld_stream(reinterpret_cast<const uint4*>(p), pol); v[0] = t.x; v[W > 1 ? 1 : 0] = t.y; v[W > 2 ? 2 : 0] = t.z; v[W > 3 ? 3 : 0] = t.w; }
    else if (W == 2) { const uint2 t = ld_stream2(reinterpret_cast<const uint2*>(p), pol); v[0] = t.x; v[W > 1 ? 1 : 0] = t.y; }
    else v[0] = p[0];
}
template <int W>
__device__ __forceinline__ void stw(uint32_t* p, const uint32_t (&v)[W]) {
    if (W == 4) *reinterpret_cast<uint4*>(p) = make_uint4(v[0], v[W > 1 ? 1 : 0], v[W > 2 ? 2 : 0], v[W > 3 ? 3 : 0]);
    else if (W == 2) *reinterpret_cast<uint2*>(p) = make_uint2(v[0], v[W > 1 ? 1 : 0]);
    else p[0] = v[0];
}

// BETA > 0: digit count known at compile time -- the loop is unrolled and all 3 * BETA
// 16-byte loads of a thread are issued before the first product, which is what keeps
// enough bytes in flight per SM to stream the key at HBM speed.  BETA = 0: runtime count.
template <int W, int BETA, bool TENS>
__global__ void __launch_bounds__(256)
inner_product_kernel(InnerProductArgs p, const ModSlot* __restrict__ slots) {
    const int row = p.row_lo + blockIdx.y;
    const ModSlot m = slots[p.ext_slot[row]];
    const size_t n = p.n;
    const int digit_of_row = row < p.l ? row / p.alpha : -1;
    const size_t erow = (size_t)p.evk_row[row];
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    if (i >= n) return;
    const int beta = BETA > 0 ? BETA : p.beta;
    const uint64_t pol = l2_evict_first_policy();
    pdl_trigger();
    // the key is static: with BETA known its loads are issued before waiting for the kernel
    // that produces the digits (complementary pipelining at kernel granularity)
    if (BETA == 0) pdl_wait();
    uint32_t ra[W], rb[W];
#pragma unroll
    for (int w = 0; w < W; ++w) ra[w] = rb[w] = 0;
    uint32_t gsrc[W];
    if (p.galois) {
#pragma unroll
        for (int w = 0; w < W; ++w) gsrc[w] = galois_src((uint32_t)i + w, p.galois, p.n, p.lg);
    }
    const bool tens = TENS && row < p.l;
    uint32_t own[W], la[W], lb[W];
#pragma unroll
    for (int w = 0; w < W; ++w) own[w] = la[w] = lb[w] = 0;
    constexpr int CH = BETA > 0 ? BETA : 4;      // digits per 64-bit accumulation chunk (four 62-bit products fit)
    for (int t0 = 0; t0 < beta; t0 += CH) {
        uint32_t d[CH][W], xa[CH][W], xb[CH][W];
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int t = t0 + c;
            if (BETA == 0 && t >= beta) {
#pragma unroll
                for (int w = 0; w < W; ++w) d[c][w] = xa[c][w] = xb[c][w] = 0;
                continue;
            }
            const uint32_t* dsrc = (p.carry && t == digit_of_row)
                                       ? p.carry + (size_t)row * n
                                       : p.raised + ((size_t)t * p.ext + row) * n;
            const uint32_t* ka = p.evk + (((size_t)t * 2 + 0) * p.evk_ext + erow) * n;
            const uint32_t* kb = p.evk + (((size_t)t * 2 + 1) * p.evk_ext + erow) * n;
            ldw_stream<W>(ka + i, pol, xa[c]);
            ldw_stream<W>(kb + i, pol, xb[c]);
        }
        if (BETA > 0) pdl_wait();
        if (tens && t0 == 0) {
            const size_t at = (size_t)row * n + i;
            uint32_t XA[W], XB[W], YA[W], YB[W];
            ldw<W>(p.tx_a + at, XA); ldw<W>(p.tx_b + at, XB);
            ldw<W>(p.ty_a + at, YA); ldw<W>(p.ty_b + at, YB);
#pragma unroll
            for (int w = 0; w < W; ++w) {
                own[w] = mul_mod(XA[w], YA[w], m);
                lb[w] = mul_mod(XB[w], YB[w], m);
                la[w] = m.fast ? reduce64((uint64_t)XA[w] * YB[w] + (uint64_t)YA[w] * XB[w], m)
                               : (uint32_t)(((uint64_t)XA[w] * YB[w] % m.q + (uint64_t)YA[w] * XB[w] % m.q) % m.q);
            }
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const int t = t0 + c;
            if (BETA == 0 && t >= beta) continue;
            if (tens && t == digit_of_row) {
#pragma unroll
                for (int w = 0; w < W; ++w) d[c][w] = own[w];
                continue;
            }
            const uint32_t* dsrc = (p.carry && t == digit_of_row)
                                       ? p.carry + (size_t)row * n
                                       : p.raised + ((size_t)t * p.ext + row) * n;
            if (p.galois) {
                // hoisted rotation: the raised digit is read through the automorphism
                // (sigma_k commutes with ModUp up to a multiple of the digit modulus)
#pragma unroll
                for (int w = 0; w < W; ++w) d[c][w] = dsrc[gsrc[w]];
            } else {
                ldw<W>(dsrc + i, d[c]);
            }
        }
        if (m.fast) {
            uint64_t sa[W], sb[W];
#pragma unroll
            for (int w = 0; w < W; ++w) { sa[w] = sb[w] = 0; }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    sa[w] = mad64(d[c][w], xa[c][w], sa[w]);
                    sb[w] = mad64(d[c][w], xb[c][w], sb[w]);
                }
            }
#pragma unroll
            for (int w = 0; w < W; ++w) {
                ra[w] = add_mod(ra[w], reduce64(sa[w], m), m.q);
                rb[w] = add_mod(rb[w], reduce64(sb[w], m), m.q);
            }
        } else {
            // any modulus below 2^32: reduce every product
#pragma unroll
            for (int c = 0; c < CH; ++c) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    ra[w] = (uint32_t)(((uint64_t)ra[w] + (uint64_t)d[c][w] * xa[c][w] % m.q) % m.q);
                    rb[w] = (uint32_t)(((uint64_t)rb[w] + (uint64_t)d[c][w] * xb[c][w] % m.q) % m.q);
                }
            }
        }
    }
    uint32_t* oa = p.acc_a + (size_t)(row - p.row_lo) * n + i;
    uint32_t* ob = p.acc_b + (size_t)(row - p.row_lo) * n + i;
    if (tens) {
        const uint32_t pm = p.pmod[row], pms = p.pmod_s[row];
#pragma unroll
        for (int w = 0; w < W; ++w) {
            ra[w] = add_mod(ra[w], shoup_mul(la[w], pm, pms, m.q), m.q);
            rb[w] = add_mod(rb[w], shoup_mul(lb[w], pm, pms, m.q), m.q);
        }
    }
    if (!TENS && p.lift_b && row < p.l) {
        const uint32_t pm = p.pmod[row], pms = p.pmod_s[row];
        const uint32_t* bsrc = p.lift_b + (size_t)row * n;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t bv = p.galois ? bsrc[gsrc[w]] : bsrc[i + w];
            rb[w] = add_mod(rb[w], shoup_mul(bv, pm, pms, m.q), m.q);
        }
    }
    if (!TENS && p.lift_qp) {
        const uint32_t* bsrc = p.lift_qp + (size_t)row * n;
#pragma unroll
        for (int w = 0; w < W; ++w) rb[w] = add_mod(rb[w], p.galois ? bsrc[gsrc[w]] : bsrc[i + w], m.q);
    }
    if (!TENS && p.lift_a && row < p.l) {
        const uint32_t pm = p.pmod[row], pms = p.pmod_s[row];
        const uint32_t* asrc = p.lift_a + (size_t)row * n;
#pragma unroll
        for (int w = 0; w < W; ++w) ra[w] = add_mod(ra[w], shoup_mul(asrc[i + w], pm, pms, m.q), m.q);
    }
    if (p.accumulate) {
#pragma unroll
        for (int w = 0; w < W; ++w) {
            ra[w] = add_mod(ra[w], oa[w], m.q);
            rb[w] = add_mod(rb[w], ob[w], m.q);
        }
    }
    stw<W>(oa, ra);
    stw<W>(ob, rb);
}

template <int BETA>
static cudaError_t inner_product_dispatch(const InnerProductArgs& a, const ModSlot* slots, int width, cudaStream_t st) {
    const bool tens = a.tx_a != nullptr;
    const bool pdl = !a.ordered;
    const size_t work = a.n / width;
    dim3 grid((unsigned)((work + 255) / 256), a.row_hi - a.row_lo);
    if (width == 4 && tens) return launch_opt_pdl(pdl, inner_product_kernel<4, BETA, true>, grid, dim3(256), 0, st, a, slots);
    if (width == 4) return launch_opt_pdl(pdl, inner_product_kernel<4, BETA, false>, grid, dim3(256), 0, st, a, slots);
    if (width == 2 && tens) return launch_opt_pdl(pdl, inner_product_kernel<2, BETA, true>, grid, dim3(256), 0, st, a, slots);
    if (width == 2) return launch_opt_pdl(pdl, inner_product_kernel<2, BETA, false>, grid, dim3(256), 0, st, a, slots);
    if (tens) return launch_opt_pdl(pdl, inner_product_kernel<1, BETA, true>, grid, dim3(256), 0, st, a, slots);
    return launch_opt_pdl(pdl, inner_product_kernel<1, BETA, false>, grid, dim3(256), 0, st, a, slots);
}

int inner_product_launch(const InnerProductArgs& a, const ModSlot* slots, cudaStream_t st) {
    const int rows = a.row_hi - a.row_lo;
    if (rows <= 0) return CKKS_OK;
    // words per thread: 4 (16-byte accesses) by default; CKKS_IP_W=2 halves the per-thread footprint
    // (registers, bytes in flight) for twice the threads
    static const int pref = [] { const char* e = getenv("CKKS_IP_W"); return e ? atoi(e) : 4; }();
    int width = a.n % 4 == 0 ? 4 : 1;
    if (pref == 2 && a.n % 2 == 0) width = 2;
    ProfScope ps("inner_product", st, 4.0 * a.n * rows * (3.0 * a.beta + 2.0));
    switch (a.beta) {
        case 1: CK(inner_product_dispatch<1>(a, slots, width, st)); break;
        case 2: CK(inner_product_dispatch<2>(a, slots, width, st)); break;
        case 3: CK(inner_product_dispatch<3>(a, slots, width, st)); break;
        case 4: CK(inner_product_dispatch<4>(a, slots, width, st)); break;
        default: CK(inner_product_dispatch<0>(a, slots, width, st)); break;
    }
    CK(cudaGetLastError());
    return CKKS_OK;
}

// Fused baby steps + inner sums of a double-hoisted BSGS linear transform (see BsgsInnerArgs).
// One thread owns two columns of one extended-basis row; per baby step it forms the rotated
// key-switch accumulator exactly as inner_product_kernel does (same exact modular arithmetic,
// so results equal the unfused ckks_ks_hoisted_raw + ckks_fused_terms_multi bit for bit) and
// multiplies it into the NG running sums.  Traffic: every key and every plaintext diagonal
// once, raised digits through L2; the 2 * nb accumulator limbs per row are never written.
// two stages (one baby step in flight ahead of the one being multiplied): measured against three with the
// bulk-copy pipeline, 370 vs 400 us per launch and 8.57 vs 8.84 ms per bootstrap -- the smaller buffer leaves
// more of the SM's unified L1 / shared memory to the gathered raised digits and one more CTA per SM
constexpr int kBsgsStages = 2;
constexpr int kBsgsThreads = 128;

// 8-byte asynchronous copy global -> shared.  No L2 cache hint: with the hint ptxas 12.9 put the
// policy descriptor of the copies inside the loop into an odd uniform register pair
// (LDGSTS ... desc[UR1]), which traps as an illegal instruction on sm_100a.
__device__ __forceinline__ void cp_async8(uint2* dst_smem, const uint32_t* src, uint64_t) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src) : "memory");
}

template <int NG, int BETA>
__global__ void __launch_bounds__(kBsgsThreads)
bsgs_inner_kernel(BsgsInnerArgs p, const ModSlot* __restrict__ slots) {
    const int row = blockIdx.y;
    const ModSlot m = slots[p.ext_slot[row]];
    const size_t n = p.n;
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    if (i >= n) return;
    const size_t erow = (size_t)p.evk_row[row];
    const bool qrow = row < p.l;
    const uint32_t pm = qrow ? p.pmod[row] : 0u, pms = qrow ? p.pmod_s[row] : 0u;
    const uint64_t pol = l2_evict_first_policy();
    const size_t half = (size_t)p.ext * n;
    const size_t at = (size_t)row * n + i;
    pdl_trigger();
    pdl_wait();
    uint64_t sa[NG][2], sb[NG][2];
#pragma unroll
    for (int g = 0; g < NG; ++g) sa[g][0] = sa[g][1] = sb[g][0] = sb[g][1] = 0;
    // Software pipeline through shared memory: the 2 BETA key words and NG plaintext words a
    // thread needs for baby step b + kBsgsStages - 1 are requested with cp.async (8 bytes each,
    // L2 evict-first) while baby step b is reduced and multiplied.  A thread reads back only what
    // it requested itself, so cp.async.wait_group is the only synchronisation; consecutive threads
    // use consecutive 8-byte slots (no bank conflicts).
    extern __shared__ uint2 s_pipe[];
    constexpr int ITEMS = 2 * BETA + NG;
    auto slot = [&](int stage, int item) -> uint2* { return s_pipe + ((size_t)(stage * ITEMS + item) * kBsgsThreads + threadIdx.x); };
    auto request = [&](int b) {
        if (b < p.nb) {
            const int stage = b % kBsgsStages;
            const uint32_t* key = p.evk[b];
            if (p.k[b] != 0) {
#pragma unroll
                for (int t = 0; t < BETA; ++t) {
                    cp_async8(slot(stage, 2 * t), key + (((size_t)t * 2 + 0) * p.evk_ext + erow) * n + i, pol);
                    cp_async8(slot(stage, 2 * t + 1), key + (((size_t)t * 2 + 1) * p.evk_ext + erow) * n + i, pol);
                }
            }
#pragma unroll
            for (int g = 0; g < NG; ++g) cp_async8(slot(stage, 2 * BETA + g), p.p[g][b] + at, pol);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int b = 0; b < kBsgsStages - 1; ++b) request(b);
    for (int b = 0; b < p.nb; ++b) {
        request(b + kBsgsStages - 1);
        asm volatile("cp.async.wait_group %0;" :: "n"(kBsgsStages - 1) : "memory");
        const int stage = b % kBsgsStages;
        uint32_t ra[2], rb[2];
        const uint32_t k = p.k[b];
        if (k == 0) {
            // the unrotated term: the ciphertext on the Q rows (its plaintext carries the factor P)
            if (qrow) {
                const uint2 av = *reinterpret_cast<const uint2*>(p.ct_a[0] + at);
                const uint2 bv = *reinterpret_cast<const uint2*>(p.ct_b[0] + at);
                ra[0] = av.x; ra[1] = av.y; rb[0] = bv.x; rb[1] = bv.y;
            } else {
                ra[0] = ra[1] = rb[0] = rb[1] = 0;
            }
        } else {
            const uint32_t g0 = galois_src((uint32_t)i, k, p.n, p.lg), g1 = galois_src((uint32_t)i + 1, k, p.n, p.lg);
            uint64_t ta[2] = {0, 0}, tb[2] = {0, 0};
#pragma unroll
            for (int t = 0; t < BETA; ++t) {
                const uint32_t* dsrc = p.raised[0] + ((size_t)t * p.ext + row) * n;
                const uint32_t d0 = dsrc[g0], d1 = dsrc[g1];
                const uint2 xa = *slot(stage, 2 * t), xb = *slot(stage, 2 * t + 1);
                ta[0] = mad64(d0, xa.x, ta[0]); ta[1] = mad64(d1, xa.y, ta[1]);
                tb[0] = mad64(d0, xb.x, tb[0]); tb[1] = mad64(d1, xb.y, tb[1]);
            }
            ra[0] = reduce64(ta[0], m); ra[1] = reduce64(ta[1], m);
            rb[0] = reduce64(tb[0], m); rb[1] = reduce64(tb[1], m);
            if (qrow) {
                const uint32_t* bsrc = p.ct_b[0] + (size_t)row * n;
                rb[0] = add_mod(rb[0], shoup_mul(bsrc[g0], pm, pms, m.q), m.q);
                rb[1] = add_mod(rb[1], shoup_mul(bsrc[g1], pm, pms, m.q), m.q);
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const uint2 pv = *slot(stage, 2 * BETA + g);
            sa[g][0] += (uint64_t)ra[0] * pv.x; sa[g][1] += (uint64_t)ra[1] * pv.y;
            sb[g][0] += (uint64_t)rb[0] * pv.x; sb[g][1] += (uint64_t)rb[1] * pv.y;
        }
        if ((b & 3) == 3) {
            // four 62-bit products + a carried residue fit 64 bits: fold and carry
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                sa[g][0] = reduce64(sa[g][0], m); sa[g][1] = reduce64(sa[g][1], m);
                sb[g][0] = reduce64(sb[g][0], m); sb[g][1] = reduce64(sb[g][1], m);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        uint32_t* o = p.out[0][g];
        *reinterpret_cast<uint2*>(o + at) = make_uint2(reduce64(sa[g][0], m), reduce64(sa[g][1], m));
        *reinterpret_cast<uint2*>(o + half + at) = make_uint2(reduce64(sb[g][0], m), reduce64(sb[g][1], m));
    }
}

// Bulk-copy (TMA) variant of the pipeline above: per baby step ONE elected thread requests the CTA's
// 1 KiB slice of every key / plaintext row with cp.async.bulk (global -> shared, completion counted in
// bytes on an mbarrier, L2 evict-first hint) instead of 128 threads issuing 2 BETA + NG 8-byte cp.async
// each; consumers wait on the stage's mbarrier parity.  Same shared layout, same arithmetic, same result.
// Needs n % 256 == 0 (a CTA's slice is 256 consecutive columns).
__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint32_t bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(dst_smem), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
}

template <int NG, int BETA, int BATCH>
__global__ void __launch_bounds__(kBsgsThreads * BATCH)
bsgs_inner_tma_kernel(BsgsInnerArgs p, const ModSlot* __restrict__ slots) {
    const int row = blockIdx.y;
    const ModSlot m = slots[p.ext_slot[row]];
    const size_t n = p.n;
    const size_t i0 = (size_t)blockIdx.x * kBsgsThreads * 2;           // first column of this CTA
    const int tx = threadIdx.x % kBsgsThreads;                         // column pair within the CTA's slice
    const int cb = BATCH == 1 ? 0 : threadIdx.x / kBsgsThreads;        // which ciphertext of the batch
    const size_t i = i0 + (size_t)tx * 2;
    const uint32_t* __restrict__ raised = p.raised[cb];
    const uint32_t* __restrict__ ct_a = p.ct_a[cb];
    const uint32_t* __restrict__ ct_b = p.ct_b[cb];
    const size_t erow = (size_t)p.evk_row[row];
    const bool qrow = row < p.l;
    const uint32_t pm = qrow ? p.pmod[row] : 0u, pms = qrow ? p.pmod_s[row] : 0u;
    const uint64_t pol = l2_evict_first_policy();
    const size_t half = (size_t)p.ext * n;
    const size_t at = (size_t)row * n + i;
    constexpr int ITEMS = 2 * BETA + NG;
    constexpr uint32_t kSlice = kBsgsThreads * sizeof(uint2);          // 1 KiB per item
    extern __shared__ __align__(128) uint2 s_pipe[];
    __shared__ __align__(8) uint64_t s_full[kBsgsStages];
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&s_full[0]);
    const uint32_t pipe0 = (uint32_t)__cvta_generic_to_shared(&s_pipe[0]);
    pdl_trigger();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < kBsgsStages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar0 + 8 * s));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_wait();
    uint64_t sa[NG][2], sb[NG][2];
#pragma unroll
    for (int g = 0; g < NG; ++g) sa[g][0] = sa[g][1] = sb[g][0] = sb[g][1] = 0;
    auto slot = [&](int stage, int item) -> const uint2* { return s_pipe + ((size_t)(stage * ITEMS + item) * kBsgsThreads + tx); };
    auto request = [&](int b) {
        if (threadIdx.x != 0 || b >= p.nb) return;
        const int stage = b % kBsgsStages;
        const uint32_t bar = bar0 + 8 * stage;
        const bool keyed = p.k[b] != 0;
        const uint32_t bytes = (uint32_t)((keyed ? 2 * BETA : 0) + NG) * kSlice;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
        const uint32_t base = pipe0 + (uint32_t)(stage * ITEMS) * kSlice;
        if (keyed) {
            const uint32_t* key = p.evk[b];
#pragma unroll
            for (int t = 0; t < BETA; ++t) {
                bulk_g2s(base + (2 * t) * kSlice, key + (((size_t)t * 2 + 0) * p.evk_ext + erow) * n + i0, kSlice, bar, pol);
                bulk_g2s(base + (2 * t + 1) * kSlice, key + (((size_t)t * 2 + 1) * p.evk_ext + erow) * n + i0, kSlice, bar, pol);
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) bulk_g2s(base + (2 * BETA + g) * kSlice, p.p[g][b] + (size_t)row * n + i0, kSlice, bar, pol);
    };
#pragma unroll
    for (int b = 0; b < kBsgsStages - 1; ++b) request(b);
    for (int b = 0; b < p.nb; ++b) {
        if (b > 0) __syncthreads();                      // everyone is done with the stage that is refilled next
        request(b + kBsgsStages - 1);
        const int stage = b % kBsgsStages;
        {
            const uint32_t bar = bar0 + 8 * stage, parity = (uint32_t)(b / kBsgsStages) & 1u;
            asm volatile("{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra D%=;\n bra W%=;\n D%=:\n}"
                         :: "r"(bar), "r"(parity) : "memory");
        }
        uint32_t ra[2], rb[2];
        const uint32_t k = p.k[b];
        if (k == 0) {
            if (qrow) {
                const uint2 av = *reinterpret_cast<const uint2*>(ct_a + at);
                const uint2 bv = *reinterpret_cast<const uint2*>(ct_b + at);
                ra[0] = av.x; ra[1] = av.y; rb[0] = bv.x; rb[1] = bv.y;
            } else {
                ra[0] = ra[1] = rb[0] = rb[1] = 0;
            }
        } else {
            const uint32_t g0 = galois_src((uint32_t)i, k, p.n, p.lg), g1 = galois_src((uint32_t)i + 1, k, p.n, p.lg);
            uint64_t ta[2] = {0, 0}, tb[2] = {0, 0};
#pragma unroll
            for (int t = 0; t < BETA; ++t) {
                const uint32_t* dsrc = raised + ((size_t)t * p.ext + row) * n;
                const uint32_t d0 = dsrc[g0], d1 = dsrc[g1];
                const uint2 xa = *slot(stage, 2 * t), xb = *slot(stage, 2 * t + 1);
                ta[0] = mad64(d0, xa.x, ta[0]); ta[1] = mad64(d1, xa.y, ta[1]);
                tb[0] = mad64(d0, xb.x, tb[0]); tb[1] = mad64(d1, xb.y, tb[1]);
            }
            ra[0] = reduce64(ta[0], m); ra[1] = reduce64(ta[1], m);
            rb[0] = reduce64(tb[0], m); rb[1] = reduce64(tb[1], m);
            if (qrow) {
                const uint32_t* bsrc = ct_b + (size_t)row * n;
                rb[0] = add_mod(rb[0], shoup_mul(bsrc[g0], pm, pms, m.q), m.q);
                rb[1] = add_mod(rb[1], shoup_mul(bsrc[g1], pm, pms, m.q), m.q);
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const uint2 pv = *slot(stage, 2 * BETA + g);
            sa[g][0] += (uint64_t)ra[0] * pv.x; sa[g][1] += (uint64_t)ra[1] * pv.y;
            sb[g][0] += (uint64_t)rb[0] * pv.x; sb[g][1] += (uint64_t)rb[1] * pv.y;
        }
        if ((b & 3) == 3) {
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                sa[g][0] = reduce64(sa[g][0], m); sa[g][1] = reduce64(sa[g][1], m);
                sb[g][0] = reduce64(sb[g][0], m); sb[g][1] = reduce64(sb[g][1], m);
            }
        }
    }
#pragma unroll
    for (int g = 0; g < NG; ++g) {
        uint32_t* o = p.out[cb][g];
        *reinterpret_cast<uint2*>(o + at) = make_uint2(reduce64(sa[g][0], m), reduce64(sa[g][1], m));
        *reinterpret_cast<uint2*>(o + half + at) = make_uint2(reduce64(sb[g][0], m), reduce64(sb[g][1], m));
    }
}

template <int NG, int BETA>
static int bsgs_launch_one(const BsgsInnerArgs& a, const ModSlot* slots, dim3 grid, cudaStream_t st) {
    const size_t sm = sizeof(uint2) * kBsgsThreads * (size_t)kBsgsStages * (2 * BETA + NG);
    // default: the bulk-copy (TMA) pipeline; CKKS_BSGS_TMA=0: per-thread cp.async (also the path for ring
    // degrees that are not a multiple of a CTA's 256 columns).  Measured at ks48: 400 vs 430 us per launch
    // run eagerly, equal inside the bootstrap graph.
    static const bool tma = [] { const char* e = getenv("CKKS_BSGS_TMA"); return !(e && e[0] == '0'); }();
    if (a.batch == 2) {
        // two ciphertexts per CTA share the staged key / plaintext slices (bulk-copy pipeline only)
        if (a.n % (2 * kBsgsThreads) != 0) { set_last_error("batched bsgs_inner needs n %% 256 == 0"); return CKKS_ERR_UNSUPPORTED; }
        if (sm > 48 * 1024)
            CK(cudaFuncSetAttribute(bsgs_inner_tma_kernel<NG, BETA, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(launch_pdl(bsgs_inner_tma_kernel<NG, BETA, 2>, grid, dim3(2 * kBsgsThreads), sm, st, a, slots));
        return CKKS_OK;
    }
    if (tma && a.n % (2 * kBsgsThreads) == 0) {
        if (sm > 48 * 1024)
            CK(cudaFuncSetAttribute(bsgs_inner_tma_kernel<NG, BETA, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        CK(launch_pdl(bsgs_inner_tma_kernel<NG, BETA, 1>, grid, dim3(kBsgsThreads), sm, st, a, slots));
        return CKKS_OK;
    }
    if (sm > 48 * 1024)
        CK(cudaFuncSetAttribute(bsgs_inner_kernel<NG, BETA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(launch_pdl(bsgs_inner_kernel<NG, BETA>, grid, dim3(kBsgsThreads), sm, st, a, slots));
    return CKKS_OK;
}

template <int NG>
static int bsgs_dispatch(const BsgsInnerArgs& a, const ModSlot* slots, dim3 grid, cudaStream_t st) {
    switch (a.beta) {
        case 1: return bsgs_launch_one<NG, 1>(a, slots, grid, st);
        case 2: return bsgs_launch_one<NG, 2>(a, slots, grid, st);
        case 3: return bsgs_launch_one<NG, 3>(a, slots, grid, st);
        case 4: return bsgs_launch_one<NG, 4>(a, slots, grid, st);
    }
    set_last_error("bsgs_inner supports 1..4 digits, got %d", a.beta);
    return CKKS_ERR_UNSUPPORTED;
}

int bsgs_inner_launch(const BsgsInnerArgs& a, const ModSlot* slots, cudaStream_t st) {
    if (a.n % 2 || a.nb < 1 || a.nb > kMaxTerms || a.ng < 1 || a.ng > kMaxGiants || a.batch < 1 || a.batch > kMaxBsgsBatch) {
        set_last_error("bsgs_inner needs even n, 1..%d baby steps, 1..%d giant steps, 1..%d ciphertexts", kMaxTerms, kMaxGiants, kMaxBsgsBatch);
        return CKKS_ERR_UNSUPPORTED;
    }
    int keyed = 0;
    for (int b = 0; b < a.nb; ++b) keyed += a.k[b] ? 1 : 0;
    // keys + plaintexts + outputs (+ the ciphertext once); raised digits are re-read through L2
    // (a batch shares the keys and plaintexts: only the outputs and the ciphertexts scale with it)
    const double limbs = (double)a.ext * (2.0 * a.beta * keyed + (double)a.nb * a.ng + 2.0 * a.ng * a.batch) + 2.0 * a.l * a.batch;
    ProfScope ps(a.batch > 1 ? "bsgs_inner_batch" : "bsgs_inner", st, 4.0 * a.n * limbs);
    dim3 grid((unsigned)((a.n / 2 + kBsgsThreads - 1) / kBsgsThreads), a.ext);
    int rc = CKKS_ERR_UNSUPPORTED;
    switch (a.ng) {
        case 1: rc = bsgs_dispatch<1>(a, slots, grid, st); break;
        case 2: rc = bsgs_dispatch<2>(a, slots, grid, st); break;
        case 3: rc = bsgs_dispatch<3>(a, slots, grid, st); break;
        case 4: rc = bsgs_dispatch<4>(a, slots, grid, st); break;
        case 5: rc = bsgs_dispatch<5>(a, slots, grid, st); break;
        case 6: rc = bsgs_dispatch<6>(a, slots, grid, st); break;
        case 7: rc = bsgs_dispatch<7>(a, slots, grid, st); break;
        case 8: rc = bsgs_dispatch<8>(a, slots, grid, st); break;
    }
    if (rc != CKKS_OK) return rc;
    CK(cudaGetLastError());
    return CKKS_OK;
}

template <bool VEC>
__global__ void __launch_bounds__(256)
moddown_epilogue_kernel(ModDownEpilogueArgs p, const ModSlot* __restrict__ slots) {
    const int row = blockIdx.y % p.l;
    const int half = blockIdx.y / p.l;                 // 0: a, 1: b
    const uint32_t q = slots[p.q_slot[row]].q;
    const uint32_t pinv = p.pinv[row], pinv_s = p.pinv_s[row];
    const size_t n = p.n;
    constexpr int W = VEC ? 4 : 1;
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    if (i >= n) return;
    const uint32_t* x = (half ? p.xq_b : p.xq_a) + (size_t)row * n + i;
    const uint32_t* c = p.conv + ((size_t)half * p.l + row) * n + i;
    const uint32_t* fsrc = half ? p.fold_b : p.fold_a;
    const uint32_t* f = fsrc ? fsrc + (size_t)row * n + (p.galois ? 0 : i) : nullptr;
    uint32_t* o = (half ? p.out_b : p.out_a) + (size_t)row * n + i;
    if (VEC) {
        const uint4 xv = *reinterpret_cast<const uint4*>(x);
        const uint4 cv = *reinterpret_cast<const uint4*>(c);
        uint4 r;
        r.x = shoup_mul(xv.x - cv.x + q, pinv, pinv_s, q);
        r.y = shoup_mul(xv.y - cv.y + q, pinv, pinv_s, q);
        r.z = shoup_mul(xv.z - cv.z + q, pinv, pinv_s, q);
        r.w = shoup_mul(xv.w - cv.w + q, pinv, pinv_s, q);
        if (f && p.galois) {
            r.x = add_mod(r.x, f[galois_src((uint32_t)i, p.galois, p.n, p.lg)], q);
            r.y = add_mod(r.y, f[galois_src((uint32_t)i + 1, p.galois, p.n, p.lg)], q);
            r.z = add_mod(r.z, f[galois_src((uint32_t)i + 2, p.galois, p.n, p.lg)], q);
            r.w = add_mod(r.w, f[galois_src((uint32_t)i + 3, p.galois, p.n, p.lg)], q);
        } else if (f) {
            const uint4 fv = *reinterpret_cast<const uint4*>(f);
            r.x = add_mod(r.x, fv.x, q); r.y = add_mod(r.y, fv.y, q);
            r.z = add_mod(r.z, fv.z, q); r.w = add_mod(r.w, fv.w, q);
        }
        *reinterpret_cast<uint4*>(o) = r;
    } else {
        uint32_t r = shoup_mul(x[0] - c[0] + q, pinv, pinv_s, q);
        if (f) r = add_mod(r, p.galois ? f[galois_src((uint32_t)i, p.galois, p.n, p.lg)] : f[0], q);
        o[0] = r;
    }
}

int moddown_epilogue_launch(const ModDownEpilogueArgs& a, const ModSlot* slots, cudaStream_t st) {
    if (a.l <= 0) return CKKS_OK;
    const bool vec = a.n % 4 == 0;
    const size_t work = vec ? a.n / 4 : a.n;
    dim3 grid((unsigned)((work + 255) / 256), 2 * a.l);
    ProfScope ps("moddown_epilogue", st, 4.0 * a.n * a.l * (a.fold_b ? 7.0 : 6.0));
    if (vec) moddown_epilogue_kernel<true><<<grid, 256, 0, st>>>(a, slots);
    else moddown_epilogue_kernel<false><<<grid, 256, 0, st>>>(a, slots);
    CK(cudaGetLastError());
    return CKKS_OK;
}

// acc0 += acc1 + ... over the [2][ext][n] accumulators of several workspace lanes
// (giant steps of a linear transform accumulate their inner products per lane); with
// lift_a / lift_b also += (P mod q_i) * lift on the Q rows of the two halves, i.e. a ciphertext
// that takes no key switch joins the accumulator before the shared ModDown; `raw` adds one more
// [2][ext][n] accumulator that already lives over Q||P (an inner sum that is not rotated).
__global__ void __launch_bounds__(256)
lane_reduce_kernel(uint4* acc0, size_t lane_stride4, int lanes, const int32_t* __restrict__ ext_slot,
                   const ModSlot* __restrict__ slots, int ext, size_t cols4, const uint4* lift_a,
                   const uint4* lift_b, const uint32_t* __restrict__ pmod,
                   const uint32_t* __restrict__ pmod_s, int l, const uint4* raw) {
    const int row = blockIdx.y % ext;
    const int half = blockIdx.y / ext;
    const uint32_t q = slots[ext_slot[row]].q;
    const uint4* lift = half ? lift_b : lift_a;
    const bool lifted = lift != nullptr && row < l;
    const uint32_t pm = lifted ? pmod[row] : 0u, pms = lifted ? pmod_s[row] : 0u;
    pdl_trigger();
    pdl_wait();
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols4; i += stride) {
        const size_t at = (size_t)blockIdx.y * cols4 + i;
        uint4 r = acc0[at];
        for (int ln = 1; ln < lanes; ++ln) {
            const uint4 v = acc0[at + (size_t)ln * lane_stride4];
            r.x = add_mod(r.x, v.x, q); r.y = add_mod(r.y, v.y, q);
            r.z = add_mod(r.z, v.z, q); r.w = add_mod(r.w, v.w, q);
        }
        if (raw) {                 // a [2][ext][n] accumulator that is already over Q||P
            const uint4 v = raw[at];
            r.x = add_mod(r.x, v.x, q); r.y = add_mod(r.y, v.y, q);
            r.z = add_mod(r.z, v.z, q); r.w = add_mod(r.w, v.w, q);
        }
        if (lifted) {
            const uint4 v = lift[(size_t)row * cols4 + i];
            r.x = add_mod(r.x, shoup_mul(v.x, pm, pms, q), q); r.y = add_mod(r.y, shoup_mul(v.y, pm, pms, q), q);
            r.z = add_mod(r.z, shoup_mul(v.z, pm, pms, q), q); r.w = add_mod(r.w, shoup_mul(v.w, pm, pms, q), q);
        }
        acc0[at] = r;
    }
}

int lane_reduce_launch(uint32_t* acc0, size_t lane_stride_words, int lanes, const int32_t* ext_slot,
                       const ModSlot* slots, int ext, size_t n, cudaStream_t st, const uint32_t* lift_a,
                       const uint32_t* lift_b, const uint32_t* pmod, const uint32_t* pmod_s, int l,
                       const uint32_t* raw) {
    if (lanes < 2 && !lift_a && !lift_b && !raw) return CKKS_OK;
    if (n % 4 || lane_stride_words % 4) { set_last_error("lane reduction needs n %% 4 == 0"); return CKKS_ERR_UNSUPPORTED; }
    ProfScope ps("lane_reduce", st, 4.0 * n * (2 * ext * (lanes + 1 + (raw ? 1 : 0)) + (lift_a ? l : 0) + (lift_b ? l : 0)));
    unsigned gx = (unsigned)((n / 4 + 255) / 256);
    CK(launch_pdl(lane_reduce_kernel, dim3(gx, 2 * ext), dim3(256), 0, st, (uint4*)acc0, lane_stride_words / 4, lanes,
                  ext_slot, slots, ext, n / 4, (const uint4*)lift_a, (const uint4*)lift_b, pmod, pmod_s, l, (const uint4*)raw));
    CK(cudaGetLastError());
    return CKKS_OK;
}

}  // namespace ckks
