// bconv.cu -- fast base conversion (ModUp / ModDown core).
//
// Reference: baseconv.py:95-151.  For every column c
//     y[k]   = a[k][c] * inv_qhat[k] mod Q_k
//     out[i] = (sum_k T[i][k] * y[k]) mod P_i           (non-centred, exact)
// The shipped N = 2^16 bases are not overflow-free (row sums up to 2.03 * 2^64,
// SURVEY 8a'.6), so the accumulator is folded every four terms: four products
// of 31-bit factors stay below 2^64, each partial sum goes through one
// Montgomery REDC, and the table is kept in Montgomery form (T * 2^32 mod P_i)
// so that the REDC factor cancels and the result is the exact canonical residue.
//
// Column-parallel: a thread keeps the l_in pre-scaled residues of one or two
// adjacent columns in registers and walks the output limbs; the table row and
// the per-limb constants are broadcast reads from shared memory, loads and
// stores are coalesced.  Several conversions (the beta digits of stage 1, the
// two polynomials of stage 3) run as one launch (blockIdx.y).
//
// bconv_fast: every modulus in (2^30, 2^31) -- all shipped parameter sets.
// bconv_generic: any modulus < 2^32 (unit-test primes), '%' arithmetic.
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace ckks {

// Output limbs are split over blockIdx.z in chunks: one ciphertext has only N = 2^16 columns,
// i.e. 256 CTAs per conversion, too few to fill 148 SMs x 8 resident CTAs unless the output
// walk is shared out (the l_in pre-scale is recomputed per chunk: l_in Shoup products against
// l_in * chunk MACs, so chunks stay >= 8 limbs).
constexpr int kTargetCtas = 148 * 8;
constexpr int kMinChunk = 8;
// Doubles of padding per row of the tensor kernel's shared table.  KP2 + 4 doubles per row removes every
// bank conflict of the A-fragment loads (1.18 M -> 2 k per full-size ModUp in ncu) and is SLOWER (32.0 /
// 21.1 us against 30.0 / 16.6 us for the two conversions of a ks48 key switch, measured twice): kept at 0.
#ifndef CKKS_BCONV_TABLE_PAD
#define CKKS_BCONV_TABLE_PAD 0
#endif
constexpr int kBconvTablePad = CKKS_BCONV_TABLE_PAD;

static int out_chunk(size_t ctas_xy, int l_out_max) {
    int z = (int)((kTargetCtas + ctas_xy - 1) / ctas_xy);
    if (z < 1) z = 1;
    int chunk = (l_out_max + z - 1) / z;
    if (chunk < kMinChunk) chunk = kMinChunk;
    if (chunk > l_out_max) chunk = l_out_max > 0 ? l_out_max : 1;
    return chunk;
}

template <int LIN, int CPT>
__global__ void __launch_bounds__(128)
bconv_fast(BconvJobs jobs, const ModSlot* __restrict__ slots, size_t cols, int chunk) {
    constexpr int G = (LIN + 3) / 4;         // groups of four terms
    constexpr int LINP = 4 * G;
    extern __shared__ uint4 sm4[];
    const BconvJob& job = jobs.job[blockIdx.y];
    const int l_out = job.tab.l_out;
    uint4* s_t = sm4;                        // [l_out][G]  Montgomery-form table rows
    uint4* s_om = sm4 + (size_t)l_out * G;   // [l_out]     {q, qinv, out row, 2q}
    uint4* s_in = s_om + l_out;              // [LIN]       {q, inv_qhat, shoup(inv_qhat), -}
    uint32_t* s_tw = reinterpret_cast<uint32_t*>(s_t);
    // only this CTA's chunk of output rows is staged
    const int i_lo = blockIdx.z * chunk, i_hi = min(l_out, i_lo + chunk);
    for (int idx = i_lo * LINP + threadIdx.x; idx < i_hi * LINP; idx += blockDim.x) {
        const int i = idx / LINP, k = idx - i * LINP;
        s_tw[idx] = k < LIN ? job.tab.t_mont[i * LIN + k] : 0u;
    }
    for (int i = i_lo + threadIdx.x; i < i_hi; i += blockDim.x) {
        const ModSlot& m = slots[job.tab.out_slot[i]];
        s_om[i] = make_uint4(m.q, m.qinv, job.out_row ? (uint32_t)job.out_row[i] : (uint32_t)i, 2u * m.q);
    }
    for (int k = threadIdx.x; k < LIN; k += blockDim.x)
        s_in[k] = make_uint4(slots[job.tab.in_slot[k]].q, job.tab.inv_qhat[k], job.tab.inv_qhat_s[k], 0u);
    __syncthreads();

    const size_t c = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * CPT;
    if (c >= cols) return;
    uint32_t y[CPT][LINP];
#pragma unroll
    for (int k = 0; k < LINP; ++k) {
        if (k < LIN) {
            const uint4 im = s_in[k];
            const uint32_t* src = job.in + (size_t)k * job.in_stride + c;
            if (CPT == 2) {
                const uint2 a = *reinterpret_cast<const uint2*>(src);
                y[0][k] = shoup_mul(a.x, im.y, im.z, im.x);
                y[CPT - 1][k] = shoup_mul(a.y, im.y, im.z, im.x);
            } else {
                y[0][k] = shoup_mul(*src, im.y, im.z, im.x);
            }
        } else {
#pragma unroll
            for (int p = 0; p < CPT; ++p) y[p][k] = 0;
        }
    }
#pragma unroll 2
    for (int i = i_lo; i < i_hi; ++i) {
        const uint4 om = s_om[i];
        uint32_t r[CPT];
#pragma unroll
        for (int p = 0; p < CPT; ++p) r[p] = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const uint4 t = s_t[(size_t)i * G + g];
#pragma unroll
            for (int p = 0; p < CPT; ++p) {
                uint64_t s = (uint64_t)t.x * y[p][4 * g];
                s += (uint64_t)t.y * y[p][4 * g + 1];
                s += (uint64_t)t.z * y[p][4 * g + 2];
                s += (uint64_t)t.w * y[p][4 * g + 3];
                uint32_t hi = (uint32_t)(s >> 32);
                hi = min(hi, hi - om.w);               // hi < 2^32 < 4q
                hi = csub(hi, om.x);
                const uint32_t part = redc((uint32_t)s, hi, om.x, om.y);
                r[p] = g == 0 ? part : add_mod(r[p], part, om.x);
            }
        }
        uint32_t* dst = job.out + (size_t)om.z * job.out_stride + c;
        if (CPT == 2) *reinterpret_cast<uint2*>(dst) = make_uint2(r[0], r[CPT - 1]);
        else *dst = r[0];
    }
}

// FP64-pipe variant.  B200 issues DFMA at the same rate as IMAD.lo (64/clk/SM,
// profiles/microbench) on a pipe that is otherwise idle here, while IMAD.WIDE
// costs ~2.8 slots of the integer FMA pipe.  Split y = y1 * 2^16 + y0: every
// T * y0, T * y1 < 2^47 and the 12-term sums stay below 2^51, exact in a
// double.  Seeding the accumulator with 2^52 leaves the integer sum in the low
// 52 mantissa bits, so no float->int conversion is issued.  With T in
// Montgomery form, V = A1_hi * (2^48 mod p) + A1_lo * 2^16 + A0 < 2^51 goes
// through one REDC and yields the exact canonical residue.
template <int LIN>
__global__ void __launch_bounds__(128)
bconv_f64(BconvJobs jobs, const ModSlot* __restrict__ slots, size_t cols, int chunk) {
    constexpr int LINP = (LIN + 1) / 2 * 2;
    extern __shared__ uint4 sm4[];
    const BconvJob& job = jobs.job[blockIdx.y];
    const int l_out = job.tab.l_out;
    double* s_t = reinterpret_cast<double*>(sm4);                                // [l_out][LINP]
    uint4* s_om = sm4 + ((size_t)l_out * LINP * sizeof(double)) / sizeof(uint4); // {q, qinv, row, 2^48 mod q}
    uint4* s_in = s_om + l_out;
    for (int idx = threadIdx.x; idx < l_out * LINP; idx += blockDim.x) {
        const int i = idx / LINP, k = idx - i * LINP;
        s_t[idx] = k < LIN ? (double)job.tab.t_mont[i * LIN + k] : 0.0;
    }
    for (int i = threadIdx.x; i < l_out; i += blockDim.x) {
        const ModSlot& m = slots[job.tab.out_slot[i]];
        const uint32_t c48 = (uint32_t)(((uint64_t)m.r1 << 16) % m.q);
        s_om[i] = make_uint4(m.q, m.qinv, job.out_row ? (uint32_t)job.out_row[i] : (uint32_t)i, c48);
    }
    for (int k = threadIdx.x; k < LIN; k += blockDim.x)
        s_in[k] = make_uint4(slots[job.tab.in_slot[k]].q, job.tab.inv_qhat[k], job.tab.inv_qhat_s[k], 0u);
    __syncthreads();

    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    double y0[LINP], y1[LINP];
#pragma unroll
    for (int k = 0; k < LINP; ++k) {
        y0[k] = y1[k] = 0.0;
        if (k < LIN) {
            const uint4 im = s_in[k];
            const uint32_t y = shoup_mul(job.in[(size_t)k * job.in_stride + c], im.y, im.z, im.x);
            y0[k] = (double)(y & 0xFFFFu);
            y1[k] = (double)(y >> 16);
        }
    }
    const double seed = 4503599627370496.0;     // 2^52
    const int i_lo = blockIdx.z * chunk, i_hi = min(l_out, i_lo + chunk);
    constexpr int U = 4;                        // outputs in flight: 2*U independent DFMA chains
    for (int i0 = i_lo; i0 < i_hi; i0 += U) {
        double a0[U], a1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a0[u] = a1[u] = seed;
#pragma unroll
        for (int k = 0; k < LINP; k += 2) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = min(i0 + u, i_hi - 1);
                const double2 t = reinterpret_cast<const double2*>(s_t + (size_t)i * LINP)[k / 2];
                a0[u] = fma(t.x, y0[k], a0[u]);
                a1[u] = fma(t.x, y1[k], a1[u]);
                a0[u] = fma(t.y, y0[k + 1], a0[u]);
                a1[u] = fma(t.y, y1[k + 1], a1[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u;
            if (i < i_hi) {
                const uint4 om = s_om[i];
                const uint64_t b0 = (uint64_t)__double_as_longlong(a0[u]) & 0xFFFFFFFFFFFFFull;
                const uint64_t b1 = (uint64_t)__double_as_longlong(a1[u]) & 0xFFFFFFFFFFFFFull;
                const uint64_t v = (uint64_t)(uint32_t)(b1 >> 32) * om.w + ((b1 & 0xFFFFFFFFull) << 16) + b0;
                job.out[(size_t)om.z * job.out_stride + c] = redc((uint32_t)v, (uint32_t)(v >> 32), om.x, om.y);
            }
        }
    }
}

// FP64 tensor-core variant (DMMA, mma.sync m8n8k4).  Measured on B200
// (profiles/microbench/dmma.cu): DMMA sustains 63.7 FMA/clk/SM, the same as DFMA, but one
// warp instruction carries 256 of them, so the contraction needs ~1 instruction per 10
// outputs instead of 12 IMAD.WIDE (2.8 integer-pipe slots each) per output.  Exactness:
// y = y1 * 2^16 + y0 and T * y = T * y0 + (T * 2^16 mod p) * y1 (mod p), the second table
// precomputed (BconvDev::t_f64k): the two halves of y are stacked along K, every term is below
// 2^47 resp. 2^46, at most 16 + 16 of them, so the WHOLE contraction is an integer below 2^52.
// It is formed in two chains (four DMMAs in flight per warp) of SUBNORMAL doubles (sub2d above): the
// chains' bit patterns are the integer partial sums, added on the integer pipe, and the total goes
// through ONE REDC against the Montgomery-form table.  (Until round 2 the operands were ordinary
// doubles, one chain seeded with 2^52 and the chains joined by an FP64 add: per 8 x 16 output tile
// that put 4 DADDs and, per column tile, 12 conversion DADDs on the FP64 pipe between the DMMAs;
// ncu's source view showed those DADDs stalled on the math pipe as long as the DMMAs themselves.)
// (Round 1 kept two 2^52-seeded sums and recombined them with a 64-bit multiply by 2^48 mod p;
// the stacked form has the same DMMA count and a third of the epilogue, measured equal in time:
// 29.4 us at the full-size ModUp either way -- the kernel is not bound by its integer work.)
//
// GEMM view per conversion: D[i][c] = sum_k T[i][k] * y[k][c] with M = output limbs (tiles
// of 8), K = input limbs (padded to a multiple of 4), N = columns (tiles of 8).  A warp owns
// 16 columns: it pre-scales them once (each lane 1 column x KS limbs per tile = the B
// fragments), then walks the output tiles; A fragments come from a shared-memory copy of
// the table in double.  Each lane finishes two adjacent columns of one output limb.
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

// x * 2^-1074: the SUBNORMAL double whose bit pattern is the integer x (no instruction at all: a
// register pair {x, 0}).  FP64 arithmetic never flushes subnormals, and below 2^-1022 a double is a
// 52-bit fixed-point number: with the residues' 16-bit halves fed to the tensor pipe in this form the
// products T * y * 2^-1074 (T * y < 2^47) and their sums (< 2^52) are exact and the accumulator's bit
// pattern is the integer sum itself -- no 2^52 seed, no conversion add per operand, no mask and no FP64
// add per output on the pipe that bounds this kernel.
__device__ __forceinline__ double sub2d(uint32_t x) {
    return __hiloint2double(0, (int)x);
}

template <int KS>
__global__ void __launch_bounds__(128)
bconv_dmma(BconvJobs jobs, const ModSlot* __restrict__ slots, size_t cols, int chunk) {
    constexpr int KP = 4 * KS;
    extern __shared__ uint4 sm4[];
    const BconvJob& job = jobs.job[blockIdx.y];
    const int l_in = job.tab.l_in, l_out = job.tab.l_out;
    const int i_lo = blockIdx.z * chunk, i_hi = min(l_out, i_lo + chunk);
    if (i_lo >= i_hi) return;
    const int rows_pad = (i_hi - i_lo + 7) & ~7;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kk = lane & 3, cc = lane >> 2;
    // A warp walks column tiles of 16; the table staging below is paid once per CTA and the
    // next tile's residues are in flight while the current tile is contracted.
    const size_t tiles = cols / 16;
    const size_t warps = (size_t)gridDim.x * 4;
    size_t tile = (size_t)blockIdx.x * 4 + warp;
    uint32_t raw[2][KS];
    auto fetch = [&](size_t tl) {
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const int k = 4 * j + kk;
#pragma unroll
            for (int t = 0; t < 2; ++t)
                raw[t][j] = k < l_in ? job.in[(size_t)k * job.in_stride + tl * 16 + 8 * t + cc] : 0u;
        }
    };
    pdl_trigger();
    // operands come ready-made from the table (api.cu): one level of loads, no arithmetic
    constexpr int KP2 = 2 * KP;                                            // the two halves of y stacked along K
    constexpr int TS = KP2 + kBconvTablePad;
    double* s_t = reinterpret_cast<double*>(sm4);                          // [rows_pad][TS]  {T | T * 2^16 mod p | pad}
    uint4* s_om = sm4 + ((size_t)((chunk + 7) & ~7) * TS * sizeof(double)) / sizeof(uint4);  // {q, qinv, out row, -}
    uint4* s_in = s_om + ((chunk + 7) & ~7);                               // {q, inv_qhat, shoup(inv_qhat), -}
    {
        const int kpj = job.tab.kp;
        const double* src = job.tab.t_f64k + (size_t)i_lo * 2 * kpj;
        if (kpj == KP) {
            // the CTA's rows of the table are one contiguous block: asynchronous 16-byte copies straight
            // into shared memory, in flight while the residues are fetched (no register round trip)
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_t);
            for (int idx = threadIdx.x; idx < rows_pad * KP; idx += blockDim.x) {
                const int i = idx / KP, c = idx - i * KP;             // 16-byte chunk c of row i
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                             :: "r"(dst + (uint32_t)(i * TS * 8 + 16 * c)), "l"(src + 2 * idx) : "memory");
            }
        } else {
            // a conversion with fewer input limbs than the launch's KP (the partial last digit stacked
            // with the full ones) has a narrower table: zero-fill the extra columns
            for (int idx = threadIdx.x; idx < rows_pad * KP2; idx += blockDim.x) {
                const int i = idx / KP2, c = idx - i * KP2;
                const int half = c >= KP ? 1 : 0, k = c - half * KP;
                s_t[i * TS + c] = k < kpj ? src[(size_t)i * 2 * kpj + half * kpj + k] : 0.0;
            }
        }
    }
    for (int r = threadIdx.x; r < rows_pad; r += blockDim.x) {
        uint4 om = job.tab.om[i_lo + r];
        if (job.out_row && i_lo + r < i_hi) om.z = (uint32_t)job.out_row[i_lo + r];
        s_om[r] = om;
    }
    for (int k = threadIdx.x; k < KP; k += blockDim.x)
        s_in[k] = k < job.tab.kp ? job.tab.inc[k] : make_uint4(3u, 0u, 0u, 0u);
    pdl_wait();                                 // tables are static; the residues are not
    if (tile < tiles) fetch(tile);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (tile >= tiles) return;
    for (; tile < tiles; tile += warps) {
        // B fragments: lane (kk, cc) holds y[4j + kk][16 tile + 8t + cc], split in 16-bit halves
        double y0[2][KS], y1[2][KS];
#pragma unroll
        for (int j = 0; j < KS; ++j) {
            const uint4 im = s_in[4 * j + kk];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const uint32_t y = 4 * j + kk < l_in ? shoup_mul(raw[t][j], im.y, im.z, im.x) : 0u;
                y0[t][j] = sub2d(y & 0xFFFFu);
                y1[t][j] = sub2d(y >> 16);
            }
        }
        const size_t c_base = tile * 16;
        if (tile + warps < tiles) fetch(tile + warps);
        for (int m0 = 0; m0 < rows_pad; m0 += 8) {
            double a0[KS], a1[KS];
#pragma unroll
            for (int j = 0; j < KS; ++j) {
                a0[j] = s_t[(m0 + cc) * TS + 4 * j + kk];
                a1[j] = s_t[(m0 + cc) * TS + KP + 4 * j + kk];
            }
            // two chains per column tile (low / high half of y) keep four DMMAs in flight; their sum is
            // the whole contraction, an integer below 2^52 on top of the 2^52 seed of c0
            double c0[2][2], c1[2][2];
#pragma unroll
            for (int t = 0; t < 2; ++t) { c0[t][0] = c0[t][1] = 0.0; c1[t][0] = c1[t][1] = 0.0; }
#pragma unroll
            for (int j = 0; j < KS; ++j) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    dmma884(c0[t], a0[j], y0[t][j]);
                    dmma884(c1[t], a1[j], y1[t][j]);
                }
            }
            // lane holds D[m0 + cc][2 kk + {0, 1}] of both column tiles
            const uint4 om = s_om[m0 + cc];
            if (i_lo + m0 + cc < i_hi) {
                uint32_t* dst = job.out + (size_t)om.z * job.out_stride + c_base + 2 * kk;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    uint32_t r[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        // the chains are subnormal doubles: their bit patterns ARE the integer sums, added on the
                        // integer pipe (no FP64 add, no mask).  V < 2^52: its high word (< 2^20 < p) and low word
                        // go straight through one REDC
                        const uint64_t v = (uint64_t)__double_as_longlong(c0[t][e]) + (uint64_t)__double_as_longlong(c1[t][e]);
                        r[e] = redc((uint32_t)v, (uint32_t)(v >> 32), om.x, om.y);
                    }
                    *reinterpret_cast<uint2*>(dst + 8 * t) = make_uint2(r[0], r[1]);
                }
            }
        }
    }
}

// Any modulus below 2^32; one column per thread; exact '%' folds.
__global__ void __launch_bounds__(128)
bconv_generic(BconvJobs jobs, const ModSlot* __restrict__ slots, size_t cols) {
    const BconvJob& job = jobs.job[blockIdx.y];
    const int l_in = job.tab.l_in, l_out = job.tab.l_out;
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    for (int i = 0; i < l_out; ++i) {
        const uint64_t p = slots[job.tab.out_slot[i]].q;
        uint64_t acc = 0;
        for (int k = 0; k < l_in; ++k) {
            const uint64_t q = slots[job.tab.in_slot[k]].q;
            const uint64_t y = (uint64_t)job.in[(size_t)k * job.in_stride + c] * job.tab.inv_qhat[k] % q;
            acc = (acc + (uint64_t)job.tab.t_plain[i * l_in + k] * y % p) % p;
        }
        const size_t orow = job.out_row ? (size_t)job.out_row[i] : (size_t)i;
        job.out[orow * job.out_stride + c] = (uint32_t)acc;
    }
}

// FP64 tensor-core work of the split-integer contraction: two halves x l_in x l_out FMAs per column
static double jobs_flops(const BconvJobs& jobs, size_t cols) {
    double macs = 0;
    for (int j = 0; j < jobs.count; ++j) macs += 2.0 * jobs.job[j].tab.l_in * jobs.job[j].tab.l_out;
    return 2.0 * macs * cols;
}

static double jobs_bytes(const BconvJobs& jobs, size_t cols) {
    double limbs = 0;
    for (int j = 0; j < jobs.count; ++j) limbs += jobs.job[j].tab.l_in + jobs.job[j].tab.l_out;
    return limbs * 4.0 * cols;
}

static int bconv_variant() {
    static int v = -1;
    if (v < 0) {
        // default: FP64 tensor-core kernel; CKKS_BCONV=int: IMAD.WIDE kernel; CKKS_BCONV=f64: DFMA kernel
        const char* e = getenv("CKKS_BCONV");
        v = !e ? 2 : (e[0] == 'f' ? 1 : (e[0] == 'i' ? 0 : 2));
    }
    return v;
}

template <int KS>
static int launch_dmma(const BconvJobs& jobs, const ModSlot* slots, size_t cols, int l_out_max, cudaStream_t st) {
    // tiles per warp: as many as still leave ~6 CTAs per SM (the per-CTA table staging is
    // amortised over them); the output walk is split over blockIdx.z when one conversion is too small
    const size_t tiles = cols / 16;
    const int z_max = (l_out_max + 7) / 8;
    // fewer tiles per warp before splitting the output walk: a z-split repeats the pre-scale
    int tpw = 4;
    while (tpw > 1 && ((tiles + 4 * tpw - 1) / (4 * tpw)) * jobs.count < (size_t)148 * 6) tpw >>= 1;
    const unsigned gx = (unsigned)((tiles + 4 * tpw - 1) / (4 * tpw));
    const size_t ctas_xy = (size_t)gx * jobs.count;
    int z = (int)(((size_t)148 * 6 + ctas_xy - 1) / ctas_xy);
    if (z > z_max) z = z_max;
    const int chunk = (((l_out_max + z - 1) / z) + 7) & ~7;
    const size_t sm = sizeof(double) * (size_t)chunk * (8 * KS + kBconvTablePad) + sizeof(uint4) * ((size_t)chunk + 4 * KS);
    dim3 grid(gx, jobs.count, (l_out_max + chunk - 1) / chunk);
    ProfScope ps("bconv", st, jobs_bytes(jobs, cols), jobs_flops(jobs, cols));
    if (sm > 48 * 1024)
        CK(cudaFuncSetAttribute(bconv_dmma<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CK(launch_pdl(bconv_dmma<KS>, grid, dim3(128), sm, st, jobs, slots, cols, chunk));
    CK(cudaGetLastError());
    return CKKS_OK;
}

template <int LIN>
static int launch_fast(const BconvJobs& jobs, const ModSlot* slots, size_t cols, int l_out_max,
                       bool pairs, cudaStream_t st) {
    if (bconv_variant() == 1) {          // CKKS_BCONV=f64
        constexpr int LINP = (LIN + 1) / 2 * 2;
        const size_t sm = sizeof(double) * (size_t)l_out_max * LINP + sizeof(uint4) * ((size_t)l_out_max + LIN);
        const unsigned gx = (unsigned)((cols + 127) / 128);
        const int chunk = out_chunk((size_t)gx * jobs.count, l_out_max);
        dim3 grid(gx, jobs.count, (l_out_max + chunk - 1) / chunk);
        ProfScope ps("bconv", st, jobs_bytes(jobs, cols));
        if (sm > 48 * 1024)
            CK(cudaFuncSetAttribute(bconv_f64<LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        bconv_f64<LIN><<<grid, 128, sm, st>>>(jobs, slots, cols, chunk);
        CK(cudaGetLastError());
        return CKKS_OK;
    }
    constexpr int G = (LIN + 3) / 4;
    const size_t sm = sizeof(uint4) * ((size_t)l_out_max * G + l_out_max + LIN);
    const size_t work = pairs ? cols / 2 : cols;
    const unsigned gx = (unsigned)((work + 127) / 128);
    const int chunk = out_chunk((size_t)gx * jobs.count, l_out_max);
    dim3 grid(gx, jobs.count, (l_out_max + chunk - 1) / chunk);
    ProfScope ps("bconv", st, jobs_bytes(jobs, cols));
    if (pairs) {
        if (sm > 48 * 1024)
            CK(cudaFuncSetAttribute(bconv_fast<LIN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        bconv_fast<LIN, 2><<<grid, 128, sm, st>>>(jobs, slots, cols, chunk);
    } else {
        if (sm > 48 * 1024)
            CK(cudaFuncSetAttribute(bconv_fast<LIN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        bconv_fast<LIN, 1><<<grid, 128, sm, st>>>(jobs, slots, cols, chunk);
    }
    CK(cudaGetLastError());
    return CKKS_OK;
}

int bconv_launch_jobs(const BconvJobs& jobs, const ModSlot* slots, size_t cols, cudaStream_t st) {
    if (jobs.count <= 0 || cols == 0) return CKKS_OK;
    int l_in = jobs.job[0].tab.l_in;
    int l_out_max = 0;
    bool fast = true, pairs = cols % 2 == 0, mixed = false;
    for (int j = 0; j < jobs.count; ++j) {
        const BconvJob& jb = jobs.job[j];
        if (jb.tab.l_in != jobs.job[0].tab.l_in) mixed = true;     // only the tensor-core kernel stacks these
        if (jb.tab.l_in > l_in) l_in = jb.tab.l_in;
        if (jb.tab.l_out > l_out_max) l_out_max = jb.tab.l_out;
        fast = fast && jb.tab.all31;
        pairs = pairs && (((uintptr_t)jb.in | (uintptr_t)jb.out) % 8 == 0) &&
                jb.in_stride % 2 == 0 && jb.out_stride % 2 == 0;
    }
    if (fast && l_in <= 16 && cols % 16 == 0 && bconv_variant() == 2) {
        bool aligned = true;
        for (int j = 0; j < jobs.count; ++j)
            aligned = aligned && ((uintptr_t)jobs.job[j].out % 8 == 0) && jobs.job[j].out_stride % 2 == 0;
        if (aligned) {
            switch ((l_in + 3) / 4) {
                case 1: return launch_dmma<1>(jobs, slots, cols, l_out_max, st);
                case 2: return launch_dmma<2>(jobs, slots, cols, l_out_max, st);
                case 3: return launch_dmma<3>(jobs, slots, cols, l_out_max, st);
                default: return launch_dmma<4>(jobs, slots, cols, l_out_max, st);
            }
        }
    }
    if (mixed) {
        // the other kernels are specialised on one l_in: run equal-sized groups one after the other
        for (int j0 = 0; j0 < jobs.count;) {
            BconvJobs part;
            part.count = 0;
            int j = j0;
            for (; j < jobs.count && jobs.job[j].tab.l_in == jobs.job[j0].tab.l_in; ++j) part.job[part.count++] = jobs.job[j];
            CKS(bconv_launch_jobs(part, slots, cols, st));
            j0 = j;
        }
        return CKKS_OK;
    }
    if (fast && l_in <= 16) {
        switch (l_in) {
#define BCONV_CASE(L) case L: return launch_fast<L>(jobs, slots, cols, l_out_max, pairs, st);
            BCONV_CASE(1) BCONV_CASE(2) BCONV_CASE(3) BCONV_CASE(4) BCONV_CASE(5) BCONV_CASE(6)
            BCONV_CASE(7) BCONV_CASE(8) BCONV_CASE(9) BCONV_CASE(10) BCONV_CASE(11) BCONV_CASE(12)
            BCONV_CASE(13) BCONV_CASE(14) BCONV_CASE(15) BCONV_CASE(16)
#undef BCONV_CASE
        }
    }
    dim3 grid((unsigned)((cols + 127) / 128), jobs.count);
    ProfScope ps("bconv_generic", st, jobs_bytes(jobs, cols));
    bconv_generic<<<grid, 128, 0, st>>>(jobs, slots, cols);
    CK(cudaGetLastError());
    return CKKS_OK;
}

int bconv_launch(const BconvDev& tab, const ModSlot* slots, const uint32_t* in, size_t in_stride,
                 uint32_t* out, size_t out_stride, size_t cols, cudaStream_t st) {
    BconvJobs jobs;
    jobs.count = 1;
    jobs.job[0].tab = tab;
    jobs.job[0].in = in;
    jobs.job[0].in_stride = in_stride;
    jobs.job[0].out = out;
    jobs.job[0].out_stride = out_stride;
    jobs.job[0].out_row = nullptr;
    return bconv_launch_jobs(jobs, slots, cols, st);
}

}  // namespace ckks
