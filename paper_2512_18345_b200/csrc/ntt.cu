// ntt.cu -- negacyclic NTT / iNTT over RNS limb matrices.
//
// Function computed (bit-exact target): reference transform.py:203-250
// (_run_stages), i.e. Cooley-Tukey forward over the bit-reversed psi-power
// table and Gentleman-Sande inverse with N^-1 folded into the last stage;
// natural order in, bit-reversed evaluation order out (SURVEY 8a').
//
// Implementations:
//  * generic: one radix-2 stage per launch straight on global memory; any N,
//    any stage range (serves ntt_two_phase with arbitrary n1 and small rings).
//  * N = 2^16 fast path: two kernels of eight stages each (the paper's
//    NTT1/NTT2 split, reference n1 = 2^8).  Each kernel runs
//    two radix-16 passes in registers (Shoup lazy butterflies, values kept in
//    [0, 2q)) with one conflict-free shared-memory transpose between them.
//  * N = 2^16, launches of few limbs: the same passes as ONE kernel over clusters of eight
//    CTAs per limb, the intermediate exchanged through distributed shared memory.
//  * N <= 2^15: one CTA per limb, the limb in shared memory.
#include <cstdlib>
#include "common.cuh"
#include "internal.h"

namespace ckks {

// ---------------------------------------------------------------------------------
// generic radix-2 stage
// ---------------------------------------------------------------------------------
__global__ void ntt_stage_generic(const uint32_t* in, uint32_t* out,
                                  const int32_t* __restrict__ row_slot,
                                  const ModSlot* __restrict__ slots, RowMap rm, uint32_t n,
                                  uint32_t lg, uint32_t s, int inverse) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= (n >> 1)) return;
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    const uint32_t* src = in + rm.in_row(blockIdx.y) * n;
    uint32_t* dst = out + rm.out_row(blockIdx.y) * n;
    if (!inverse) {
        const uint32_t t = n >> (s + 1);
        const uint32_t g = b / t, j = b - g * t;
        const uint32_t i0 = g * 2 * t + j, i1 = i0 + t;
        const uint2 w = m.fwd[(1u << s) + g];
        const uint32_t x = src[i0], y = src[i1];
        const uint32_t v = shoup_mul(y, w.x, w.y, q);
        dst[i0] = add_mod(x, v, q);
        dst[i1] = sub_mod(x, v, q);
    } else {
        const uint32_t t = 1u << s, groups = n >> (s + 1);
        const uint32_t g = b >> s, j = b & (t - 1);
        const uint32_t i0 = g * 2 * t + j, i1 = i0 + t;
        uint2 w = m.inv[groups + g];
        const uint32_t x = src[i0], y = src[i1];
        uint32_t total = add_mod(x, y, q);
        const uint32_t diff = sub_mod(x, y, q);
        if (s == lg - 1) {
            total = shoup_mul(total, m.n_inv, m.n_inv_s, q);
            w = make_uint2(m.w_last, m.w_last_s);
        }
        dst[i0] = total;
        dst[i1] = shoup_mul(diff, w.x, w.y, q);
    }
}

// ---------------------------------------------------------------------------------
// radix-16 register passes
// ---------------------------------------------------------------------------------
// Forward: values enter in [0, 2q) and leave in [0, 2q).  `v` = y * w mod q, canonical.
__device__ __forceinline__ void ct_bfly(uint32_t& x, uint32_t& y, uint32_t v, uint32_t q) {
    const uint32_t xc = csub(x, q);
    x = xc + v;
    y = xc - v + q;
}

// Four Cooley-Tukey stages on 16 registers.  MUL(s, g, y) returns y * w mod q in
// [0, q) for the twiddle of local stage s (0..3), local group g (0 .. 2^s - 1).
template <class MUL>
__device__ __forceinline__ void ct16(uint32_t (&v)[16], uint32_t q, MUL mul) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {              // fixed trip count: always fully unrolled
            const int half = 8 >> s;
            const int g = b >> (3 - s), j = b & (half - 1);
            const int i0 = g * 2 * half + j;
            ct_bfly(v[i0], v[i0 + half], mul(s, g, v[i0 + half]), q);
        }
    }
}

// Four Gentleman-Sande stages on 16 registers, canonical in and out.
// MUL(s, g, d): d * w mod q in [0, q) for local stage s (pair distance 2^s),
// local group g (0 .. (8 >> s) - 1); d may be any 32-bit value.
template <int STAGES = 4, class MUL>
__device__ __forceinline__ void gs16(uint32_t (&v)[16], uint32_t q, MUL mul) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int t = 1 << s;
            const int g = b >> s, j = b & (t - 1);
            const int i0 = g * 2 * t + j;
            const uint32_t x = v[i0], y = v[i0 + t];
            v[i0] = csub(x + y, q);
            v[i0 + t] = mul(s, g, x - y + q);
        }
    }
}

// Multiplier functors.  Table form: one Shoup multiplication by a stored
// {w, w'} pair.  Split form (the contiguous phase's last / first four stages):
// w = X[s] * YZ[s][e][g] with X per 256-block and YZ a 240-entry per-modulus
// table, two chained Shoup multiplications and no per-butterfly table traffic
// (the on-the-fly idea of reference transform.py:126-169 with a three-way split).
#define TW_MUL(expr) [&](int s, int gi, uint32_t y) { const uint2 w = (expr); return shoup_mul(y, w.x, w.y, q); }

// ---------------------------------------------------------------------------------
// N = 2^16, strided phase: 256-point transforms down the columns of the
// 256 x 256 view (element (j, c) at j*256 + c).  A CTA owns COLS adjacent
// columns; thread (g, c) holds 16 rows.  Tile row j is stored at padded row
// j + (j >> 4) so that both register layouts (j = g + 16m and j = 16g + m) hit
// 32 distinct banks per warp.
// ---------------------------------------------------------------------------------
constexpr int kN16 = 65536;

template <int COLS>
__global__ void __launch_bounds__(16 * COLS)
ntt16_fwd_strided(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                  const ModSlot* __restrict__ slots, RowMap rm) {
    __shared__ uint2 s_tw[256];
    __shared__ uint32_t tile[271 * COLS];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    pdl_trigger();
    // twiddles go through a register and are stored only after the data loads are in flight: the
    // in-order issue would otherwise serialise the table's latency with the data's
    static_assert(16 * COLS == 256, "one twiddle pair per thread");
    const uint2 tw_stage = m.fwd[tid];
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + blockIdx.x * COLS + c;
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = src[(g + 16 * k) * 256];
    s_tw[tid] = tw_stage;
    __syncthreads();
    // stages 0..3: rows j = g + 16k, group index = k >> (4 - s): uniform twiddles
    ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(g + 17 * k) * COLS + c] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[(17 * g + k) * COLS + c];
    // stages 4..7: rows j = 16g + k
    ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + blockIdx.x * COLS + c;
#pragma unroll
    for (int k = 0; k < 16; ++k) dst[(16 * g + k) * 256] = csub(v[k], q);
}

template <int COLS>
__global__ void __launch_bounds__(16 * COLS)
ntt16_inv_strided(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                  const ModSlot* __restrict__ slots, RowMap rm) {
    __shared__ uint2 s_tw[256];
    __shared__ uint32_t tile[271 * COLS];
    const int tid = threadIdx.x;
    const int c = tid % COLS, g = tid / COLS;
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    pdl_trigger();
    // twiddles go through a register and are stored only after the data loads are in flight: the
    // in-order issue would otherwise serialise the table's latency with the data's
    static_assert(16 * COLS == 256, "one twiddle pair per thread");
    const uint2 tw_stage = m.inv[tid];
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + blockIdx.x * COLS + c;
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = src[(16 * g + k) * 256];
    s_tw[tid] = tw_stage;
    __syncthreads();
    // global stages 8..11 = 256-point GS stages 0..3 on rows j = 16g + k
    gs16(v, q, TW_MUL(s_tw[(16 + g) * (8 >> s) + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(17 * g + k) * COLS + c] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[(g + 17 * k) * COLS + c];
    // global stages 12..14 on rows j = g + 16k, then the last stage with N^-1
    gs16<3>(v, q, TW_MUL(s_tw[(8 >> s) + gi]));
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + blockIdx.x * COLS + c;
    const uint32_t ninv = m.n_inv, ninv_s = m.n_inv_s, wl = m.w_last, wl_s = m.w_last_s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t x = v[j], y = v[j + 8];
        const uint32_t total = csub(x + y, q);
        const uint32_t diff = x - y + q;
        dst[(g + 16 * j) * 256] = shoup_mul(total, ninv, ninv_s, q);
        dst[(g + 16 * (j + 8)) * 256] = shoup_mul(diff, wl, wl_s, q);
    }
}

// ---------------------------------------------------------------------------------
// N = 2^16, contiguous phase: 256 independent 256-point transforms on
// consecutive 1 KiB blocks.  A CTA owns 16 blocks (16 KiB); thread (blk, e)
// holds 16 elements.  Tile element e of block blk is stored at
// blk*272 + e + (e >> 4).
//
// Twiddles.  The four stages next to the data (forward 12..15, inverse 0..3)
// use N/2 + N/4 + N/8 + N/16 distinct twiddles per limb.  For the 16 consecutive
// elements a thread holds in that pass they are the table entries
//     [idx0], [2 idx0 .. +2), [4 idx0 .. +4), [8 idx0 .. +8),   idx0 = (256 + B) * 16 + e,
// i.e. 15 Shoup pairs = 120 B in five aligned vector loads (8 + 16 + 32 + 64 B),
// consecutive threads reading consecutive addresses.  They are fetched with the
// data at kernel start.  (An earlier version rebuilt them on the fly from a
// 240-entry split table with a second Shoup product per butterfly; on B200 the
// integer multiplier -- the fmaheavy pipe -- is the busiest unit of this kernel
// while L2 has headroom, so table reads win.)  The other four stages need 15
// twiddles per block, staged through shared memory by the block's own lanes.
// ---------------------------------------------------------------------------------
struct Tw15 {
    uint2 t1, t2[2], t4[4], t8[8];
};

__device__ __forceinline__ void ld256(const void* p, uint32_t (&r)[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}

__device__ __forceinline__ void st256(void* p, const uint32_t (&r)[8]) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__device__ __forceinline__ void load_tw15(const uint2* __restrict__ tab, uint32_t idx0, Tw15& t) {
    t.t1 = __ldg(tab + idx0);
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(tab + 2 * idx0));
    t.t2[0] = make_uint2(a.x, a.y);
    t.t2[1] = make_uint2(a.z, a.w);
    uint32_t r[8];
    ld256(tab + 4 * idx0, r);
#pragma unroll
    for (int j = 0; j < 4; ++j) t.t4[j] = make_uint2(r[2 * j], r[2 * j + 1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        ld256(tab + 8 * idx0 + 4 * h, r);
#pragma unroll
        for (int j = 0; j < 4; ++j) t.t8[4 * h + j] = make_uint2(r[2 * j], r[2 * j + 1]);
    }
}

// EPI: the ModDown epilogue (reference keyswitch.py:412-418, :452) runs on the transform's
// registers instead of a separate pass: the rows are conv = NTT(BConv_{P->Q}(..)) of both
// halves, and the kernel stores (x_Q - conv) * P^-1 (+ fold) straight into the result, so conv
// is never written or re-read.
template <bool EPI>
__global__ void __launch_bounds__(256, EPI ? 5 : 6)
ntt16_fwd_contig(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                 const ModSlot* __restrict__ slots, RowMap rm, ModDownEpilogueArgs ep) {
    __shared__ uint32_t tile[16 * 272];
    __shared__ uint2 s_blk[16][16];      // per block: the 15 twiddles of stages 8..11
    const int tid = threadIdx.x;
    const int e = tid & 15, blk = tid >> 4;
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    const uint32_t B = blockIdx.x * 16 + blk;          // 256-element block index within the limb
    const bool ep_single = EPI && ep.halves == 1;
    const int ep_row = EPI ? blockIdx.y % ep.l : 0, ep_half = (EPI && !ep_single) ? (blockIdx.y / ep.l) & 1 : 0;
    const size_t ep_g = EPI ? blockIdx.y / ((ep_single ? 1 : 2) * ep.l) : 0;      // element of a batched ModDown
    const size_t ep_at = (size_t)ep_row * kN16 + B * 256 + 16 * e;
    pdl_trigger();
    if (EPI) {
        // x_Q (and the folded polynomial) are needed only after the last stage: pull their
        // lines into L2 now
        asm volatile("prefetch.global.L2 [%0];" :: "l"((ep_half ? ep.xq_b : ep.xq_a) + ep_g * ep.xq_stride + ep_at));
        const uint32_t* f = ep_half ? ep.fold_b : ep.fold_a;
        if (f && !ep.galois) asm volatile("prefetch.global.L2 [%0];" :: "l"(f + ep_at));
    }
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + B * 256;
    const uint2* __restrict__ fwd = m.fwd;
    // the 16 threads of a 256-block stage that block's table entries themselves: the whole
    // kernel then only needs warp-level synchronisation (a block's exchange is half a warp)
    uint2 tw_stage = make_uint2(0u, 0u);
    if (e < 15) {
        const int st = 31 - __clz(e + 1);              // local stage, group = e + 1 - 2^st
        tw_stage = fwd[((256 + B) << st) + (e + 1 - (1 << st))];
    }
    Tw15 tw;
    load_tw15(fwd, (256 + B) * 16 + e, tw);
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = src[e + 16 * k];
    s_blk[blk][e] = tw_stage;                          // stored once the data loads are in flight
    __syncwarp();
    // global stages 8..11: elements e + 16k, slot = (256 + B) * 2^s + group
    ct16(v, q, TW_MUL(s_blk[blk][(1 << s) - 1 + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[blk * 272 + e + 17 * k] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[blk * 272 + 17 * e + k];
    // global stages 12..15: elements 16e + k, slot = ((256 + B) * 16 + e) * 2^s + group
    ct16(v, q, TW_MUL(s == 0 ? tw.t1 : (s == 1 ? tw.t2[gi & 1] : (s == 2 ? tw.t4[gi & 3] : tw.t8[gi & 7]))));
    if (EPI) {
        const uint32_t pinv = ep.pinv[ep_row], pinv_s = ep.pinv_s[ep_row];
        const uint32_t* x = (ep_half ? ep.xq_b : ep.xq_a) + ep_g * ep.xq_stride + ep_at;
        const uint32_t* fsrc = ep_half ? ep.fold_b : ep.fold_a;
        uint32_t* o = (ep_half ? ep.out_b : ep.out_a) + ep_g * ep.out_stride + ep_at;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t xv[8], r[8];
            ld256(x + 8 * h, xv);
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = shoup_mul(xv[k] - csub(v[8 * h + k], q) + q, pinv, pinv_s, q);
            if (fsrc && ep.galois) {
                const uint32_t* f = fsrc + (size_t)ep_row * kN16;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    r[k] = add_mod(r[k], f[galois_src(B * 256 + 16 * e + 8 * h + k, ep.galois, kN16, 16)], q);
            } else if (fsrc) {
                uint32_t fv[8];
                ld256(fsrc + ep_at + 8 * h, fv);
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = add_mod(r[k], fv[k], q);
            }
            st256(o + 8 * h, r);
        }
        return;
    }
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = csub(v[8 * h + k], q);
        st256(dst + 8 * h, r);
    }
}

// MUL: the transform's input is the element-wise product in (.) in2 of two evaluation-domain
// polynomials (the d2 = a1 * a2 term of HMult), formed on load instead of by a tensor pass.
template <bool MUL>
__global__ void __launch_bounds__(256, MUL ? 3 : 6)
ntt16_inv_contig(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                 const ModSlot* __restrict__ slots, RowMap rm, const uint32_t* in2) {
    __shared__ uint32_t tile[16 * 272];
    __shared__ uint2 s_blk[16][16];      // per block: the 15 twiddles of stages 4..7, laid out 8 | 4 | 2 | 1
    const int tid = threadIdx.x;
    const int e = tid & 15, blk = tid >> 4;
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    const uint32_t B = blockIdx.x * 16 + blk;
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
    const uint2* __restrict__ inv = m.inv;
    pdl_trigger();
    uint2 tw_stage = make_uint2(0u, 0u);
    if (e < 15) {
        // stage s of 4..7 has (8 >> s) groups
        const int st = e < 8 ? 0 : (e < 12 ? 1 : (e < 14 ? 2 : 3));
        const int off = st == 0 ? 0 : (st == 1 ? 8 : (st == 2 ? 12 : 14));
        tw_stage = inv[(256 + B) * (8 >> st) + (e - off)];
    }
    Tw15 tw;
    load_tw15(inv, (256 + B) * 16 + e, tw);
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t r[8];
        ld256(src + 8 * h, r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * h + k] = r[k];
    }
    s_blk[blk][e] = tw_stage;                          // stored once the data loads are in flight
    if (MUL) {
        const uint32_t* src2 = in2 + rm.in_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t r[8];
            ld256(src2 + 8 * h, r);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[8 * h + k] = mul_mod(v[8 * h + k], r[k], m);
        }
    }
    __syncwarp();
    // global stages 0..3 on elements 16e + k: slot = ((256 + B) * 16 + e) * (8 >> s) + group
    gs16(v, q, TW_MUL(s == 0 ? tw.t8[gi & 7] : (s == 1 ? tw.t4[gi & 3] : (s == 2 ? tw.t2[gi & 1] : tw.t1))));
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[blk * 272 + 17 * e + k] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[blk * 272 + e + 17 * k];
    // global stages 4..7 on elements e + 16k: slot = (256 + B) * (8 >> s) + group
    gs16(v, q, TW_MUL(s_blk[blk][(s == 0 ? 0 : (s == 1 ? 8 : (s == 2 ? 12 : 14))) + gi]));
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + B * 256;
#pragma unroll
    for (int k = 0; k < 16; ++k) dst[e + 16 * k] = v[k];
}

// ---------------------------------------------------------------------------------
// N = 2^16, single pass over a thread-block cluster (the transform the
// two-kernel split of transform.py:290-323 / PAPER.md:355-365 approximates).  A cluster of
// eight CTAs owns one limb; each CTA keeps 1/8 of it (32 KiB) in shared memory and the
// intermediate of the two phases never goes to global memory: it is exchanged through
// distributed shared memory (st.shared::cluster into the CTA that owns the element in the
// other phase's layout).
//
//   forward:  CTA r loads columns [32r, 32r + 32) of the 256 x 256 view (128-byte row
//             segments), runs stages 0..7 as the strided phase does, sends row j to CTA
//             j / 32, then runs stages 8..15 on its 32 contiguous 256-blocks and stores them
//             (or the ModDown epilogue's result) as one contiguous 32 KiB piece.
//   inverse:  the mirror image: blocks [32r, 32r + 32) in, stages 0..7, column c to CTA
//             c / 32, stages 8..15 with N^-1 folded into the last, 128-byte row segments out.
//
// Same butterflies, same twiddle slots and the same register passes as the two-kernel
// path (bit-exact to it and to _run_stages), half its global traffic, one launch.
// 512 threads x 16 residues; thread layouts: strided passes (g, c) = (tid / 32, tid % 32),
// contiguous passes (blk, e) = (tid / 16, tid % 16).
// ---------------------------------------------------------------------------------
constexpr int kClusterCtas = 8;
// Default policy of ntt_launch (see cluster_max_rows()): measured on B200 (profiles/ntt_cluster_ab.py,
// r2l_ntt_cluster_ab.json) the single launch wins up to ~28 limbs (2 rows: 6.4 vs 11.5 us inverse, 28
// rows: 12.7 vs 15.0 us) and loses above (192 rows: 63 vs 48 us: two cluster barriers and a 21 B/clk/SM
// DSMEM exchange per CTA cost more than the global round trip they replace).
constexpr int kClusterDefaultMaxRows = 28;
constexpr int kClusterThreads = 512;
constexpr int kXbufWords = 32 * 272;           // 32 blocks, padded as in the contiguous kernels
constexpr int kTileWords = 256 * 32;
constexpr size_t kClusterSmem = sizeof(uint32_t) * (kXbufWords + kTileWords) + sizeof(uint2) * (256 + 32 * 16);

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
// the first barrier phase only says "every CTA of the cluster is running" (no data is handed over): relaxed,
// so that it costs no memory fence (the release form compiles to MEMBAR.ALL.GPU + ERRBAR)
__device__ __forceinline__ void cluster_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait_relaxed() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}

template <bool EPI, int OCC>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterThreads, OCC)
ntt16_fwd_cluster(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                  const ModSlot* __restrict__ slots, RowMap rm, ModDownEpilogueArgs ep) {
    extern __shared__ __align__(16) uint32_t dyn_smem[];
    uint32_t* tile = dyn_smem;                               // [256][32]  strided-phase transpose
    uint32_t* xbuf = dyn_smem + kTileWords;                  // [32][272]  this CTA's blocks, filled by the cluster
    uint2* s_tw = reinterpret_cast<uint2*>(xbuf + kXbufWords);       // [256]     twiddles of stages 0..7
    uint2* s_blk = s_tw + 256;                               // [32][16]  per block: twiddles of stages 8..11
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_ctarank();
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    const uint2* __restrict__ fwd = m.fwd;
    const int e = tid & 15, blk = tid >> 4;                  // contiguous-phase coordinates
    const uint32_t B = rank * 32 + blk;
    const bool ep_single = EPI && ep.halves == 1;
    const int ep_row = EPI ? blockIdx.y % ep.l : 0, ep_half = (EPI && !ep_single) ? (blockIdx.y / ep.l) & 1 : 0;
    const size_t ep_g = EPI ? blockIdx.y / ((ep_single ? 1 : 2) * ep.l) : 0;
    const size_t ep_at = (size_t)ep_row * kN16 + B * 256 + 16 * e;
    pdl_trigger();
    cluster_arrive_relaxed();                                // (1) "this CTA is running"
    if (EPI) {
        asm volatile("prefetch.global.L2 [%0];" :: "l"((ep_half ? ep.xq_b : ep.xq_a) + ep_g * ep.xq_stride + ep_at));
        const uint32_t* f = ep_half ? ep.fold_b : ep.fold_a;
        if (f && !ep.galois) asm volatile("prefetch.global.L2 [%0];" :: "l"(f + ep_at));
    }
    // table entries go through registers and are stored after the data loads are in flight
    const uint2 tw_stage = fwd[tid & 255];
    uint2 blk_stage = make_uint2(0u, 0u);
    if (e < 15) {
        const int st = 31 - __clz(e + 1);
        blk_stage = fwd[((256 + B) << st) + (e + 1 - (1 << st))];
    }
    const int c = tid & 31, g = tid >> 5;                    // strided-phase coordinates
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + rank * 32 + c;
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = src[(g + 16 * k) * 256];
    if (tid < 256) s_tw[tid] = tw_stage;
    s_blk[blk * 16 + e] = blk_stage;
    __syncthreads();
    ct16(v, q, TW_MUL(s_tw[(1 << s) + gi]));                 // stages 0..3, rows g + 16k
#pragma unroll
    for (int k = 0; k < 16; ++k) tile[(g + 16 * k) * 32 + c] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = tile[(16 * g + k) * 32 + c];
    ct16(v, q, TW_MUL(s_tw[(16 << s) + (g << s) + gi]));     // stages 4..7, rows 16g + k
    // row j = 16g + k is block j of the contiguous phase: it belongs to CTA j / 32 = g / 2
    cluster_wait_relaxed();                                  // (1) every CTA of the cluster is running
    {
        const uint32_t at = smem_addr(xbuf + (16 * (g & 1)) * 272 + rank * 32 + c);
        const uint32_t remote = map_to_rank(at, g >> 1);
#pragma unroll
        for (int k = 0; k < 16; ++k) st_cluster(remote + k * 272 * 4, v[k]);
    }
    cluster_arrive();                                        // (2) my rows are delivered
    Tw15 tw;
    load_tw15(fwd, (256 + B) * 16 + e, tw);
    cluster_wait();                                          // (2) my blocks are complete
    uint32_t* xb = xbuf + blk * 272;
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xb[e + 16 * k];
    __syncwarp();
    ct16(v, q, TW_MUL(s_blk[blk * 16 + (1 << s) - 1 + gi]));  // stages 8..11, elements e + 16k
#pragma unroll
    for (int k = 0; k < 16; ++k) xb[e + 17 * k] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xb[17 * e + k];
    // stages 12..15, elements 16e + k
    ct16(v, q, TW_MUL(s == 0 ? tw.t1 : (s == 1 ? tw.t2[gi & 1] : (s == 2 ? tw.t4[gi & 3] : tw.t8[gi & 7]))));
    if (EPI) {
        const uint32_t pinv = ep.pinv[ep_row], pinv_s = ep.pinv_s[ep_row];
        const uint32_t* x = (ep_half ? ep.xq_b : ep.xq_a) + ep_g * ep.xq_stride + ep_at;
        const uint32_t* fsrc = ep_half ? ep.fold_b : ep.fold_a;
        uint32_t* o = (ep_half ? ep.out_b : ep.out_a) + ep_g * ep.out_stride + ep_at;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t xv[8], r[8];
            ld256(x + 8 * h, xv);
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = shoup_mul(xv[k] - csub(v[8 * h + k], q) + q, pinv, pinv_s, q);
            if (fsrc && ep.galois) {
                const uint32_t* f = fsrc + (size_t)ep_row * kN16;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    r[k] = add_mod(r[k], f[galois_src(B * 256 + 16 * e + 8 * h + k, ep.galois, kN16, 16)], q);
            } else if (fsrc) {
                uint32_t fv[8];
                ld256(fsrc + ep_at + 8 * h, fv);
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = add_mod(r[k], fv[k], q);
            }
            st256(o + 8 * h, r);
        }
        return;
    }
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t r[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) r[k] = csub(v[8 * h + k], q);
        st256(dst + 8 * h, r);
    }
}

template <bool MUL, int OCC>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterThreads, OCC)
ntt16_inv_cluster(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                  const ModSlot* __restrict__ slots, RowMap rm, const uint32_t* in2) {
    extern __shared__ __align__(16) uint32_t dyn_smem[];
    uint32_t* cbuf = dyn_smem;                               // [32][272]  contiguous-phase transposes, later [256][32]
    uint32_t* xt = dyn_smem + kXbufWords;                    // [256][32]  this CTA's columns, filled by the cluster
    uint2* s_tw = reinterpret_cast<uint2*>(xt + kTileWords);
    uint2* s_blk = s_tw + 256;
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_ctarank();
    const ModSlot& m = slots[row_slot[blockIdx.y]];
    const uint32_t q = m.q;
    const uint2* __restrict__ inv = m.inv;
    const int e = tid & 15, blk = tid >> 4;
    const uint32_t B = rank * 32 + blk;
    const uint32_t* src = in + rm.in_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
    pdl_trigger();
    cluster_arrive_relaxed();                                // (1)
    const uint2 tw_stage = inv[tid & 255];
    uint2 blk_stage = make_uint2(0u, 0u);
    if (e < 15) {
        const int st = e < 8 ? 0 : (e < 12 ? 1 : (e < 14 ? 2 : 3));
        const int off = st == 0 ? 0 : (st == 1 ? 8 : (st == 2 ? 12 : 14));
        blk_stage = inv[(256 + B) * (8 >> st) + (e - off)];
    }
    Tw15 tw;
    load_tw15(inv, (256 + B) * 16 + e, tw);
    uint32_t v[16];
    pdl_wait();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t r[8];
        ld256(src + 8 * h, r);
#pragma unroll
        for (int k = 0; k < 8; ++k) v[8 * h + k] = r[k];
    }
    if (tid < 256) s_tw[tid] = tw_stage;                     // stored once the data loads are in flight
    s_blk[blk * 16 + e] = blk_stage;
    if (MUL) {
        const uint32_t* src2 = in2 + rm.in_row(blockIdx.y) * kN16 + B * 256 + 16 * e;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t r[8];
            ld256(src2 + 8 * h, r);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[8 * h + k] = mul_mod(v[8 * h + k], r[k], m);
        }
    }
    __syncwarp();
    // stages 0..3 on elements 16e + k
    gs16(v, q, TW_MUL(s == 0 ? tw.t8[gi & 7] : (s == 1 ? tw.t4[gi & 3] : (s == 2 ? tw.t2[gi & 1] : tw.t1))));
    uint32_t* cb = cbuf + blk * 272;
#pragma unroll
    for (int k = 0; k < 16; ++k) cb[17 * e + k] = v[k];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cb[e + 17 * k];
    // stages 4..7 on elements e + 16k
    gs16(v, q, TW_MUL(s_blk[blk * 16 + (s == 0 ? 0 : (s == 1 ? 8 : (s == 2 ? 12 : 14))) + gi]));
    // element e + 16k of block B is (row B, column e + 16k) of the 256 x 256 view: its column
    // belongs to CTA (e + 16k) / 32 = k / 2.  Rows are stored with the two 16-word halves
    // swapped on odd rows so that the two blocks of a warp hit different banks.
    cluster_wait_relaxed();                                  // (1)
    {
        const uint32_t sw = 16 * (B & 1);
        const uint32_t at0 = smem_addr(xt + B * 32 + (e ^ sw)), at1 = smem_addr(xt + B * 32 + ((e + 16) ^ sw));
#pragma unroll
        for (int k = 0; k < 16; ++k) st_cluster(map_to_rank((k & 1) ? at1 : at0, k >> 1), v[k]);
    }
    cluster_arrive();                                        // (2)
    const int c = tid & 31, g = tid >> 5;
    uint32_t* dst = out + rm.out_row(blockIdx.y) * kN16 + rank * 32 + c;
    const uint32_t ninv = m.n_inv, ninv_s = m.n_inv_s, wl = m.w_last, wl_s = m.w_last_s;
    cluster_wait();                                          // (2): also orders s_tw and frees cbuf
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = xt[(16 * g + k) * 32 + (c ^ (16 * (k & 1)))];
    // global stages 8..11 on rows 16g + k
    gs16(v, q, TW_MUL(s_tw[(16 + g) * (8 >> s) + gi]));
#pragma unroll
    for (int k = 0; k < 16; ++k) cbuf[(16 * g + k) * 32 + c] = v[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = cbuf[(g + 16 * k) * 32 + c];
    // global stages 12..14 on rows g + 16k, then the last stage with N^-1
    gs16<3>(v, q, TW_MUL(s_tw[(8 >> s) + gi]));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t x = v[j], y = v[j + 8];
        const uint32_t total = csub(x + y, q);
        const uint32_t diff = x - y + q;
        dst[(g + 16 * j) * 256] = shoup_mul(total, ninv, ninv_s, q);
        dst[(g + 16 * (j + 8)) * 256] = shoup_mul(diff, wl, wl_s, q);
    }
}

// ---------------------------------------------------------------------------------
// N <= 2^15: the whole limb lives in one CTA's shared memory (N * 4 B <= 128 KiB), so
// the transform is ONE launch: radix-4 steps (two stages per barrier) on the
// shared copy, same butterflies and twiddle slots as _run_stages.  Serves
// BASELINE config 1 (N = 2^13) and the small parameter sets of the tests.
// ---------------------------------------------------------------------------------
template <bool INV>
__global__ void __launch_bounds__(1024, 1)
ntt_small_kernel(const uint32_t* in, uint32_t* out, const int32_t* __restrict__ row_slot,
                 const ModSlot* __restrict__ slots, RowMap rm, uint32_t n, uint32_t lg) {
    extern __shared__ uint32_t sm[];
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    const ModSlot& m = slots[row_slot[blockIdx.x]];
    const uint32_t q = m.q;
    const uint2* __restrict__ tw = INV ? m.inv : m.fwd;
    pdl_trigger();
    const uint32_t* src = in + rm.in_row(blockIdx.x) * n;
    uint32_t* dst = out + rm.out_row(blockIdx.x) * n;
    pdl_wait();
    if (n >= 4) {
        for (uint32_t i = tid; i < n / 4; i += nt)
            reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
        for (uint32_t i = tid; i < n; i += nt) sm[i] = src[i];
    }
    __syncthreads();
    if (!INV) {
        // Cooley-Tukey, values kept in [0, 2q)
        uint32_t s = 0;
        while (s < lg) {
            if (s + 2 <= lg) {
                const uint32_t lh = lg - s - 2, h = 1u << lh;           // h = quarter of the stage-s group
                for (uint32_t b = tid; b < n / 4; b += nt) {
                    const uint32_t g = b >> lh, j = b & (h - 1);
                    const uint32_t i0 = (g << (lh + 2)) + j;
                    uint32_t a = sm[i0], bb = sm[i0 + h], c = sm[i0 + 2 * h], d = sm[i0 + 3 * h];
                    const uint2 w1 = tw[(1u << s) + g];
                    const uint2 w2 = tw[(2u << s) + 2 * g], w3 = tw[(2u << s) + 2 * g + 1];
                    ct_bfly(a, c, shoup_mul(c, w1.x, w1.y, q), q);
                    ct_bfly(bb, d, shoup_mul(d, w1.x, w1.y, q), q);
                    ct_bfly(a, bb, shoup_mul(bb, w2.x, w2.y, q), q);
                    ct_bfly(c, d, shoup_mul(d, w3.x, w3.y, q), q);
                    sm[i0] = a; sm[i0 + h] = bb; sm[i0 + 2 * h] = c; sm[i0 + 3 * h] = d;
                }
                s += 2;
            } else {
                const uint32_t lt = lg - s - 1, t = 1u << lt;
                for (uint32_t b = tid; b < n / 2; b += nt) {
                    const uint32_t g = b >> lt, j = b & (t - 1);
                    const uint32_t i0 = (g << (lt + 1)) + j;
                    uint32_t x = sm[i0], y = sm[i0 + t];
                    const uint2 w = tw[(1u << s) + g];
                    ct_bfly(x, y, shoup_mul(y, w.x, w.y, q), q);
                    sm[i0] = x; sm[i0 + t] = y;
                }
                s += 1;
            }
            __syncthreads();
        }
        if (n >= 4) {
            for (uint32_t i = tid; i < n / 4; i += nt) {
                uint4 v = reinterpret_cast<const uint4*>(sm)[i];
                v.x = csub(v.x, q); v.y = csub(v.y, q); v.z = csub(v.z, q); v.w = csub(v.w, q);
                reinterpret_cast<uint4*>(dst)[i] = v;
            }
        } else {
            for (uint32_t i = tid; i < n; i += nt) dst[i] = csub(sm[i], q);
        }
        return;
    }
    // Gentleman-Sande, canonical values; the last stage carries N^-1 (transform.py:243-246)
    uint32_t s = 0;
    while (s + 1 < lg) {
        if (s + 3 <= lg) {
            const uint32_t t = 1u << s;
            const uint32_t g1 = n >> (s + 1), g2 = n >> (s + 2);
            for (uint32_t b = tid; b < n / 4; b += nt) {
                const uint32_t G = b >> s, j = b & (t - 1);
                const uint32_t i0 = (G << (s + 2)) + j;
                const uint32_t a = sm[i0], bb = sm[i0 + t], c = sm[i0 + 2 * t], d = sm[i0 + 3 * t];
                const uint2 w0 = tw[g1 + 2 * G], w1 = tw[g1 + 2 * G + 1], w2 = tw[g2 + G];
                const uint32_t a1 = csub(a + bb, q), b1 = shoup_mul(a - bb + q, w0.x, w0.y, q);
                const uint32_t c1 = csub(c + d, q), d1 = shoup_mul(c - d + q, w1.x, w1.y, q);
                sm[i0] = csub(a1 + c1, q);
                sm[i0 + 2 * t] = shoup_mul(a1 - c1 + q, w2.x, w2.y, q);
                sm[i0 + t] = csub(b1 + d1, q);
                sm[i0 + 3 * t] = shoup_mul(b1 - d1 + q, w2.x, w2.y, q);
            }
            s += 2;
        } else {
            const uint32_t t = 1u << s, g1 = n >> (s + 1);
            for (uint32_t b = tid; b < n / 2; b += nt) {
                const uint32_t g = b >> s, j = b & (t - 1);
                const uint32_t i0 = (g << (s + 1)) + j;
                const uint32_t x = sm[i0], y = sm[i0 + t];
                const uint2 w = tw[g1 + g];
                sm[i0] = csub(x + y, q);
                sm[i0 + t] = shoup_mul(x - y + q, w.x, w.y, q);
            }
            s += 1;
        }
        __syncthreads();
    }
    {
        const uint32_t half = n >> 1;
        const uint32_t ninv = m.n_inv, ninv_s = m.n_inv_s, wl = m.w_last, wl_s = m.w_last_s;
        for (uint32_t j = tid; j < half; j += nt) {
            const uint32_t x = sm[j], y = sm[j + half];
            dst[j] = shoup_mul(csub(x + y, q), ninv, ninv_s, q);
            dst[j + half] = shoup_mul(x - y + q, wl, wl_s, q);
        }
    }
}

constexpr uint32_t kSmallMaxN = 32768;

// ---------------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------------
static int launch_generic(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                          const ModSlot* slots, RowMap rm, int rows, uint32_t n, int inverse,
                          uint32_t s_lo, uint32_t s_hi, cudaStream_t st) {
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    if (s_lo >= s_hi) {
        if (rm.in || rm.out) {
            set_last_error("empty stage range with a row map is not supported");
            return CKKS_ERR_ARG;
        }
        if (in != out)
            CK(cudaMemcpyAsync(out, in, sizeof(uint32_t) * (size_t)rows * n, cudaMemcpyDeviceToDevice, st));
        return CKKS_OK;
    }
    const uint32_t half = n >> 1;
    const uint32_t threads = half < 256 ? (half < 32 ? 32 : half) : 256;
    // gridDim.y is capped at 65535: walk tall stacks (e.g. exhaustive small-ring tests) in slabs
    for (int r0 = 0; r0 < rows; r0 += 65535) {
        const int cnt = rows - r0 < 65535 ? rows - r0 : 65535;
        dim3 grid((half + threads - 1) / threads, cnt);
        const RowMap rm_first{rm.in ? rm.in + r0 : nullptr, rm.out ? rm.out + r0 : nullptr};
        const RowMap rm_rest{rm_first.out, rm_first.out};
        const size_t off_in = rm.in ? 0 : (size_t)r0 * n, off_out = rm.out ? 0 : (size_t)r0 * n;
        for (uint32_t s = s_lo; s < s_hi; ++s) {
            const bool first = s == s_lo;
            // one radix-2 stage per launch: the transform's 2 * R * N * 4 bytes spread over its stages
            ProfScope ps("ntt_generic_stage", st, 8.0 * cnt * n / (double)(s_hi - s_lo));
            ntt_stage_generic<<<grid, threads, 0, st>>>(first ? in + off_in : out + off_out,
                                                        out + off_out, row_slot + r0, slots,
                                                        first ? rm_first : rm_rest, n, lg, s, inverse);
        }
    }
    CK(cudaGetLastError());
    return CKKS_OK;
}

static int launch_small(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                        const ModSlot* slots, RowMap rm, int rows, uint32_t n, uint32_t lg,
                        int inverse, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        CK(cudaFuncSetAttribute(ntt_small_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmallMaxN * 4)));
        CK(cudaFuncSetAttribute(ntt_small_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kSmallMaxN * 4)));
        attr_set = true;
    }
    const uint32_t quads = n / 4;
    const uint32_t threads = quads < 32 ? 32 : (quads > 1024 ? 1024 : quads);
    ProfScope ps(inverse ? "ntt_small_inv" : "ntt_small_fwd", st, 8.0 * rows * n);
    if (inverse) CK(launch_pdl(ntt_small_kernel<true>, dim3(rows), dim3(threads), (size_t)n * 4, st, in, out, row_slot, slots, rm, n, lg));
    else CK(launch_pdl(ntt_small_kernel<false>, dim3(rows), dim3(threads), (size_t)n * 4, st, in, out, row_slot, slots, rm, n, lg));
    return CKKS_OK;
}

bool ntt_can_fuse_moddown(uint32_t n) { return n == (uint32_t)kN16; }

// Which N = 2^16 launches take the single-pass cluster kernels: those of at most
// CKKS_NTT_CLUSTER_MAX_ROWS limbs (0: none, the two-kernel path everywhere).
static int g_cluster_max_rows = -1, g_cluster_occ = -1;      // -1: not decided yet (environment, then default)
static int cluster_max_rows() {
    if (g_cluster_max_rows < 0) {
        const char* s = getenv("CKKS_NTT_CLUSTER_MAX_ROWS");
        g_cluster_max_rows = s ? atoi(s) : kClusterDefaultMaxRows;
        if (g_cluster_max_rows < 0) g_cluster_max_rows = 0;
    }
    return g_cluster_max_rows;
}
static int cluster_occ() {
    if (g_cluster_occ < 0) {
        const char* s = getenv("CKKS_NTT_CLUSTER_OCC");
        g_cluster_occ = (s && atoi(s) == 3) ? 3 : 2;
    }
    return g_cluster_occ;
}
void ntt_policy(int max_rows, int occ, int* max_rows_now, int* occ_now) {
    if (max_rows >= 0) g_cluster_max_rows = max_rows;
    if (occ == 2 || occ == 3) g_cluster_occ = occ;
    if (max_rows_now) *max_rows_now = cluster_max_rows();
    if (occ_now) *occ_now = cluster_occ();
}
static int cluster_attrs() {
    static bool done = false;
    if (done) return CKKS_OK;
    const int bytes = (int)kClusterSmem;
    CK(cudaFuncSetAttribute(ntt16_fwd_cluster<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_fwd_cluster<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_fwd_cluster<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_fwd_cluster<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_inv_cluster<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_inv_cluster<false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_inv_cluster<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    CK(cudaFuncSetAttribute(ntt16_inv_cluster<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = true;
    return CKKS_OK;
}

int ntt_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot, const ModSlot* slots,
               RowMap rm, int rows, uint32_t n, int inverse, cudaStream_t st,
               const ModDownEpilogueArgs* epi, const uint32_t* mul_in) {
    if (rows <= 0) return CKKS_OK;
    if (mul_in && (!inverse || n != (uint32_t)kN16)) {
        set_last_error("product-on-load needs an inverse N = 2^16 transform");
        return CKKS_ERR_ARG;
    }
    const int epi_unit = epi ? (epi->halves == 1 ? 1 : 2) * epi->l : 1;
    if (epi && (inverse || !ntt_can_fuse_moddown(n) || rows % epi_unit != 0 ||
                (rows != epi_unit && (epi->fold_a || epi->fold_b)))) {
        set_last_error("fused ModDown epilogue needs a forward N = 2^16 transform over (a multiple of) 2 l rows");
        return CKKS_ERR_ARG;
    }
    if (n == (uint32_t)kN16 && rows <= cluster_max_rows()) {
        // single-pass transform, one cluster of eight CTAs per limb: 2 * R * N * 4 bytes in ONE launch
        CKS(cluster_attrs());
        const dim3 grid(kClusterCtas, rows), block(kClusterThreads);
        const bool occ3 = cluster_occ() == 3;
        if (!inverse) {
            if (epi) {
                ProfScope ps("ntt16_fwd_cluster_moddown", st, 4.0 * rows * kN16 * (epi->fold_b ? 3.5 : 3.0));
                if (occ3) CK(launch_pdl(ntt16_fwd_cluster<true, 3>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, *epi));
                else CK(launch_pdl(ntt16_fwd_cluster<true, 2>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, *epi));
            } else {
                ProfScope ps("ntt16_fwd_cluster", st, 8.0 * rows * kN16);
                if (occ3) CK(launch_pdl(ntt16_fwd_cluster<false, 3>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, ModDownEpilogueArgs{}));
                else CK(launch_pdl(ntt16_fwd_cluster<false, 2>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, ModDownEpilogueArgs{}));
            }
        } else {
            ProfScope ps("ntt16_inv_cluster", st, (mul_in ? 12.0 : 8.0) * rows * kN16);
            if (mul_in) {
                if (occ3) CK(launch_pdl(ntt16_inv_cluster<true, 3>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, mul_in));
                else CK(launch_pdl(ntt16_inv_cluster<true, 2>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, mul_in));
            } else {
                if (occ3) CK(launch_pdl(ntt16_inv_cluster<false, 3>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, (const uint32_t*)nullptr));
                else CK(launch_pdl(ntt16_inv_cluster<false, 2>, grid, block, kClusterSmem, st, in, out, row_slot, slots, rm, (const uint32_t*)nullptr));
            }
        }
        CK(cudaGetLastError());
        return CKKS_OK;
    }
    if (n == (uint32_t)kN16) {
        constexpr int COLS = 16;
        dim3 g_str(256 / COLS, rows), g_con(16, rows);
        const RowMap rm2{rm.out, rm.out};
        if (!inverse) {
            // algorithmic bytes: 2 * R * N * 4 per TRANSFORM; the first kernel of the pair is
            // charged the transform's read, the second its write (what passes between them is the
            // implementation's own traffic)
            { ProfScope ps("ntt16_fwd_strided", st, 4.0 * rows * kN16);
              CK(launch_pdl(ntt16_fwd_strided<COLS>, g_str, dim3(16 * COLS), 0, st, in, out, row_slot, slots, rm)); }
            if (epi) {
                // instead of the transform's write: reads x_Q (+ fold on half the rows), writes the result
                ProfScope ps("ntt16_fwd_contig_moddown", st, 4.0 * rows * kN16 * (epi->fold_b ? 2.5 : 2.0));
                CK(launch_pdl(ntt16_fwd_contig<true>, g_con, dim3(256), 0, st, out, out, row_slot, slots, rm2, *epi));
            } else {
                ProfScope ps("ntt16_fwd_contig", st, 4.0 * rows * kN16);
                CK(launch_pdl(ntt16_fwd_contig<false>, g_con, dim3(256), 0, st, out, out, row_slot, slots, rm2, ModDownEpilogueArgs{}));
            }
        } else {
            { ProfScope ps("ntt16_inv_contig", st, (mul_in ? 8.0 : 4.0) * rows * kN16);
              if (mul_in) CK(launch_pdl(ntt16_inv_contig<true>, g_con, dim3(256), 0, st, in, out, row_slot, slots, rm, mul_in));
              else CK(launch_pdl(ntt16_inv_contig<false>, g_con, dim3(256), 0, st, in, out, row_slot, slots, rm, (const uint32_t*)nullptr)); }
            { ProfScope ps("ntt16_inv_strided", st, 4.0 * rows * kN16);
              CK(launch_pdl(ntt16_inv_strided<COLS>, g_str, dim3(16 * COLS), 0, st, out, out, row_slot, slots, rm2)); }
        }
        CK(cudaGetLastError());
        return CKKS_OK;
    }
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    if (n <= kSmallMaxN) return launch_small(in, out, row_slot, slots, rm, rows, n, lg, inverse, st);
    return launch_generic(in, out, row_slot, slots, rm, rows, n, inverse, 0, lg, st);
}

int ntt_stages_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                      const ModSlot* slots, int rows, uint32_t n, int inverse, uint32_t s_lo,
                      uint32_t s_hi, cudaStream_t st) {
    const RowMap rm{nullptr, nullptr};
    if (rows <= 0) return CKKS_OK;
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    if (n == (uint32_t)kN16 && s_hi - s_lo == 8 && (s_lo == 0 || s_lo == 8)) {
        // the engine's own phase split: run the matching fast kernel alone
        constexpr int COLS = 16;
        dim3 g_str(256 / COLS, rows), g_con(16, rows);
        const bool strided = inverse ? (s_lo == 8) : (s_lo == 0);
        if (!inverse && strided) ntt16_fwd_strided<COLS><<<g_str, 16 * COLS, 0, st>>>(in, out, row_slot, slots, rm);
        if (!inverse && !strided) ntt16_fwd_contig<false><<<g_con, 256, 0, st>>>(in, out, row_slot, slots, rm, ModDownEpilogueArgs{});
        if (inverse && !strided) ntt16_inv_contig<false><<<g_con, 256, 0, st>>>(in, out, row_slot, slots, rm, nullptr);
        if (inverse && strided) ntt16_inv_strided<COLS><<<g_str, 16 * COLS, 0, st>>>(in, out, row_slot, slots, rm);
        CK(cudaGetLastError());
        return CKKS_OK;
    }
    return launch_generic(in, out, row_slot, slots, rm, rows, n, inverse, s_lo, s_hi, st);
}

}  // namespace ckks
