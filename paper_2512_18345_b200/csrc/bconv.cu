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
// Column-parallel: one thread per column keeps the l_in pre-scaled residues in
// registers and walks the output limbs; the table row is a broadcast read from
// shared memory, stores are fully coalesced.  Several conversions (the beta
// digits of stage 1, the two polynomials of stage 3) run as one launch.
#include "common.cuh"
#include "internal.h"

namespace ckks {

struct OutMod {
    uint32_t q, qinv, fast, pad;
};

template <int LIN>
__global__ void __launch_bounds__(256)
bconv_kernel(BconvJobs jobs, const ModSlot* __restrict__ slots, size_t cols) {
    extern __shared__ uint32_t smem[];
    const BconvJob& job = jobs.job[blockIdx.y];
    const int l_in = job.tab.l_in, l_out = job.tab.l_out;
    // shared: table rows padded to LIN words, then per-output modulus constants
    uint32_t* s_t = smem;                                   // [l_out][LIN]
    OutMod* s_mod = reinterpret_cast<OutMod*>(smem + (size_t)l_out * LIN);
    for (int idx = threadIdx.x; idx < l_out * LIN; idx += blockDim.x) {
        const int i = idx / LIN, k = idx - i * LIN;
        uint32_t v = 0;
        if (k < l_in) {
            const bool fast = slots[job.tab.out_slot[i]].fast;
            v = fast ? job.tab.t_mont[i * l_in + k] : job.tab.t_plain[i * l_in + k];
        }
        s_t[idx] = v;
    }
    for (int i = threadIdx.x; i < l_out; i += blockDim.x) {
        const ModSlot& m = slots[job.tab.out_slot[i]];
        s_mod[i] = OutMod{m.q, m.qinv, m.fast, 0};
    }
    __syncthreads();

    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    uint32_t y[LIN];
#pragma unroll
    for (int k = 0; k < LIN; ++k) {
        y[k] = 0;
        if (k < l_in) {
            const ModSlot& m = slots[job.tab.in_slot[k]];
            const uint32_t a = job.in[(size_t)k * job.in_stride + c];
            y[k] = m.q >> 31 ? (uint32_t)((uint64_t)a * job.tab.inv_qhat[k] % m.q)
                             : shoup_mul(a, job.tab.inv_qhat[k], job.tab.inv_qhat_s[k], m.q);
        }
    }
    for (int i = 0; i < l_out; ++i) {
        const OutMod om = s_mod[i];
        const uint32_t* trow = s_t + (size_t)i * LIN;
        uint32_t r = 0;
        if (om.fast && job.tab.all31) {
#pragma unroll
            for (int k0 = 0; k0 < LIN; k0 += 4) {
                uint64_t s = 0;
#pragma unroll
                for (int k = k0; k < k0 + 4 && k < LIN; ++k) s += (uint64_t)trow[k] * y[k];
                uint32_t hi = (uint32_t)(s >> 32);
                hi = min(hi, hi - 2u * om.q);
                hi = csub(hi, om.q);
                r = add_mod(r, redc((uint32_t)s, hi, om.q, om.qinv), om.q);
            }
        } else {
            // small or 32-bit target modulus (unit tests): exact 128-bit-free fold
            uint64_t acc = 0;
#pragma unroll
            for (int k = 0; k < LIN; ++k) acc = (acc + (uint64_t)trow[k] * y[k] % om.q) % om.q;
            r = (uint32_t)acc;
        }
        const size_t orow = job.out_row ? (size_t)job.out_row[i] : (size_t)i;
        job.out[orow * job.out_stride + c] = r;
    }
}

int bconv_launch_jobs(const BconvJobs& jobs, const ModSlot* slots, size_t cols, cudaStream_t st) {
    if (jobs.count <= 0 || cols == 0) return CKKS_OK;
    const int l_in = jobs.job[0].tab.l_in;
    int l_out_max = 0;
    for (int j = 0; j < jobs.count; ++j) {
        if (jobs.job[j].tab.l_in != l_in) {
            set_last_error("stacked conversions must share l_in");
            return CKKS_ERR_ARG;
        }
        if (jobs.job[j].tab.l_out > l_out_max) l_out_max = jobs.job[j].tab.l_out;
    }
    dim3 grid((unsigned)((cols + 255) / 256), jobs.count);
#define BCONV_GO(LIN)                                                                      \
    do {                                                                                   \
        size_t sm = (size_t)l_out_max * LIN * 4 + (size_t)l_out_max * sizeof(OutMod);      \
        if (sm > 48 * 1024)                                                                \
            CK(cudaFuncSetAttribute(bconv_kernel<LIN>,                                     \
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));\
        ProfScope ps("bconv", st);                                                      \
        bconv_kernel<LIN><<<grid, 256, sm, st>>>(jobs, slots, cols);                       \
    } while (0)
    if (l_in <= 1) BCONV_GO(1);
    else if (l_in <= 2) BCONV_GO(2);
    else if (l_in <= 4) BCONV_GO(4);
    else if (l_in <= 8) BCONV_GO(8);
    else if (l_in <= 12) BCONV_GO(12);
    else if (l_in <= 16) BCONV_GO(16);
    else if (l_in <= 24) BCONV_GO(24);
    else if (l_in <= 32) BCONV_GO(32);
    else {
        set_last_error("base conversion from %d limbs is not supported (max 32)", l_in);
        return CKKS_ERR_UNSUPPORTED;
    }
#undef BCONV_GO
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
