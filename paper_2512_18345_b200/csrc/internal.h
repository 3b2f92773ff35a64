// internal.h -- declarations shared between the translation units of
// libckks_b200.so (not part of the C ABI; see include/ckks_b200.h for that).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace ckks {

struct ModSlot;

void set_last_error(const char* fmt, ...);

#define CK(call)                                                                        \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::ckks::set_last_error("%s failed at %s:%d: %s", #call, __FILE__, __LINE__, \
                                   cudaGetErrorString(_e));                             \
            return CKKS_ERR_CUDA;                                                       \
        }                                                                               \
    } while (0)

#define CKS(call)                         \
    do {                                  \
        int _s = (call);                  \
        if (_s != CKKS_OK) return _s;     \
    } while (0)

// Launch with programmatic stream serialisation (see common.cuh pdl_*): the launch latency
// and the table-loading prologue of kernel N+1 overlap the tail of kernel N; inside CUDA
// graphs this becomes a programmatic dependency edge.  CKKS_PDL=0 falls back to ordinary
// launches (the kernels' pdl_* calls are then no-ops).
bool pdl_enabled();
// `pdl` false: an ordinary, fully stream-ordered launch (for a kernel that reads, before its
// pdl_wait(), memory its stream predecessor may have written -- see InnerProductArgs::ordered).
template <class... P, class... A>
inline cudaError_t launch_opt_pdl(bool pdl, void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, P(args)...);
}
template <class... P, class... A>
inline cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
    return launch_opt_pdl(true, kernel, grid, block, smem, st, static_cast<A&&>(args)...);
}

// Logical row r of a launch lives at physical row in[r] of the source buffer
// and out[r] of the destination (identity when null).  Lets the key-switch
// pipeline transform scattered limbs (e.g. the converted rows of a raised
// digit) in place without an assembly copy (reference keyswitch.py:283-293).
struct RowMap {
    const int32_t* in;
    const int32_t* out;
    __host__ __device__ size_t in_row(unsigned r) const { return in ? (size_t)in[r] : (size_t)r; }
    __host__ __device__ size_t out_row(unsigned r) const { return out ? (size_t)out[r] : (size_t)r; }
};

// Optional per-kernel timing (api.cu): when enabled through ckks_profile_enable
// every launch site below is bracketed by CUDA events on its own stream.
struct ProfScope {
    cudaStream_t st;
    bool live;
    // alg_bytes: algorithmic bytes of the launch (operand limbs read + written once,
    // tables and twiddles excluded: SURVEY 8d / Appendix A convention)
    // alg_flops: floating-point operations of a tensor-core launch (2 per FMA), 0 otherwise
    ProfScope(const char* name, cudaStream_t stream, double alg_bytes = 0.0, double alg_flops = 0.0);
    ~ProfScope();
};

// ntt.cu
struct ModDownEpilogueArgs;
// epi != null (forward, N = 2^16, rows = 2 l only): the last kernel applies the ModDown
// epilogue to its registers and stores the key-switch result instead of the transform.
int ntt_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot, const ModSlot* slots,
               RowMap rm, int rows, uint32_t n, int inverse, cudaStream_t st,
               const ModDownEpilogueArgs* epi = nullptr, const uint32_t* mul_in = nullptr);
// mul_in != null (inverse, N = 2^16 only): the input is in (.) mul_in, multiplied on load.
bool ntt_can_fuse_moddown(uint32_t n);
// Which N = 2^16 launches take the single-pass cluster kernels (at most max_rows limbs; 0: none)
// and at how many CTAs per SM (2 or 3); negative / other values leave a setting as it is.
void ntt_policy(int max_rows, int occ, int* max_rows_now, int* occ_now);
int ntt_stages_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                      const ModSlot* slots, int rows, uint32_t n, int inverse, uint32_t s_lo,
                      uint32_t s_hi, cudaStream_t st);

// elementwise.cu
int elementwise_launch(const uint32_t* a, const uint32_t* b, uint32_t* out, const int32_t* row_slot,
                       const ModSlot* slots, int rows, size_t cols, int kind, cudaStream_t st);
int automorphism_eval_launch(const uint32_t* in, uint32_t* out, int rows, uint32_t n, uint32_t k,
                             cudaStream_t st);
int automorphism_coeff_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                              const ModSlot* slots, int rows, uint32_t n, uint32_t k, cudaStream_t st);

int lift2_centered_launch(const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                          const ModSlot* slots, int32_t slot0, int32_t slot1, uint32_t inv,
                          int rows, size_t n, cudaStream_t st);
int pmult_acc_launch(const uint32_t* x, const uint32_t* p, uint32_t* acc, const int32_t* row_slot,
                     const ModSlot* slots, int rows, size_t cols, int first, cudaStream_t st);

constexpr int kMaxTerms = 16;
struct FusedTerms {
    int count;
    const uint32_t* x[kMaxTerms];   // ciphertexts [2][rows][n]
    const uint32_t* xb[kMaxTerms];  // b half of term t when it does not sit at x[t] + rows * n (a mod-dropped
                                    // ciphertext keeps its halves a full level apart); null: adjacent
    const uint32_t* p[kMaxTerms];   // plaintexts [rows][n] or null
};
int fused_terms_launch(const FusedTerms& terms, uint32_t* out, const int32_t* row_slot,
                       const ModSlot* slots, int rows, size_t cols, cudaStream_t st);
constexpr int kMaxGiants = 8;
struct FusedMulti {
    int nb, ng;
    const uint32_t* x[kMaxTerms];               // baby-step ciphertexts [2][rows][n]
    const uint32_t* p[kMaxGiants][kMaxTerms];   // plaintext diagonal of (giant g, baby b), or `zero`
    const uint32_t* zero;                       // [rows][n] zeros standing in for absent diagonals
    uint32_t* out[kMaxGiants];                  // [2][rows][n] each
};
int fused_terms_multi_launch(const FusedMulti& a, const int32_t* row_slot, const ModSlot* slots,
                             int rows, size_t cols, cudaStream_t st);
int tensor_launch(const uint32_t* xa, const uint32_t* xb, const uint32_t* ya, const uint32_t* yb,
                  uint32_t* out, const int32_t* row_slot, const ModSlot* slots, int rows, size_t cols,
                  cudaStream_t st);

// bconv.cu
// Device image of one conversion table (reference baseconv.py:37-54).
struct BconvDev {
    int l_in, l_out;
    uint32_t all31;             // sources < 2^31 and targets in (2^30, 2^31): bconv_fast applies
    const int32_t* in_slot;     // [l_in]   context slots of the source basis
    const int32_t* out_slot;    // [l_out]  context slots of the target basis
    const uint32_t* inv_qhat;   // [l_in]   (Q*/Q_j)^-1 mod Q_j
    const uint32_t* inv_qhat_s; // [l_in]   Shoup companions
    const uint32_t* t_mont;     // [l_out][l_in]  (Q*/Q_j) * 2^32 mod P_i  (Montgomery form)
    const uint32_t* t_plain;    // [l_out][l_in]  (Q*/Q_j) mod P_i
    // ready-made operands of the FP64 tensor-core kernel (one load level in its prologue):
    int kp;                     // l_in rounded up to a multiple of 4
    const double* t_f64;        // [l_out rounded up to 8][kp]  t_mont as doubles, zero padded
    const double* t_f64k;       // [l_out rounded up to 8][2 kp]  {t_mont | t_mont * 2^16 mod P_i}: the two 16-bit
                                //   halves of y stacked along K, so ONE accumulator holds the whole sum (< 2^52)
    const uint4* om;            // [l_out rounded up to 8]  {P_i, -P_i^-1.. (qinv), i, 2^48 mod P_i}
    const uint4* inc;           // [kp]  {Q_k, inv_qhat, shoup(inv_qhat), 0}; padding {3, 0, 0, 0}
};

struct BconvJob {
    BconvDev tab;
    const uint32_t* in;         // source limb k at in + k * in_stride
    size_t in_stride;
    uint32_t* out;              // target limb i at out + out_row[i] * out_stride
    size_t out_stride;
    const int32_t* out_row;     // null: identity
};

constexpr int kMaxBconvJobs = 8;
struct BconvJobs {
    int count;
    BconvJob job[kMaxBconvJobs];
};

int bconv_launch_jobs(const BconvJobs& jobs, const ModSlot* slots, size_t cols, cudaStream_t st);
int bconv_launch(const BconvDev& tab, const ModSlot* slots, const uint32_t* in, size_t in_stride,
                 uint32_t* out, size_t out_stride, size_t cols, cudaStream_t st);

// keyswitch.cu
struct InnerProductArgs {
    const uint32_t* carry;      // ct.a rows (null: every row comes from `raised`)
    const uint32_t* raised;     // [beta][ext][n]
    const uint32_t* evk;        // [beta_total][2][evk_ext][n]
    uint32_t* acc_a;            // row r - row_lo at acc_a + (r - row_lo) * n
    uint32_t* acc_b;
    const int32_t* ext_slot;    // [ext] context slot of every active extended-basis row
    const int32_t* evk_row;     // [ext] row of the key matrix holding active row r
    int l, alpha, beta, ext, evk_ext;
    int row_lo, row_hi;
    uint32_t n;
    uint32_t galois, lg;        // galois != 0: read digit columns through X -> X^galois (hoisting)
    int accumulate;             // add into acc instead of overwriting it
    // The kernel issues its switching-key loads BEFORE griddepcontrol.wait (the key is static
    // inside a pipeline whose earlier kernels are ModUp stages).  When the inner product is the
    // FIRST kernel of an ABI call its stream predecessor is unknown -- it may be the kernel that
    // wrote the key (key generation, the stacking copy of SwitchingKey.matrix()) -- so those entry
    // points set `ordered` and the kernel is launched without the programmatic attribute.
    int ordered;
    // tensor mode (all four non-null): the operands of an HMult; the kernel forms d2 = xa*ya (the
    // carried digit rows), d1 = xa*yb + ya*xb and d0 = xb*yb itself and lifts P*d1, P*d0 into
    // the accumulators, so no tensor pass and no (d0, d1, d2) buffers exist.  carry, lift_a and
    // lift_b are ignored.
    const uint32_t *tx_a, *tx_b, *ty_a, *ty_b;
    const uint32_t* lift_a;     // non-null: add (P mod q_i) * lift_a to the Q rows of acc_a (no automorphism)
    const uint32_t* lift_b;     // non-null: add (P mod q_i) * sigma(lift_b) to the Q rows of acc_b, i.e.
    const uint32_t* pmod;       //   fold the rotated ciphertext's b-part into the Q||P accumulator
    const uint32_t* pmod_s;     //   (double hoisting: no ModDown per rotation)
    const uint32_t* lift_qp;    // non-null: [ext][n], already over Q||P: add sigma(lift_qp) to EVERY row of acc_b as
                                //   it is (the b half of a giant step's inner sum never leaves Q||P)
};
int inner_product_launch(const InnerProductArgs& a, const ModSlot* slots, cudaStream_t st);

struct ModDownEpilogueArgs {
    const uint32_t* xq_a;       // [l][n] accumulator Q part (a half)
    const uint32_t* xq_b;
    const uint32_t* conv;       // [2][l][n]  NTT(BConv_{P->Q}(INTT(x_P)))
    const uint32_t* fold_a;     // polynomial to add into the a half (null: none)
    const uint32_t* fold_b;     // ct.b to add into the b half (null: none)
    uint32_t* out_a;
    uint32_t* out_b;
    const int32_t* q_slot;      // [l]
    const uint32_t* pinv;       // [l]  P^-1 mod q_i
    const uint32_t* pinv_s;     // [l]  Shoup companions
    int l;
    uint32_t n;
    uint32_t galois, lg;        // galois != 0: fold_b is read through X -> X^galois
    // batched ModDown (several accumulators in one launch, rows = batch * 2 l): element g reads
    // xq_* + g * xq_stride and writes out_* + g * out_stride (words); 0 for a single ModDown
    size_t xq_stride, out_stride;
    // 1: every element is ONE polynomial (a halves only: rows = batch * l, element g reads
    // xq_a + g * xq_stride and writes out_a + g * out_stride); 0 or 2: both halves
    int halves;
};
// All baby steps of a double-hoisted BSGS linear transform fused with all giant-step inner
// sums: for every baby step b the Q||P accumulator u_b of the rotation sigma_{k_b} of the
// ciphertext (inner product of the raised digits with key b, P * sigma(ct_b) lifted in; k_b = 0:
// the ciphertext itself on the Q rows) is formed in registers and immediately multiplied into
// out[g] += p[g][b] (.) u_b.  The u_b are never written.
constexpr int kMaxBsgsBatch = 2;
struct BsgsInnerArgs {
    // `batch` independent ciphertexts at the same level go through the same keys and diagonals in
    // ONE launch (CTAs of 128 * batch threads: every key / plaintext slice is fetched into shared
    // memory once and multiplied into each ciphertext's sums: the L2-aware multi-polynomial grouping
    // of the paper, PAPER.md "scheduling", done inside the kernel).  Element c uses raised[c],
    // ct_a[c], ct_b[c] and out[c][*].
    int batch;
    const uint32_t* raised[kMaxBsgsBatch];      // [beta][ext][n]
    const uint32_t* ct_a[kMaxBsgsBatch];        // [l][n]
    const uint32_t* ct_b[kMaxBsgsBatch];        // [l][n]
    const int32_t* ext_slot;                    // [ext]
    const int32_t* evk_row;                     // [ext]
    const uint32_t* pmod;                       // [l]  P mod q_i
    const uint32_t* pmod_s;
    int l, alpha, beta, ext, evk_ext;
    uint32_t n, lg;
    int nb, ng;
    uint32_t k[kMaxTerms];                      // automorphism index of baby step b (0: none)
    const uint32_t* evk[kMaxTerms];             // its switching key [beta_total][2][evk_ext][n] (unused for k = 0)
    const uint32_t* p[kMaxGiants][kMaxTerms];   // plaintext diagonal over Q||P, or `zero`
    uint32_t* out[kMaxBsgsBatch][kMaxGiants];   // [2][ext][n] each
};
int bsgs_inner_launch(const BsgsInnerArgs& a, const ModSlot* slots, cudaStream_t st);

int moddown_epilogue_launch(const ModDownEpilogueArgs& a, const ModSlot* slots, cudaStream_t st);
int lane_reduce_launch(uint32_t* acc0, size_t lane_stride_words, int lanes, const int32_t* ext_slot,
                       const ModSlot* slots, int ext, size_t n, cudaStream_t st,
                       const uint32_t* lift_a = nullptr, const uint32_t* lift_b = nullptr,
                       const uint32_t* pmod = nullptr, const uint32_t* pmod_s = nullptr, int l = 0,
                       const uint32_t* raw = nullptr);

}  // namespace ckks
