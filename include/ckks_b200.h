/*
 * ckks_b200.h -- C ABI of libckks_b200.so, the sm_100a engine behind the
 * rnscope-compatible Python package paper_2512_18345_b200.
 *
 * The reference (rnscope 0.1.0, /root/reference/pkg/src/rnscope) has no FFI
 * layer: its boundary is the Python module API of rns / transform / baseconv /
 * keyswitch.  Each entry point below names the reference routine whose work it
 * takes over (paths relative to that package).  The Python side performs the
 * reference's structural checks and raises its exception types; these
 * functions only validate what they need to launch safely.
 *
 * Conventions
 *  - all `const uint32_t*` / `uint32_t*` data arguments are DEVICE pointers to
 *    row-major limb matrices of 32-bit residues in [0, q) (the RNSV wire
 *    layout, vectors.py:3-14); `row_slot` arguments are DEVICE int32 arrays of
 *    modulus slots (one per row) obtained from ckks_modulus_register;
 *  - `stream` is a cudaStream_t passed as void* (0 = default stream); every
 *    call only enqueues work and is CUDA-graph capturable unless noted;
 *  - functions return CKKS_OK (0) or a CKKS_ERR_* code; ckks_last_error()
 *    returns a thread-local description of the last failure;
 *  - nothing here falls back to the CPU: without a CUDA device
 *    ckks_ctx_create fails with CKKS_ERR_CUDA.
 */
#ifndef CKKS_B200_H
#define CKKS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKKS_OK 0
#define CKKS_ERR_ARG 1
#define CKKS_ERR_CUDA 2
#define CKKS_ERR_UNSUPPORTED 3
#define CKKS_ERR_STATE 4

typedef struct ckks_ctx ckks_ctx;

/* ABI version of this header; bumped on any signature change. */
int ckks_abi_version(void);
const char* ckks_last_error(void);

/* Per-kernel device timing, the engine's analogue of the reference's op
 * counters (instrument.py:11-32).  While enabled, every kernel launch is
 * bracketed by CUDA events on its stream (do not enable during graph
 * capture).  ckks_profile_read synchronises and writes one line
 * "<kernel> <launches> <total_ms> <algorithmic_bytes> <tensor_flops>" per kernel class
 * into buf (bytes: operand limbs read + written once, tables excluded; tensor_flops: FP64
 * tensor-core operations of the base-conversion contraction, 2 per FMA, 0 for other kernels). */
int ckks_profile_enable(int on);
int ckks_profile_read(char* buf, size_t cap);

/* ---- context ---------------------------------------------------------------- */

/* One context per process per GPU: owns the modulus slots, twiddle tables,
 * conversion tables and key-switch plans (the reference keeps these in
 * functools.lru_cache: transform.py:121-123,184-186, keyswitch.py:221-223). */
int ckks_ctx_create(int device, ckks_ctx** out);
void ckks_ctx_destroy(ckks_ctx* ctx);

/* Workspace lanes.  Key-switch plans work out of one device arena; with
 * `lanes` > 1 the arena is replicated so that calls issued on different
 * streams (independent rotations, the two EvalMod branches of a bootstrap) can
 * run concurrently: select a lane, then enqueue on that lane's stream.
 * ckks_set_lanes reallocates (not capturable); ckks_select_lane is host state
 * only. */
int ckks_set_lanes(ckks_ctx* ctx, int lanes);
int ckks_select_lane(ckks_ctx* ctx, int lane);

/* The arena is reallocated (it MOVES) when the lane count changes or a plan needs more words
 * than any plan before it.  A CUDA graph captured earlier holds raw pointers into the old
 * arena: ckks_arena_generation returns a counter that changes with every reallocation, so a
 * holder of such a graph can refuse to replay it (Bootstrapper.capture does);
 * ckks_arena_reserve grows the arena to `words_per_lane` up front (e.g. the full-level plan's
 * size) so that later plans never move it. */
int ckks_arena_generation(ckks_ctx* ctx, uint64_t* generation);
int ckks_arena_reserve(ckks_ctx* ctx, size_t words_per_lane);

/* Register modulus q for ring degree n with psi a primitive 2n-th root of
 * unity mod q (already squared down to order 2n, transform.py:88-96) and build
 * its device twiddle tables: fwd[t] = psi^bitrev(t), inv[t] = psi^-bitrev(t),
 * N^-1 (transform.py:76-118, Modulus rns.py:85-113).  n = 0 or psi = 0
 * registers the modulus for element-wise / conversion use only.  Idempotent
 * per (q, n, psi).  Not capturable (allocates, copies). */
int ckks_modulus_register(ckks_ctx* ctx, uint32_t q, uint32_t n, uint32_t psi, int32_t* slot);

/* A slot whose twiddle tables are the CALLER's (n words each, residues mod q, schedule order of
 * transform.py:43-49) instead of powers of a root: `ntt(limb, m, table)` in the reference uses
 * whatever table it is handed (transform.py:253-276), which is what its twiddle-corruption
 * negative control relies on (verify.py:51-57).  Always a fresh slot.  Not capturable. */
int ckks_modulus_register_tables(ckks_ctx* ctx, uint32_t q, uint32_t n, const uint32_t* fwd,
                                 const uint32_t* inv, uint32_t n_inv, int32_t* slot);

/* Copy a slot's tables back to the host (TwiddleTable.fwd/inv/n_inv,
 * transform.py:43-64); fwd/inv hold n words each. */
int ckks_modulus_tables(ckks_ctx* ctx, int32_t slot, uint32_t* fwd, uint32_t* inv, uint32_t* n_inv);

/* ---- transforms: transform.py:203-323 --------------------------------------- */

/* ntt_polynomial (transform.py:279-287): whole transform of `rows` limbs of
 * degree n; row r uses modulus slot row_slot[r].  in may equal out. */
int ckks_ntt(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, const int32_t* row_slot, int rows,
             uint32_t n, int inverse, void* stream);

/* Scheduling of the N = 2^16 transform (no effect on results): launches of at most
 * cluster_max_rows limbs run as ONE kernel over thread-block clusters of eight CTAs per
 * limb (the intermediate of transform.py:290-323's two phases is exchanged through
 * distributed shared memory), taller ones as the two-kernel split; 0 = two kernels
 * everywhere.  ctas_per_sm is 2 or 3.  Negative arguments leave a setting unchanged; the
 * current values are returned through the pointers (may be null).  Process-wide host state:
 * set it before capturing graphs.  Environment defaults: CKKS_NTT_CLUSTER_MAX_ROWS,
 * CKKS_NTT_CLUSTER_OCC. */
int ckks_ntt_policy(int cluster_max_rows, int ctas_per_sm, int* cluster_max_rows_now, int* ctas_per_sm_now);

/* _run_stages over [stage_lo, stage_hi) (transform.py:203-250), the building
 * block of ntt_two_phase (transform.py:290-323). */
int ckks_ntt_stages(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                    int rows, uint32_t n, int inverse, uint32_t stage_lo, uint32_t stage_hi,
                    void* stream);

/* ---- element-wise and automorphism: rns.py:243-320 -------------------------- */

/* poly_elementwise (rns.py:243-258); kind 0 add, 1 sub, 2 mul. */
int ckks_elementwise(ckks_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out,
                     const int32_t* row_slot, int rows, size_t cols, int kind, void* stream);

/* automorphism, evaluation domain (rns.py:313-320): out[:, t] = in[:, perm_k(t)]. */
int ckks_automorphism_eval(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, int rows, uint32_t n,
                           uint32_t k, void* stream);

/* automorphism, coefficient domain (rns.py:306-312). */
int ckks_automorphism_coeff(ckks_ctx* ctx, const uint32_t* in, uint32_t* out,
                            const int32_t* row_slot, int rows, uint32_t n, uint32_t k, void* stream);

/* ---- CKKS additions without a reference counterpart -------------- */

/* Exact centred lift (bootstrapping ModRaise): in [2][n] coefficient-domain
 * limbs over slots slot0, slot1 -> out [rows][n], out[i] = centred value mod
 * modulus row_slot[i]. */
int ckks_lift2_centered(ckks_ctx* ctx, const uint32_t* in, int32_t slot0, int32_t slot1,
                        uint32_t* out, const int32_t* row_slot, int rows, size_t n, void* stream);

/* acc (+)= x (.) p on both halves of a ciphertext: x, acc [2][rows][cols], p
 * [rows][cols]; first != 0 overwrites acc (the PMult-accumulate inner loop of
 * the BSGS linear transforms; each product is poly_elementwise "mul"). */
int ckks_pmult_accumulate(ckks_ctx* ctx, const uint32_t* x, const uint32_t* p, uint32_t* acc,
                          const int32_t* row_slot, int rows, size_t cols, int first, void* stream);

/* out = sum_t x[t] (.) p[t] over `count` <= 16 (ciphertext, plaintext) pairs in one
 * pass; x[t] are DEVICE pointers to [2][rows][cols] ciphertexts, p[t] to
 * [rows][cols] plaintexts or NULL (term = x[t]); the pointer arrays themselves
 * are HOST arrays.  The inner sum of a BSGS linear transform (each product is
 * poly_elementwise "mul", each sum "add", rns.py:243-258). */
int ckks_fused_terms(ckks_ctx* ctx, int count, const uint32_t* const* x, const uint32_t* const* p,
                     uint32_t* out, const int32_t* row_slot, int rows, size_t cols, void* stream);
/* The same with the two halves of every term given separately: xa[t], xb[t] are [rows][cols] each
 * (xb NULL, or xb[t] NULL: the b half follows the a half as in ckks_fused_terms).  For ciphertexts
 * whose halves are not adjacent -- a ciphertext with limbs dropped keeps them a full level apart --
 * so that no gathering copy is needed. */
int ckks_fused_terms_halves(ckks_ctx* ctx, int count, const uint32_t* const* xa, const uint32_t* const* xb,
                            const uint32_t* const* p, uint32_t* out, const int32_t* row_slot, int rows,
                            size_t cols, void* stream);

/* All giant-step inner sums of a BSGS linear transform in one pass:
 * out[g] = sum_b x[b] (.) p[g * nb + b] for g < ng <= 8, b < nb <= 16; x[b] and out[g]
 * are [2][rows][cols] ciphertexts, p[.] [rows][cols] plaintexts or NULL (diagonal
 * absent: `zero`, a DEVICE [rows][cols] matrix of zeros, is read in its place, so it may
 * be NULL only when no p[.] is); pointer arrays are HOST arrays.  Same arithmetic as ng
 * calls of ckks_fused_terms, but every x[b] is read once. */
int ckks_fused_terms_multi(ckks_ctx* ctx, int nb, int ng, const uint32_t* const* x,
                           const uint32_t* const* p, const uint32_t* zero, uint32_t* const* out,
                           const int32_t* row_slot, int rows, size_t cols, void* stream);

/* Tensor product (front of HMult): x, y [2][rows][cols] -> out [3][rows][cols] =
 * (b1*b2, a1*b2 + a2*b1, a1*a2). */
int ckks_tensor(ckks_ctx* ctx, const uint32_t* x, const uint32_t* y, uint32_t* out,
                const int32_t* row_slot, int rows, size_t cols, void* stream);
/* Same with the four halves as separate [rows][cols] matrices (ciphertexts whose a and b parts
 * are views of larger allocations, e.g. after dropping limbs). */
int ckks_tensor_halves(ckks_ctx* ctx, const uint32_t* xa, const uint32_t* xb, const uint32_t* ya,
                       const uint32_t* yb, uint32_t* out, const int32_t* row_slot, int rows, size_t cols,
                       void* stream);

/* ---- base conversion: baseconv.py:57-151 ------------------------------------ */

/* build_bconv_table (baseconv.py:57-85) for source slots -> target slots.
 * Not capturable. */
int ckks_bconv_table_create(ckks_ctx* ctx, const int32_t* in_slot, int l_in, const int32_t* out_slot,
                            int l_out, int32_t* table);

/* Host copy of T (l_out x l_in) and inv_qhat (l_in), BConvTable.t / .inv_qhat. */
int ckks_bconv_table_read(ckks_ctx* ctx, int32_t table, uint32_t* t, uint32_t* inv_qhat);

/* convert (baseconv.py:147-151): in [l_in][cols] -> out [l_out][cols], exact
 * non-centred fast base conversion. */
int ckks_bconv(ckks_ctx* ctx, int32_t table, const uint32_t* in, uint32_t* out, size_t cols,
               void* stream);

/* ---- key switching: keyswitch.py:186-453 ------------------------------------ */

/* _KsTables (keyswitch.py:186-218) plus device workspace for one shape:
 * `l` active Q limbs (slots q_slot[l]) in digits of `alpha`, P basis p_slot[alpha].
 * Key matrices passed to this plan are [beta][2][evk_ext][n]; active Q row i is
 * key row i and P row j is key row evk_p_off + j (evk_ext = L + alpha and
 * evk_p_off = L for a key generated at the full level L).  Not capturable. */
int ckks_ks_plan_create(ckks_ctx* ctx, uint32_t n, int l, int alpha, const int32_t* q_slot,
                        const int32_t* p_slot, int evk_ext, int evk_p_off, int32_t* plan);

/* ModDown-only plan: the stage-3 machinery for `l` Q limbs and an arbitrary
 * `alpha`-limb P basis, without raise tables or stage-1/2 workspace.  With
 * alpha = 1 and P = {q_last} ckks_ks_stage3 on this plan is RNS rescaling
 * (drop the last limb): (x_i - NTT(INTT(x_last) mod q_i)) * q_last^-1, the
 * composition of reference primitives recorded as the rescale oracle
 * (SURVEY 8c).  Not capturable. */
int ckks_moddown_plan_create(ckks_ctx* ctx, uint32_t n, int l, int alpha, const int32_t* q_slot,
                             const int32_t* p_slot, int32_t* plan);

/* keyswitch_stage1 (keyswitch.py:297-315): a [l][n] evaluation domain ->
 * raised [beta][l+alpha][n], digit limbs carried through. */
int ckks_ks_stage1(ckks_ctx* ctx, int32_t plan, const uint32_t* a, uint32_t* raised, void* stream);

/* keyswitch_stage2 / stage2_p_part / stage2_q_part (keyswitch.py:318-384) on
 * extended-basis rows [row_lo, row_hi): acc_a, acc_b are [row_hi-row_lo][n]. */
int ckks_ks_stage2(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, const uint32_t* evk,
                   int row_lo, int row_hi, uint32_t* acc_a, uint32_t* acc_b, void* stream);

/* keyswitch_stage3 (keyswitch.py:422-441): ModDown of both accumulator halves. */
int ckks_ks_stage3(ckks_ctx* ctx, int32_t plan, const uint32_t* q_a, const uint32_t* q_b,
                   const uint32_t* p_a, const uint32_t* p_b, uint32_t* out_a, uint32_t* out_b,
                   void* stream);

/* keyswitch (keyswitch.py:444-453): all three stages on the plan's workspace;
 * out_b = delta.b + ct_b when ct_b is non-null.  evk as for the plan. */
int ckks_keyswitch(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* ct_b,
                   const uint32_t* evk, uint32_t* out_a, uint32_t* out_b, void* stream);

/* Hoisted rotation: with `raised` = ckks_ks_stage1(ct_a) computed once, returns the key
 * switch of the rotated ciphertext (sigma_k(ct_a), sigma_k(ct_b)) for the Galois key
 * `evk` of X -> X^k: the raised digits and ct_b are read through the automorphism
 * inside the inner-product and ModDown kernels, so each further rotation of the same
 * ciphertext skips the whole of stage 1.  sigma_k commutes with ModUp only up to a
 * multiple of the digit modulus, so the limbs differ from
 * ckks_keyswitch(automorphism(ct)) by key-switch noise, not bit for bit (the reference
 * has no hoisting, PAPER.md:616 notes Cheddar does). */
int ckks_ks_hoisted(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, uint32_t k,
                    const uint32_t* evk, const uint32_t* ct_b, uint32_t* out_a, uint32_t* out_b,
                    void* stream);

/* Double hoisting: like ckks_ks_hoisted but WITHOUT the ModDown -- writes the Q||P
 * accumulator of the rotated ciphertext, out_qp [2][l+alpha][n], with (P mod q_i) *
 * sigma_k(ct_b) already folded into the Q rows of its b half, so that
 * ModDown(out_qp) = hrot(ct).  Sums of plaintext products of several such accumulators
 * (the inner sums of a BSGS linear transform, plaintexts encoded over Q||P) then need one
 * ModDown per sum (ckks_ks_stage3 on the pieces of the buffer) instead of one per
 * rotation.  k = 0 applies no automorphism. */
int ckks_ks_hoisted_raw(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, uint32_t k,
                        const uint32_t* evk, const uint32_t* ct_b, uint32_t* out_qp, void* stream);

/* Relinearisation fused with the rescale that follows it: key switch of d2 under evk,
 * plus (d1, d0) lifted into the Q||P accumulator, then ONE ModDown by P * (the k dropped
 * limbs) through `md_plan` = ckks_moddown_plan_create(l - k limbs, P' = dropped limbs then
 * P).  Output [l-k][n] per half.  Equals rescale(relinearize(d0, d1, d2)) up to the rounding
 * of one division instead of two. */
int ckks_ks_relin_rescale(ckks_ctx* ctx, int32_t ks_plan, int32_t md_plan, const uint32_t* d2,
                          const uint32_t* d1, const uint32_t* d0, const uint32_t* evk,
                          uint32_t* out_a, uint32_t* out_b, void* stream);

/* Key switches whose results are summed (giant steps of a BSGS linear transform) can
 * share one ModDown: ckks_ks_accumulate runs stages 1-2 of keyswitch.py:444-453 for
 * (ct_a, evk) and adds the Q||P accumulator into the current lane's workspace (first !=
 * 0 overwrites); ckks_ks_finish sums the accumulators of lanes [c, c + lanes_used), c the
 * currently selected lane (0 unless the caller itself runs inside a lane group), runs
 * stage 3 once on lane c and adds fold_a / fold_b (may be NULL) to the two halves.
 * ModDown is linear up to its rounding, so this equals the sum of separate key switches
 * up to key-switch noise. */
int ckks_ks_accumulate(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* evk,
                       int first, void* stream);
/* HMult + relinearise + rescale from the four operand halves (each [l][n]) without a tensor
 * pass or (d0, d1, d2) buffers: values equal ckks_tensor + ckks_ks_relin_rescale bit for bit.
 * (add_a, add_b), both or neither NULL: a ciphertext over the l - k output limbs added to the
 * result inside the ModDown epilogue (poly_elementwise "add" without its own pass).
 * N = 2^16 only (CKKS_ERR_UNSUPPORTED otherwise: use the two-call route). */
int ckks_hmult_relin_rescale(ckks_ctx* ctx, int32_t ks_plan, int32_t md_plan, const uint32_t* xa,
                             const uint32_t* xb, const uint32_t* ya, const uint32_t* yb,
                             const uint32_t* evk, const uint32_t* add_a, const uint32_t* add_b,
                             uint32_t* out_a, uint32_t* out_b, void* stream);

/* Baby steps and inner sums of a double-hoisted BSGS linear transform in one pass:
 * out[g] = sum_b p[g * nb + b] (.) u_b, u_b = the ckks_ks_hoisted_raw accumulator of rotation
 * k[b] with key evk[b] (k[b] = 0: the ciphertext (ct_a, ct_b) on the Q rows, zero on the P
 * rows; evk[b] ignored).  The u_b are formed in registers and never written; values equal
 * ckks_ks_hoisted_raw + ckks_fused_terms_multi bit for bit.  p[.] are [l+alpha][n] plaintexts
 * over Q||P (NULL: `zero` is read), out[g] are [2][l+alpha][n]; nb <= 16, ng <= 8; k, evk, p,
 * out are HOST arrays. */
int ckks_bsgs_inner(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, const uint32_t* ct_a,
                    const uint32_t* ct_b, int nb, const uint32_t* k, const uint32_t* const* evk, int ng,
                    const uint32_t* const* p, const uint32_t* zero, uint32_t* const* out, void* stream);

/* The same for `batch` (<= 2) independent ciphertexts at the same level, through the same keys and
 * diagonals, in ONE launch: each key / plaintext slice is staged in shared memory once and
 * multiplied into every ciphertext's sums (the reference batches key switches in a loop,
 * keyswitch.py:456-459; the paper's L2-aware multi-polynomial grouping is this sharing).  raised,
 * ct_a, ct_b: host arrays of `batch` device pointers; out: host array [batch][ng], element c's
 * results at out[c * ng + g].  Values equal `batch` calls of ckks_bsgs_inner bit for bit.
 * Needs n % 256 == 0 (CKKS_ERR_UNSUPPORTED otherwise: call ckks_bsgs_inner per ciphertext). */
int ckks_bsgs_inner_batch(ckks_ctx* ctx, int32_t plan, int batch, const uint32_t* const* raised,
                          const uint32_t* const* ct_a, const uint32_t* const* ct_b, int nb, const uint32_t* k,
                          const uint32_t* const* evk, int ng, const uint32_t* const* p, const uint32_t* zero,
                          uint32_t* const* out, void* stream);

/* ckks_ks_stage3 (ModDown) of `count` <= 4 accumulators in one set of launches: qp is
 * [count][2][l + alpha][n] (Q rows then P rows per half), out [count][2][l][n]; element g uses the
 * workspace of lane (current + g), so count lanes from the current one must exist and be idle.
 * Same limbs as count calls of ckks_ks_stage3.  N = 2^16 only. */
int ckks_ks_stage3_batch(ckks_ctx* ctx, int32_t plan, int count, const uint32_t* qp, uint32_t* out,
                         void* stream);

/* ckks_ks_accumulate for the rotation sigma_k of (ct_a, ct_b) without materialising it: the
 * automorphism is a gather inside the inner product and P * sigma_k(ct_b) is lifted into the b
 * accumulator (no separate automorphism pass, no separate sum of the b parts). */
int ckks_ks_accumulate_rot(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* ct_b,
                           uint32_t k, const uint32_t* evk, int first, void* stream);

/* The a halves only of `count` Q||P accumulators (same layout as ckks_ks_stage3_batch's input,
 * b halves skipped); out is [count][l][n]. */
int ckks_ks_stage3_batch_a(ckks_ctx* ctx, int32_t plan, int count, const uint32_t* qp, uint32_t* out,
                           void* stream);

/* ckks_ks_accumulate_rot for an inner sum kept over Q||P: ct_a = ModDown of its a half ([l][n]),
 * b_qp its b half as it is ([l + alpha][n]), added to the b accumulator through X -> X^k without
 * a ModDown or a lift (composition of keyswitch.py:318-332 and rns.py:295-320). */
int ckks_ks_accumulate_rot_qp(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* b_qp,
                              uint32_t k, const uint32_t* evk, int first, void* stream);
int ckks_ks_finish(ckks_ctx* ctx, int32_t plan, int lanes_used, const uint32_t* fold_a,
                   const uint32_t* fold_b, uint32_t* out_a, uint32_t* out_b, void* stream);

/* ckks_ks_finish and the rescale that follows it as one division: (fold_a, fold_b) joins the
 * accumulator times P, raw_qp (may be NULL; a [2][l + alpha][n] accumulator already over Q||P)
 * as it is, and `md_plan` = ckks_moddown_plan_create(Q_{l-k}, {q_{l-k}..q_{l-1}} U P)
 * divides by P * q_{l-1} ... q_{l-k}; outputs have l - k rows (same value as ks_finish +
 * rescale up to the rounding of the division). */
int ckks_ks_finish_rescale(ckks_ctx* ctx, int32_t plan, int32_t md_plan, int lanes_used,
                           const uint32_t* fold_a, const uint32_t* fold_b, const uint32_t* raw_qp,
                           uint32_t* out_a, uint32_t* out_b, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CKKS_B200_H */
