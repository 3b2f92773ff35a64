/*
 * oracle/ckks_oracle.c -- CPU restatement of the rnscope hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_2512_18345_b200/ may import,
 * link or execute this file; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it, as the checker or
 * as the timed CPU baseline.
 *
 * Every function follows one routine of the reference package (paths are
 * relative to /root/reference/pkg/src/rnscope/) and is pinned against that
 * routine's real outputs through tests/golden/ (see tests/golden/make_golden.py
 * and tests/test_oracle_golden.py).  Arithmetic is deliberately the plain
 * "(a op b) % q" of the NumPy code -- no Montgomery, no Shoup, no laziness --
 * so that it is an independent statement of the maths the CUDA path must hit.
 *
 * Residues are uint32 on the wire (vectors.py:3-14); all products are formed
 * in uint64 / unsigned __int128 so every step is exact.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* Worker threads of the parallel loops below.  Launchers such as torchrun export
 * OMP_NUM_THREADS=1 to every rank; the CPU baseline is meant to use every host thread it is
 * given, so bench.py sets the count explicitly.  Returns the count in effect (1 without OpenMP). */
#ifdef _OPENMP
#include <omp.h>
int orc_set_threads(int n) {
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
}
#else
int orc_set_threads(int n) { (void)n; return 1; }
#endif

typedef struct {
    uint32_t q;
    uint32_t n_inv;
    uint32_t *fwd;   /* fwd[t] = psi^bitrev(t)      transform.py:99  */
    uint32_t *inv;   /* inv[t] = psi^-bitrev(t)     transform.py:100 */
} orc_modulus;

typedef struct {
    uint32_t n;
    uint32_t lg;
    int n_mod;
    orc_modulus *mod;
} orc_ctx;

static inline uint32_t mulmod(uint32_t a, uint32_t b, uint32_t q) {
    return (uint32_t)(((uint64_t)a * b) % q);
}

static uint32_t powmod(uint32_t base, uint64_t e, uint32_t q) {
    uint64_t acc = 1 % q, b = base % q;
    while (e) {
        if (e & 1) acc = acc * b % q;
        b = b * b % q;
        e >>= 1;
    }
    return (uint32_t)acc;
}

static uint32_t bitrev(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* transform.py:76-118 build_twiddle_table (tables only; seeds are derived on
 * demand by orc_otf_twiddle).  psi has order 2*mod_n; when mod_n > n it is
 * squared down (transform.py:90-96). */
orc_ctx *orc_create(uint32_t n, int n_mod, const uint64_t *q, const uint64_t *psi,
                    const uint64_t *mod_n) {
    orc_ctx *c = (orc_ctx *)calloc(1, sizeof(orc_ctx));
    c->n = n;
    c->lg = 0;
    while ((1u << c->lg) < n) c->lg++;
    c->n_mod = n_mod;
    c->mod = (orc_modulus *)calloc((size_t)n_mod, sizeof(orc_modulus));
    for (int i = 0; i < n_mod; ++i) {
        orc_modulus *m = &c->mod[i];
        m->q = (uint32_t)q[i];
        m->fwd = (uint32_t *)malloc(sizeof(uint32_t) * n);
        m->inv = (uint32_t *)malloc(sizeof(uint32_t) * n);
        if (n >= 2 && psi[i] != 0 && (m->q - 1) % (2ull * n) == 0) {
            uint32_t root = (uint32_t)psi[i];
            uint64_t order = 2 * mod_n[i];
            while (order > 2ull * n) { root = mulmod(root, root, m->q); order >>= 1; }
            uint32_t root_inv = powmod(root, (uint64_t)m->q - 2, m->q);
            uint32_t *pw = (uint32_t *)malloc(sizeof(uint32_t) * n);
            uint32_t *pwi = (uint32_t *)malloc(sizeof(uint32_t) * n);
            uint32_t acc = 1 % m->q, acci = 1 % m->q;
            for (uint32_t k = 0; k < n; ++k) {
                pw[k] = acc; pwi[k] = acci;
                acc = mulmod(acc, root, m->q);
                acci = mulmod(acci, root_inv, m->q);
            }
            for (uint32_t t = 0; t < n; ++t) {
                uint32_t r = bitrev(t, c->lg);
                m->fwd[t] = pw[r];
                m->inv[t] = pwi[r];
            }
            free(pw); free(pwi);
            m->n_inv = powmod(n % m->q, (uint64_t)m->q - 2, m->q);
        } else {
            memset(m->fwd, 0, sizeof(uint32_t) * n);
            memset(m->inv, 0, sizeof(uint32_t) * n);
            m->n_inv = 0;
        }
    }
    return c;
}

void orc_destroy(orc_ctx *c) {
    if (!c) return;
    for (int i = 0; i < c->n_mod; ++i) { free(c->mod[i].fwd); free(c->mod[i].inv); }
    free(c->mod);
    free(c);
}

void orc_get_twiddles(const orc_ctx *c, int mod, uint32_t *fwd, uint32_t *inv, uint32_t *n_inv) {
    memcpy(fwd, c->mod[mod].fwd, sizeof(uint32_t) * c->n);
    memcpy(inv, c->mod[mod].inv, sizeof(uint32_t) * c->n);
    *n_inv = c->mod[mod].n_inv;
}

/* transform.py:203-250 _run_stages over stages [s_lo, s_hi) of one row. */
static void run_stages(uint32_t *a, const orc_modulus *m, uint32_t n, uint32_t lg,
                       int inverse, uint32_t s_lo, uint32_t s_hi) {
    const uint64_t q = m->q;
    for (uint32_t s = s_lo; s < s_hi; ++s) {
        if (!inverse) {
            uint32_t groups = 1u << s, t = n >> (s + 1);
            for (uint32_t g = 0; g < groups; ++g) {
                uint64_t w = m->fwd[groups + g];
                uint32_t *x = a + (size_t)g * 2 * t, *y = x + t;
                for (uint32_t j = 0; j < t; ++j) {
                    uint64_t v = (uint64_t)y[j] * w % q;
                    uint64_t hi = ((uint64_t)x[j] + q - v) % q;
                    x[j] = (uint32_t)(((uint64_t)x[j] + v) % q);
                    y[j] = (uint32_t)hi;
                }
            }
        } else {
            uint32_t groups = n >> (s + 1), t = 1u << s;
            int last = (s == lg - 1);
            for (uint32_t g = 0; g < groups; ++g) {
                uint64_t w = m->inv[groups + g];
                if (last) w = w * m->n_inv % q;            /* transform.py:243-246 */
                uint32_t *x = a + (size_t)g * 2 * t, *y = x + t;
                for (uint32_t j = 0; j < t; ++j) {
                    uint64_t total = ((uint64_t)x[j] + y[j]) % q;
                    uint64_t diff = ((uint64_t)x[j] + q - y[j]) % q;
                    if (last) total = total * m->n_inv % q;
                    x[j] = (uint32_t)total;
                    y[j] = (uint32_t)(diff * w % q);
                }
            }
        }
    }
}

/* transform.py:279-287 ntt_polynomial: rows may carry distinct moduli. In place. */
void orc_ntt(const orc_ctx *c, uint32_t *data, const int32_t *row_mod, int rows, int inverse) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < rows; ++r)
        run_stages(data + (size_t)r * c->n, &c->mod[row_mod[r]], c->n, c->lg, inverse, 0, c->lg);
}

/* transform.py:290-323 ntt_two_phase, table twiddles; the inter-phase copy is
 * the explicit buffer handoff of :320. */
void orc_ntt_two_phase(const orc_ctx *c, uint32_t *data, const int32_t *row_mod, int rows,
                       int inverse, uint32_t n1) {
    uint32_t h1 = 0;
    while ((1u << h1) < n1) h1++;
    uint32_t split = inverse ? c->lg - h1 : h1;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < rows; ++r) {
        uint32_t *row = data + (size_t)r * c->n;
        run_stages(row, &c->mod[row_mod[r]], c->n, c->lg, inverse, 0, split);
        uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * c->n);
        memcpy(tmp, row, sizeof(uint32_t) * c->n);
        run_stages(tmp, &c->mod[row_mod[r]], c->n, c->lg, inverse, split, c->lg);
        memcpy(row, tmp, sizeof(uint32_t) * c->n);
        free(tmp);
    }
}

/* transform.py:126-151 generate_twiddle: slot (stage*block + index) from the
 * two O(sqrt N) seed arrays, one modular multiplication. */
uint32_t orc_otf_twiddle(const orc_ctx *c, int mod, uint32_t slot, int inverse) {
    const orc_modulus *m = &c->mod[mod];
    uint32_t lg = c->lg, h = lg / 2, block = 1u << h;
    const uint32_t *tab = inverse ? m->inv : m->fwd;
    /* psi (or psi^-1) = table slot whose exponent is 1: bitrev(t)=1 -> t = n/2 */
    uint32_t psi = lg ? tab[c->n >> 1] : 1;
    uint32_t hi_step = h ? powmod(psi, 1ull << (lg - h), m->q) : psi;
    uint32_t lo_idx = slot & (block - 1), hi_idx = slot >> h;
    uint32_t lo_rev = h ? bitrev(lo_idx, h) : 0;
    uint32_t hi_rev = (lg - h) ? bitrev(hi_idx, lg - h) : 0;
    uint32_t lo = powmod(hi_step, lo_rev, m->q);   /* fwd_seed_lo[lo_rev]  :114 */
    uint32_t hi = powmod(psi, hi_rev, m->q);       /* fwd_seed_hi[hi_rev]  :115 */
    return mulmod(lo, hi, m->q);
}

/* rns.py:243-258 poly_elementwise. kind: 0 add, 1 sub, 2 mul. */
void orc_elementwise(const orc_ctx *c, const uint32_t *a, const uint32_t *b, uint32_t *out,
                     const int32_t *row_mod, int rows, int kind) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; ++r) {
        const uint64_t q = c->mod[row_mod[r]].q;
        const uint32_t *x = a + (size_t)r * c->n, *y = b + (size_t)r * c->n;
        uint32_t *o = out + (size_t)r * c->n;
        for (uint32_t j = 0; j < c->n; ++j) {
            uint64_t v;
            if (kind == 0) v = ((uint64_t)x[j] + y[j]) % q;
            else if (kind == 1) v = ((uint64_t)x[j] + q - y[j]) % q;
            else v = (uint64_t)x[j] * y[j] % q;
            o[j] = (uint32_t)v;
        }
    }
}

/* rns.py:261-265, :306-312 coefficient-domain automorphism X -> X^k. */
void orc_automorphism_coeff(const orc_ctx *c, const uint32_t *in, uint32_t *out,
                            const int32_t *row_mod, int rows, uint32_t k) {
    const uint32_t n = c->n;
    for (int r = 0; r < rows; ++r) {
        const uint32_t q = c->mod[row_mod[r]].q;
        const uint32_t *src = in + (size_t)r * n;
        uint32_t *dst = out + (size_t)r * n;
        for (uint32_t i = 0; i < n; ++i) {
            uint64_t j = ((uint64_t)i * k) % (2ull * n);
            uint32_t v = src[i];
            if (j >= n) v = (uint32_t)(((uint64_t)q - v) % q);
            dst[j % n] = v;
        }
    }
}

/* rns.py:268-292 _evaluation_permutation: probe -> INTT -> coefficient
 * automorphism -> NTT, read off the source column of every output column.
 * Returns 0 on success, 1 if the probe did not come back as a permutation. */
int orc_eval_permutation(const orc_ctx *c, int probe_mod, uint32_t k, int32_t *perm) {
    const uint32_t n = c->n;
    uint32_t *buf = (uint32_t *)malloc(sizeof(uint32_t) * n);
    uint32_t *shuf = (uint32_t *)malloc(sizeof(uint32_t) * n);
    int32_t rm = probe_mod;
    for (uint32_t i = 0; i < n; ++i) buf[i] = i;
    run_stages(buf, &c->mod[probe_mod], n, c->lg, 1, 0, c->lg);
    orc_automorphism_coeff(c, buf, shuf, &rm, 1, k);
    run_stages(shuf, &c->mod[probe_mod], n, c->lg, 0, 0, c->lg);
    unsigned char *seen = (unsigned char *)calloc(n, 1);
    int bad = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (shuf[i] >= n || seen[shuf[i]]) { bad = 1; break; }
        seen[shuf[i]] = 1;
        perm[i] = (int32_t)shuf[i];
    }
    free(seen); free(buf); free(shuf);
    return bad;
}

/* rns.py:313-320 evaluation-domain automorphism: column gather. */
void orc_gather_columns(const orc_ctx *c, const uint32_t *in, uint32_t *out, int rows,
                        const int32_t *perm) {
    const uint32_t n = c->n;
    for (int r = 0; r < rows; ++r)
        for (uint32_t t = 0; t < n; ++t)
            out[(size_t)r * n + t] = in[(size_t)r * n + perm[t]];
}

/* baseconv.py:57-85 build_bconv_table, with the big products folded mod p. */
static void bconv_table(const uint32_t *qs, int l_in, const uint32_t *ps, int l_out,
                        uint32_t *t /* l_out*l_in */, uint32_t *inv_qhat /* l_in */) {
    for (int j = 0; j < l_in; ++j) {
        uint64_t h = 1 % qs[j];
        for (int k = 0; k < l_in; ++k)
            if (k != j) h = h * (qs[k] % qs[j]) % qs[j];
        inv_qhat[j] = powmod((uint32_t)h, (uint64_t)qs[j] - 2, qs[j]);
        if (qs[j] == 2) inv_qhat[j] = 1;
    }
    for (int i = 0; i < l_out; ++i)
        for (int j = 0; j < l_in; ++j) {
            uint64_t h = 1 % ps[i];
            for (int k = 0; k < l_in; ++k)
                if (k != j) h = h * (qs[k] % ps[i]) % ps[i];
            t[i * l_in + j] = (uint32_t)h;
        }
}

void orc_bconv_table(const uint32_t *qs, int l_in, const uint32_t *ps, int l_out,
                     uint32_t *t, uint32_t *inv_qhat) {
    bconv_table(qs, l_in, ps, l_out, t, inv_qhat);
}

/* baseconv.py:95-151 _prescale + bconv / bconv_with_intermediate_reduction:
 * out[i] = (sum_k T[i][k] * (a[k]*inv_qhat[k] % Q_k)) % P_i, exact (the two
 * reference paths agree bit for bit, tests/test_baseconv.py:102-108), so a
 * 128-bit accumulator states both. Non-centred, no float correction. */
void orc_bconv(const uint32_t *qs, int l_in, const uint32_t *ps, int l_out,
               const uint32_t *in, uint32_t *out, size_t cols) {
    uint32_t *t = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l_in * l_out);
    uint32_t *inv = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l_in);
    bconv_table(qs, l_in, ps, l_out, t, inv);
    uint32_t *y = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l_in * cols);
#pragma omp parallel for schedule(static)
    for (int k = 0; k < l_in; ++k)
        for (size_t c = 0; c < cols; ++c)
            y[(size_t)k * cols + c] = mulmod(in[(size_t)k * cols + c], inv[k], qs[k]);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < l_out; ++i)
        for (size_t c = 0; c < cols; ++c) {
            u128 acc = 0;
            for (int k = 0; k < l_in; ++k)
                acc += (u128)t[i * l_in + k] * y[(size_t)k * cols + c];
            out[(size_t)i * cols + c] = (uint32_t)(acc % ps[i]);
        }
    free(t); free(inv); free(y);
}

/* ---- key switching, keyswitch.py:256-453 -------------------------------- */

typedef struct {
    int l, alpha, dnum;
    const int32_t *q_idx;   /* l     context modulus indices of the Q basis */
    const int32_t *p_idx;   /* alpha context modulus indices of the P basis */
} ks_shape;

static uint32_t mod_q(const orc_ctx *c, int idx) { return c->mod[idx].q; }

/* keyswitch.py:256-315 keyswitch_stage1 / _raise_group with B = beta.
 * a: [l][n] evaluation domain. raised: [dnum][l+alpha][n].
 * Generalised to levels that are not a multiple of alpha (the reference enforces
 * L = dnum * alpha, params.py:40): digit t covers rows [t*alpha, min(l, (t+1)*alpha)), so
 * the last digit may be partial; dnum = ceil(l / alpha).  At l = dnum * alpha this is the
 * reference's routine verbatim (pinned at l in {12, 24, 36, 48}, tests/golden). */
void orc_ks_stage1(const orc_ctx *c, int l, int alpha, int dnum, const int32_t *q_idx,
                   const int32_t *p_idx, const uint32_t *a, uint32_t *raised) {
    const uint32_t n = c->n;
    const int ext = l + alpha;
    /* :267-270 INTT of all digit rows (the stack is just the input rows) */
    uint32_t *coeff = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l * n);
    memcpy(coeff, a, sizeof(uint32_t) * (size_t)l * n);
    orc_ntt(c, coeff, q_idx, l, 1);
    uint32_t *conv = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)ext * n);
    uint32_t *qs = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)alpha);
    uint32_t *ps = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)ext);
    int32_t *target = (int32_t *)malloc(sizeof(int32_t) * (size_t)ext);
    for (int t = 0; t < dnum; ++t) {
        const int lo = t * alpha, hi = (lo + alpha < l) ? lo + alpha : l;
        /* :196-201 raise target = complementary Q limbs then P limbs */
        int cnt = 0;
        for (int i = 0; i < l; ++i)
            if (i < lo || i >= hi) target[cnt++] = q_idx[i];
        for (int i = 0; i < alpha; ++i) target[cnt++] = p_idx[i];
        for (int i = lo; i < hi; ++i) qs[i - lo] = mod_q(c, q_idx[i]);
        for (int i = 0; i < cnt; ++i) ps[i] = mod_q(c, target[i]);
        orc_bconv(qs, hi - lo, ps, cnt, coeff + (size_t)lo * n, conv, n);        /* :276 */
        orc_ntt(c, conv, target, cnt, 0);                                        /* :278 */
        /* :283-293 assemble: carried digit rows from the input, rest from conv */
        uint32_t *out = raised + (size_t)t * ext * n;
        int src = 0;
        for (int row = 0; row < ext; ++row) {
            if (row >= lo && row < hi)
                memcpy(out + (size_t)row * n, a + (size_t)row * n, sizeof(uint32_t) * n);
            else
                memcpy(out + (size_t)row * n, conv + (size_t)(src++) * n, sizeof(uint32_t) * n);
        }
    }
    free(coeff); free(conv); free(qs); free(ps); free(target);
}

/* keyswitch.py:318-355 _stage2_accumulate / keyswitch_stage2 on rows
 * [row_lo, row_hi) of the extended basis.
 * raised: [dnum][ext][n]; evk: [dnum][2][ext][n] (pair t: a then b);
 * acc_a, acc_b: [row_hi-row_lo][n]. */
void orc_ks_stage2(const orc_ctx *c, int l, int alpha, int dnum, const int32_t *q_idx,
                   const int32_t *p_idx, const uint32_t *raised, const uint32_t *evk,
                   int row_lo, int row_hi, uint32_t *acc_a, uint32_t *acc_b) {
    const uint32_t n = c->n;
    const int ext = l + alpha;
#pragma omp parallel for schedule(static)
    for (int row = row_lo; row < row_hi; ++row) {
        const uint64_t q = mod_q(c, row < l ? q_idx[row] : p_idx[row - l]);
        uint32_t *oa = acc_a + (size_t)(row - row_lo) * n;
        uint32_t *ob = acc_b + (size_t)(row - row_lo) * n;
        for (uint32_t j = 0; j < n; ++j) {
            uint64_t sa = 0, sb = 0;
            for (int t = 0; t < dnum; ++t) {
                uint64_t d = raised[((size_t)t * ext + row) * n + j];
                uint64_t ka = evk[(((size_t)t * 2 + 0) * ext + row) * n + j];
                uint64_t kb = evk[(((size_t)t * 2 + 1) * ext + row) * n + j];
                sa = (sa + d * ka % q) % q;   /* :329 */
                sb = (sb + d * kb % q) % q;   /* :330 */
            }
            oa[j] = (uint32_t)sa;
            ob[j] = (uint32_t)sb;
        }
    }
}

/* keyswitch.py:387-441 _moddown_group / keyswitch_stage3 for one polynomial.
 * xq: [l][n], xp: [alpha][n] evaluation domain -> out [l][n]. */
void orc_ks_moddown(const orc_ctx *c, int l, int alpha, const int32_t *q_idx,
                    const int32_t *p_idx, const uint32_t *xq, const uint32_t *xp,
                    uint32_t *out) {
    const uint32_t n = c->n;
    uint32_t *pc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)alpha * n);
    uint32_t *conv = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l * n);
    uint32_t *ps = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)alpha);
    uint32_t *qs = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)l);
    memcpy(pc, xp, sizeof(uint32_t) * (size_t)alpha * n);
    orc_ntt(c, pc, p_idx, alpha, 1);                       /* :402 */
    for (int i = 0; i < alpha; ++i) ps[i] = mod_q(c, p_idx[i]);
    for (int i = 0; i < l; ++i) qs[i] = mod_q(c, q_idx[i]);
    orc_bconv(ps, alpha, qs, l, pc, conv, n);              /* :408 */
    orc_ntt(c, conv, q_idx, l, 0);                         /* :409 */
#pragma omp parallel for schedule(static)
    for (int i = 0; i < l; ++i) {
        const uint64_t q = qs[i];
        uint64_t pprod = 1 % q;                            /* :205-208 P^-1 mod q_i */
        for (int k = 0; k < alpha; ++k) pprod = pprod * (ps[k] % q) % q;
        const uint64_t pinv = powmod((uint32_t)pprod, q - 2, (uint32_t)q);
        for (uint32_t j = 0; j < n; ++j) {
            uint64_t d = ((uint64_t)xq[(size_t)i * n + j] + q - conv[(size_t)i * n + j]) % q;
            out[(size_t)i * n + j] = (uint32_t)(d * pinv % q);   /* :416 */
        }
    }
    free(pc); free(conv); free(ps); free(qs);
}

/* keyswitch.py:444-453 keyswitch. Optional dumps (may be NULL) follow the
 * names of dump_pipeline_vectors (:462-490).
 * evk: [dnum][2][ext][n].  raised_out: [dnum][ext][n]; acc_out: [2][ext][n]
 * (a rows then b rows, each Q part then P part). */
void orc_keyswitch(const orc_ctx *c, int l, int alpha, int dnum, const int32_t *q_idx,
                   const int32_t *p_idx, const uint32_t *ct_a, const uint32_t *ct_b,
                   const uint32_t *evk, uint32_t *out_a, uint32_t *out_b,
                   uint32_t *raised_out, uint32_t *acc_out) {
    const uint32_t n = c->n;
    const int ext = l + alpha;
    uint32_t *raised = raised_out ? raised_out
                                  : (uint32_t *)malloc(sizeof(uint32_t) * (size_t)dnum * ext * n);
    uint32_t *acc = acc_out ? acc_out : (uint32_t *)malloc(sizeof(uint32_t) * 2 * (size_t)ext * n);
    uint32_t *acc_a = acc, *acc_b = acc + (size_t)ext * n;
    orc_ks_stage1(c, l, alpha, dnum, q_idx, p_idx, ct_a, raised);
    orc_ks_stage2(c, l, alpha, dnum, q_idx, p_idx, raised, evk, 0, ext, acc_a, acc_b);
    orc_ks_moddown(c, l, alpha, q_idx, p_idx, acc_a, acc_a + (size_t)l * n, out_a);
    orc_ks_moddown(c, l, alpha, q_idx, p_idx, acc_b, acc_b + (size_t)l * n, out_b);
    orc_elementwise(c, out_b, ct_b, out_b, q_idx, l, 0);   /* :452 fold ct.b */
    if (!raised_out) free(raised);
    if (!acc_out) free(acc);
}

/* ---- extensions for circuits above the reference's entry points -------------------------
 * The reference stops at keyswitch() (keyswitch.py:444-453); HRot, HMult + relinearise,
 * rescale, hoisting and bootstrapping are compositions of its primitives.  The
 * routines below restate the composed steps the CUDA engine fuses, each as plain loops over
 * the same "(a op b) % q" arithmetic, so that whole circuits can be replayed on the CPU. */

/* Register one more modulus after orc_create (tables as in orc_create).  Returns its index. */
int orc_add_modulus(orc_ctx *c, uint64_t q, uint64_t psi, uint64_t mod_n) {
    const uint32_t n = c->n;
    c->mod = (orc_modulus *)realloc(c->mod, sizeof(orc_modulus) * (size_t)(c->n_mod + 1));
    orc_modulus *m = &c->mod[c->n_mod];
    m->q = (uint32_t)q;
    m->fwd = (uint32_t *)calloc(n, sizeof(uint32_t));
    m->inv = (uint32_t *)calloc(n, sizeof(uint32_t));
    m->n_inv = 0;
    if (n >= 2 && psi != 0 && (m->q - 1) % (2ull * n) == 0) {
        uint32_t root = (uint32_t)psi;
        uint64_t order = 2 * mod_n;
        while (order > 2ull * n) { root = mulmod(root, root, m->q); order >>= 1; }
        uint32_t root_inv = powmod(root, (uint64_t)m->q - 2, m->q);
        uint32_t *pw = (uint32_t *)malloc(sizeof(uint32_t) * n);
        uint32_t *pwi = (uint32_t *)malloc(sizeof(uint32_t) * n);
        uint32_t acc = 1 % m->q, acci = 1 % m->q;
        for (uint32_t k = 0; k < n; ++k) {
            pw[k] = acc; pwi[k] = acci;
            acc = mulmod(acc, root, m->q);
            acci = mulmod(acci, root_inv, m->q);
        }
        for (uint32_t t = 0; t < n; ++t) {
            uint32_t r = bitrev(t, c->lg);
            m->fwd[t] = pw[r];
            m->inv[t] = pwi[r];
        }
        free(pw); free(pwi);
        m->n_inv = powmod(n % m->q, (uint64_t)m->q - 2, m->q);
    }
    return c->n_mod++;
}

/* transform.py:203-250 _run_stages on an explicit stage range (ntt_two_phase's halves). */
void orc_ntt_stages(const orc_ctx *c, uint32_t *data, const int32_t *row_mod, int rows,
                    int inverse, uint32_t s_lo, uint32_t s_hi) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < rows; ++r)
        run_stages(data + (size_t)r * c->n, &c->mod[row_mod[r]], c->n, c->lg, inverse, s_lo, s_hi);
}

/* keyswitch.py:318-332 _stage2_accumulate, generalised the way the engine uses it:
 *  - the ciphertext may live at l <= L limbs while the key is the full-level one: active
 *    extended-basis row r reads key row evk_row[r] of a key with evk_ext rows per polynomial;
 *  - perm != NULL: the digits are read through the evaluation-domain automorphism
 *    (rns.py:313-320 out[:, t] = in[:, perm[t]]): hoisted rotation;
 *  - lift_a / lift_b != NULL: (P mod q_i) * lift is added on the Q rows (lift_b through perm),
 *    i.e. a polynomial that takes no key switch joins the Q||P accumulator;
 *  - accumulate: add into acc instead of overwriting it.
 * raised: [beta][ext][n]; evk: [beta_total][2][evk_ext][n]; acc_a, acc_b: [ext][n]. */
void orc_inner_product(const orc_ctx *c, int l, int beta, int ext, const int32_t *ext_idx,
                       const uint32_t *raised, const uint32_t *evk, int evk_ext,
                       const int32_t *evk_row, const int32_t *perm, const uint32_t *lift_a,
                       const uint32_t *lift_b, const uint32_t *pmod, int accumulate,
                       uint32_t *acc_a, uint32_t *acc_b) {
    const uint32_t n = c->n;
#pragma omp parallel for schedule(static)
    for (int row = 0; row < ext; ++row) {
        const uint64_t q = mod_q(c, ext_idx[row]);
        const size_t er = (size_t)evk_row[row];
        uint32_t *oa = acc_a + (size_t)row * n, *ob = acc_b + (size_t)row * n;
        for (uint32_t j = 0; j < n; ++j) {
            const uint32_t src = perm ? (uint32_t)perm[j] : j;
            uint64_t sa = 0, sb = 0;
            for (int t = 0; t < beta; ++t) {
                uint64_t d = raised[((size_t)t * ext + row) * n + src];
                uint64_t ka = evk[(((size_t)t * 2 + 0) * evk_ext + er) * n + j];
                uint64_t kb = evk[(((size_t)t * 2 + 1) * evk_ext + er) * n + j];
                sa = (sa + d * ka % q) % q;
                sb = (sb + d * kb % q) % q;
            }
            if (row < l && lift_a) sa = (sa + (uint64_t)lift_a[(size_t)row * n + j] * pmod[row] % q) % q;
            if (row < l && lift_b) sb = (sb + (uint64_t)lift_b[(size_t)row * n + src] * pmod[row] % q) % q;
            if (accumulate) { sa = (sa + oa[j]) % q; sb = (sb + ob[j]) % q; }
            oa[j] = (uint32_t)sa;
            ob[j] = (uint32_t)sb;
        }
    }
}

/* acc (+)= x (.) p on both halves of a ciphertext: x, acc [2][rows][n], p [rows][n]
 * (chains of rns.py:243-258 poly_elementwise mul / add). */
void orc_pmult_acc(const orc_ctx *c, const uint32_t *x, const uint32_t *p, uint32_t *acc,
                   const int32_t *row_mod, int rows, int first) {
    const uint32_t n = c->n;
#pragma omp parallel for schedule(static)
    for (int r = 0; r < 2 * rows; ++r) {
        const int row = r % rows;
        const uint64_t q = mod_q(c, row_mod[row]);
        const uint32_t *xs = x + (size_t)r * n, *ps = p + (size_t)row * n;
        uint32_t *o = acc + (size_t)r * n;
        for (uint32_t j = 0; j < n; ++j) {
            uint64_t v = (uint64_t)xs[j] * ps[j] % q;
            if (!first) v = (v + o[j]) % q;
            o[j] = (uint32_t)v;
        }
    }
}

/* ModRaise: the value v in (-q0 q1 / 2, q0 q1 / 2] with v = in[0] mod q0 = in[1] mod q1
 * (Garner lift of two coefficient-domain limbs, centred), reduced modulo every target row. */
void orc_lift2_centered(const orc_ctx *c, const uint32_t *in, int mod0, int mod1, uint32_t *out,
                        const int32_t *row_mod, int rows) {
    const uint32_t n = c->n;
    const uint64_t q0 = mod_q(c, mod0), q1 = mod_q(c, mod1);
    const uint64_t q0_inv = powmod((uint32_t)(q0 % q1), q1 - 2, (uint32_t)q1);
    const u128 big = (u128)q0 * q1;
#pragma omp parallel for schedule(static)
    for (uint32_t j = 0; j < n; ++j) {
        const uint64_t r0 = in[j], r1 = in[(size_t)n + j];
        const uint64_t d = (r1 + q1 - r0 % q1) % q1;
        const u128 v = (u128)r0 + (u128)q0 * (d * q0_inv % q1);
        const int neg = v > big / 2;
        const u128 mag = neg ? big - v : v;
        for (int i = 0; i < rows; ++i) {
            const uint64_t q = mod_q(c, row_mod[i]);
            uint64_t r = (uint64_t)(mag % q);
            if (neg && r) r = q - r;
            out[(size_t)i * n + j] = (uint32_t)r;
        }
    }
}

/* out = in + (P mod q_i) * lift on rows < l (rows >= l copied): a polynomial over Q joins a
 * Q||P accumulator.  in may alias out. */
void orc_add_lifted(const orc_ctx *c, const uint32_t *in, const uint32_t *lift,
                    const uint32_t *pmod, const int32_t *ext_idx, int l, int ext, uint32_t *out) {
    const uint32_t n = c->n;
#pragma omp parallel for schedule(static)
    for (int row = 0; row < ext; ++row) {
        const uint64_t q = mod_q(c, ext_idx[row]);
        for (uint32_t j = 0; j < n; ++j) {
            uint64_t v = in[(size_t)row * n + j];
            if (row < l) v = (v + (uint64_t)lift[(size_t)row * n + j] * pmod[row] % q) % q;
            out[(size_t)row * n + j] = (uint32_t)v;
        }
    }
}
