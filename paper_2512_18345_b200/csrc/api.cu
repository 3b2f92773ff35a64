// api.cu -- context, table construction and the extern "C" surface declared
// in include/ckks_b200.h.  Host code here is setup only (tables are built once
// per modulus / basis pair / key-switch shape and cached on the device); the
// hot calls at the bottom just enqueue kernels on the caller's stream.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "../../include/ckks_b200.h"

namespace ckks {

static thread_local char g_err[512] = "";

void set_last_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("CKKS_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

// ---- optional kernel timing ----------------------------------------------------------
struct ProfRec { int name; cudaEvent_t a, b; double bytes, flops; };
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<std::string> g_prof_names;
static std::vector<cudaEvent_t> g_prof_pool;

static cudaEvent_t prof_event() {
    if (!g_prof_pool.empty()) { cudaEvent_t e = g_prof_pool.back(); g_prof_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

ProfScope::ProfScope(const char* name, cudaStream_t stream, double alg_bytes, double alg_flops) : st(stream), live(g_prof_on) {
    if (!live) return;
    int id = -1;
    for (size_t i = 0; i < g_prof_names.size(); ++i)
        if (g_prof_names[i] == name) id = (int)i;
    if (id < 0) { id = (int)g_prof_names.size(); g_prof_names.push_back(name); }
    ProfRec r{id, prof_event(), prof_event(), alg_bytes, alg_flops};
    cudaEventRecord(r.a, st);
    g_prof.push_back(r);
}

ProfScope::~ProfScope() {
    if (live) cudaEventRecord(g_prof.back().b, st);
}

// ---- host number theory (setup only) -----------------------------------------------
static inline uint32_t h_mulmod(uint32_t a, uint32_t b, uint32_t q) {
    return (uint32_t)((uint64_t)a * b % q);
}
static uint32_t h_powmod(uint32_t b, uint64_t e, uint32_t q) {
    uint64_t acc = 1 % q, x = b % q;
    for (; e; e >>= 1) {
        if (e & 1) acc = acc * x % q;
        x = x * x % q;
    }
    return (uint32_t)acc;
}
static inline uint32_t h_inv(uint32_t a, uint32_t q) { return h_powmod(a, (uint64_t)q - 2, q); }
static inline uint32_t h_shoup(uint32_t w, uint32_t q) { return (uint32_t)(((uint64_t)w << 32) / q); }
static uint32_t h_bitrev(uint32_t x, uint32_t bits) {
    uint32_t r = 0;
    for (uint32_t i = 0; i < bits; ++i) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}
static bool h_is_prime(uint32_t n) {
    if (n < 2) return false;
    for (uint32_t p : {2u, 3u, 5u, 7u, 11u, 13u, 17u, 19u, 23u, 29u, 31u, 37u}) {
        if (n == p) return true;
        if (n % p == 0) return false;
    }
    uint32_t d = n - 1, r = 0;
    while (!(d & 1)) { d >>= 1; ++r; }
    for (uint32_t a : {2u, 3u, 5u, 7u}) {   // deterministic below 3.2e9; 11 added for 2^32
        uint32_t x = h_powmod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool comp = true;
        for (uint32_t i = 1; i < r && comp; ++i) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    uint32_t x = h_powmod(11, d, n);
    if (!(x == 1 || x == n - 1)) {
        bool comp = true;
        for (uint32_t i = 1; i < r && comp; ++i) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) comp = false;
        }
        if (comp) return false;
    }
    return true;
}

template <class T>
static int upload(const std::vector<T>& h, T** d) {
    *d = nullptr;
    if (h.empty()) return CKKS_OK;
    CK(cudaMalloc((void**)d, sizeof(T) * h.size()));
    CK(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return CKKS_OK;
}

struct BconvTable {
    int l_in = 0, l_out = 0;
    std::vector<uint32_t> t_plain, inv_qhat;      // host copies for ckks_bconv_table_read
    BconvDev dev{};
    std::vector<void*> owned;
};

constexpr int kMaxMergedDrop = 4;   // limbs a fused relinearise+rescale may drop

struct KsPlan {
    uint32_t n = 0;
    int l = 0, alpha = 0, beta = 0, ext = 0, evk_ext = 0;
    int32_t *d_q_slot = nullptr, *d_p_slot = nullptr, *d_ext_slot = nullptr, *d_evk_row = nullptr;
    std::vector<int> digit_lo, digit_hi;           // Q rows [lo, hi) of digit t
    std::vector<int32_t> raise_table;              // table id per digit
    std::vector<int32_t*> d_raise_out_row;         // per digit: ext row of every converted limb
    int s1_rows = 0;
    int32_t *d_s1_row = nullptr, *d_s1_slot = nullptr;
    int32_t moddown_table = -1;
    int32_t *d_s3_in_row = nullptr, *d_s3_p_slot = nullptr, *d_s3_q_slot = nullptr;
    uint32_t *d_pinv = nullptr, *d_pinv_s = nullptr;
    uint32_t *d_pmod = nullptr, *d_pmod_s = nullptr;   // P mod q_i (and Shoup companion)
    // workspace: word offsets into the context's shared arena (bound at call time)
    size_t off_coeff = 0, off_raised = 0, off_acc = 0, off_conv = 0, off_pc = 0, ws_words = 0;
    uint32_t *ws_coeff = nullptr, *ws_raised = nullptr, *ws_acc = nullptr, *ws_conv = nullptr,
             *ws_pc = nullptr;
    bool moddown_only = false;
    // row maps of batched ModDowns (ckks_ks_stage3_batch), by batch size; built on first use
    struct BatchMaps { int32_t *in_row, *pc_row, *p_slot, *conv_row, *q_slot; size_t lane_words; };
    std::map<int, BatchMaps> s3_batch;            // key: count * 4 + halves
};

}  // namespace ckks

using namespace ckks;

struct ckks_ctx {
    int device = 0;
    static constexpr int kMaxSlots = 4096;
    ModSlot* d_slots = nullptr;
    std::vector<ModSlot> h_slots;
    std::map<std::tuple<uint32_t, uint32_t, uint32_t>, int32_t> slot_index;
    std::vector<std::unique_ptr<BconvTable>> tables;
    std::vector<std::unique_ptr<KsPlan>> plans;
    std::vector<void*> owned;
    // One workspace arena shared by every plan (calls on one stream serialise); it only
    // grows at plan creation, never in the hot path.  Graphs captured before a later,
    // larger plan is created must be re-captured.
    uint32_t* ws = nullptr;
    size_t ws_words = 0;          // words per lane
    // Bumped whenever the arena is (re)allocated.  Anything that recorded raw pointers into it
    // (a captured CUDA graph) remembers the generation and must not be replayed after a change:
    // ckks_arena_generation lets callers check (Bootstrapper.capture / replay do).
    uint64_t ws_generation = 0;
    // Lanes: independent copies of the arena so that key switches issued on different
    // streams (independent rotations, the two EvalMod branches) can overlap.
    int lanes = 1;
    int lane = 0;
};

static int check_ctx(ckks_ctx* ctx) {
    if (!ctx) { set_last_error("null context"); return CKKS_ERR_ARG; }
    CK(cudaSetDevice(ctx->device));
    return CKKS_OK;
}

static int check_slot(ckks_ctx* ctx, int32_t s) {
    if (s < 0 || s >= (int32_t)ctx->h_slots.size()) {
        set_last_error("modulus slot %d out of range", s);
        return CKKS_ERR_ARG;
    }
    return CKKS_OK;
}

extern "C" {

int ckks_abi_version(void) { return 1; }
const char* ckks_last_error(void) { return g_err; }

int ckks_profile_enable(int on) {
    for (auto& r : g_prof) { g_prof_pool.push_back(r.a); g_prof_pool.push_back(r.b); }
    g_prof.clear();
    g_prof_on = on != 0;
    return CKKS_OK;
}

int ckks_profile_read(char* buf, size_t cap) {
    if (!buf || cap == 0) { set_last_error("null profile buffer"); return CKKS_ERR_ARG; }
    CK(cudaDeviceSynchronize());
    std::vector<double> total(g_prof_names.size(), 0.0);
    std::vector<int> count(g_prof_names.size(), 0);
    std::vector<double> bytes(g_prof_names.size(), 0.0), flops(g_prof_names.size(), 0.0);
    for (auto& r : g_prof) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        total[r.name] += ms;
        count[r.name] += 1;
        bytes[r.name] += r.bytes;
        flops[r.name] += r.flops;
    }
    size_t at = 0;
    buf[0] = 0;
    for (size_t i = 0; i < g_prof_names.size(); ++i) {
        if (!count[i]) continue;
        int w = snprintf(buf + at, cap - at, "%s %d %.6f %.0f %.0f\n", g_prof_names[i].c_str(), count[i], total[i], bytes[i], flops[i]);
        if (w < 0 || (size_t)w >= cap - at) break;
        at += (size_t)w;
    }
    return CKKS_OK;
}

int ckks_set_lanes(ckks_ctx* ctx, int lanes) {
    CKS(check_ctx(ctx));
    if (lanes < 1 || lanes > 16) { set_last_error("lane count %d out of range [1, 16]", lanes); return CKKS_ERR_ARG; }
    if (lanes != ctx->lanes) {
        CK(cudaDeviceSynchronize());
        if (ctx->ws) CK(cudaFree(ctx->ws));
        ctx->ws = nullptr;
        ctx->lanes = lanes;
        ctx->lane = 0;
        ctx->ws_generation++;
        if (ctx->ws_words) CK(cudaMalloc((void**)&ctx->ws, sizeof(uint32_t) * ctx->ws_words * lanes));
    }
    return CKKS_OK;
}

int ckks_arena_generation(ckks_ctx* ctx, uint64_t* generation) {
    if (!ctx || !generation) { set_last_error("null argument"); return CKKS_ERR_ARG; }
    *generation = ctx->ws_generation;
    return CKKS_OK;
}

int ckks_arena_reserve(ckks_ctx* ctx, size_t words_per_lane) {
    CKS(check_ctx(ctx));
    if (words_per_lane > ctx->ws_words) {
        CK(cudaDeviceSynchronize());
        if (ctx->ws) CK(cudaFree(ctx->ws));
        ctx->ws = nullptr;
        ctx->ws_words = 0;
        ctx->ws_generation++;
        CK(cudaMalloc((void**)&ctx->ws, sizeof(uint32_t) * words_per_lane * ctx->lanes));
        ctx->ws_words = words_per_lane;
    }
    return CKKS_OK;
}

int ckks_select_lane(ckks_ctx* ctx, int lane) {
    if (!ctx || lane < 0 || lane >= ctx->lanes) { set_last_error("lane %d out of range", lane); return CKKS_ERR_ARG; }
    ctx->lane = lane;
    return CKKS_OK;
}

int ckks_ctx_create(int device, ckks_ctx** out) {
    if (!out) { set_last_error("null out pointer"); return CKKS_ERR_ARG; }
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= 0) {
        set_last_error("no CUDA device available (%s); this engine has no CPU fallback",
                       e != cudaSuccess ? cudaGetErrorString(e) : "device count is 0");
        return CKKS_ERR_CUDA;
    }
    if (device < 0 || device >= count) { set_last_error("device %d out of range", device); return CKKS_ERR_ARG; }
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0) {
        // the library holds sm_100a SASS only (no PTX, no other cubin): fail here, not at the
        // first launch with "no kernel image"
        set_last_error("device %d is sm_%d%d; libckks_b200 is built for sm_100a (B200) only", device,
                       prop.major, prop.minor);
        return CKKS_ERR_UNSUPPORTED;
    }
    auto ctx = new ckks_ctx();
    ctx->device = device;
    if (cudaMalloc((void**)&ctx->d_slots, sizeof(ModSlot) * ckks_ctx::kMaxSlots) != cudaSuccess) {
        delete ctx;
        set_last_error("cudaMalloc of the modulus slot table failed");
        return CKKS_ERR_CUDA;
    }
    *out = ctx;
    return CKKS_OK;
}

void ckks_ctx_destroy(ckks_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (void* p : ctx->owned) cudaFree(p);
    for (auto& t : ctx->tables)
        for (void* p : t->owned) cudaFree(p);
    for (auto& pl : ctx->plans) {
        for (void* p : {(void*)pl->d_q_slot, (void*)pl->d_p_slot, (void*)pl->d_ext_slot,
                        (void*)pl->d_evk_row, (void*)pl->d_s1_row, (void*)pl->d_s1_slot,
                        (void*)pl->d_s3_in_row, (void*)pl->d_s3_p_slot, (void*)pl->d_s3_q_slot,
                        (void*)pl->d_pinv, (void*)pl->d_pinv_s, (void*)pl->d_pmod, (void*)pl->d_pmod_s})
            cudaFree(p);
        for (int32_t* p : pl->d_raise_out_row) cudaFree(p);
    }
    cudaFree(ctx->ws);
    cudaFree(ctx->d_slots);
    delete ctx;
}

int ckks_modulus_register(ckks_ctx* ctx, uint32_t q, uint32_t n, uint32_t psi, int32_t* slot) {
    CKS(check_ctx(ctx));
    if (!slot) { set_last_error("null slot pointer"); return CKKS_ERR_ARG; }
    if (q < 3 || !(q & 1) || !h_is_prime(q)) { set_last_error("%u is not an odd prime", q); return CKKS_ERR_ARG; }
    if (n < 2 || psi == 0) { n = 0; psi = 0; }
    auto key = std::make_tuple(q, n, psi);
    auto it = ctx->slot_index.find(key);
    if (it != ctx->slot_index.end()) { *slot = it->second; return CKKS_OK; }
    if ((int)ctx->h_slots.size() >= ckks_ctx::kMaxSlots) { set_last_error("modulus slot table full"); return CKKS_ERR_STATE; }

    ModSlot m{};
    m.q = q;
    uint32_t qinv = q;                                  // Newton: q * qinv = 1 mod 2^32
    for (int i = 0; i < 5; ++i) qinv *= 2u - q * qinv;
    m.qinv = qinv;
    m.r1 = (uint32_t)((1ull << 32) % q);
    m.r2 = h_mulmod(m.r1, m.r1, q);
    m.r1s = h_shoup(m.r1, q);
    m.r2s = h_shoup(m.r2, q);
    m.fast = (q > (1u << 30) && q < (1u << 31)) ? 1u : 0u;
    m.n = 0;
    if (n) {
        if (n & (n - 1)) { set_last_error("ring degree %u is not a power of two", n); return CKKS_ERR_ARG; }
        if (q >> 31) {
            set_last_error("modulus %u needs 32 bits; the transform kernels require q < 2^31", q);
            return CKKS_ERR_UNSUPPORTED;
        }
        if ((q - 1) % (2ull * n)) { set_last_error("%u is not NTT-friendly for degree %u", q, n); return CKKS_ERR_ARG; }
        if (h_powmod(psi, n, q) != q - 1) { set_last_error("%u is not a primitive %u-th root mod %u", psi, 2 * n, q); return CKKS_ERR_ARG; }
        uint32_t lg = 0;
        while ((1u << lg) < n) ++lg;
        const uint32_t psi_inv = h_inv(psi, q);
        std::vector<uint32_t> pw(n), pwi(n);
        uint32_t a = 1, b = 1;
        for (uint32_t k = 0; k < n; ++k) {
            pw[k] = a; pwi[k] = b;
            a = h_mulmod(a, psi, q);
            b = h_mulmod(b, psi_inv, q);
        }
        std::vector<uint2> fwd(n), inv(n);
        for (uint32_t t = 0; t < n; ++t) {
            const uint32_t r = h_bitrev(t, lg);
            fwd[t] = make_uint2(pw[r], h_shoup(pw[r], q));
            inv[t] = make_uint2(pwi[r], h_shoup(pwi[r], q));
        }
        uint2 *d_fwd, *d_inv;
        CKS(upload(fwd, &d_fwd));
        CKS(upload(inv, &d_inv));
        ctx->owned.push_back(d_fwd);
        ctx->owned.push_back(d_inv);
        m.fwd = d_fwd;
        m.inv = d_inv;
        m.n = n;
        m.n_inv = h_inv(n % q, q);
        m.n_inv_s = h_shoup(m.n_inv, q);
        m.w_last = h_mulmod(inv[1].x, m.n_inv, q);
        m.w_last_s = h_shoup(m.w_last, q);
    }
    const int32_t id = (int32_t)ctx->h_slots.size();
    CK(cudaMemcpy(ctx->d_slots + id, &m, sizeof(ModSlot), cudaMemcpyHostToDevice));
    ctx->h_slots.push_back(m);
    ctx->slot_index[key] = id;
    *slot = id;
    return CKKS_OK;
}

int ckks_modulus_register_tables(ckks_ctx* ctx, uint32_t q, uint32_t n, const uint32_t* fwd_w,
                                 const uint32_t* inv_w, uint32_t n_inv, int32_t* slot) {
    CKS(check_ctx(ctx));
    if (!slot || !fwd_w || !inv_w) { set_last_error("null pointer"); return CKKS_ERR_ARG; }
    if (q < 3 || !(q & 1) || (q >> 31)) { set_last_error("custom tables need an odd modulus below 2^31, got %u", q); return CKKS_ERR_ARG; }
    if (n < 2 || (n & (n - 1))) { set_last_error("ring degree %u is not a power of two >= 2", n); return CKKS_ERR_ARG; }
    if ((int)ctx->h_slots.size() >= ckks_ctx::kMaxSlots) { set_last_error("modulus slot table full"); return CKKS_ERR_STATE; }
    ModSlot m{};
    m.q = q;
    uint32_t qinv = q;
    for (int i = 0; i < 5; ++i) qinv *= 2u - q * qinv;
    m.qinv = qinv;
    m.r1 = (uint32_t)((1ull << 32) % q);
    m.r2 = h_mulmod(m.r1, m.r1, q);
    m.r1s = h_shoup(m.r1, q);
    m.r2s = h_shoup(m.r2, q);
    m.fast = (q > (1u << 30) && q < (1u << 31)) ? 1u : 0u;
    std::vector<uint2> fwd(n), inv(n);
    for (uint32_t t = 0; t < n; ++t) {
        if (fwd_w[t] >= q || inv_w[t] >= q) { set_last_error("table entry %u is not a residue mod %u", t, q); return CKKS_ERR_ARG; }
        fwd[t] = make_uint2(fwd_w[t], h_shoup(fwd_w[t], q));
        inv[t] = make_uint2(inv_w[t], h_shoup(inv_w[t], q));
    }
    uint2 *d_fwd, *d_inv;
    CKS(upload(fwd, &d_fwd));
    CKS(upload(inv, &d_inv));
    ctx->owned.push_back(d_fwd);
    ctx->owned.push_back(d_inv);
    m.fwd = d_fwd;
    m.inv = d_inv;
    m.n = n;
    m.n_inv = n_inv % q;
    m.n_inv_s = h_shoup(m.n_inv, q);
    m.w_last = h_mulmod(inv[1].x, m.n_inv, q);       // transform.py:243-246: the last stage's twiddle carries N^-1
    m.w_last_s = h_shoup(m.w_last, q);
    const int32_t id = (int32_t)ctx->h_slots.size();
    CK(cudaMemcpy(ctx->d_slots + id, &m, sizeof(ModSlot), cudaMemcpyHostToDevice));
    ctx->h_slots.push_back(m);                       // not entered in slot_index: never returned for (q, n, psi)
    *slot = id;
    return CKKS_OK;
}

int ckks_modulus_tables(ckks_ctx* ctx, int32_t slot, uint32_t* fwd, uint32_t* inv, uint32_t* n_inv) {
    CKS(check_ctx(ctx));
    CKS(check_slot(ctx, slot));
    const ModSlot& m = ctx->h_slots[slot];
    if (!m.n) { set_last_error("slot %d has no transform tables", slot); return CKKS_ERR_STATE; }
    std::vector<uint2> tmp(m.n);
    CK(cudaMemcpy(tmp.data(), m.fwd, sizeof(uint2) * m.n, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < m.n; ++i) fwd[i] = tmp[i].x;
    CK(cudaMemcpy(tmp.data(), m.inv, sizeof(uint2) * m.n, cudaMemcpyDeviceToHost));
    for (uint32_t i = 0; i < m.n; ++i) inv[i] = tmp[i].x;
    *n_inv = m.n_inv;
    return CKKS_OK;
}

// ---- transforms ----------------------------------------------------------------------

int ckks_ntt(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, const int32_t* row_slot, int rows,
             uint32_t n, int inverse, void* stream) {
    CKS(check_ctx(ctx));
    if (n < 2 || (n & (n - 1))) { set_last_error("ring degree %u is not a power of two >= 2", n); return CKKS_ERR_ARG; }
    return ntt_launch(in, out, row_slot, ctx->d_slots, RowMap{nullptr, nullptr}, rows, n, inverse,
                      (cudaStream_t)stream);
}

int ckks_ntt_policy(int cluster_max_rows, int ctas_per_sm, int* cluster_max_rows_now, int* ctas_per_sm_now) {
    ntt_policy(cluster_max_rows, ctas_per_sm, cluster_max_rows_now, ctas_per_sm_now);
    return CKKS_OK;
}

int ckks_ntt_stages(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, const int32_t* row_slot,
                    int rows, uint32_t n, int inverse, uint32_t stage_lo, uint32_t stage_hi,
                    void* stream) {
    CKS(check_ctx(ctx));
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    if (n < 2 || (n & (n - 1)) || stage_lo > stage_hi || stage_hi > lg) {
        set_last_error("bad stage range [%u, %u) for degree %u", stage_lo, stage_hi, n);
        return CKKS_ERR_ARG;
    }
    return ntt_stages_launch(in, out, row_slot, ctx->d_slots, rows, n, inverse, stage_lo, stage_hi,
                             (cudaStream_t)stream);
}

// ---- element-wise ---------------------------------------------------------------------

int ckks_elementwise(ckks_ctx* ctx, const uint32_t* a, const uint32_t* b, uint32_t* out,
                     const int32_t* row_slot, int rows, size_t cols, int kind, void* stream) {
    CKS(check_ctx(ctx));
    return elementwise_launch(a, b, out, row_slot, ctx->d_slots, rows, cols, kind, (cudaStream_t)stream);
}

int ckks_automorphism_eval(ckks_ctx* ctx, const uint32_t* in, uint32_t* out, int rows, uint32_t n,
                           uint32_t k, void* stream) {
    CKS(check_ctx(ctx));
    if (!(k & 1) || n == 0 || (n & (n - 1))) { set_last_error("automorphism needs odd k and power-of-two n"); return CKKS_ERR_ARG; }
    return automorphism_eval_launch(in, out, rows, n, k & (2 * n - 1), (cudaStream_t)stream);
}

int ckks_automorphism_coeff(ckks_ctx* ctx, const uint32_t* in, uint32_t* out,
                            const int32_t* row_slot, int rows, uint32_t n, uint32_t k, void* stream) {
    CKS(check_ctx(ctx));
    if (!(k & 1) || n == 0 || (n & (n - 1))) { set_last_error("automorphism needs odd k and power-of-two n"); return CKKS_ERR_ARG; }
    return automorphism_coeff_launch(in, out, row_slot, ctx->d_slots, rows, n, k & (2 * n - 1),
                                     (cudaStream_t)stream);
}

int ckks_lift2_centered(ckks_ctx* ctx, const uint32_t* in, int32_t slot0, int32_t slot1,
                        uint32_t* out, const int32_t* row_slot, int rows, size_t n, void* stream) {
    CKS(check_ctx(ctx));
    CKS(check_slot(ctx, slot0));
    CKS(check_slot(ctx, slot1));
    const uint32_t q0 = ctx->h_slots[slot0].q, q1 = ctx->h_slots[slot1].q;
    if (q0 == q1 || (q0 >> 31) || (q1 >> 31)) { set_last_error("lift needs two distinct moduli below 2^31"); return CKKS_ERR_ARG; }
    return lift2_centered_launch(in, out, row_slot, ctx->d_slots, slot0, slot1, h_inv(q0 % q1, q1),
                                 rows, n, (cudaStream_t)stream);
}

int ckks_pmult_accumulate(ckks_ctx* ctx, const uint32_t* x, const uint32_t* p, uint32_t* acc,
                          const int32_t* row_slot, int rows, size_t cols, int first, void* stream) {
    CKS(check_ctx(ctx));
    return pmult_acc_launch(x, p, acc, row_slot, ctx->d_slots, rows, cols, first, (cudaStream_t)stream);
}

int ckks_fused_terms_halves(ckks_ctx* ctx, int count, const uint32_t* const* xa, const uint32_t* const* xb,
                            const uint32_t* const* p, uint32_t* out, const int32_t* row_slot, int rows,
                            size_t cols, void* stream) {
    CKS(check_ctx(ctx));
    if (count < 1 || count > kMaxTerms || !xa || !p) { set_last_error("term count %d out of range [1, %d]", count, kMaxTerms); return CKKS_ERR_ARG; }
    FusedTerms t{};
    t.count = count;
    for (int i = 0; i < count; ++i) { t.x[i] = xa[i]; t.xb[i] = xb ? xb[i] : nullptr; t.p[i] = p[i]; }
    return fused_terms_launch(t, out, row_slot, ctx->d_slots, rows, cols, (cudaStream_t)stream);
}

int ckks_fused_terms(ckks_ctx* ctx, int count, const uint32_t* const* x, const uint32_t* const* p,
                     uint32_t* out, const int32_t* row_slot, int rows, size_t cols, void* stream) {
    return ckks_fused_terms_halves(ctx, count, x, nullptr, p, out, row_slot, rows, cols, stream);
}

int ckks_fused_terms_multi(ckks_ctx* ctx, int nb, int ng, const uint32_t* const* x,
                           const uint32_t* const* p, const uint32_t* zero, uint32_t* const* out,
                           const int32_t* row_slot, int rows, size_t cols, void* stream) {
    CKS(check_ctx(ctx));
    if (nb < 1 || nb > kMaxTerms || ng < 1 || ng > kMaxGiants || !x || !p || !out) {
        set_last_error("fused_terms_multi: %d terms x %d outputs out of range [1, %d] x [1, %d]", nb, ng, kMaxTerms, kMaxGiants);
        return CKKS_ERR_ARG;
    }
    FusedMulti a{};
    a.nb = nb;
    a.ng = ng;
    for (int b = 0; b < nb; ++b) a.x[b] = x[b];
    for (int g = 0; g < ng; ++g) {
        a.out[g] = out[g];
        for (int b = 0; b < nb; ++b) {
            a.p[g][b] = p[(size_t)g * nb + b] ? p[(size_t)g * nb + b] : zero;
            if (!a.p[g][b]) { set_last_error("fused_terms_multi: absent diagonal (%d, %d) but no zero plaintext given", g, b); return CKKS_ERR_ARG; }
        }
    }
    a.zero = zero;
    return fused_terms_multi_launch(a, row_slot, ctx->d_slots, rows, cols, (cudaStream_t)stream);
}

int ckks_tensor(ckks_ctx* ctx, const uint32_t* x, const uint32_t* y, uint32_t* out,
                const int32_t* row_slot, int rows, size_t cols, void* stream) {
    CKS(check_ctx(ctx));
    const size_t half = (size_t)rows * cols;
    return tensor_launch(x, x + half, y, y + half, out, row_slot, ctx->d_slots, rows, cols, (cudaStream_t)stream);
}

int ckks_tensor_halves(ckks_ctx* ctx, const uint32_t* xa, const uint32_t* xb, const uint32_t* ya,
                       const uint32_t* yb, uint32_t* out, const int32_t* row_slot, int rows, size_t cols,
                       void* stream) {
    CKS(check_ctx(ctx));
    return tensor_launch(xa, xb, ya, yb, out, row_slot, ctx->d_slots, rows, cols, (cudaStream_t)stream);
}

// ---- base conversion ------------------------------------------------------------------

int ckks_bconv_table_create(ckks_ctx* ctx, const int32_t* in_slot, int l_in, const int32_t* out_slot,
                            int l_out, int32_t* table) {
    CKS(check_ctx(ctx));
    if (l_in < 1 || l_out < 1 || !in_slot || !out_slot || !table) { set_last_error("bad conversion shape %d -> %d", l_in, l_out); return CKKS_ERR_ARG; }
    std::vector<uint32_t> qs(l_in), ps(l_out);
    for (int j = 0; j < l_in; ++j) { CKS(check_slot(ctx, in_slot[j])); qs[j] = ctx->h_slots[in_slot[j]].q; }
    for (int i = 0; i < l_out; ++i) { CKS(check_slot(ctx, out_slot[i])); ps[i] = ctx->h_slots[out_slot[i]].q; }
    auto tab = std::make_unique<BconvTable>();
    tab->l_in = l_in;
    tab->l_out = l_out;
    tab->inv_qhat.resize(l_in);
    tab->t_plain.resize((size_t)l_in * l_out);
    std::vector<uint32_t> inv_s(l_in), t_mont((size_t)l_in * l_out);
    uint32_t all31 = 1;
    for (int j = 0; j < l_in; ++j) {
        uint64_t h = 1 % qs[j];
        for (int k = 0; k < l_in; ++k)
            if (k != j) h = h * (qs[k] % qs[j]) % qs[j];
        if (h == 0) { set_last_error("source moduli are not pairwise coprime"); return CKKS_ERR_ARG; }
        tab->inv_qhat[j] = h_inv((uint32_t)h, qs[j]);
        inv_s[j] = h_shoup(tab->inv_qhat[j], qs[j]);
        if (qs[j] >> 31) all31 = 0;
    }
    for (int i = 0; i < l_out; ++i)
        for (int j = 0; j < l_in; ++j) {
            uint64_t h = 1 % ps[i];
            for (int k = 0; k < l_in; ++k)
                if (k != j) h = h * (qs[k] % ps[i]) % ps[i];
            if (!(ps[i] > (1u << 30) && ps[i] < (1u << 31))) all31 = 0;   // fast kernel range
            tab->t_plain[(size_t)i * l_in + j] = (uint32_t)h;
            t_mont[(size_t)i * l_in + j] = (uint32_t)((h << 32) % ps[i]);
        }
    std::vector<int32_t> in_s(in_slot, in_slot + l_in), out_s(out_slot, out_slot + l_out);
    int32_t *d_in, *d_out;
    uint32_t *d_inv, *d_invs, *d_tm, *d_tp;
    CKS(upload(in_s, &d_in));
    CKS(upload(out_s, &d_out));
    CKS(upload(tab->inv_qhat, &d_inv));
    CKS(upload(inv_s, &d_invs));
    CKS(upload(t_mont, &d_tm));
    CKS(upload(tab->t_plain, &d_tp));
    // operands of bconv_dmma in their final form
    const int kp = (l_in + 3) & ~3, lo8 = (l_out + 7) & ~7;
    std::vector<double> t_f64((size_t)lo8 * kp, 0.0);
    std::vector<uint4> om(lo8, make_uint4(3u, 0u, 0u, 0u)), inc(kp, make_uint4(3u, 0u, 0u, 0u));
    for (int i = 0; i < l_out; ++i) {
        for (int j = 0; j < l_in; ++j) t_f64[(size_t)i * kp + j] = (double)t_mont[(size_t)i * l_in + j];
        const ModSlot& m = ctx->h_slots[out_slot[i]];
        om[i] = make_uint4(m.q, m.qinv, (uint32_t)i, (uint32_t)(((uint64_t)m.r1 << 16) % m.q));
    }
    for (int j = 0; j < l_in; ++j) inc[j] = make_uint4(qs[j], tab->inv_qhat[j], inv_s[j], 0u);
    // K-stacked table of the tensor-core kernel: T * y = T * y0 + (T * 2^16 mod p) * y1 (mod p); every
    // term < 2^47 resp. 2^46, at most 16 + 16 of them: the sum stays below 2^52 and is exact in ONE double
    std::vector<double> t_f64k((size_t)lo8 * 2 * kp, 0.0);
    for (int i = 0; i < l_out; ++i)
        for (int j = 0; j < l_in; ++j) {
            const uint64_t tm = t_mont[(size_t)i * l_in + j];
            t_f64k[(size_t)i * 2 * kp + j] = (double)tm;
            t_f64k[(size_t)i * 2 * kp + kp + j] = (double)((tm << 16) % ps[i]);
        }
    double *d_tf, *d_tfk;
    uint4 *d_om, *d_inc;
    CKS(upload(t_f64, &d_tf));
    CKS(upload(t_f64k, &d_tfk));
    CKS(upload(om, &d_om));
    CKS(upload(inc, &d_inc));
    tab->owned = {d_in, d_out, d_inv, d_invs, d_tm, d_tp, d_tf, d_tfk, d_om, d_inc};
    tab->dev = BconvDev{l_in, l_out, all31, d_in, d_out, d_inv, d_invs, d_tm, d_tp, kp, d_tf, d_tfk, d_om, d_inc};
    *table = (int32_t)ctx->tables.size();
    ctx->tables.push_back(std::move(tab));
    return CKKS_OK;
}

static int check_table(ckks_ctx* ctx, int32_t t) {
    if (t < 0 || t >= (int32_t)ctx->tables.size()) { set_last_error("conversion table %d out of range", t); return CKKS_ERR_ARG; }
    return CKKS_OK;
}

int ckks_bconv_table_read(ckks_ctx* ctx, int32_t table, uint32_t* t, uint32_t* inv_qhat) {
    CKS(check_ctx(ctx));
    CKS(check_table(ctx, table));
    const BconvTable& tab = *ctx->tables[table];
    memcpy(t, tab.t_plain.data(), sizeof(uint32_t) * tab.t_plain.size());
    memcpy(inv_qhat, tab.inv_qhat.data(), sizeof(uint32_t) * tab.inv_qhat.size());
    return CKKS_OK;
}

int ckks_bconv(ckks_ctx* ctx, int32_t table, const uint32_t* in, uint32_t* out, size_t cols,
               void* stream) {
    CKS(check_ctx(ctx));
    CKS(check_table(ctx, table));
    return bconv_launch(ctx->tables[table]->dev, ctx->d_slots, in, cols, out, cols, cols,
                        (cudaStream_t)stream);
}

// ---- key switching --------------------------------------------------------------------

static int plan_create(ckks_ctx* ctx, uint32_t n, int l, int alpha, const int32_t* q_slot,
                       const int32_t* p_slot, int evk_ext, int evk_p_off, bool moddown_only,
                       int32_t* plan) {
    CKS(check_ctx(ctx));
    if (l < 1 || alpha < 1 || !q_slot || !p_slot || !plan || evk_p_off < l || evk_ext < evk_p_off + alpha) {
        set_last_error("bad key-switch shape l=%d alpha=%d evk_ext=%d evk_p_off=%d", l, alpha, evk_ext, evk_p_off);
        return CKKS_ERR_ARG;
    }
    for (int i = 0; i < l + alpha; ++i) {
        const int32_t s = i < l ? q_slot[i] : p_slot[i - l];
        CKS(check_slot(ctx, s));
        if (ctx->h_slots[s].n != n) { set_last_error("slot %d has no tables for degree %u", s, n); return CKKS_ERR_ARG; }
    }
    auto pl = std::make_unique<KsPlan>();
    pl->n = n; pl->l = l; pl->alpha = alpha; pl->ext = l + alpha; pl->evk_ext = evk_ext;
    pl->beta = moddown_only ? 0 : (l + alpha - 1) / alpha;
    pl->moddown_only = moddown_only;
    const int ext = pl->ext;
    std::vector<int32_t> qv(q_slot, q_slot + l), pv(p_slot, p_slot + alpha), extv, evk_row;
    extv = qv;
    extv.insert(extv.end(), pv.begin(), pv.end());
    for (int i = 0; i < l; ++i) evk_row.push_back(i);
    for (int j = 0; j < alpha; ++j) evk_row.push_back(evk_p_off + j);
    CKS(upload(qv, &pl->d_q_slot));
    CKS(upload(pv, &pl->d_p_slot));
    CKS(upload(extv, &pl->d_ext_slot));
    CKS(upload(evk_row, &pl->d_evk_row));
    // stage 1: one raise table per digit (keyswitch.py:193-202)
    std::vector<int32_t> s1_row, s1_slot;
    for (int t = 0; t < pl->beta; ++t) {
        const int lo = t * alpha, hi = std::min(l, lo + alpha);
        pl->digit_lo.push_back(lo);
        pl->digit_hi.push_back(hi);
        std::vector<int32_t> target, out_row;
        for (int r = 0; r < ext; ++r) {
            if (r >= lo && r < hi) continue;
            target.push_back(extv[r]);
            out_row.push_back(r);
            s1_row.push_back(t * ext + r);
            s1_slot.push_back(extv[r]);
        }
        int32_t tab;
        CKS(ckks_bconv_table_create(ctx, qv.data() + lo, hi - lo, target.data(), (int)target.size(), &tab));
        pl->raise_table.push_back(tab);
        int32_t* d_or;
        CKS(upload(out_row, &d_or));
        pl->d_raise_out_row.push_back(d_or);
    }
    pl->s1_rows = (int)s1_row.size();
    CKS(upload(s1_row, &pl->d_s1_row));
    CKS(upload(s1_slot, &pl->d_s1_slot));
    // stage 3: P -> Q table, P^-1 mod q_i (keyswitch.py:203-208)
    CKS(ckks_bconv_table_create(ctx, pv.data(), alpha, qv.data(), l, &pl->moddown_table));
    std::vector<uint32_t> pinv(l), pinv_s(l), pmod(l), pmod_s(l);
    for (int i = 0; i < l; ++i) {
        const uint32_t q = ctx->h_slots[qv[i]].q;
        uint64_t prod = 1 % q;
        for (int j = 0; j < alpha; ++j) prod = prod * (ctx->h_slots[pv[j]].q % q) % q;
        if (prod == 0) { set_last_error("P and Q bases share a modulus"); return CKKS_ERR_ARG; }
        pinv[i] = h_inv((uint32_t)prod, q);
        pinv_s[i] = h_shoup(pinv[i], q);
        pmod[i] = (uint32_t)prod;
        pmod_s[i] = h_shoup(pmod[i], q);
    }
    CKS(upload(pmod, &pl->d_pmod));
    CKS(upload(pmod_s, &pl->d_pmod_s));
    CKS(upload(pinv, &pl->d_pinv));
    CKS(upload(pinv_s, &pl->d_pinv_s));
    std::vector<int32_t> s3_in_row, s3_p_slot, s3_q_slot;
    for (int h = 0; h < 2; ++h) {
        for (int j = 0; j < alpha; ++j) { s3_in_row.push_back(h * ext + l + j); s3_p_slot.push_back(pv[j]); }
        for (int i = 0; i < l; ++i) s3_q_slot.push_back(qv[i]);
    }
    CKS(upload(s3_in_row, &pl->d_s3_in_row));
    CKS(upload(s3_p_slot, &pl->d_s3_p_slot));
    CKS(upload(s3_q_slot, &pl->d_s3_q_slot));
    // workspace: carve the shared arena (grown here if needed, never in the hot path)
    {
        const size_t nn = n;
        size_t at = 0;
        pl->off_coeff = at;  at += moddown_only ? 0 : nn * l;
        pl->off_raised = at; at += moddown_only ? 0 : nn * pl->beta * ext;
        pl->off_acc = at;    at += moddown_only ? 0 : nn * 2 * ext;
        pl->off_conv = at;   at += nn * 2 * l;
        pl->off_pc = at;     at += nn * 2 * (alpha + (moddown_only ? 0 : kMaxMergedDrop));
        pl->ws_words = at;
        if (at > ctx->ws_words) {
            CK(cudaDeviceSynchronize());
            if (ctx->ws) CK(cudaFree(ctx->ws));
            ctx->ws = nullptr;
            ctx->ws_words = 0;
            ctx->ws_generation++;
            CK(cudaMalloc((void**)&ctx->ws, sizeof(uint32_t) * at * ctx->lanes));
            ctx->ws_words = at;
        }
    }
    *plan = (int32_t)ctx->plans.size();
    ctx->plans.push_back(std::move(pl));
    return CKKS_OK;
}

static int get_plan(ckks_ctx* ctx, int32_t id, KsPlan** out) {
    CKS(check_ctx(ctx));
    if (id < 0 || id >= (int32_t)ctx->plans.size()) { set_last_error("key-switch plan %d out of range", id); return CKKS_ERR_ARG; }
    KsPlan* pl = ctx->plans[id].get();
    uint32_t* base = ctx->ws + (size_t)ctx->lane * ctx->ws_words;
    pl->ws_coeff = base + pl->off_coeff;
    pl->ws_raised = base + pl->off_raised;
    pl->ws_acc = base + pl->off_acc;
    pl->ws_conv = base + pl->off_conv;
    pl->ws_pc = base + pl->off_pc;
    *out = pl;
    return CKKS_OK;
}

static int need_full_plan(KsPlan* pl) {
    if (pl->moddown_only) { set_last_error("plan was created for ModDown / rescale only"); return CKKS_ERR_STATE; }
    return CKKS_OK;
}

// ModUp of every digit into `raised` (keyswitch.py:256-294).  With
// carry_copy the digit's own limbs are copied through; the fused pipeline
// skips that copy and lets stage 2 read them from the input directly.
static int stage1_core(ckks_ctx* ctx, KsPlan* pl, const uint32_t* a, uint32_t* raised,
                       bool carry_copy, cudaStream_t st, const uint32_t* mul_in = nullptr) {
    const size_t n = pl->n;
    // mul_in: the polynomial to switch is a (.) mul_in, formed while the inverse transform loads
    CKS(ntt_launch(a, pl->ws_coeff, pl->d_q_slot, ctx->d_slots, RowMap{nullptr, nullptr}, pl->l,
                   pl->n, 1, st, nullptr, mul_in));
    for (int t0 = 0; t0 < pl->beta;) {
        // all digits in one launch, the partial last digit included (bconv_launch_jobs splits
        // unequal sizes itself when the kernel in use cannot stack them)
        BconvJobs jobs;
        jobs.count = 0;
        int t = t0;
        for (; t < pl->beta && jobs.count < kMaxBconvJobs; ++t) {
            BconvJob& j = jobs.job[jobs.count++];
            j.tab = ctx->tables[pl->raise_table[t]]->dev;
            j.in = pl->ws_coeff + (size_t)pl->digit_lo[t] * n;
            j.in_stride = n;
            j.out = raised + (size_t)t * pl->ext * n;
            j.out_stride = n;
            j.out_row = pl->d_raise_out_row[t];
        }
        CKS(bconv_launch_jobs(jobs, ctx->d_slots, n, st));
        t0 = t;
    }
    CKS(ntt_launch(raised, raised, pl->d_s1_slot, ctx->d_slots, RowMap{pl->d_s1_row, pl->d_s1_row},
                   pl->s1_rows, pl->n, 0, st));
    if (carry_copy)
        for (int t = 0; t < pl->beta; ++t) {
            const size_t lo = pl->digit_lo[t], cnt = pl->digit_hi[t] - pl->digit_lo[t];
            CK(cudaMemcpyAsync(raised + ((size_t)t * pl->ext + lo) * n, a + lo * n,
                               sizeof(uint32_t) * cnt * n, cudaMemcpyDeviceToDevice, st));
        }
    return CKKS_OK;
}

static uint32_t log2u(uint32_t n) {
    uint32_t lg = 0;
    while ((1u << lg) < n) ++lg;
    return lg;
}

static int stage3_core(ckks_ctx* ctx, KsPlan* pl, const uint32_t* q_a, const uint32_t* q_b,
                       const uint32_t* p_a, const uint32_t* p_b, const uint32_t* fold_b,
                       uint32_t* out_a, uint32_t* out_b, cudaStream_t st, uint32_t galois = 0,
                       const uint32_t* fold_a = nullptr, uint32_t* ws_conv = nullptr,
                       uint32_t* ws_pc = nullptr) {
    const size_t n = pl->n;
    if (!ws_conv) ws_conv = pl->ws_conv;     // a plan borrowed by another plan's call works in
    if (!ws_pc) ws_pc = pl->ws_pc;           // the caller's workspace (arena layouts differ)
    const RowMap id{nullptr, nullptr};
    if (p_b == p_a + (size_t)pl->ext * n) {
        // accumulator laid out [2][ext][n]: both P parts in one launch through the row map
        CKS(ntt_launch(p_a - (size_t)pl->l * n, ws_pc, pl->d_s3_p_slot, ctx->d_slots,
                       RowMap{pl->d_s3_in_row, nullptr}, 2 * pl->alpha, pl->n, 1, st));
    } else {
        CKS(ntt_launch(p_a, ws_pc, pl->d_s3_p_slot, ctx->d_slots, id, pl->alpha, pl->n, 1, st));
        CKS(ntt_launch(p_b, ws_pc + (size_t)pl->alpha * n, pl->d_s3_p_slot, ctx->d_slots, id,
                       pl->alpha, pl->n, 1, st));
    }
    BconvJobs jobs;
    jobs.count = 2;
    for (int h = 0; h < 2; ++h) {
        BconvJob& j = jobs.job[h];
        j.tab = ctx->tables[pl->moddown_table]->dev;
        j.in = ws_pc + (size_t)h * pl->alpha * n;
        j.in_stride = n;
        j.out = ws_conv + (size_t)h * pl->l * n;
        j.out_stride = n;
        j.out_row = nullptr;
    }
    CKS(bconv_launch_jobs(jobs, ctx->d_slots, n, st));
    ModDownEpilogueArgs e{};
    e.xq_a = q_a; e.xq_b = q_b; e.conv = ws_conv; e.fold_a = fold_a; e.fold_b = fold_b;
    e.out_a = out_a; e.out_b = out_b;
    e.q_slot = pl->d_q_slot; e.pinv = pl->d_pinv; e.pinv_s = pl->d_pinv_s;
    e.l = pl->l; e.n = pl->n;
    e.galois = galois; e.lg = log2u(pl->n);
    if (ntt_can_fuse_moddown(pl->n))       // epilogue applied inside the transform's last kernel
        return ntt_launch(ws_conv, ws_conv, pl->d_s3_q_slot, ctx->d_slots, id, 2 * pl->l, pl->n, 0, st, &e);
    CKS(ntt_launch(ws_conv, ws_conv, pl->d_s3_q_slot, ctx->d_slots, id, 2 * pl->l, pl->n, 0, st));
    return moddown_epilogue_launch(e, ctx->d_slots, st);
}

static InnerProductArgs ip_args(KsPlan* pl, const uint32_t* carry, const uint32_t* raised,
                                const uint32_t* evk, int row_lo, int row_hi, uint32_t* acc_a,
                                uint32_t* acc_b) {
    InnerProductArgs a{};
    a.carry = carry; a.raised = raised; a.evk = evk; a.acc_a = acc_a; a.acc_b = acc_b;
    a.ext_slot = pl->d_ext_slot; a.evk_row = pl->d_evk_row;
    a.l = pl->l; a.alpha = pl->alpha; a.beta = pl->beta; a.ext = pl->ext; a.evk_ext = pl->evk_ext;
    a.row_lo = row_lo; a.row_hi = row_hi; a.n = pl->n;
    a.galois = 0; a.lg = log2u(pl->n); a.accumulate = 0; a.ordered = 0;
    a.lift_a = nullptr; a.lift_b = nullptr; a.pmod = nullptr; a.pmod_s = nullptr; a.lift_qp = nullptr;
    return a;
}

int ckks_ks_plan_create(ckks_ctx* ctx, uint32_t n, int l, int alpha, const int32_t* q_slot,
                        const int32_t* p_slot, int evk_ext, int evk_p_off, int32_t* plan) {
    return plan_create(ctx, n, l, alpha, q_slot, p_slot, evk_ext, evk_p_off, false, plan);
}

int ckks_moddown_plan_create(ckks_ctx* ctx, uint32_t n, int l, int alpha, const int32_t* q_slot,
                             const int32_t* p_slot, int32_t* plan) {
    return plan_create(ctx, n, l, alpha, q_slot, p_slot, l + alpha, l, true, plan);
}

int ckks_ks_stage1(ckks_ctx* ctx, int32_t plan, const uint32_t* a, uint32_t* raised, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    return stage1_core(ctx, pl, a, raised, true, (cudaStream_t)stream);
}

int ckks_ks_stage2(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, const uint32_t* evk,
                   int row_lo, int row_hi, uint32_t* acc_a, uint32_t* acc_b, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (row_lo < 0 || row_hi > pl->ext || row_lo > row_hi) { set_last_error("bad row range [%d, %d)", row_lo, row_hi); return CKKS_ERR_ARG; }
    InnerProductArgs ip = ip_args(pl, nullptr, raised, evk, row_lo, row_hi, acc_a, acc_b);
    ip.ordered = 1;           // first kernel of the call: its predecessor may have written the key
    return inner_product_launch(ip, ctx->d_slots, (cudaStream_t)stream);
}

int ckks_ks_stage3(ckks_ctx* ctx, int32_t plan, const uint32_t* q_a, const uint32_t* q_b,
                   const uint32_t* p_a, const uint32_t* p_b, uint32_t* out_a, uint32_t* out_b,
                   void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    return stage3_core(ctx, pl, q_a, q_b, p_a, p_b, nullptr, out_a, out_b, (cudaStream_t)stream);
}

int ckks_keyswitch(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* ct_b,
                   const uint32_t* evk, uint32_t* out_a, uint32_t* out_b, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, ct_a, pl->ws_raised, false, st));
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    CKS(inner_product_launch(ip_args(pl, ct_a, pl->ws_raised, evk, 0, pl->ext, acc_a, acc_b),
                             ctx->d_slots, st));
    return stage3_core(ctx, pl, acc_a, acc_b, acc_a + (size_t)pl->l * n, acc_b + (size_t)pl->l * n,
                       ct_b, out_a, out_b, st);
}

int ckks_ks_hoisted(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, uint32_t k,
                    const uint32_t* evk, const uint32_t* ct_b, uint32_t* out_a, uint32_t* out_b,
                    void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (!(k & 1)) { set_last_error("automorphism index must be odd"); return CKKS_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    InnerProductArgs ip = ip_args(pl, nullptr, raised, evk, 0, pl->ext, acc_a, acc_b);
    ip.galois = k & (2 * pl->n - 1);
    if (ip.galois == 1) ip.galois = 0;           // X -> X: the plain inner product, no gather
    ip.ordered = 1;
    CKS(inner_product_launch(ip, ctx->d_slots, st));
    return stage3_core(ctx, pl, acc_a, acc_b, acc_a + (size_t)pl->l * n, acc_b + (size_t)pl->l * n,
                       ct_b, out_a, out_b, st, ip.galois);
}

int ckks_ks_hoisted_raw(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, uint32_t k,
                        const uint32_t* evk, const uint32_t* ct_b, uint32_t* out_qp, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (k != 0 && !(k & 1)) { set_last_error("automorphism index must be odd (or 0 for none)"); return CKKS_ERR_ARG; }
    const size_t n = pl->n;
    InnerProductArgs ip = ip_args(pl, nullptr, raised, evk, 0, pl->ext, out_qp, out_qp + (size_t)pl->ext * n);
    ip.galois = k & (2 * pl->n - 1);
    ip.lift_b = ct_b;
    ip.pmod = pl->d_pmod;
    ip.pmod_s = pl->d_pmod_s;
    ip.ordered = 1;
    return inner_product_launch(ip, ctx->d_slots, (cudaStream_t)stream);
}

static int bsgs_inner_core(ckks_ctx* ctx, int32_t plan, int batch, const uint32_t* const* raised,
                           const uint32_t* const* ct_a, const uint32_t* const* ct_b, int nb, const uint32_t* k,
                           const uint32_t* const* evk, int ng, const uint32_t* const* p, const uint32_t* zero,
                           uint32_t* const* out, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (nb < 1 || nb > kMaxTerms || ng < 1 || ng > kMaxGiants || !k || !evk || !p || !out) {
        set_last_error("bsgs_inner: %d baby x %d giant steps out of range [1, %d] x [1, %d]", nb, ng, kMaxTerms, kMaxGiants);
        return CKKS_ERR_ARG;
    }
    if (batch < 1 || batch > kMaxBsgsBatch || !raised || !ct_a || !ct_b) {
        set_last_error("bsgs_inner: batch of %d ciphertexts out of range [1, %d]", batch, kMaxBsgsBatch);
        return CKKS_ERR_ARG;
    }
    BsgsInnerArgs a{};
    a.batch = batch;
    for (int c = 0; c < batch; ++c) {
        if (!raised[c] || !ct_a[c] || !ct_b[c]) { set_last_error("bsgs_inner: null operand in batch element %d", c); return CKKS_ERR_ARG; }
        a.raised[c] = raised[c]; a.ct_a[c] = ct_a[c]; a.ct_b[c] = ct_b[c];
    }
    a.ext_slot = pl->d_ext_slot; a.evk_row = pl->d_evk_row; a.pmod = pl->d_pmod; a.pmod_s = pl->d_pmod_s;
    a.l = pl->l; a.alpha = pl->alpha; a.beta = pl->beta; a.ext = pl->ext; a.evk_ext = pl->evk_ext;
    a.n = pl->n; a.lg = log2u(pl->n);
    a.nb = nb; a.ng = ng;
    for (int b = 0; b < nb; ++b) {
        if (k[b] != 0 && !(k[b] & 1)) { set_last_error("automorphism index must be odd (or 0 for none)"); return CKKS_ERR_ARG; }
        a.k[b] = k[b] & (2 * pl->n - 1);
        a.evk[b] = evk[b];
        if (a.k[b] && !a.evk[b]) { set_last_error("bsgs_inner: rotation %d has no key", b); return CKKS_ERR_ARG; }
    }
    for (int g = 0; g < ng; ++g) {
        for (int c = 0; c < batch; ++c) {
            a.out[c][g] = out[(size_t)c * ng + g];
            if (!a.out[c][g]) { set_last_error("bsgs_inner: null output (%d, %d)", c, g); return CKKS_ERR_ARG; }
        }
        for (int b = 0; b < nb; ++b) {
            a.p[g][b] = p[(size_t)g * nb + b] ? p[(size_t)g * nb + b] : zero;
            if (!a.p[g][b]) { set_last_error("bsgs_inner: absent diagonal (%d, %d) but no zero plaintext given", g, b); return CKKS_ERR_ARG; }
        }
    }
    return bsgs_inner_launch(a, ctx->d_slots, (cudaStream_t)stream);
}

int ckks_bsgs_inner(ckks_ctx* ctx, int32_t plan, const uint32_t* raised, const uint32_t* ct_a,
                    const uint32_t* ct_b, int nb, const uint32_t* k, const uint32_t* const* evk, int ng,
                    const uint32_t* const* p, const uint32_t* zero, uint32_t* const* out, void* stream) {
    return bsgs_inner_core(ctx, plan, 1, &raised, &ct_a, &ct_b, nb, k, evk, ng, p, zero, out, stream);
}

int ckks_bsgs_inner_batch(ckks_ctx* ctx, int32_t plan, int batch, const uint32_t* const* raised,
                          const uint32_t* const* ct_a, const uint32_t* const* ct_b, int nb, const uint32_t* k,
                          const uint32_t* const* evk, int ng, const uint32_t* const* p, const uint32_t* zero,
                          uint32_t* const* out, void* stream) {
    return bsgs_inner_core(ctx, plan, batch, raised, ct_a, ct_b, nb, k, evk, ng, p, zero, out, stream);
}

// Relinearisation (or any key switch) fused with the rescale that follows it: the
// polynomials the switched pair is added to (d1, d0) are lifted into the Q||P accumulator
// (times P on the Q rows), and ONE ModDown divides by P * q_{l-1} * ... * q_{l-k}: the
// accumulator rows [l-k, l+alpha) are contiguous, so they serve as the "P part" of a
// ModDown plan built for Q_{l-k} with P' = {q_{l-k}..q_{l-1}} U P.
int ckks_ks_relin_rescale(ckks_ctx* ctx, int32_t ks_plan, int32_t md_plan, const uint32_t* d2,
                          const uint32_t* d1, const uint32_t* d0, const uint32_t* evk,
                          uint32_t* out_a, uint32_t* out_b, void* stream) {
    KsPlan *pl, *md;
    CKS(get_plan(ctx, ks_plan, &pl));
    CKS(need_full_plan(pl));
    CKS(get_plan(ctx, md_plan, &md));
    if (md->n != pl->n || md->l + md->alpha != pl->ext || md->l >= pl->l) {
        set_last_error("ModDown plan (l=%d, alpha=%d) does not tile the key-switch accumulator (l=%d, ext=%d)",
                       md->l, md->alpha, pl->l, pl->ext);
        return CKKS_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, d2, pl->ws_raised, false, st));
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    InnerProductArgs ip = ip_args(pl, d2, pl->ws_raised, evk, 0, pl->ext, acc_a, acc_b);
    ip.lift_a = d1;
    ip.lift_b = d0;
    ip.pmod = pl->d_pmod;
    ip.pmod_s = pl->d_pmod_s;
    CKS(inner_product_launch(ip, ctx->d_slots, st));
    if (md->alpha > pl->alpha + kMaxMergedDrop) { set_last_error("merged rescale drops more than %d limbs", kMaxMergedDrop); return CKKS_ERR_UNSUPPORTED; }
    return stage3_core(ctx, md, acc_a, acc_b, acc_a + (size_t)md->l * n, acc_b + (size_t)md->l * n,
                       nullptr, out_a, out_b, st, 0, nullptr, pl->ws_conv, pl->ws_pc);
}

// HMult + relinearise + rescale without a tensor pass: d2 = xa * ya is formed while the first
// inverse transform loads, and the inner product forms the carried rows of d2 and the lifted
// d1 = xa * yb + ya * xb, d0 = xb * yb from the four operand halves.  Same values as ckks_tensor +
// ckks_ks_relin_rescale (exact modular arithmetic), five limb transfers per row and one launch less.
int ckks_hmult_relin_rescale(ckks_ctx* ctx, int32_t ks_plan, int32_t md_plan, const uint32_t* xa,
                             const uint32_t* xb, const uint32_t* ya, const uint32_t* yb,
                             const uint32_t* evk, const uint32_t* add_a, const uint32_t* add_b,
                             uint32_t* out_a, uint32_t* out_b, void* stream) {
    KsPlan *pl, *md;
    CKS(get_plan(ctx, ks_plan, &pl));
    CKS(need_full_plan(pl));
    CKS(get_plan(ctx, md_plan, &md));
    if (md->n != pl->n || md->l + md->alpha != pl->ext || md->l >= pl->l) {
        set_last_error("ModDown plan (l=%d, alpha=%d) does not tile the key-switch accumulator (l=%d, ext=%d)",
                       md->l, md->alpha, pl->l, pl->ext);
        return CKKS_ERR_ARG;
    }
    if (pl->n != 65536) { set_last_error("fused HMult needs N = 2^16 (product-on-load transform)"); return CKKS_ERR_UNSUPPORTED; }
    if (md->alpha > pl->alpha + kMaxMergedDrop) { set_last_error("merged rescale drops more than %d limbs", kMaxMergedDrop); return CKKS_ERR_UNSUPPORTED; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, xa, pl->ws_raised, false, st, ya));
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    InnerProductArgs ip = ip_args(pl, nullptr, pl->ws_raised, evk, 0, pl->ext, acc_a, acc_b);
    ip.tx_a = xa; ip.tx_b = xb; ip.ty_a = ya; ip.ty_b = yb;
    ip.pmod = pl->d_pmod;
    ip.pmod_s = pl->d_pmod_s;
    CKS(inner_product_launch(ip, ctx->d_slots, st));
    // (add_a, add_b): a ciphertext at the output level added inside the ModDown epilogue
    return stage3_core(ctx, md, acc_a, acc_b, acc_a + (size_t)md->l * n, acc_b + (size_t)md->l * n,
                       add_b, out_a, out_b, st, 0, add_a, pl->ws_conv, pl->ws_pc);
}

// ModDown of `count` Q||P accumulators at once (the inner sums of the moving giant steps of a
// BSGS transform): the same five kernels as ckks_ks_stage3, each over count times the rows, instead
// of count chains of five small launches.  Element g works in the arena of lane (current + g); qp
// is [count][2][l + alpha][n], out [count][2][l][n].  N = 2^16, count <= 4.
static int stage3_batch_core(ckks_ctx* ctx, int32_t plan, int count, int halves, const uint32_t* qp,
                             uint32_t* out, cudaStream_t st) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    if (count < 1 || halves * count > kMaxBconvJobs || ctx->lane + count > ctx->lanes) {
        set_last_error("batched ModDown of %d accumulators needs that many lanes from the current one and at most %d polynomials",
                       count, kMaxBconvJobs);
        return CKKS_ERR_ARG;
    }
    if (!ntt_can_fuse_moddown(pl->n) || ctx->ws_words % pl->n) { set_last_error("batched ModDown needs N = 2^16"); return CKKS_ERR_UNSUPPORTED; }
    const size_t n = pl->n;
    const int l = pl->l, alpha = pl->alpha, ext = pl->ext;
    const int key = count * 4 + halves;
    auto it = pl->s3_batch.find(key);
    if (it == pl->s3_batch.end() || it->second.lane_words != ctx->ws_words) {
        // rows of element g: accumulator at g * 2 ext (+ ext for the b half), workspace at g lanes
        const int32_t lane_rows = (int32_t)(ctx->ws_words / n);
        std::vector<int32_t> in_row, pc_row, p_slot, conv_row, q_slot;
        std::vector<int32_t> ps(2 * alpha), qs(2 * l);
        CK(cudaMemcpy(ps.data(), pl->d_s3_p_slot, sizeof(int32_t) * 2 * alpha, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(qs.data(), pl->d_s3_q_slot, sizeof(int32_t) * 2 * l, cudaMemcpyDeviceToHost));
        for (int g = 0; g < count; ++g)
            for (int h = 0; h < halves; ++h) {
                for (int j = 0; j < alpha; ++j) {
                    in_row.push_back(g * 2 * ext + h * ext + l + j);
                    pc_row.push_back(g * lane_rows + h * alpha + j);
                    p_slot.push_back(ps[h * alpha + j]);
                }
                for (int i = 0; i < l; ++i) {
                    conv_row.push_back(g * lane_rows + h * l + i);
                    q_slot.push_back(qs[h * l + i]);
                }
            }
        KsPlan::BatchMaps m{};
        CKS(upload(in_row, &m.in_row));
        CKS(upload(pc_row, &m.pc_row));
        CKS(upload(p_slot, &m.p_slot));
        CKS(upload(conv_row, &m.conv_row));
        CKS(upload(q_slot, &m.q_slot));
        m.lane_words = ctx->ws_words;
        for (void* ptr : {(void*)m.in_row, (void*)m.pc_row, (void*)m.p_slot, (void*)m.conv_row, (void*)m.q_slot})
            ctx->owned.push_back(ptr);
        it = pl->s3_batch.insert_or_assign(key, m).first;
    }
    const KsPlan::BatchMaps& m = it->second;
    CKS(ntt_launch(qp, pl->ws_pc, m.p_slot, ctx->d_slots, RowMap{m.in_row, m.pc_row}, count * halves * alpha, pl->n, 1, st));
    BconvJobs jobs;
    jobs.count = halves * count;
    for (int g = 0; g < count; ++g)
        for (int h = 0; h < halves; ++h) {
            BconvJob& j = jobs.job[halves * g + h];
            j.tab = ctx->tables[pl->moddown_table]->dev;
            j.in = pl->ws_pc + (size_t)g * ctx->ws_words + (size_t)h * alpha * n;
            j.in_stride = n;
            j.out = pl->ws_conv + (size_t)g * ctx->ws_words + (size_t)h * l * n;
            j.out_stride = n;
            j.out_row = nullptr;
        }
    CKS(bconv_launch_jobs(jobs, ctx->d_slots, n, st));
    ModDownEpilogueArgs e{};
    e.xq_a = qp; e.xq_b = qp + (size_t)ext * n; e.conv = pl->ws_conv; e.fold_a = nullptr; e.fold_b = nullptr;
    e.out_a = out; e.out_b = out + (size_t)l * n;
    e.q_slot = pl->d_q_slot; e.pinv = pl->d_pinv; e.pinv_s = pl->d_pinv_s;
    e.l = l; e.n = pl->n; e.galois = 0; e.lg = log2u(pl->n);
    e.xq_stride = (size_t)2 * ext * n;
    e.out_stride = (size_t)halves * l * n;
    e.halves = halves;
    return ntt_launch(pl->ws_conv, pl->ws_conv, m.q_slot, ctx->d_slots, RowMap{m.conv_row, m.conv_row},
                      count * halves * l, pl->n, 0, st, &e);
}

int ckks_ks_stage3_batch(ckks_ctx* ctx, int32_t plan, int count, const uint32_t* qp, uint32_t* out,
                         void* stream) {
    return stage3_batch_core(ctx, plan, count, 2, qp, out, (cudaStream_t)stream);
}

// The a halves only: qp is still [count][2][l + alpha][n] (the b halves are skipped), out is
// [count][l][n].  For giant steps whose b half stays over Q||P (ckks_ks_accumulate_rot_qp).
int ckks_ks_stage3_batch_a(ckks_ctx* ctx, int32_t plan, int count, const uint32_t* qp, uint32_t* out,
                           void* stream) {
    return stage3_batch_core(ctx, plan, count, 1, qp, out, (cudaStream_t)stream);
}

// ---- giant steps sharing one ModDown ---------------------------------------------------
// ModDown is linear up to its rounding, so the key switches of several independent
// ciphertexts that are summed afterwards (the giant steps of a BSGS linear transform)
// can add their stage-2 accumulators over Q||P and be scaled down once.

int ckks_ks_accumulate(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* evk,
                       int first, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, ct_a, pl->ws_raised, false, st));
    InnerProductArgs ip = ip_args(pl, ct_a, pl->ws_raised, evk, 0, pl->ext, pl->ws_acc,
                                  pl->ws_acc + (size_t)pl->ext * n);
    ip.accumulate = first ? 0 : 1;
    return inner_product_launch(ip, ctx->d_slots, st);
}

// Same for a ROTATED ciphertext without materialising the rotation: ModUp of the unrotated a
// part, the automorphism applied as a gather inside the inner product (sigma_k commutes with
// ModUp up to a multiple of the digit modulus), and P * sigma_k(ct_b) lifted into the b
// accumulator, so the shared ModDown returns sum_g KS(sigma_g(a_g)) + sigma_g(b_g).
int ckks_ks_accumulate_rot(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* ct_b,
                           uint32_t k, const uint32_t* evk, int first, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (!(k & 1)) { set_last_error("automorphism index must be odd"); return CKKS_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, ct_a, pl->ws_raised, false, st));
    InnerProductArgs ip = ip_args(pl, ct_a, pl->ws_raised, evk, 0, pl->ext, pl->ws_acc,
                                  pl->ws_acc + (size_t)pl->ext * n);
    ip.galois = k & (2 * pl->n - 1);
    ip.lift_b = ct_b;
    ip.pmod = pl->d_pmod;
    ip.pmod_s = pl->d_pmod_s;
    ip.accumulate = first ? 0 : 1;
    return inner_product_launch(ip, ctx->d_slots, st);
}

// Giant step of a double-hoisted BSGS transform whose inner sum (u_a, u_b) lives over Q||P: only
// u_a is scaled down (ct_a = ModDown(u_a), [l][n]) and switched; u_b ([ext][n]) is added to the
// b accumulator through the automorphism AS IT IS -- no ModDown, no lift by P, one rounding less
// than ckks_ks_accumulate_rot on (ModDown(u_a), ModDown(u_b)).
int ckks_ks_accumulate_rot_qp(ckks_ctx* ctx, int32_t plan, const uint32_t* ct_a, const uint32_t* b_qp,
                              uint32_t k, const uint32_t* evk, int first, void* stream) {
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    if (!(k & 1)) { set_last_error("automorphism index must be odd"); return CKKS_ERR_ARG; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(stage1_core(ctx, pl, ct_a, pl->ws_raised, false, st));
    InnerProductArgs ip = ip_args(pl, ct_a, pl->ws_raised, evk, 0, pl->ext, pl->ws_acc,
                                  pl->ws_acc + (size_t)pl->ext * n);
    ip.galois = k & (2 * pl->n - 1);
    ip.lift_qp = b_qp;
    ip.accumulate = first ? 0 : 1;
    return inner_product_launch(ip, ctx->d_slots, st);
}

int ckks_ks_finish(ckks_ctx* ctx, int32_t plan, int lanes_used, const uint32_t* fold_a,
                   const uint32_t* fold_b, uint32_t* out_a, uint32_t* out_b, void* stream) {
    // the accumulators of lanes [current lane, current lane + lanes_used) are summed into the
    // current lane's (the caller's home lane; 0 outside nested forks)
    if (!ctx || lanes_used < 1 || ctx->lane + lanes_used > ctx->lanes) { set_last_error("bad lane count %d", lanes_used); return CKKS_ERR_ARG; }
    KsPlan* pl;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(lane_reduce_launch(pl->ws_acc, ctx->ws_words, lanes_used, pl->d_ext_slot, ctx->d_slots, pl->ext, n, st));
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    return stage3_core(ctx, pl, acc_a, acc_b, acc_a + (size_t)pl->l * n, acc_b + (size_t)pl->l * n,
                       fold_b, out_a, out_b, st, 0, fold_a);
}

// ckks_ks_finish followed by a rescale by the top limbs, as ONE division: (fold_a, fold_b) is
// lifted into the accumulator (times P) during the lane reduction, raw_qp (a [2][ext][n]
// accumulator already over Q||P, e.g. the unrotated inner sum) is added as is, and the ModDown plan
// `md_plan` (Q_{l-k} with P' = {q_{l-k}..q_{l-1}} U P, as in ckks_ks_relin_rescale) divides
// everything by P * q_{l-1} ... q_{l-k}.  out_a / out_b have l - k rows.
int ckks_ks_finish_rescale(ckks_ctx* ctx, int32_t plan, int32_t md_plan, int lanes_used,
                           const uint32_t* fold_a, const uint32_t* fold_b, const uint32_t* raw_qp,
                           uint32_t* out_a, uint32_t* out_b, void* stream) {
    if (!ctx || lanes_used < 1 || ctx->lane + lanes_used > ctx->lanes) { set_last_error("bad lane count %d", lanes_used); return CKKS_ERR_ARG; }
    KsPlan *pl, *md;
    CKS(get_plan(ctx, plan, &pl));
    CKS(need_full_plan(pl));
    CKS(get_plan(ctx, md_plan, &md));
    if (md->n != pl->n || md->l + md->alpha != pl->ext || md->l >= pl->l) {
        set_last_error("ModDown plan (l=%d, alpha=%d) does not tile the key-switch accumulator (l=%d, ext=%d)",
                       md->l, md->alpha, pl->l, pl->ext);
        return CKKS_ERR_ARG;
    }
    if (md->alpha > pl->alpha + kMaxMergedDrop) { set_last_error("merged rescale drops more than %d limbs", kMaxMergedDrop); return CKKS_ERR_UNSUPPORTED; }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t n = pl->n;
    CKS(lane_reduce_launch(pl->ws_acc, ctx->ws_words, lanes_used, pl->d_ext_slot, ctx->d_slots, pl->ext, n, st,
                           fold_a, fold_b, pl->d_pmod, pl->d_pmod_s, pl->l, raw_qp));
    uint32_t* acc_a = pl->ws_acc;
    uint32_t* acc_b = pl->ws_acc + (size_t)pl->ext * n;
    return stage3_core(ctx, md, acc_a, acc_b, acc_a + (size_t)md->l * n, acc_b + (size_t)md->l * n,
                       nullptr, out_a, out_b, st, 0, nullptr, pl->ws_conv, pl->ws_pc);
}

}  // extern "C"
