// C-ABI of libhespmm_b200.so (include/hespmm_b200.h): context/table setup,
// key management, primitive wrappers, the CSR x CSC planner and the batched
// SpMSpM executor.  Host code here only orchestrates; all limb arithmetic is
// in the sm_100a kernels of ops.cu / ntt.cuh.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/hespmm_b200.h"
#include "ops.cuh"

typedef unsigned __int128 u128;

namespace hs {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static u64 powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = (u64)((u128)r * b % q);
        b = (u64)((u128)b * b % q);
        e >>= 1;
    }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a % q, q - 2, q); }
static int bitlen(u64 q) { return 64 - __builtin_clzll(q); }
static u32 brev(u32 x, int bits) {
    u32 y = 0;
    for (int i = 0; i < bits; i++) { y = (y << 1) | (x & 1); x >>= 1; }
    return y;
}
static ulonglong2 shoup_pair(u64 w, u64 q) {
    ulonglong2 r;
    r.x = w;
    r.y = (u64)(((u128)w << 64) / q);
    return r;
}

PrimeConst make_prime_const(u64 q, u32 n) {
    PrimeConst P{};
    P.q = q;
    P.two_q = 2 * q;
    P.k = (u32)bitlen(q);
    P.mu64 = (u64)(((u128)1 << (63 + P.k)) / q);
    u64 inv = 1;                                   // Newton: q * inv == 1 mod 2^64
    for (int i = 0; i < 7; i++) inv *= 2 - q * inv;
    P.qinv_neg = (u64)0 - inv;
    P.r_mod = (u64)(((u128)1 << 64) % q);
    P.r2_mod = (u64)((u128)P.r_mod * P.r_mod % q);
    P.m64 = (u64)(((u128)1 << 64) / q);
    P.r_sh = (u64)(((u128)P.r_mod << 64) / q);
    if (n) {
        P.n_inv = invmod(n, q);
        P.n_inv_sh = (u64)(((u128)P.n_inv << 64) / q);
    }
    return P;
}

// psi: first g in [2, 1000) whose g^((q-1)/2n) has order exactly 2n
// (reference params.py:75-84).
static u64 find_psi(u64 q, u64 n) {
    u64 order = 2 * n;
    if ((q - 1) % order) return 0;
    u64 e = (q - 1) / order;
    for (u64 g = 2; g < 1000; g++) {
        u64 psi = powmod(g, e, q);
        if (powmod(psi, n, q) == q - 1) return psi;
    }
    return 0;
}

static bool is_prime_u64(u64 x) {
    if (x < 2) return false;
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    for (u64 p : bases)
        if (x % p == 0) return x == p;
    u64 d = x - 1;
    int r = 0;
    while (!(d & 1)) { d >>= 1; r++; }
    for (u64 a : bases) {
        u64 y = powmod(a, d, x);
        if (y == 1 || y == x - 1) continue;
        bool comp = true;
        for (int i = 0; i < r - 1; i++) {
            y = (u64)((u128)y * y % x);
            if (y == x - 1) { comp = false; break; }
        }
        if (comp) return false;
    }
    return true;
}

}  // namespace hs

using namespace hs;

#define CHECK_LAUNCH()                                                                 \
    do {                                                                               \
        cudaError_t e_ = cudaGetLastError();                                           \
        if (e_ != cudaSuccess) {                                                       \
            set_error(std::string("kernel launch failed: ") + cudaGetErrorString(e_)); \
            return (hs_status)HS_CUDA_ERROR;                                           \
        }                                                                              \
    } while (0)

#define ST(s) ((cudaStream_t)(s))

extern "C" {

const char* hs_last_error(void) { return g_err.c_str(); }
const char* hs_version(void) { return "hespmm_b200 0.1.0 (sm_100a)"; }
int64_t hs_launch_count(void) { return (int64_t)launch_count(); }

hs_status hs_ctx_create(hs_ctx** out, int device, uint32_t n, uint32_t levels,
                        const uint64_t* chain, uint64_t aux) {
    *out = nullptr;
    if (n < 8 || (n & (n - 1)) || n > (1u << 17)) {
        set_error("ring degree must be a power of two in [8, 2^17], got " + std::to_string(n));
        return (hs_status)HS_PARAMETER_ERROR;
    }
    if (levels < 1 || levels > 62) {
        set_error("levels must be in [1, 62]");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    HS_CUDA(cudaSetDevice(device));
    {
        // The runner's per-call work buffers come from the stream-ordered pool;
        // keep freed blocks cached instead of returning them to the driver at
        // every synchronisation (re-mapping GBs per matmul costs 100s of ms).
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    hs_ctx* c = new hs_ctx();
    c->device = device;
    c->n = n;
    c->log_n = __builtin_ctz(n);
    c->L = (int)levels;
    const int L = c->L, P = L + 2;
    c->primes.assign(chain, chain + L + 1);
    c->primes.push_back(aux);
    for (u64 q : c->primes) {
        // < 2^60: the kernels keep lazy residues in [0, 8q) and test signs (8q < 2^63)
        if (q >= (1ull << 60) || q < 3 || (q - 1) % (2ull * n) || !is_prime_u64(q)) {
            set_error("non-NTT-friendly prime (or >= 2^60) " + std::to_string(q));
            delete c;
            return (hs_status)HS_PARAMETER_ERROR;
        }
    }
    // per-prime constants and twiddles
    std::vector<ulonglong2> tw((size_t)P * n), itw((size_t)P * n);
    std::vector<double2> twd((size_t)P * n), itwd((size_t)P * n);
    std::vector<u64> pw(n), ipw(n);
    c->pc.resize(P);
    // NTT butterflies (both directions) on the FP64 pipe for primes <= 2^50 + 2^40 (every
    // scaling prime of a scale_bits <= 50 chain; ntt.cuh unit_butterflies_f64
    // states the bounds).  HS_NTT_F64=0 keeps every prime on the integer path.
    const char* f64env = getenv("HS_NTT_F64");
    // (the A/B-only fused ModUp + inner-product kernel finishes integer-path
    // forward NTTs itself, so it keeps every prime on the integer path)
    const bool f64_on = !(f64env && f64env[0] == '0') && !getenv("HS_MODUP_FUSED");
    for (int p = 0; p < P; p++) {
        u64 q = c->primes[p];
        c->pc[p] = make_prime_const(q, n);
        if (f64_on && q <= (1ull << 50) + (1ull << 40)) c->pc[p].pad |= PC_F64;
        u64 psi = find_psi(q, n);
        if (!psi) {
            set_error("no primitive 2n-th root for prime " + std::to_string(q));
            delete c;
            return (hs_status)HS_PARAMETER_ERROR;
        }
        u64 ipsi = invmod(psi, q);
        pw[0] = ipw[0] = 1;
        for (u32 k = 1; k < n; k++) {
            pw[k] = (u64)((u128)pw[k - 1] * psi % q);
            ipw[k] = (u64)((u128)ipw[k - 1] * ipsi % q);
        }
        for (u32 i = 0; i < n; i++) {
            u32 r = brev(i, c->log_n);
            tw[(size_t)p * n + i] = shoup_pair(pw[r], q);
            // w < 2^51 is exact in a double; RN(w / q) by one IEEE division of exact operands
            twd[(size_t)p * n + i] = make_double2((double)pw[r], (double)pw[r] / (double)q);
            itwd[(size_t)p * n + i] = make_double2((double)ipw[r], (double)ipw[r] / (double)q);
            itw[(size_t)p * n + i] = shoup_pair(ipw[r], q);
        }
    }
    // key-switch and rescale constants (reference context.py:39-53)
    // df: [L+1] digit factors, then [L+1] digit factors times 2^64 (for a
    // Montgomery-form digit source, csrc/ops.cu SrcTensor)
    std::vector<ulonglong2> df(2 * (L + 1)), auxinv(L + 1), qlinv((size_t)(L + 1) * (L + 1));
    c->df.resize(L + 1);
    c->auxinv.resize(L + 1);
    c->qlinv.assign((size_t)(L + 1) * (L + 1), 0);
    for (int i = 0; i <= L; i++) {
        u64 qi = c->primes[i], prod = 1;
        for (int j = 0; j <= L; j++)
            if (j != i) prod = (u64)((u128)prod * (c->primes[j] % qi) % qi);
        c->df[i] = invmod(prod, qi);
        df[i] = shoup_pair(c->df[i], qi);
        df[L + 1 + i] = shoup_pair((u64)(((u128)c->df[i] << 64) % qi), qi);
        c->auxinv[i] = invmod(aux % qi, qi);
        auxinv[i] = shoup_pair(c->auxinv[i], qi);
    }
    for (int lvl = 0; lvl <= L; lvl++)
        for (int i = 0; i < lvl; i++) {
            u64 v = invmod(c->primes[lvl] % c->primes[i], c->primes[i]);
            c->qlinv[(size_t)lvl * (L + 1) + i] = v;
            qlinv[(size_t)lvl * (L + 1) + i] = shoup_pair(v, c->primes[i]);
        }
    // one device blob: pc | tw | itw | df | auxinv | qlinv
    size_t off_pc = 0;
    size_t off_tw = (off_pc + P * sizeof(PrimeConst) + 255) & ~(size_t)255;
    size_t off_itw = off_tw + tw.size() * sizeof(ulonglong2);
    size_t off_df = off_itw + itw.size() * sizeof(ulonglong2);
    size_t off_ai = off_df + df.size() * sizeof(ulonglong2);
    size_t off_ql = off_ai + auxinv.size() * sizeof(ulonglong2);
    size_t off_twd = off_ql + qlinv.size() * sizeof(ulonglong2);
    off_twd = (off_twd + 255) & ~(size_t)255;
    size_t off_itwd = off_twd + twd.size() * sizeof(double2);
    size_t total = off_itwd + itwd.size() * sizeof(double2);
    cudaError_t e = cudaMalloc(&c->d_blob, total);
    if (e != cudaSuccess) {
        set_error(std::string("cudaMalloc tables: ") + cudaGetErrorString(e));
        delete c;
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    char* base = (char*)c->d_blob;
    cudaMemcpy(base + off_pc, c->pc.data(), P * sizeof(PrimeConst), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_tw, tw.data(), tw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_itw, itw.data(), itw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_df, df.data(), df.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_ai, auxinv.data(), auxinv.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_ql, qlinv.data(), qlinv.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + off_twd, twd.data(), twd.size() * sizeof(double2), cudaMemcpyHostToDevice);
    e = cudaMemcpy(base + off_itwd, itwd.data(), itwd.size() * sizeof(double2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        set_error(std::string("table upload: ") + cudaGetErrorString(e));
        cudaFree(c->d_blob);
        delete c;
        return (hs_status)HS_CUDA_ERROR;
    }
    Dev& d = c->dev;
    d.n = n;
    d.log_n = c->log_n;
    d.L = L;
    d.aux_q = aux;
    d.pc = (const PrimeConst*)(base + off_pc);
    d.tw = (const ulonglong2*)(base + off_tw);
    d.itw = (const ulonglong2*)(base + off_itw);
    d.df = (const ulonglong2*)(base + off_df);
    d.dfR = d.df + (L + 1);
    d.auxinv = (const ulonglong2*)(base + off_ai);
    d.qlinv = (const ulonglong2*)(base + off_ql);
    d.twd = (const double2*)(base + off_twd);
    d.itwd = (const double2*)(base + off_itwd);
    *out = c;
    return (hs_status)HS_OK;
}

void hs_ctx_destroy(hs_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->relin.d) cudaFree(c->relin.d);
    for (auto& kv : c->galois) cudaFree(kv.second.d);
    for (void* p : {(void*)c->d_jump, (void*)c->d_zig, (void*)c->d_thr, (void*)c->d_sk, (void*)c->d_kskf})
        if (p) cudaFree(p);
    if (c->d_blob) cudaFree(c->d_blob);
    if (c->d_kg_err) cudaFree(c->d_kg_err);
    for (u64* b : c->kpool_buf) cudaFree(b);
    for (auto e : c->kpool_gen_ev) cudaEventDestroy(e);
    for (auto e : c->kpool_use_ev) cudaEventDestroy(e);
    if (c->kpool_side) cudaStreamDestroy(c->kpool_side);
    for (auto s : c->kg_stream)
        if (s) cudaStreamDestroy(s);
    for (auto e : c->kg_event)
        if (e) cudaEventDestroy(e);
    delete c;
}

hs_status hs_ctx_tables(const hs_ctx* c, uint32_t p, uint64_t* roots, uint64_t* roots_sh,
                        uint64_t* iroots, uint64_t* iroots_sh, uint64_t* n_inv, uint64_t* mu) {
    if (!c || p >= c->primes.size()) {
        set_error("prime index out of range");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    const u32 n = c->n;
    std::vector<ulonglong2> tw(n), itw(n);
    cudaMemcpy(tw.data(), c->dev.tw + (size_t)p * n, n * sizeof(ulonglong2), cudaMemcpyDeviceToHost);
    HS_CUDA(cudaMemcpy(itw.data(), c->dev.itw + (size_t)p * n, n * sizeof(ulonglong2),
                       cudaMemcpyDeviceToHost));
    for (u32 i = 0; i < n; i++) {
        if (roots) roots[i] = tw[i].x;
        if (roots_sh) roots_sh[i] = tw[i].y;
        if (iroots) iroots[i] = itw[i].x;
        if (iroots_sh) iroots_sh[i] = itw[i].y;
    }
    u64 q = c->primes[p];
    if (n_inv) *n_inv = c->pc[p].n_inv;
    if (mu) *mu = (u64)(((u128)1 << (2 * bitlen(q))) / q);   // reference Barrett mu
    return (hs_status)HS_OK;
}

// ------------------------------------------------------------------ keys

static KeyBuf* key_slot(hs_ctx* c, int kind, uint32_t step, bool create) {
    if (kind == 0) {
        if (!c->relin.d && create) {
            if (cudaMalloc(&c->relin.d, c->key_bytes()) != cudaSuccess) return nullptr;
        }
        return c->relin.d ? &c->relin : nullptr;
    }
    auto it = c->galois.find(step);
    if (it != c->galois.end()) return &it->second;
    if (!create) return nullptr;
    KeyBuf kb;
    if (cudaMalloc(&kb.d, c->key_bytes()) != cudaSuccess) return nullptr;
    return &(c->galois[step] = kb);
}

static bool key_args_ok(hs_ctx* c, int kind, uint32_t step) {
    if (kind != 0 && kind != 1) {
        set_error("key kind must be 0 (relin) or 1 (galois)");
        return false;
    }
    if (kind == 1 && (step == 0 || step >= c->n / 2)) {
        set_error("rotation step " + std::to_string(step) + " out of range");
        return false;
    }
    return true;
}

hs_status hs_key_upload(hs_ctx* c, int kind, uint32_t step, const uint64_t* key, int on_host,
                        void* stream) {
    if (!key_args_ok(c, kind, step)) return (hs_status)HS_PARAMETER_ERROR;
    KeyBuf* kb = key_slot(c, kind, step, true);
    if (!kb) {
        set_error("out of device memory for key");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    HS_CUDA(cudaMemcpyAsync(kb->d, key, c->key_bytes(),
                            on_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ST(stream)));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

}  // extern "C"

namespace hs {
// HESP container KSK record (reference ckks/serial.py:48-66): u32 digits,
// then per digit the b poly and the a poly, each = u32 count followed by
// count x (u32 byte size = 8n, 8n bytes of little-endian uint64 limbs).
// Limbs sit at 4-byte (not 8-byte) alignment, so words are read as u32 pairs.
__global__ void hesp_ksk_gather_kernel(const unsigned* raw, u64* key, int L, u32 n) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int limb = blockIdx.y;                       // (c * (L+1) + i) * (L+2) + m
    const int m = limb % (L + 2), ci = limb / (L + 2);
    const int i = ci % (L + 1), c = ci / (L + 1);
    const size_t limb_rec = 4 + (size_t)8 * n;          // bytes
    const size_t poly_rec = 4 + (size_t)(L + 2) * limb_rec;
    const size_t off = 4 + (size_t)i * 2 * poly_rec + (size_t)c * poly_rec + 4 + (size_t)m * limb_rec + 4 +
                       (size_t)8 * j;                   // bytes from the record start
    const unsigned* w = raw + off / 4;
    key[(size_t)limb * n + j] = (u64)w[0] | ((u64)w[1] << 32);
}
}  // namespace hs

extern "C" {

hs_status hs_key_upload_hesp(hs_ctx* c, int kind, uint32_t step, const uint8_t* rec, int64_t rec_bytes,
                             void* stream) {
    if (!key_args_ok(c, kind, step)) return (hs_status)HS_PARAMETER_ERROR;
    const int L = c->L;
    const u32 n = c->n;
    const size_t limb_rec = 4 + (size_t)8 * n, poly_rec = 4 + (size_t)(L + 2) * limb_rec;
    const size_t need = 4 + (size_t)(L + 1) * 2 * poly_rec;
    if ((size_t)rec_bytes != need || ((uintptr_t)rec & 3)) {
        set_error("hs_key_upload_hesp: record size " + std::to_string(rec_bytes) + " != " +
                  std::to_string(need) + " (or misaligned)");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    KeyBuf* kb = key_slot(c, kind, step, true);
    if (!kb) {
        set_error("out of device memory for key");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    hesp_ksk_gather_kernel<<<dim3((n + 255) / 256, 2 * (L + 1) * (L + 2)), 256, 0, ST(stream)>>>(
        (const unsigned*)rec, kb->d, L, n);
    note_launch();
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_key_generate(hs_ctx* c, int kind, uint32_t step, const uint64_t* a, const int64_t* e,
                          const uint64_t* target, const uint64_t* sk, void* stream) {
    if (!key_args_ok(c, kind, step)) return (hs_status)HS_PARAMETER_ERROR;
    KeyBuf* kb = key_slot(c, kind, step, true);
    if (!kb) {
        set_error("out of device memory for key");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    const int L = c->L;
    const u32 n = c->n;
    const size_t half = (size_t)(L + 1) * (L + 2) * n;
    cudaStream_t st = ST(stream);
    // a component straight into the key; e limbs (NTT) into the b half, then combine in place
    HS_CUDA(cudaMemcpyAsync(kb->d + half, a, half * sizeof(u64), cudaMemcpyDeviceToDevice, st));
    u64* ntt_e = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&ntt_e, half * sizeof(u64), st));
    for (int i = 0; i <= L; i++)
        signed_to_limbs(c->dev, (const long long*)e + (size_t)i * n, L + 2, prime_map_range(0, L + 2),
                        ntt_e + (size_t)i * (L + 2) * n, st);
    ntt_plain(c->dev, ntt_e, nullptr, (L + 1) * (L + 2), prime_map_range(0, L + 2), true, st);
    // KSK factors p * (Q_L / q_i) mod q_m (context.py:45-48)
    std::vector<ulonglong2> f((size_t)(L + 1) * (L + 1));
    for (int i = 0; i <= L; i++)
        for (int m = 0; m <= L; m++) {
            u64 qm = c->primes[m], v = c->primes[L + 1] % qm;
            for (int j = 0; j <= L; j++)
                if (j != i) v = (u64)((u128)v * (c->primes[j] % qm) % qm);
            f[(size_t)i * (L + 1) + m] = shoup_pair(v, qm);
        }
    ulonglong2* d_f = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&d_f, f.size() * sizeof(ulonglong2), st));
    HS_CUDA(cudaMemcpyAsync(d_f, f.data(), f.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice, st));
    ksk_combine(c->dev, kb->d, ntt_e, target, sk, d_f, st);
    CHECK_LAUNCH();
    HS_CUDA(cudaStreamSynchronize(st));   // f is a stack vector
    cudaFreeAsync(ntt_e, st);
    cudaFreeAsync(d_f, st);
    return (hs_status)HS_OK;
}

hs_status hs_key_download(hs_ctx* c, int kind, uint32_t step, uint64_t* out, void* stream) {
    if (!key_args_ok(c, kind, step)) return (hs_status)HS_PARAMETER_ERROR;
    KeyBuf* kb = key_slot(c, kind, step, false);
    if (!kb) {
        set_error("no such key");
        return (hs_status)HS_KEY_MISSING;
    }
    HS_CUDA(cudaMemcpyAsync(out, kb->d, c->key_bytes(), cudaMemcpyDeviceToDevice, ST(stream)));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

int hs_key_has(const hs_ctx* c, int kind, uint32_t step) {
    if (kind == 0) return c->relin.d != nullptr;
    return c->galois.count(step) ? 1 : 0;
}

hs_status hs_key_drop(hs_ctx* c, int kind, uint32_t step) {
    if (kind == 0) {
        if (c->relin.d) cudaFree(c->relin.d);
        c->relin.d = nullptr;
    } else {
        auto it = c->galois.find(step);
        if (it != c->galois.end()) {
            cudaFree(it->second.d);
            c->galois.erase(it);
        }
    }
    return (hs_status)HS_OK;
}

int64_t hs_key_count(const hs_ctx* c) { return (int64_t)c->galois.size() + (c->relin.d ? 1 : 0); }

// ----------------------------------------------------------- limb kernels

static bool prime_range_ok(hs_ctx* c, int first, int count) {
    if (first < 0 || count < 0 || first + count > c->L + 2 || count > 64) {
        set_error("prime range out of bounds");
        return false;
    }
    return true;
}

hs_status hs_ntt(hs_ctx* c, uint64_t* data, int32_t nitems, int32_t nlimbs, int32_t first,
                 int32_t inverse, void* stream) {
    if (!prime_range_ok(c, first, nlimbs)) return (hs_status)HS_PARAMETER_ERROR;
    ntt_plain(c->dev, data, nullptr, nitems * nlimbs, prime_map_range(first, nlimbs), !inverse,
              ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_signed_to_ntt(hs_ctx* c, const int64_t* coeffs, int32_t nlimbs, int32_t first,
                           uint64_t* out, void* stream) {
    if (!prime_range_ok(c, first, nlimbs)) return (hs_status)HS_PARAMETER_ERROR;
    PrimeMap pm = prime_map_range(first, nlimbs);
    signed_to_limbs(c->dev, (const long long*)coeffs, nlimbs, pm, out, ST(stream));
    ntt_plain(c->dev, out, nullptr, nlimbs, pm, true, ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_seam_op(int32_t op, uint64_t count, const uint64_t* a, const uint64_t* b, uint64_t* out,
                     uint64_t q, uint64_t s, uint64_t q_src, void* stream) {
    if (op < 0 || op > SEAM_EXTEND || q < 3 || q >= (1ull << 60)) {
        set_error("bad seam op or modulus");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    seam_op(op, count, a, b, out, make_prime_const(q, 0), s, q_src, ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

}  // extern "C"

namespace {
__global__ void zip_kernel(const u64* a, const u64* b, ulonglong2* out, u32 n) {
    u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = make_ulonglong2(a[k], b[k]);
}
struct SeamTables {
    PrimeConst* pc = nullptr;
    ulonglong2* tw = nullptr;
};
}  // namespace

extern "C" {

hs_status hs_seam_ntt(uint64_t* a, uint32_t n, uint64_t q, const uint64_t* roots,
                      const uint64_t* roots_sh, uint64_t n_inv, int32_t inverse, void* stream) {
    if (n < 8 || (n & (n - 1)) || n > (1u << 17)) {
        set_error("bad ring degree");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    if (q < 3 || q >= (1ull << 60)) {
        set_error("bad modulus (the kernels need q < 2^60)");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    // Tables are rebuilt per call from the caller's arrays (the seam is for API
    // compatibility, not the hot path), so no stale cache can alias them.
    cudaStream_t st = ST(stream);
    PrimeConst P = make_prime_const(q, n);
    P.n_inv = n_inv;
    P.n_inv_sh = (u64)(((u128)n_inv << 64) / q);
    SeamTables t;
    HS_CUDA(cudaMallocAsync((void**)&t.pc, sizeof(PrimeConst), st));
    HS_CUDA(cudaMallocAsync((void**)&t.tw, (size_t)n * sizeof(ulonglong2), st));
    HS_CUDA(cudaMemcpyAsync(t.pc, &P, sizeof(P), cudaMemcpyHostToDevice, st));
    zip_kernel<<<(n + 255) / 256, 256, 0, st>>>(roots, roots_sh, t.tw, n);
    note_launch();
    Dev d{};
    d.n = n;
    d.log_n = __builtin_ctz(n);
    d.L = -1;
    d.pc = t.pc;
    d.tw = t.tw;
    d.itw = t.tw;
    PrimeMap pm = prime_map_range(0, 1);
    ntt_plain(d, a, nullptr, 1, pm, !inverse, st);
    CHECK_LAUNCH();
    HS_CUDA(cudaStreamSynchronize(st));   // P lives on this stack frame
    cudaFreeAsync(t.pc, st);
    cudaFreeAsync(t.tw, st);
    return (hs_status)HS_OK;
}

// -------------------------------------------------------- CKKS primitives

static bool level_ok(hs_ctx* c, uint32_t level) {
    if ((int)level > c->L) {
        set_error("level " + std::to_string(level) + " outside chain bounds");
        return false;
    }
    return true;
}

hs_status hs_eval_add(hs_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out, uint32_t level,
                      void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    add_batch(c->dev, 1, level, 2, strided(a, 0), strided(b, 0), strided(out, 0), ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_eval_mult_ct(hs_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out3,
                          uint32_t level, void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    tensor_batch(c->dev, 1, level, strided(a, 0), strided(b, 0), strided(out3, 0), ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_eval_mult_pt(hs_ctx* c, const uint64_t* ct, const uint64_t* pt, uint64_t* out,
                          uint32_t npoly, uint32_t level, int32_t pt_mont, void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    mult_pt_batch(c->dev, 1, level, npoly, strided(ct, 0), strided(pt, 0), strided(out, 0),
                  pt_mont != 0, ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

}  // extern "C"

template <class T>
static hs_status alloc_async(T** p, size_t count, cudaStream_t st) {
    HS_CUDA(cudaMallocAsync((void**)p, count * sizeof(T), st));
    return (hs_status)HS_OK;
}

static hs_status key_ptr_array(hs_ctx* c, const std::vector<const u64*>& keys, const u64*** out,
                               cudaStream_t st) {
    if (alloc_async(out, keys.size(), st)) return (hs_status)HS_OUT_OF_MEMORY;
    HS_CUDA(cudaMemcpyAsync((void*)*out, keys.data(), keys.size() * sizeof(u64*),
                            cudaMemcpyHostToDevice, st));
    return (hs_status)HS_OK;
}

extern "C" {

hs_status hs_relinearize(hs_ctx* c, const uint64_t* ct3, uint64_t* out, uint32_t level, void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    if (!c->relin.d) {
        set_error("no relinearization key in bundle");
        return (hs_status)HS_KEY_MISSING;
    }
    cudaStream_t st = ST(stream);
    u64* scratch;
    const u64** keys;
    if (alloc_async(&scratch, ks_scratch_elems(1, level, c->n), st)) return (hs_status)HS_OUT_OF_MEMORY;
    if (key_ptr_array(c, {c->relin.d}, &keys, st)) return (hs_status)HS_CUDA_ERROR;
    relin_batch(c->dev, 1, level, strided(ct3, 0), keys, strided(out, 0), scratch, st);
    CHECK_LAUNCH();
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(scratch, st);
    cudaFreeAsync((void*)keys, st);
    return (hs_status)HS_OK;
}

hs_status hs_rescale(hs_ctx* c, const uint64_t* ct, uint64_t* out, uint32_t npoly, uint32_t level,
                     void* stream) {
    if (level == 0) {
        set_error("modulus chain exhausted: cannot rescale at level 0");
        return (hs_status)HS_EVAL_ERROR;
    }
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    cudaStream_t st = ST(stream);
    u64* T;
    if (alloc_async(&T, rescale_scratch_elems(1, npoly, c->n), st)) return (hs_status)HS_OUT_OF_MEMORY;
    rescale_batch(c->dev, 1, level, npoly, strided(ct, 0), strided(out, 0), ItemPtr{nullptr, nullptr, 0},
                  T, st);
    CHECK_LAUNCH();
    cudaFreeAsync(T, st);
    return (hs_status)HS_OK;
}

static u32 galois_elt(u32 step, u32 n) { return (u32)powmod(5, step, 2ull * n); }

hs_status hs_eval_rotate(hs_ctx* c, const uint64_t* ct, uint64_t* out, uint32_t level, uint32_t step,
                         void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    auto it = c->galois.find(step);
    if (it == c->galois.end()) {
        set_error("missing Galois key for step " + std::to_string(step));
        return (hs_status)HS_KEY_MISSING;
    }
    cudaStream_t st = ST(stream);
    u64* scratch;
    const u64** keys;
    u32* gal;
    u32 g = galois_elt(step, c->n);
    if (alloc_async(&scratch, ks_scratch_elems(1, level, c->n), st)) return (hs_status)HS_OUT_OF_MEMORY;
    if (key_ptr_array(c, {it->second.d}, &keys, st)) return (hs_status)HS_CUDA_ERROR;
    if (alloc_async(&gal, 1, st)) return (hs_status)HS_OUT_OF_MEMORY;
    HS_CUDA(cudaMemcpyAsync(gal, &g, sizeof(u32), cudaMemcpyHostToDevice, st));
    rotate_batch(c->dev, 1, level, strided(ct, 0), gal, keys, strided(out, 0), scratch, st);
    CHECK_LAUNCH();
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(scratch, st);
    cudaFreeAsync((void*)keys, st);
    cudaFreeAsync(gal, st);
    return (hs_status)HS_OK;
}

hs_status hs_eval_rotate_hoisted(hs_ctx* c, const uint64_t* ct, uint64_t* const* outs,
                                 const uint32_t* steps, int32_t nsteps, uint32_t level, void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    if (nsteps <= 0) return (hs_status)HS_OK;
    std::vector<const u64*> keys(nsteps);
    std::vector<u32> gal(nsteps);
    for (int k = 0; k < nsteps; k++) {
        auto it = c->galois.find(steps[k]);
        if (it == c->galois.end()) {
            set_error("missing Galois key for step " + std::to_string(steps[k]));
            return (hs_status)HS_KEY_MISSING;
        }
        keys[k] = it->second.d;
        gal[k] = galois_elt(steps[k], c->n);
    }
    cudaStream_t st = ST(stream);
    u64* scratch;
    const u64** d_keys;
    u32* d_gal;
    u64** d_outs;
    if (alloc_async(&scratch, ks_hoisted_scratch_elems(nsteps, level, c->n), st))
        return (hs_status)HS_OUT_OF_MEMORY;
    if (key_ptr_array(c, keys, &d_keys, st)) return (hs_status)HS_CUDA_ERROR;
    if (alloc_async(&d_gal, nsteps, st) || alloc_async(&d_outs, nsteps, st))
        return (hs_status)HS_OUT_OF_MEMORY;
    HS_CUDA(cudaMemcpyAsync(d_gal, gal.data(), nsteps * sizeof(u32), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_outs, outs, nsteps * sizeof(u64*), cudaMemcpyHostToDevice, st));
    rotate_hoisted(c->dev, nsteps, level, ct, d_gal, d_keys, table((const u64* const*)d_outs), scratch,
                   st);
    CHECK_LAUNCH();
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(scratch, st);
    cudaFreeAsync((void*)d_keys, st);
    cudaFreeAsync(d_gal, st);
    cudaFreeAsync(d_outs, st);
    return (hs_status)HS_OK;
}

hs_status hs_encrypt(hs_ctx* c, const int64_t* v, const int64_t* e0, const int64_t* e1,
                     const uint64_t* pk_b, const uint64_t* pk_a, const uint64_t* pt, uint32_t level,
                     uint64_t* ct, void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_PARAMETER_ERROR;
    cudaStream_t st = ST(stream);
    const int nl = level + 1;
    const size_t lim = (size_t)nl * c->n;
    u64* tmp;
    if (alloc_async(&tmp, 3 * lim, st)) return (hs_status)HS_OUT_OF_MEMORY;
    PrimeMap pm = prime_map_range(0, nl);
    signed_to_limbs(c->dev, (const long long*)v, nl, pm, tmp, st);
    signed_to_limbs(c->dev, (const long long*)e0, nl, pm, tmp + lim, st);
    signed_to_limbs(c->dev, (const long long*)e1, nl, pm, tmp + 2 * lim, st);
    ntt_plain(c->dev, tmp, nullptr, 3 * nl, pm, true, st);
    encrypt_combine(c->dev, nl, tmp, pk_b, pk_a, tmp + lim, tmp + 2 * lim, pt, ct, st);
    CHECK_LAUNCH();
    cudaFreeAsync(tmp, st);
    return (hs_status)HS_OK;
}

hs_status hs_decrypt(hs_ctx* c, const uint64_t* ct, const uint64_t* sk, uint32_t level, uint64_t* pt,
                     void* stream) {
    if (!level_ok(c, level)) return (hs_status)HS_EVAL_ERROR;
    decrypt_combine(c->dev, level + 1, ct, sk, pt, ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

hs_status hs_to_montgomery(hs_ctx* c, uint64_t* data, int32_t nitems, int32_t nlimbs, int32_t first,
                           int32_t inverse, void* stream) {
    if (!prime_range_ok(c, first, nlimbs)) return (hs_status)HS_PARAMETER_ERROR;
    to_montgomery(c->dev, data, (size_t)nitems * nlimbs, prime_map_range(first, nlimbs), inverse != 0,
                  ST(stream));
    CHECK_LAUNCH();
    return (hs_status)HS_OK;
}

}  // extern "C"
