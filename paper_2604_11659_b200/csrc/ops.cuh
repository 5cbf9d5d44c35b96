// Declarations of the device operations (ops.cu) used by the C-ABI layer.
#pragma once
#include "ntt.cuh"

namespace hs {

// Limb index within an item -> prime index.
struct PrimeMap {
    unsigned char p[64];
    int nl;
};

// Per-item pointer: table of pointers, or base + b * stride.
struct ItemPtr {
    const u64* const* tab;
    const u64* base;
    size_t stride;
    HS_DEV const u64* at(int b) const { return tab ? tab[b] : base + (size_t)b * stride; }
    HS_DEV u64* atw(int b) const { return const_cast<u64*>(at(b)); }
};

inline ItemPtr strided(const u64* base, size_t stride) { return ItemPtr{nullptr, base, stride}; }
inline ItemPtr table(const u64* const* tab) { return ItemPtr{tab, nullptr, 0}; }

PrimeConst make_prime_const(u64 q, u32 n);
long long launch_count();

// In-step kernel timer (bench.py's roofline line).  hs_probe_arm(kind) arms
// one kernel class; every launch of that class then records a CUDA event
// pair on its own launching stream around it, with the launch's algorithmic
// DRAM bytes and integer work (butterflies or 64x64 MACs).  hs_probe_read
// synchronises and returns {launches, total ms, bytes, work}.
enum ProbeKind { PROBE_NONE = 0, PROBE_MODUP = 1, PROBE_KS_INNER = 2, PROBE_KEYGEN = 3, PROBE_KINDS = 4 };
struct ProbeScope {
    int slot = -1;
    cudaStream_t st;
    ProbeScope(int kind, cudaStream_t st, double bytes, double work, int launches = 1);
    ~ProbeScope();
};
inline PrimeMap prime_map_range(int first, int count) {
    PrimeMap m{};
    m.nl = count;
    for (int i = 0; i < count && i < 64; i++) m.p[i] = (unsigned char)(first + i);
    return m;
}

// ---- batched transforms
void ntt_plain(const Dev& d, u64* buf, const u64* src, int njobs, const PrimeMap& pm, bool fwd,
               cudaStream_t st);

// ---- key switching
// Scratch (u64 elements) needed by key_switch_* for B items at level l.
size_t ks_scratch_elems(int B, int l, u32 n);
size_t ks_hoisted_scratch_elems(int R, int l, u32 n);

// Relinearize B degree-2 cts stored as [3][l+1][n] (ItemPtr ct3) -> out [2][l+1][n].
void relin_batch(const Dev& d, int B, int l, ItemPtr ct3, const u64* const* keys, ItemPtr out,
                 u64* scratch, cudaStream_t st);
// mult_ct fused with relinearize: out = relin(a (x) b) for B pairs at level l.
void mult_relin_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, const u64* const* keys,
                      ItemPtr out, u64* scratch, cudaStream_t st);
// mult_relin then rescale (with the mask product) of the result, merged:
// out = rescale(relin(a * b)) * mask at level l-1; top receives limb l only.
void mult_relin_rescale_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, const u64* const* keys,
                              ItemPtr mask_mont, ItemPtr top, ItemPtr out, u64* scratch, u64* U,
                              cudaStream_t st);
// Rotation of B cts at level l by Galois elements gal[b] with keys[b].
void rotate_batch(const Dev& d, int B, int l, ItemPtr ct, const u32* gal, const u64* const* keys,
                  ItemPtr out, u64* scratch, cudaStream_t st);
// Rotate B items and add them into acc [2][l+1][n] (one ModDown NTT per
// output limb); false (nothing launched) when the scratch is too small.
bool rotate_accumulate(const Dev& d, int B, int l, ItemPtr ct, const u32* gal, const u64* const* keys,
                       u64* acc, u64* scratch, cudaStream_t st, int nkeys);
// Same, items sorted by key in G runs: gs[0..G] (device) = run starts,
// head[b] (device) = 1 for the first item of a run.  ModUp and the inner
// product of the chain moduli run once per run (SURVEY P4 + linearity).
bool rotate_accumulate_grouped(const Dev& d, int B, int G, const int* gs, const unsigned char* head, int l,
                               ItemPtr ct, const u32* gal, const u64* const* keys, u64* acc, u64* scratch,
                               cudaStream_t st);
// Hoisted rotations of ONE source ct into R outputs (one per step).
void rotate_hoisted(const Dev& d, int R, int l, const u64* src, const u32* gal,
                    const u64* const* keys, ItemPtr out, u64* scratch, cudaStream_t st);

// ---- rescale (optionally fused with a plaintext-mask multiply after it)
size_t rescale_scratch_elems(int B, int npoly, u32 n);
void rescale_batch(const Dev& d, int B, int l, int npoly, ItemPtr in, ItemPtr out,
                   ItemPtr mask_mont, u64* scratch, cudaStream_t st);

// ---- elementwise
void tensor_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, ItemPtr out, cudaStream_t st);
void mult_pt_batch(const Dev& d, int B, int l, int npoly, ItemPtr ct, ItemPtr pt, ItemPtr out,
                   bool pt_mont, cudaStream_t st);
void add_batch(const Dev& d, int B, int l, int npoly, ItemPtr a, ItemPtr b, ItemPtr out,
               cudaStream_t st);
// acc[poly][m] += sum_b src(b)[poly][m]   (mod q_m), nl limbs per poly
void accumulate(const Dev& d, int B, int nl, int npoly, ItemPtr src, u64* acc, cudaStream_t st);
void to_montgomery(const Dev& d, u64* buf, size_t nlimb_total, const PrimeMap& pm, bool inverse,
                   cudaStream_t st);
// limbs[l][j] = coeffs[j] mod q_{pm[l]} for signed int64 coefficients
void signed_to_limbs(const Dev& d, const long long* coeffs, int nl, const PrimeMap& pm, u64* out,
                     cudaStream_t st);
// KSK assembly: b[i][m] = ntt_e[i][m] + [m<=L] f[i][m] target[m] - a[i][m] sk[m]
void ksk_combine(const Dev& d, u64* key, const u64* ntt_e, const u64* target, const u64* sk,
                 const ulonglong2* f, cudaStream_t st);
// Encryption combine: c0 = v pk_b + e0 + pt ; c1 = v pk_a + e1 (all NTT form, nl limbs)
void encrypt_combine(const Dev& d, int nl, const u64* v, const u64* pkb, const u64* pka,
                     const u64* e0, const u64* e1, const u64* pt, u64* ct, cudaStream_t st);
// Decrypt: pt[i] = c0[i] + c1[i] s[i]
void decrypt_combine(const Dev& d, int nl, const u64* ct, const u64* sk, u64* pt, cudaStream_t st);

// ---- on-device Galois key generation (keygen.cu)
void keygen_streams(const Dev& d, int K, const void* streams, u64* const* a_out, long long* e_out,
                    const void* jump, const void* zig, const u64* thr, cudaStream_t st);
size_t keygen_par_scratch_bytes(int K, u32 n, int L);
void keygen_streams_parallel(const Dev& d, int K, const void* streams, u64* const* a_out,
                             long long* e_out, const void* jump, const void* zig, const u64* thr,
                             void* scratch, int* err, cudaStream_t st);
void shoup_companions(const Dev& d, const u64* v, u64* sh, int nl, cudaStream_t st);
void keygen_assemble(const Dev& d, int K, u64* const* keys, const long long* e, const u32* gal,
                     const u64* sk, const ulonglong2* f, u64* skp, cudaStream_t st);
size_t keygen_assemble_scratch_bytes(int K, const Dev& d);

// data[i] mod q for limbs after an integer-sum collective
void reduce_mod(const Dev& d, u64* data, int npoly, int nl, cudaStream_t st);

// Seam kernels (single prime given by value, nlimb limbs of n)
enum SeamOp { SEAM_ADD, SEAM_SUB, SEAM_NEG, SEAM_MUL, SEAM_SCALAR, SEAM_FMA, SEAM_EXTEND };
void seam_op(int op, size_t count, const u64* a, const u64* b, u64* out, PrimeConst P, u64 s,
             u64 q_src, cudaStream_t st);

}  // namespace hs
