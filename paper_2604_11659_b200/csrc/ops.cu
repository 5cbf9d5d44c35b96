#include <algorithm>
// Device operations of the encrypted SpMSpM path: limb kernels, key
// switching (decompose -> ModUp -> key inner product -> ModDown), rescale,
// tensor product, NTT-domain Galois automorphism, accumulation.
//
// Reference semantics (paths relative to /root/reference/pkg/src/hespmm/):
//   key switch     ckks/context.py:462-498
//   relinearize    ckks/context.py:363-380 (+ _digits_from_ntt :454-460)
//   rescale        ckks/context.py:382-399
//   eval_rotate    ckks/context.py:401-452
//   mult_ct / pt   ckks/context.py:334-361
// Every kernel writes canonical residues, so results are bit-identical to
// the reference regardless of the (lazy) reduction strategy used inside.
#include "ops.cuh"

#include <atomic>
#include <cstdlib>
#include <vector>

namespace hs {

static std::atomic<long long> g_launches{0};
void note_launch(int count) { g_launches += count; }
long long launch_count() { return g_launches.load(); }

// ---- in-step kernel timer
namespace {
struct ProbeRec {
    cudaEvent_t e0, e1;
    int kind, launches;
    double bytes, work;
};
std::vector<ProbeRec> g_probe;       // event pool; [0, g_probe_used) recorded since the last read
size_t g_probe_used = 0;
int g_probe_kind = 0;                // bit k arms kind k
}  // namespace

ProbeScope::ProbeScope(int kind, cudaStream_t s, double bytes, double work, int launches) : st(s) {
    if (kind == PROBE_NONE || !((g_probe_kind >> kind) & 1)) return;
    if (g_probe_used == g_probe.size()) {
        ProbeRec r{};
        if (cudaEventCreate(&r.e0) != cudaSuccess || cudaEventCreate(&r.e1) != cudaSuccess) return;
        g_probe.push_back(r);
    }
    slot = (int)g_probe_used++;
    ProbeRec& r = g_probe[slot];
    r.kind = kind;
    r.launches = launches;
    r.bytes = bytes;
    r.work = work;
    cudaEventRecord(r.e0, st);
}
ProbeScope::~ProbeScope() {
    if (slot >= 0) cudaEventRecord(g_probe[slot].e1, st);
}
void probe_arm(int mask) {
    g_probe_kind = mask;
    g_probe_used = 0;
}
// {launches, total ms, algorithmic bytes, integer work} of the launches of
// `kind` recorded since the last arm (arming again clears the record).
int probe_read(int kind, double* out4) {
    out4[0] = out4[1] = out4[2] = out4[3] = 0.0;
    for (size_t k = 0; k < g_probe_used; k++) {
        ProbeRec& r = g_probe[k];
        if (r.kind != kind) continue;
        if (cudaEventSynchronize(r.e1) != cudaSuccess) return 1;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.e0, r.e1) != cudaSuccess) return 1;
        out4[0] += r.launches;
        out4[1] += ms;
        out4[2] += r.bytes;
        out4[3] += r.work;
    }
    return 0;
}

// =========================================================== helpers

HS_DEV u64 canon4(u64 v, const PrimeConst& P) {    // [0,4q) -> [0,q)
    return csub(csub(v, P.two_q), P.q);
}

// 128-bit multiply-accumulate (hi:lo) += a*b.
HS_DEV void mac128(u64& lo, u64& hi, u64 a, u64 b) {
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\t"
        "madc.hi.u64 %1, %2, %3, %1;"
        : "+l"(lo), "+l"(hi)
        : "l"(a), "l"(b));
}

// Montgomery reduction of a 128-bit accumulator: returns X * 2^-64 mod q.
HS_DEV u64 redc128(u64 lo, u64 hi, const PrimeConst& P) {
    hi = reduce64(hi, P);                    // X' = (hi mod q) 2^64 + lo < q 2^64
    u64 m = lo * P.qinv_neg;
    u64 r = hi + mulhi64(m, P.q) + (lo != 0ull);
    return csub(r, P.q);
}

// Key inner products: keys are kept in standard form, so the REDC result
// X 2^-64 is brought back with one Montgomery product by 2^128 mod q --
// one conversion per output instead of one per key element.
HS_DEV u64 redc128_std(u64 lo, u64 hi, const PrimeConst& P) {
    return mont_mul(redc128(lo, hi, P), P.r2_mod, P.q, P.qinv_neg);
}

// hi 2^64 + lo mod q for any hi, lo < 2^64: hi (2^64 mod q) by Shoup plus
// lo mod q (Barrett), one exact canonical result.  Cheaper than REDC + the
// Montgomery correction (redc128_std) for standard-form keys.
HS_DEV u64 reduce128(u64 lo, u64 hi, const PrimeConst& P) {
    // approximate quotients (ntt.cuh): each part in [0, 4q), sum < 8q
    const u64 t = shoup_ax(hi, P.r_mod, P.r_sh, 0ull - P.q) + reduce64_lazy(lo, P);
    return csub(csub(csub(t, P.two_q << 1), P.two_q), P.q);
}

// Barrett reduction of a 128-bit value x < 2 q^2 (same estimate as mul_mod).
HS_DEV u64 barrett128(u64 lo, u64 hi, const PrimeConst& P) {
    u64 q1 = (hi << (65 - P.k)) | (lo >> (P.k - 1));
    u64 qt = mulhi64(q1, P.mu64);
    u64 r = lo - qt * P.q;
    r = csub(r, P.two_q);
    r = csub(r, P.q);
    return csub(r, P.q);
}

// NTT-domain Galois automorphism X -> X^g: out[k] = in[perm(k)].
// Slot k of a limb holds a(psi^(2 brev(k) + 1)) (bit-reversed output order of
// the reference NTT), so out[k] = in[k'] with 2 brev(k') + 1 = (2 brev(k) + 1) g
// mod 2n.  Pure index map, no sign flips; equals the reference's
// INTT -> signed coefficient permutation -> NTT (context.py:416-452).
HS_DEV u32 galois_perm(u32 k, u32 g, int log_n) {
    u32 br = __brev(k) >> (32 - log_n);
    u32 e = (u32)((((u64)(2 * br + 1)) * g) & ((2ull << log_n) - 1));
    return __brev((e - 1) >> 1) >> (32 - log_n);
}

// =========================================================== plain NTT jobs
// Job interface (ntt.cuh): Ctx make(jb) once per CTA; prime/load/scratch/store.

template <bool FWD>
struct JobPlain {
    u64* buf;           // [jobs][n], in place
    const u64* src;     // optional separate source (same layout) or nullptr
    PrimeMap pm;
    u32 n;
    struct Ctx {
        const u64* src;
        u64* dst;
        int p;
    };
    HS_DEV Ctx make(int jb) const {
        return Ctx{(src ? src : buf) + (size_t)jb * n, buf + (size_t)jb * n, pm.p[jb % pm.nl]};
    }
    HS_DEV int prime(const Ctx& c) const { return c.p; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst&) const { return c.src[j]; }
    HS_DEV u64* scratch(const Ctx& c) const { return c.dst; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        c.dst[j] = FWD ? canon4(v, P) : shoup(v, P.n_inv, P.n_inv_sh, P.q);
    }
};

void ntt_plain(const Dev& d, u64* buf, const u64* src, int njobs, const PrimeMap& pm, bool fwd,
               cudaStream_t st) {
    if (fwd) launch_ntt<true>(d, JobPlain<true>{buf, src, pm, d.n}, njobs, st);
    else launch_ntt<false>(d, JobPlain<false>{buf, src, pm, d.n}, njobs, st);
}

// Inverse NTT of limb `limb` of each item of an ItemPtr set, written to dst.
// Item jb = b*npoly + poly reads ptr(b) + (poly*nl + limb)*n.
struct JobInvGather {
    ItemPtr in;
    int npoly, nl, limb, prime_idx;
    u64* dst;           // [jobs][n]
    u32 n;
    struct Ctx {
        const u64* src;
        u64* dst;
    };
    HS_DEV Ctx make(int jb) const {
        const int b = jb / npoly, poly = jb % npoly;
        return Ctx{in.at(b) + ((size_t)poly * nl + limb) * n, dst + (size_t)jb * n};
    }
    HS_DEV int prime(const Ctx&) const { return prime_idx; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst&) const { return __ldg(c.src + j); }
    HS_DEV u64* scratch(const Ctx& c) const { return c.dst; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        c.dst[j] = shoup(v, P.n_inv, P.n_inv_sh, P.q);
    }
};

// =========================================================== key switching
// Work buffers for a batch of B items at level l (all compact):
//   E   [B][l+1][l+2][n]  ModUp output, NTT domain; slot l+1 is the aux prime;
//                         slot i of digit i holds x_i * df_i (never lifted).
//   D   [B][l+1][n]       digits in coefficient domain.
//   ACC [B][2][l+2][n]    key inner products (b then a component).
//   T   [B][2][n]         INTT of ACC aux limbs.

// Digit sources: the NTT-domain limb x_i that is decomposed (bound per CTA).
struct SrcPlain {      // x = ct(b).poly[i]
    ItemPtr ct;
    int poly;
    struct B {
        const u64* x;
    };
    HS_DEV B bind(int b, int i, int l, u32 n, const Dev&) const {
        return B{ct.at(b) + ((size_t)poly * (l + 1) + i) * n};
    }
    HS_DEV u64 x(const B& s, u32 j, const Dev&, const PrimeConst&) const { return __ldg(s.x + j); }
};
struct SrcPerm {       // x = automorphism_g(ct(b).c1)[i]
    ItemPtr ct;
    const u32* gal;
    struct B {
        const u64* x;
        u32 g;
    };
    HS_DEV B bind(int b, int i, int l, u32 n, const Dev&) const {
        return B{ct.at(b) + ((size_t)(l + 1) + i) * n, gal[b]};
    }
    HS_DEV u64 x(const B& s, u32 j, const Dev& d, const PrimeConst&) const {
        return __ldg(s.x + galois_perm(j, s.g, d.log_n));
    }
};
struct SrcTensor {     // x = d2 = a1 * b1 of the tensor product of two cts
    // Montgomery product a1 b1 2^-64 (cheaper than Barrett); the 2^64 is
    // folded into the digit factor the decomposition applies next (dfR).
    static constexpr bool kMont = true;
    ItemPtr a, bb;
    struct B {
        const u64* a;
        const u64* b;
    };
    HS_DEV B bind(int b, int i, int l, u32 n, const Dev&) const {
        const size_t o = ((size_t)(l + 1) + i) * n;
        return B{a.at(b) + o, bb.at(b) + o};
    }
    HS_DEV u64 x(const B& s, u32 j, const Dev&, const PrimeConst& P) const {
        return mont_mul_lazy(__ldg(s.a + j), __ldg(s.b + j), P.q, P.qinv_neg);    // [0, 2q)
    }
};

template <class S, class = void>
struct SrcMont { static constexpr bool value = false; };
template <class S>
struct SrcMont<S, std::void_t<decltype(S::kMont)>> { static constexpr bool value = S::kMont; };

template <class Src>
struct JobDecompose {                       // inverse NTT, job = b*(l+1)+i
    Src src;
    u64* E;
    u64* D;
    const ulonglong2* df;
    int l;
    u32 n;
    Dev d;
    struct Ctx {
        typename Src::B s;
        u64* e;              // E[b][i][i]
        u64* dd;             // D[b][i]
        ulonglong2 w;        // digit factor
        int i;
    };
    HS_DEV Ctx make(int jb) const {
        const int b = jb / (l + 1), i = jb % (l + 1);
        return Ctx{src.bind(b, i, l, n, d), E + ((size_t)jb * (l + 2) + i) * n, D + (size_t)jb * n,
                   SrcMont<Src>::value ? d.dfR[i] : df[i], i};
    }
    HS_DEV int prime(const Ctx& c) const { return c.i; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        const u64 v = shoup(src.x(c.s, j, d, P), c.w.x, c.w.y, P.q);
        c.e[j] = v;
        return v;
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.dd; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        c.dd[j] = shoup(v, P.n_inv, P.n_inv_sh, P.q);
    }
};

#ifndef HS_LIFT_LAZY
#define HS_LIFT_LAZY 1           // ModUp loaders lift into [0, 4q) (approximate Barrett)
#endif
struct JobModUp {                           // forward NTT, job = (b*(l+1)+i)*(l+1)+t
    const u64* D;
    u64* E;
    int l, L;
    u32 n;
    const PrimeConst* pc;
    struct Ctx {
        const u64* d;        // digit i (coefficient domain, mod q_i)
        u64* e;              // E[b][i][m]
        u64 qsrc;
        int pm;
        bool small;          // q_i / 2 < q_m: the lift needs no reduction
    };
    HS_DEV Ctx make(int jb) const {
        const int t = jb % (l + 1);
        const int bi = jb / (l + 1);
        const int i = bi % (l + 1);
        const int m = t < i ? t : t + 1;     // m in [0, l+1] \ {i}; l+1 = aux
        const int pm = m <= l ? m : L + 1;
        const u64 qs = pc[i].q;
        return Ctx{D + (size_t)bi * n, E + ((size_t)bi * (l + 2) + m) * n, qs, pm, (qs >> 1) < pc[pm].q};
    }
    HS_DEV int prime(const Ctx& c) const { return c.pm; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
#if HS_LIFT_LAZY
        return lift_lazy(__ldg(c.d + j), c.qsrc, P);           // [0, 4q): forward loader
#else
        return lift_mod_sel(__ldg(c.d + j), c.qsrc, P, c.small);
#endif
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.e; }
    // E stays in [0, 4q): the inner product only needs sum_i e k < 2^128 with
    // hi < 2^63 (reduce128), i.e. (l+1) 4q^2 < 2^127 -- no canonicalisation.
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst&) const { c.e[j] = v; }
};

// Key inner product: ACC[b][c][m] = sum_i E[b][i][m][perm(k)] * K_b[c][i][m].
// Keys are stored in standard form; redc128_std turns the 128-bit sum into
// the plain residue.  Streaming kernel (HBM/L2 bound): each thread owns two
// adjacent coefficients so key rows move as 16-byte loads and more loads are
// in flight per thread.  grid = (ceil(n/512), l+2, B).
constexpr int KSI_T = 256;
#ifndef KSI_UNROLL
#define KSI_UNROLL 2
#endif
constexpr int kKsiUnroll = KSI_UNROLL;

#ifndef KSI_IPB
#define KSI_IPB 4                    // A/B cfg2: 1 -> 126.3 ms, 2 -> 125.0, 4 -> 124.7
#endif
constexpr int kKsiIpb = KSI_IPB;             // items per CTA (loads of the next item overlap)

#ifndef KSI_MINB
#define KSI_MINB 4                   // A/B cfg2: 4 -> 121 ms, 5 -> 125, 6 -> 133
#endif
__global__ void __launch_bounds__(KSI_T, KSI_MINB)
ks_inner_kernel(Dev d, int l, int B, const u64* __restrict__ E, size_t e_item_stride,
                const u64* const* __restrict__ keys, const u32* __restrict__ gal,
                u64* __restrict__ ACC) {
    const u32 n = d.n;
    const u32 k = 2 * (blockIdx.x * KSI_T + threadIdx.x);
    const int m = blockIdx.y;
    if (k >= n) return;
    const int pm = m <= l ? m : d.L + 1;
    const PrimeConst P = d.pc[pm];
    const size_t estride = (size_t)(l + 2) * n;                    // one digit of E
    const size_t kstride = (size_t)(d.L + 2) * n;                  // one digit of a key
    const size_t kst2 = kstride / 2;
#pragma unroll
    for (int bb = 0; bb < kKsiIpb; bb++) {
        const int b = blockIdx.z * kKsiIpb + bb;
        if (b >= B) break;
        const u32 g = gal ? gal[b] : 0u;
        const u32 src0 = g ? galois_perm(k, g, d.log_n) : k;
        const u32 src1 = g ? galois_perm(k + 1, g, d.log_n) : k + 1;
        const u64* __restrict__ Ei = E + (size_t)b * e_item_stride + (size_t)m * n;
        const u64* key = keys[b];
        const ulonglong2* __restrict__ kb = (const ulonglong2*)(key + (size_t)pm * n + k);
        const ulonglong2* __restrict__ ka =
            (const ulonglong2*)(key + (size_t)(d.L + 1) * kstride + (size_t)pm * n + k);
        u64 lb0 = 0, hb0 = 0, la0 = 0, ha0 = 0, lb1 = 0, hb1 = 0, la1 = 0, ha1 = 0;
#pragma unroll kKsiUnroll
        for (int i = 0; i <= l; i++, Ei += estride, kb += kst2, ka += kst2) {
            u64 e0, e1;
            if (g) {
                e0 = __ldg(Ei + src0);
                e1 = __ldg(Ei + src1);
            } else {
                const ulonglong2 ee = __ldg((const ulonglong2*)(Ei + k));
                e0 = ee.x;
                e1 = ee.y;
            }
            const ulonglong2 vb = __ldg(kb), va = __ldg(ka);
            mac128(lb0, hb0, e0, vb.x);
            mac128(lb1, hb1, e1, vb.y);
            mac128(la0, ha0, e0, va.x);
            mac128(la1, ha1, e1, va.y);
        }
        u64* out = ACC + (size_t)b * 2 * (l + 2) * n;
        *(ulonglong2*)(out + (size_t)m * n + k) =
            make_ulonglong2(reduce128(lb0, hb0, P), reduce128(lb1, hb1, P));
        *(ulonglong2*)(out + ((size_t)(l + 2) + m) * n + k) =
            make_ulonglong2(reduce128(la0, ha0, P), reduce128(la1, ha1, P));
    }
}

static dim3 ks_inner_grid(const Dev& d, int l, int B) {
    return dim3((d.n + 2 * KSI_T - 1) / (2 * KSI_T), l + 2, (B + kKsiIpb - 1) / kKsiIpb);
}

// ---- the key inner product with bulk-async (TMA engine) row streaming.
//
// Same sums as ks_inner_kernel for the un-permuted case (every pair-batch key
// switch): ACC[b][c][m][k] = sum_i E[b][i][m][k] * K_b[c][i][m][k].  One CTA
// owns a 256-coefficient column tile of one target modulus m for KSI2_IPB
// consecutive items.  A producer warp streams the rows of each (item, digit)
// -- E (2 KB), key b-half (2 KB), key a-half (2 KB) -- into a KSI2_NST-stage
// shared-memory ring with cp.async.bulk (no registers, no address math in the
// consumers), completion signalled on per-stage mbarriers; 4 consumer warps
// (2 coefficients per thread) wait on a stage, multiply-accumulate in 128
// bits, and release it on an "empty" mbarrier.  Grid x = item group (fastest),
// so the CTAs sharing a key tile (the relinearisation key: every item) run
// back to back and the key rows come from L2 after the first read
// (E is streamed with an evict-first hint, keys with evict-last).
constexpr int KSI2_CT = 128;                 // consumer threads
constexpr int KSI2_C = 2 * KSI2_CT;          // coefficients per tile
constexpr int KSI2_ROWB = KSI2_C * 8;        // bytes per row tile
#ifndef KSI2_NST
#define KSI2_NST 6
#endif
#ifndef KSI2_IPB
#define KSI2_IPB 2
#endif
constexpr int kKsi2Nst = KSI2_NST, kKsi2Ipb = KSI2_IPB;
constexpr size_t KSI2_SMEM = (size_t)kKsi2Nst * 3 * KSI2_ROWB;

HS_DEV u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
HS_DEV void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
HS_DEV void mbar_wait(u32 bar, u32 parity) {
    u32 ok;
    do {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(bar), "r"(parity)
                     : "memory");
    } while (!ok);
}
HS_DEV void mbar_arrive(u32 bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
HS_DEV void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
HS_DEV void bulk_g2s(u32 dst, const void* src, u32 bytes, u32 bar, u64 policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}

__global__ void __launch_bounds__(KSI2_CT + 32)
ks_inner_tma_kernel(Dev d, int l, int B, const u64* __restrict__ E, size_t e_item_stride,
                    const u64* const* __restrict__ keys, u64* __restrict__ ACC,
                    const int* __restrict__ imap, int m0) {
    extern __shared__ __align__(128) unsigned char ksi2_smem[];
    __shared__ __align__(8) unsigned long long bars[2 * kKsi2Nst];     // full, empty
    const u32 n = d.n;
    const int m = m0 + (int)blockIdx.z;
    const u32 col0 = blockIdx.y * KSI2_C;
    const int b0 = blockIdx.x * kKsi2Ipb;
    const int nb = min(kKsi2Ipb, B - b0);
    const int pm = m <= l ? m : d.L + 1;
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u32 smb = smem_u32(ksi2_smem);
    const u32 full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[kKsi2Nst]);
    if (tid == 0) {
        for (int s = 0; s < kKsi2Nst; s++) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, KSI2_CT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == KSI2_CT / 32) {                                     // producer warp
        if (lane == 0) {
            u64 pol_e, pol_k;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_e));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_k));
            const size_t kstride = (size_t)(d.L + 2) * n;
            int s = 0;
            u32 ph = 0;                                             // parity of the ring's current lap
            int t = 0;
            for (int bb = 0; bb < nb; bb++) {
                const int b = imap ? imap[b0 + bb] : b0 + bb;         // physical item slot
                const u64* key = keys[b];
                const u64* er = E + (size_t)b * e_item_stride + (size_t)m * n + col0;
                const u64* kbr = key + (size_t)pm * n + col0;
                const u64* kar = key + (size_t)(d.L + 1) * kstride + (size_t)pm * n + col0;
                for (int i = 0; i <= l; i++, t++) {
                    if (t >= kKsi2Nst) mbar_wait(empty0 + 8 * s, ph ^ 1);
                    const u32 full = full0 + 8 * s;
                    const u32 dst = smb + (u32)(s * 3 * KSI2_ROWB);
                    mbar_expect_tx(full, 3 * KSI2_ROWB);
                    bulk_g2s(dst, er + (size_t)i * (l + 2) * n, KSI2_ROWB, full, pol_e);
                    bulk_g2s(dst + KSI2_ROWB, kbr + (size_t)i * kstride, KSI2_ROWB, full, pol_k);
                    bulk_g2s(dst + 2 * KSI2_ROWB, kar + (size_t)i * kstride, KSI2_ROWB, full, pol_k);
                    if (++s == kKsi2Nst) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }
    // consumers
    const PrimeConst P = d.pc[pm];
    const u32 k = col0 + 2 * tid;
    int s = 0;
    u32 ph = 0;
    for (int bb = 0; bb < nb; bb++) {
        u64 lb0 = 0, hb0 = 0, la0 = 0, ha0 = 0, lb1 = 0, hb1 = 0, la1 = 0, ha1 = 0;
        for (int i = 0; i <= l; i++) {
            mbar_wait(full0 + 8 * s, ph);
            const ulonglong2* row = (const ulonglong2*)(ksi2_smem + s * 3 * KSI2_ROWB);
            const ulonglong2 ee = row[tid];
            const ulonglong2 vb = row[KSI2_CT + tid];
            const ulonglong2 va = row[2 * KSI2_CT + tid];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * s);
            if (++s == kKsi2Nst) {
                s = 0;
                ph ^= 1;
            }
            mac128(lb0, hb0, ee.x, vb.x);
            mac128(lb1, hb1, ee.y, vb.y);
            mac128(la0, ha0, ee.x, va.x);
            mac128(la1, ha1, ee.y, va.y);
        }
        const int b = imap ? imap[b0 + bb] : b0 + bb;
        u64* out = ACC + (size_t)b * 2 * (l + 2) * n;
        *(ulonglong2*)(out + (size_t)m * n + k) = make_ulonglong2(reduce128(lb0, hb0, P), reduce128(lb1, hb1, P));
        *(ulonglong2*)(out + ((size_t)(l + 2) + m) * n + k) =
            make_ulonglong2(reduce128(la0, ha0, P), reduce128(la1, ha1, P));
    }
}

// ks_inner over B un-permuted items: the bulk-async kernel when the ring has
// whole 256-coefficient tiles (HS_KSI_LDG=1 selects the LDG kernel, A/B).
// imap (device, optional): logical item -> physical item slot (E, keys, ACC);
// targets m0 .. m0+mcnt-1 (default: all l+2).  Only the bulk-async kernel
// takes imap / a target subset.
static bool ks_inner_tma_ok(const Dev& d) {
    static const bool ldg = getenv("HS_KSI_LDG") != nullptr;
    return !ldg && d.n % KSI2_C == 0;
}
static void launch_ks_inner(const Dev& d, int l, int B, const u64* E, size_t e_item_stride,
                            const u64* const* keys, u64* ACC, cudaStream_t st,
                            const int* imap = nullptr, int m0 = 0, int mcnt = -1) {
    if (mcnt < 0) mcnt = l + 2;
    if (!ks_inner_tma_ok(d)) {
        ks_inner_kernel<<<ks_inner_grid(d, l, B), KSI_T, 0, st>>>(d, l, B, E, e_item_stride, keys, nullptr,
                                                                 ACC);
    } else {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(ks_inner_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)KSI2_SMEM);
            attr = true;
        }
        const dim3 grid((B + kKsi2Ipb - 1) / kKsi2Ipb, d.n / KSI2_C, mcnt);
        ks_inner_tma_kernel<<<grid, KSI2_CT + 32, KSI2_SMEM, st>>>(d, l, B, E, e_item_stride, keys, ACC,
                                                                   imap, m0);
    }
    note_launch();
}

// ModDown addends (what is added to the key-switch output), bound per CTA.
struct AddNone {
    struct B {};
    HS_DEV B bind(int, int, int, int, const Dev&) const { return B{}; }
    HS_DEV u64 v(const B&, u32, const Dev&, const PrimeConst&) const { return 0; }
};
struct AddTensor {     // relinearize after mult_ct: d0 = a0 b0, d1 = a0 b1 + a1 b0
    ItemPtr a, bb;
    // one code path for both polys: x0 y0 + x1 y1 with (x1, y1) absent for d0
    // (the inlined epilogue is instruction-cache bound, not ALU bound)
    struct B {
        const u64 *x0, *y0, *x1, *y1;
    };
    HS_DEV B bind(int b, int poly, int m, int l, const Dev& d) const {
        const u64* A = a.at(b);
        const u64* Bp = bb.at(b);
        const size_t o0 = (size_t)m * d.n, o1 = ((size_t)(l + 1) + m) * d.n;
        return poly ? B{A + o0, Bp + o1, A + o1, Bp + o0} : B{A + o0, Bp + o0, nullptr, nullptr};
    }
    HS_DEV u64 v(const B& s, u32 j, const Dev&, const PrimeConst& P) const {
        u64 lo = 0, hi = 0;
        mac128(lo, hi, __ldg(s.x0 + j), __ldg(s.y0 + j));
        const u64 x1 = s.x1 ? __ldg(s.x1 + j) : 0ull, y1 = s.x1 ? __ldg(s.y1 + j) : 0ull;
        mac128(lo, hi, x1, y1);
        return barrett128(lo, hi, P);
    }
};
struct AddPoly {       // d0/d1 taken from a stored ct (npoly polys at level l)
    ItemPtr ct;
    struct B {
        const u64* p;
    };
    HS_DEV B bind(int b, int poly, int m, int l, const Dev& d) const {
        return B{ct.at(b) + ((size_t)poly * (l + 1) + m) * d.n};
    }
    HS_DEV u64 v(const B& s, u32 j, const Dev&, const PrimeConst&) const { return __ldg(s.p + j); }
};
struct AddPermC0 {     // rotation: automorphism_g(c0) on poly 0
    ItemPtr ct;
    const u32* gal;
    struct B {
        const u64* c0;
        u32 g;
    };
    HS_DEV B bind(int b, int poly, int m, int l, const Dev& d) const {
        return B{poly ? nullptr : ct.at(b) + (size_t)m * d.n, poly ? 0u : gal[b]};
    }
    HS_DEV u64 v(const B& s, u32 j, const Dev& d, const PrimeConst&) const {
        return s.c0 ? __ldg(s.c0 + galois_perm(j, s.g, d.log_n)) : 0ull;
    }
};

template <class Add>
struct JobModDown {                          // forward NTT, job = (b*2+c)*nm+(m-m0)
    const u64* T;
    const u64* ACC;
    ItemPtr out;                             // per item ct [2][l+1][n]
    Add add;
    int l;
    Dev d;
    int m0, nm;                              // limbs m0 .. m0+nm-1 (all: 0, l+1)
    struct Ctx {
        const u64* t;        // INTT of the aux accumulator (coefficients mod p)
        const u64* acc;      // ACC[b][c][m]
        u64* out;            // out(b)[c][m]
        typename Add::B add;
        ulonglong2 w;        // p^-1 mod q_m
        int m;
        bool small;          // p / 2 < q_m
    };
    HS_DEV Ctx make(int jb) const {
        const int bc = jb / nm, m = m0 + jb % nm;
        const int b = bc >> 1, c = bc & 1;
        return Ctx{T + (size_t)bc * d.n, ACC + ((size_t)bc * (l + 2) + m) * d.n,
                   out.atw(b) + ((size_t)c * (l + 1) + m) * d.n, add.bind(b, c, m, l, d), d.auxinv[m], m,
                   (d.aux_q >> 1) < d.pc[m].q};
    }
    HS_DEV int prime(const Ctx& c) const { return c.m; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        return lift_mod_sel(__ldg(c.t + j), d.aux_q, P, c.small);
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.out; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        // (acc - v) p^-1 + addend, one canonicalisation: acc < q, v < 4q
        const u64 r = shoup_lazy(__ldg(c.acc + j) + (P.two_q << 1) - v, c.w.x, c.w.y, P.q);   // [0, 2q)
        c.out[j] = csub(csub(r + add.v(c.add, j, d, P), P.two_q), P.q);
    }
};

size_t ks_scratch_elems(int B, int l, u32 n) {
    return (size_t)B * n * ((size_t)(l + 1) * (l + 2) + (l + 1) + 2 * (l + 2) + 2);
}

size_t ks_hoisted_scratch_elems(int R, int l, u32 n) {
    return (size_t)n * ((size_t)(l + 1) * (l + 2) + (l + 1) + (size_t)R * (2 * (l + 2) + 2));
}

// ModDown of ACC (B items) into out with addend.
template <class Add>
static void mod_down(const Dev& d, int B, int l, const u64* ACC, u64* T, const Add& add,
                     ItemPtr out, cudaStream_t st) {
    launch_ntt<false>(d, JobInvGather{strided(ACC, (size_t)(l + 2) * d.n), 1, l + 2, l + 1,
                                      d.L + 1, T, d.n},
                      B * 2, st);
    launch_ntt<true>(d, JobModDown<Add>{T, ACC, out, add, l, d, 0, l + 1}, B * 2 * (l + 1), st);
}

// Fused ModUp second pass + key inner product.  One CTA owns a contiguous
// 2048-element tile of target modulus m for item b; for every digit i it
// finishes the NTT of lift(digit_i) on that tile in shared memory (the first
// pass already ran, writing lazy values into E[b][i][m]) and folds the tile
// into 128-bit accumulators against the key tile; the ModUp output is never
// written back to HBM.  Digit i == m contributes x_i * df_i (already in E).
template <int LA, int LB, int MINB>
__global__ void __launch_bounds__(NTT_THREADS, MINB)
modup_inner_kernel(Dev d, int l, const u64* __restrict__ E, const u64* const* __restrict__ keys,
                   u64* __restrict__ ACC) {
    constexpr int H = NTT_TILE >> LB;
    __shared__ u64 sm[NTT_TILE + NTT_TILE / 8];
    const u32 n = d.n;
    const int m = blockIdx.y, b = blockIdx.z;
    const int pm = m <= l ? m : d.L + 1;
    const PrimeConst P = d.pc[pm];
    const ulonglong2* __restrict__ tw = d.tw + (size_t)pm * n;
    const u32 hi0 = blockIdx.x * H;
    const u32 j0 = hi0 << LB;
    const u32 t = threadIdx.x;
    const size_t kst = (size_t)(d.L + 2) * n;
    const u64* __restrict__ key = keys[b];
    const u64* kb = key + (size_t)pm * n + j0;
    const u64* ka = key + (size_t)(d.L + 1) * kst + (size_t)pm * n + j0;
    const u64* Eb = E + (size_t)b * (l + 1) * (l + 2) * n;
    u64 lb[NTT_EPT], hb[NTT_EPT], la[NTT_EPT], ha[NTT_EPT];
#pragma unroll
    for (int k = 0; k < NTT_EPT; k++) lb[k] = hb[k] = la[k] = ha[k] = 0;
    for (int i = 0; i <= l; i++) {
        const u64* src = Eb + ((size_t)i * (l + 2) + m) * n + j0;
        u64 ext[NTT_EPT];
        if (i == m) {
#pragma unroll
            for (int k = 0; k < NTT_EPT; k++) ext[k] = src[t + k * NTT_THREADS];
        } else {
            // pass A leaves lazy values (ntt.cuh invariants): back to [0, 4q)
#pragma unroll
            for (int k = 0; k < NTT_EPT; k++)
                sm[spad(t + k * NTT_THREADS)] = reduce64_lazy(src[t + k * NTT_THREADS], P);
            __syncthreads();
            ntt_rounds_fwd<LB, H, 1>(sm, tw, hi0, LA, P.q, P.two_q);
#pragma unroll
            for (int k = 0; k < NTT_EPT; k++) ext[k] = canon4(sm[spad(t + k * NTT_THREADS)], P);
            __syncthreads();
        }
        const u64* kbi = kb + (size_t)i * kst;
        const u64* kai = ka + (size_t)i * kst;
#pragma unroll
        for (int k = 0; k < NTT_EPT; k++) {
            mac128(lb[k], hb[k], ext[k], kbi[t + k * NTT_THREADS]);
            mac128(la[k], ha[k], ext[k], kai[t + k * NTT_THREADS]);
        }
    }
    u64* out = ACC + (size_t)b * 2 * (l + 2) * n + j0;
#pragma unroll
    for (int k = 0; k < NTT_EPT; k++) {
        out[(size_t)m * n + t + k * NTT_THREADS] = redc128_std(lb[k], hb[k], P);
        out[(size_t)(l + 2 + m) * n + t + k * NTT_THREADS] = redc128_std(la[k], ha[k], P);
    }
}

template <int LA, int LB>
static void launch_modup_inner(const Dev& d, int B, int l, u64* D, u64* E, const u64* const* keys,
                               u64* ACC, cudaStream_t st) {
    const u32 n = d.n;
    JobModUp job{D, E, l, d.L, n, d.pc};
    constexpr int CA = NTT_TILE >> LA;
    const int njobs = B * (l + 1) * (l + 1);
    for (int base = 0; base < njobs; base += 65535) {
        const int cnt = njobs - base < 65535 ? njobs - base : 65535;
        ntt_pass_kernel<true, true, false, LA, 1, CA, NTT_EPT16, LA + LB, 0, JobModUp>
            <<<dim3(n / NTT_TILE, cnt), NTT_TILE / NTT_EPT16, 0, st>>>(d, job, base);
        note_launch();
    }
    // HS_MODUP_MINB=1 trades occupancy for registers (A/B knob for profiling)
    static const int minb = getenv("HS_MODUP_MINB") ? atoi(getenv("HS_MODUP_MINB")) : 2;
    if (minb == 1)
        modup_inner_kernel<LA, LB, 1><<<dim3(n / NTT_TILE, l + 2, B), NTT_THREADS, 0, st>>>(d, l, E, keys, ACC);
    else
        modup_inner_kernel<LA, LB, 2><<<dim3(n / NTT_TILE, l + 2, B), NTT_THREADS, 0, st>>>(d, l, E, keys, ACC);
    note_launch();
}

// ModUp + inner product for B items (E must hold x_i df_i in slot (i, i)).
// Algorithmic DRAM bytes of one ks_inner launch: E read once, each of the
// nkeys distinct keys read once (repeat uses hit L2), ACC written once.
static double ks_inner_bytes(const Dev& d, int l, int B, int nkeys) {
    const double limb = 8.0 * d.n, ml = (double)(l + 1) * (l + 2);
    return B * ml * limb + nkeys * 2.0 * ml * limb + B * 2.0 * (l + 2) * limb;
}

static void modup_and_inner(const Dev& d, int B, int l, u64* D, u64* E, const u64* const* keys,
                            u64* ACC, cudaStream_t st, int nkeys) {
    // Default: ModUp as a batched two-pass NTT writing E, then the streaming
    // inner-product kernel (both run at high occupancy).  HS_MODUP_FUSED=1
    // selects the fused pass-B + inner-product kernel (no E round trip, but
    // 128-bit accumulators cap it at 25% occupancy).
    static const bool fused = getenv("HS_MODUP_FUSED") != nullptr;
    if (!fused) {
        const double jobs = (double)B * (l + 1) * (l + 1), n = d.n;
        {
            // algorithmic (unique) bytes: pass A reads each digit once (its l+1
            // lifts re-read it from L2) and writes one limb per job; pass B
            // reads and writes one limb per job
            ProbeScope ps(PROBE_MODUP, st, (3.0 * jobs + (double)B * (l + 1)) * 8.0 * n,
                          jobs * (n / 2) * d.log_n, 2);
            launch_ntt<true>(d, JobModUp{D, E, l, d.L, d.n, d.pc}, B * (l + 1) * (l + 1), st);
        }
        {
            ProbeScope ps(PROBE_KS_INNER, st, ks_inner_bytes(d, l, B, nkeys),
                          (double)B * 2 * (l + 1) * (l + 2) * n);
            launch_ks_inner(d, l, B, E, (size_t)(l + 1) * (l + 2) * d.n, keys, ACC, st);
        }
        return;
    }
    switch (d.log_n) {
        case 12: launch_modup_inner<6, 6>(d, B, l, D, E, keys, ACC, st); return;
        case 13: launch_modup_inner<6, 7>(d, B, l, D, E, keys, ACC, st); return;
        case 14: launch_modup_inner<7, 7>(d, B, l, D, E, keys, ACC, st); return;
        case 15: launch_modup_inner<7, 8>(d, B, l, D, E, keys, ACC, st); return;
        case 16: launch_modup_inner<8, 8>(d, B, l, D, E, keys, ACC, st); return;
        case 17: launch_modup_inner<8, 9>(d, B, l, D, E, keys, ACC, st); return;
        default: break;
    }
    // small rings: whole-limb single-pass NTT, then the plain inner product
    launch_ntt<true>(d, JobModUp{D, E, l, d.L, d.n, d.pc}, B * (l + 1) * (l + 1), st);
    ks_inner_kernel<<<ks_inner_grid(d, l, B), KSI_T, 0, st>>>(d, l, B, E, (size_t)(l + 1) * (l + 2) * d.n, keys,
                                                             nullptr, ACC);
    note_launch();
}

template <class Src, class Add>
static void key_switch_batch(const Dev& d, int B, int l, const Src& src, const Add& add,
                             const u64* const* keys, ItemPtr out, u64* scratch, cudaStream_t st,
                             int nkeys) {
    const u32 n = d.n;
    u64* E = scratch;
    u64* D = E + (size_t)B * (l + 1) * (l + 2) * n;
    u64* ACC = D + (size_t)B * (l + 1) * n;
    u64* T = ACC + (size_t)B * 2 * (l + 2) * n;
    launch_ntt<false>(d, JobDecompose<Src>{src, E, D, d.df, l, n, d}, B * (l + 1), st);
    modup_and_inner(d, B, l, D, E, keys, ACC, st, nkeys);
    mod_down(d, B, l, ACC, T, add, out, st);
}

void relin_batch(const Dev& d, int B, int l, ItemPtr ct3, const u64* const* keys, ItemPtr out,
                 u64* scratch, cudaStream_t st) {
    key_switch_batch(d, B, l, SrcPlain{ct3, 2}, AddPoly{ct3}, keys, out, scratch, st, 1);
}

void mult_relin_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, const u64* const* keys,
                      ItemPtr out, u64* scratch, cudaStream_t st) {
    key_switch_batch(d, B, l, SrcTensor{a, b}, AddTensor{a, b}, keys, out, scratch, st, 1);
}

// ModDown followed by rescale, merged.  Both subtract the NTT of a lifted
// coefficient vector and scale; the NTT mod q_m is linear, so for m < l
//   out_m = (acc_m - NTT_m(lift_p T)) p^-1 + add_m                (ModDown)
//   r_m   = (out_m - NTT_m(lift_ql u)) q_l^-1 mask_m,  u = INTT(out_l)
//         = (acc_m p^-1 + add_m - NTT_m(lift_p(T) p^-1 + lift_ql(u))) q_l^-1 mask_m
// -- exact modular identities, so r_m is the same residue the two separate
// steps produce (hespmm/ckks/context.py key switch then rescale).  Only limb
// l of the relinearised ct is formed; one forward NTT per (item, poly, m < l)
// replaces two.
template <class Add>
struct JobModDownRescale {                   // forward NTT, job = (b*2+c)*l+m, m < l
    const u64* T;                            // [bc][n] INTT of the aux accumulator (mod p)
    const u64* U;                            // [bc][n] INTT of out limb l (mod q_l)
    const u64* ACC;
    ItemPtr out, mask;                       // out per item [2][l][n]; mask [l][n] (Montgomery)
    Add add;
    int l;
    Dev d;
    const ulonglong2* qlinv;                 // row for level l
    struct Ctx {
        const u64 *t, *u, *acc, *mask;
        u64* out;
        typename Add::B add;
        ulonglong2 wp, wl;   // p^-1, q_l^-1 mod q_m
        u64 ql;
        int m;
    };
    HS_DEV Ctx make(int jb) const {
        const int bc = jb / l, m = jb % l;
        const int b = bc >> 1, c = bc & 1;
        const bool has_mask = mask.tab || mask.base;
        return Ctx{T + (size_t)bc * d.n, U + (size_t)bc * d.n, ACC + ((size_t)bc * (l + 2) + m) * d.n,
                   has_mask ? mask.at(b) + (size_t)m * d.n : nullptr, out.atw(b) + ((size_t)c * l + m) * d.n,
                   add.bind(b, c, m, l, d), d.auxinv[m], qlinv[m], d.pc[l].q, m};
    }
    HS_DEV int prime(const Ctx& c) const { return c.m; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        const u64 tp = shoup_lazy(lift_lazy(__ldg(c.t + j), d.aux_q, P), c.wp.x, c.wp.y, P.q);  // [0, 2q)
        return csub(tp + lift_lazy(__ldg(c.u + j), c.ql, P), P.two_q);                          // [0, 4q)
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.out; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        const u64 y = shoup_lazy(__ldg(c.acc + j), c.wp.x, c.wp.y, P.q) + add.v(c.add, j, d, P);  // [0, 3q)
        u64 r = shoup_lazy(y + (P.two_q << 1) - v, c.wl.x, c.wl.y, P.q);                         // [0, 2q)
        const u64 mk = c.mask ? __ldg(c.mask + j) : P.r_mod;
        r = mont_mul_lazy(r, mk, P.q, P.qinv_neg);                                               // [0, 2q)
        c.out[j] = csub(r, P.q);
    }
};

// u = INTT(out_l) of the relinearised ct's top limb without forming out_l:
// out_l = (acc_l - NTT_l(lift_p T)) p^-1 + add_l, so by linearity
//   INTT(out_l) = INTT(acc_l p^-1 + add_l) - lift_l(T) p^-1      (mod q_l)
// -- one inverse NTT instead of a forward NTT followed by an inverse one.
template <class Add>
struct JobTopU {                             // inverse NTT, job = b*2+c, prime l
    const u64* T;
    const u64* ACC;
    u64* U;                                  // [bc][n]
    Add add;
    int l;
    Dev d;
    struct Ctx {
        const u64 *t, *acc;
        u64* u;
        typename Add::B add;
        ulonglong2 w;        // p^-1 mod q_l
    };
    HS_DEV Ctx make(int bc) const {
        return Ctx{T + (size_t)bc * d.n, ACC + ((size_t)bc * (l + 2) + l) * d.n, U + (size_t)bc * d.n,
                   add.bind(bc >> 1, bc & 1, l, l, d), d.auxinv[l]};
    }
    HS_DEV int prime(const Ctx&) const { return l; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        return shoup_lazy(__ldg(c.acc + j), c.w.x, c.w.y, P.q) + add.v(c.add, j, d, P);   // [0, 3q)
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.u; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        const u64 y = shoup(v, P.n_inv, P.n_inv_sh, P.q);
        const u64 t = shoup(lift_mod(__ldg(c.t + j), d.aux_q, P), c.w.x, c.w.y, P.q);
        c.u[j] = sub_mod(y, t, P.q);
    }
};

void mult_relin_rescale_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, const u64* const* keys,
                              ItemPtr mask_mont, ItemPtr top, ItemPtr out, u64* scratch, u64* U,
                              cudaStream_t st) {
    const u32 n = d.n;
    u64* E = scratch;
    u64* D = E + (size_t)B * (l + 1) * (l + 2) * n;
    u64* ACC = D + (size_t)B * (l + 1) * n;
    u64* T = ACC + (size_t)B * 2 * (l + 2) * n;
    const AddTensor add{a, b};
    launch_ntt<false>(d, JobDecompose<SrcTensor>{SrcTensor{a, b}, E, D, d.df, l, n, d}, B * (l + 1), st);
    modup_and_inner(d, B, l, D, E, keys, ACC, st, 1);       // the relin key, shared
    launch_ntt<false>(d, JobInvGather{strided(ACC, (size_t)(l + 2) * n), 1, l + 2, l + 1, d.L + 1, T, n},
                      B * 2, st);
    // u = INTT of limb l of the relinearised ct
    static const bool top_fwd = getenv("HS_TOPLIMB_FWD") != nullptr;   // A/B: old two-transform path
    if (top_fwd) {
        launch_ntt<true>(d, JobModDown<AddTensor>{T, ACC, top, add, l, d, l, 1}, B * 2, st);
        launch_ntt<false>(d, JobInvGather{top, 2, l + 1, l, l, U, n}, B * 2, st);
    } else {
        launch_ntt<false>(d, JobTopU<AddTensor>{T, ACC, U, add, l, d}, B * 2, st);
    }
    launch_ntt<true>(d,
                     JobModDownRescale<AddTensor>{T, U, ACC, out, mask_mont, add, l, d,
                                                  d.qlinv + (size_t)l * (d.L + 1)},
                     B * 2 * l, st);
}

void rotate_batch(const Dev& d, int B, int l, ItemPtr ct, const u32* gal, const u64* const* keys,
                  ItemPtr out, u64* scratch, cudaStream_t st) {
    key_switch_batch(d, B, l, SrcPerm{ct, gal}, AddPermC0{ct, gal}, keys, out, scratch, st, B);
}

// Rotate B items and add them all into acc ([2][l+1][n]), with ONE ModDown
// NTT per output limb instead of one per item.  ModDown of item b is
//   out_b,m = (acc_b,m - NTT_m(lift_p T_b)) p^-1 + add_b,m
// and the NTT mod q_m is linear, so
//   sum_b out_b,m = (sum_b acc_b,m - NTT_m(sum_b lift_p T_b)) p^-1 + sum_b add_b,m
// -- the same residues as rotating each item and adding (the reference's
// per-item eval_rotate + eval_add, hespmm/engine.py accumulation loop).
// rot_partial_kernel sums, per chunk of items, the coefficient/NTT vectors
// F = [S0, S1, A0, A1, Z0, Z1] (acc per poly, addend per poly = permuted c0
// and 0, lifted T per poly); accum_fold_kernel adds the chunks onto F, whose
// A slots start as the running sum acc; JobRotAcc runs the NTT of Z and the
// ModDown epilogue, overwriting acc (its scratch between the two passes).
__global__ void __launch_bounds__(256)
rot_partial_kernel(Dev d, int B, int l, int chunk, ItemPtr ct, const u32* __restrict__ gal,
                   const u64* __restrict__ ACC, const u64* __restrict__ T, u64* __restrict__ part,
                   const unsigned char* __restrict__ head) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int m = blockIdx.y;
    const PrimeConst P = d.pc[m];
    const int b0 = blockIdx.z * chunk, b1 = min(B, b0 + chunk);
    const size_t acc_item = (size_t)2 * (l + 2) * n;
    u64 s0 = 0, s1 = 0, a0 = 0, z0 = 0, z1 = 0;
    for (int b = b0; b < b1; b++) {
        if (!head || head[b]) {            // grouped: the head slot holds its group's sum
            const u64* A = ACC + (size_t)b * acc_item + (size_t)m * n + k;
            s0 = add_mod(s0, __ldg(A), P.q);
            s1 = add_mod(s1, __ldg(A + (size_t)(l + 2) * n), P.q);
        }
        a0 = add_mod(a0, __ldg(ct.at(b) + (size_t)m * n + galois_perm(k, gal[b], d.log_n)), P.q);
        z0 = add_mod(z0, lift_mod(__ldg(T + (size_t)b * 2 * n + k), d.aux_q, P), P.q);
        z1 = add_mod(z1, lift_mod(__ldg(T + ((size_t)b * 2 + 1) * n + k), d.aux_q, P), P.q);
    }
    const size_t ls = (size_t)(l + 1) * n;              // one slot [l+1][n]
    u64* dst = part + (size_t)blockIdx.z * 6 * ls + (size_t)m * n + k;
    dst[0] = s0;
    dst[ls] = s1;
    dst[2 * ls] = a0;
    dst[3 * ls] = 0ull;
    dst[4 * ls] = z0;
    dst[5 * ls] = z1;
}

struct JobRotAcc {                           // forward NTT, job = c*(l+1)+m
    const u64* F;                            // [6][l+1][n] folded sums
    u64* acc;                                // [2][l+1][n]
    int l;
    Dev d;
    struct Ctx {
        const u64 *z, *s, *a;
        u64* out;
        ulonglong2 w;        // p^-1 mod q_m
        int m;
    };
    HS_DEV Ctx make(int jb) const {
        const int c = jb / (l + 1), m = jb % (l + 1);
        const size_t ls = (size_t)(l + 1) * d.n, o = (size_t)m * d.n;
        return Ctx{F + (4 + c) * ls + o, F + c * ls + o, F + (2 + c) * ls + o, acc + (size_t)c * ls + o,
                   d.auxinv[m], m};
    }
    HS_DEV int prime(const Ctx& c) const { return c.m; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst&) const { return __ldg(c.z + j); }
    HS_DEV u64* scratch(const Ctx& c) const { return c.out; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        const u64 r = shoup_lazy(__ldg(c.s + j) + (P.two_q << 1) - v, c.w.x, c.w.y, P.q);   // [0, 2q)
        c.out[j] = csub(csub(r + __ldg(c.a + j), P.two_q), P.q);
    }
};

__global__ void accum_fold_kernel(Dev d, int nl, int nchunks, const u64* part, u64* acc);

bool rotate_accumulate(const Dev& d, int B, int l, ItemPtr ct, const u32* gal, const u64* const* keys,
                       u64* acc, u64* scratch, cudaStream_t st, int nkeys) {
    const u32 n = d.n;
    const int nl = l + 1;
    const size_t ls = (size_t)nl * n;
    // F and the chunk partials reuse the E region of the scratch (free after
    // the inner product): room for F plus at least one chunk
    const long cap = (long)((size_t)B * (l + 1) * (l + 2) * n / (6 * ls)) - 1;
    if (B <= 0 || cap < 1) return false;
    u64* E = scratch;
    u64* D = E + (size_t)B * (l + 1) * (l + 2) * n;
    u64* ACC = D + (size_t)B * (l + 1) * n;
    u64* T = ACC + (size_t)B * 2 * (l + 2) * n;
    launch_ntt<false>(d, JobDecompose<SrcPerm>{SrcPerm{ct, gal}, E, D, d.df, l, n, d}, B * (l + 1), st);
    modup_and_inner(d, B, l, D, E, keys, ACC, st, nkeys);
    launch_ntt<false>(d, JobInvGather{strided(ACC, (size_t)(l + 2) * n), 1, l + 2, l + 1, d.L + 1, T, n},
                      B * 2, st);
    const int cols = (int)((n + 255) / 256) * nl;
    int nchunks = std::max(1, std::min((B + 7) / 8, (148 * 8 + cols - 1) / cols));
    nchunks = (int)std::min<long>(nchunks, cap);
    const int chunk = (B + nchunks - 1) / nchunks;
    nchunks = (B + chunk - 1) / chunk;
    u64* F = E;
    u64* part = F + 6 * ls;
    cudaMemsetAsync(F, 0, 2 * ls * sizeof(u64), st);
    cudaMemcpyAsync(F + 2 * ls, acc, 2 * ls * sizeof(u64), cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(F + 4 * ls, 0, 2 * ls * sizeof(u64), st);
    rot_partial_kernel<<<dim3((n + 255) / 256, nl, nchunks), 256, 0, st>>>(d, B, l, chunk, ct, gal, ACC, T, part,
                                                                         nullptr);
    accum_fold_kernel<<<dim3((n + 255) / 256, 6 * nl), 256, 0, st>>>(d, nl, nchunks, part, F);
    note_launch(2);
    launch_ntt<true>(d, JobRotAcc{F, acc, l, d}, 2 * nl, st);
    return true;
}

// ---- rotate-and-accumulate with items grouped by key.
// Items [0, B) are sorted by rotation step, so the items sharing a Galois key
// form runs (groups gs[g] .. gs[g+1]-1).  Only the SUM over items of the
// rotated cts is needed, and for every chain modulus m <= l everything after
// the digits' lifts is linear:
//   sum_b acc_b,m = sum_i NTT_m(sum_b lift_m(x_b,i)) * K_g[i][m]   (m != i)
//                 + (sum_b x_b,i df_i) * K_g[i][i]                 (m == i)
// so the ModUp NTTs and the inner product of a chain modulus run once per
// group (into the group head's slots), not once per item.  The aux modulus
// stays per item: ModDown lifts T_b = INTT_p(acc_b,p) item by item (a
// non-linear step), so each item keeps its own aux digit transforms and aux
// accumulator.  Exact identities mod q_m: the residues equal the per-item
// rotations summed (the reference's eval_rotate + eval_add).
struct JobModUpGroup {                       // forward NTT, job = (g*(l+1)+i)*l + t
    const u64* D;                            // head slot of each group: signed sum (group_sum_kernel)
    u64* E;
    const int* gs;                           // [G+1] group starts (items)
    int l;
    u32 n;
    const PrimeConst* pc;
    struct Ctx {
        const u64* d;        // D[b0][i]: sum over the group of the centred digits (int64)
        u64* e;              // E[b0][i][m]
        int pm;
    };
    HS_DEV Ctx make(int jb) const {
        const int t = jb % l, gi = jb / l;
        const int i = gi % (l + 1), g = gi / (l + 1);
        const int m = t < i ? t : t + 1;     // m in [0, l] \ {i}
        const int b0 = gs[g];
        return Ctx{D + ((size_t)b0 * (l + 1) + i) * n, E + (((size_t)b0 * (l + 1) + i) * (l + 2) + m) * n, m};
    }
    HS_DEV int prime(const Ctx& c) const { return c.pm; }
    // sum_b lift_m(x_b) = (sum_b centred(x_b)) mod q_m: one signed reduction
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        const long long v = (long long)__ldg(c.d + j);
        const u64 t = reduce64(v < 0 ? 0ull - (u64)v : (u64)v, P);
        return (v < 0 && t) ? P.q - t : t;
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.e; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst&) const { c.e[j] = v; }   // [0, 4q)
};

struct JobModUpAux {                         // forward NTT, job = b*(l+1)+i: the aux target only
    const u64* D;
    u64* E;
    int l, L;
    u32 n;
    const PrimeConst* pc;
    struct Ctx {
        const u64* d;
        u64* e;
        u64 qsrc;
    };
    HS_DEV Ctx make(int jb) const {
        const int i = jb % (l + 1);
        return Ctx{D + (size_t)jb * n, E + ((size_t)jb * (l + 2) + l + 1) * n, pc[i].q};
    }
    HS_DEV int prime(const Ctx&) const { return L + 1; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
#if HS_LIFT_LAZY
        return lift_lazy(__ldg(c.d + j), c.qsrc, P);
#else
        return lift_mod(__ldg(c.d + j), c.qsrc, P);
#endif
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.e; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst&) const { c.e[j] = v; }
};

// Per group and digit i: D[b0][i] := sum_b centred(x_b,i) as int64 (|sum| <
// 16 q_i / 2 < 2^63 with at most 16 items per group), and
// E[b0][i][i] := sum_b E[b][i][i] (x_b,i df_i, canonical).  Runs after the
// per-item aux ModUp, which still reads every item's own digit.
__global__ void __launch_bounds__(256) group_sum_kernel(Dev d, int l, const int* __restrict__ gs, u64* D,
                                                        u64* E) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * 256 + threadIdx.x;
    const int i = blockIdx.y, g = blockIdx.z;
    const int b0 = gs[g], b1 = gs[g + 1];
    if (k >= n) return;
    const u64 q = d.pc[i].q, half = q >> 1;
    const size_t ditem = (size_t)(l + 1) * n, od = (size_t)i * n + k;
    long long sum = 0;
    for (int b = b0; b < b1; b++) {
        const u64 x = D[(size_t)b * ditem + od];
        sum += x > half ? (long long)x - (long long)q : (long long)x;
    }
    D[(size_t)b0 * ditem + od] = (u64)sum;
    if (b1 - b0 < 2) return;
    const size_t item = (size_t)(l + 1) * (l + 2) * n, o = ((size_t)i * (l + 2) + i) * n + k;
    u64 acc = E[(size_t)b0 * item + o];
    for (int b = b0 + 1; b < b1; b++) acc = add_mod(acc, __ldg(E + (size_t)b * item + o), q);
    E[(size_t)b0 * item + o] = acc;
}

bool rotate_accumulate_grouped(const Dev& d, int B, int G, const int* gs, const unsigned char* head, int l,
                               ItemPtr ct, const u32* gal, const u64* const* keys, u64* acc, u64* scratch,
                               cudaStream_t st) {
    const u32 n = d.n;
    const int nl = l + 1;
    const size_t ls = (size_t)nl * n;
    const long cap = (long)((size_t)B * (l + 1) * (l + 2) * n / (6 * ls)) - 1;
    if (B <= 0 || G <= 0 || cap < 1 || !ks_inner_tma_ok(d) || l < 1) return false;
    u64* E = scratch;
    u64* D = E + (size_t)B * (l + 1) * (l + 2) * n;
    u64* ACC = D + (size_t)B * (l + 1) * n;
    u64* T = ACC + (size_t)B * 2 * (l + 2) * n;
    const size_t e_item = (size_t)(l + 1) * (l + 2) * n;
    launch_ntt<false>(d, JobDecompose<SrcPerm>{SrcPerm{ct, gal}, E, D, d.df, l, n, d}, B * (l + 1), st);
    {
        const double jobs = (double)G * (l + 1) * l + (double)B * (l + 1), nn = n;
        ProbeScope ps(PROBE_MODUP, st, (3.0 * jobs + 2.0 * B * (l + 1)) * 8.0 * nn, jobs * (nn / 2) * d.log_n, 4);
        launch_ntt<true>(d, JobModUpAux{D, E, l, d.L, n, d.pc}, B * (l + 1), st);
        group_sum_kernel<<<dim3((n + 255) / 256, l + 1, G), 256, 0, st>>>(d, l, gs, D, E);
        note_launch();
        launch_ntt<true>(d, JobModUpGroup{D, E, gs, l, n, d.pc}, G * (l + 1) * l, st);
    }
    {
        const double limb = 8.0 * n;
        const double bytes = (double)G * (l + 1) * (l + 1) * limb + (double)B * (l + 1) * limb +
                             (double)G * 2 * (l + 1) * (l + 2) * limb + (double)B * 2 * (l + 2) * limb;
        ProbeScope ps(PROBE_KS_INNER, st, bytes, 2.0 * ((double)G * (l + 1) * (l + 1) + (double)B * (l + 1)) * n, 2);
        launch_ks_inner(d, l, G, E, e_item, keys, ACC, st, gs, 0, l + 1);     // chain moduli, per group
        launch_ks_inner(d, l, B, E, e_item, keys, ACC, st, nullptr, l + 1, 1); // aux modulus, per item
    }
    launch_ntt<false>(d, JobInvGather{strided(ACC, (size_t)(l + 2) * n), 1, l + 2, l + 1, d.L + 1, T, n},
                      B * 2, st);
    const int cols = (int)((n + 255) / 256) * nl;
    int nchunks = std::max(1, std::min((B + 7) / 8, (148 * 8 + cols - 1) / cols));
    nchunks = (int)std::min<long>(nchunks, cap);
    const int chunk = (B + nchunks - 1) / nchunks;
    nchunks = (B + chunk - 1) / chunk;
    u64* F = E;
    u64* part = F + 6 * ls;
    cudaMemsetAsync(F, 0, 2 * ls * sizeof(u64), st);
    cudaMemcpyAsync(F + 2 * ls, acc, 2 * ls * sizeof(u64), cudaMemcpyDeviceToDevice, st);
    cudaMemsetAsync(F + 4 * ls, 0, 2 * ls * sizeof(u64), st);
    rot_partial_kernel<<<dim3((n + 255) / 256, nl, nchunks), 256, 0, st>>>(d, B, l, chunk, ct, gal, ACC, T, part,
                                                                         head);
    accum_fold_kernel<<<dim3((n + 255) / 256, 6 * nl), 256, 0, st>>>(d, nl, nchunks, part, F);
    note_launch(2);
    launch_ntt<true>(d, JobRotAcc{F, acc, l, d}, 2 * nl, st);
    return true;
}

// Hoisted rotations (P3 of SURVEY.md): decompose + ModUp the source once; per
// step only the automorphism-gathered inner product and ModDown remain.
void rotate_hoisted(const Dev& d, int R, int l, const u64* src, const u32* gal,
                    const u64* const* keys, ItemPtr out, u64* scratch, cudaStream_t st) {
    const u32 n = d.n;
    u64* E = scratch;
    u64* D = E + (size_t)(l + 1) * (l + 2) * n;
    u64* ACC = D + (size_t)(l + 1) * n;
    u64* T = ACC + (size_t)R * 2 * (l + 2) * n;
    ItemPtr s = strided(src, 0);
    launch_ntt<false>(d, JobDecompose<SrcPlain>{SrcPlain{s, 1}, E, D, d.df, l, n, d}, l + 1, st);
    launch_ntt<true>(d, JobModUp{D, E, l, d.L, n, d.pc}, (l + 1) * (l + 1), st);
    ks_inner_kernel<<<ks_inner_grid(d, l, R), KSI_T, 0, st>>>(d, l, R, E, 0, keys, gal, ACC);
    note_launch();
    mod_down(d, R, l, ACC, T, AddPermC0{s, gal}, out, st);
}

// =========================================================== rescale

struct JobRescale {                          // forward NTT, job = (b*npoly+c)*l+i
    const u64* T;
    ItemPtr in, out, mask;
    int l, npoly;
    const PrimeConst* pc;
    const ulonglong2* qlinv;                 // row for level l
    u32 n;
    struct Ctx {
        const u64* t;        // INTT of the last limb (coefficients mod q_l)
        const u64* x;        // in(b)[c][i]
        u64* out;            // out(b)[c][i]
        const u64* mask;     // mask(b)[i] (Montgomery form) or null
        ulonglong2 w;        // q_l^-1 mod q_i
        u64 ql;
        int i;
        bool small;          // q_l / 2 < q_i
    };
    HS_DEV Ctx make(int jb) const {
        const int bc = jb / l, i = jb % l;
        const int b = bc / npoly, c = bc % npoly;
        const bool has_mask = mask.tab || mask.base;
        return Ctx{T + (size_t)bc * n, in.at(b) + ((size_t)c * (l + 1) + i) * n,
                   out.atw(b) + ((size_t)c * l + i) * n, has_mask ? mask.at(b) + (size_t)i * n : nullptr,
                   qlinv[i], pc[l].q, i, (pc[l].q >> 1) < pc[i].q};
    }
    HS_DEV int prime(const Ctx& c) const { return c.i; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        return lift_mod_sel(__ldg(c.t + j), c.ql, P, c.small);
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.out; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        u64 r = shoup_lazy(__ldg(c.x + j) + (P.two_q << 1) - v, c.w.x, c.w.y, P.q);    // [0, 2q)
        // mask in Montgomery form; no mask = Montgomery one (2^64 mod q): one code path
        const u64 mk = c.mask ? __ldg(c.mask + j) : P.r_mod;
        r = mont_mul_lazy(r, mk, P.q, P.qinv_neg);                                    // [0, 2q)
        c.out[j] = csub(r, P.q);
    }
};

size_t rescale_scratch_elems(int B, int npoly, u32 n) { return (size_t)B * npoly * n; }

void rescale_batch(const Dev& d, int B, int l, int npoly, ItemPtr in, ItemPtr out,
                   ItemPtr mask_mont, u64* T, cudaStream_t st) {
    launch_ntt<false>(d, JobInvGather{in, npoly, l + 1, l, l, T, d.n}, B * npoly, st);
    JobRescale jr{T, in, out, mask_mont, l, npoly, d.pc, d.qlinv + (size_t)l * (d.L + 1), d.n};
    launch_ntt<true>(d, jr, B * npoly * l, st);
}

// =========================================================== elementwise

__global__ void tensor_kernel(Dev d, int l, ItemPtr a, ItemPtr b, ItemPtr out) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, it = blockIdx.z;
    if (k >= n) return;
    const PrimeConst P = d.pc[i];
    const size_t nl = l + 1;
    const u64* A = a.at(it);
    const u64* B = b.at(it);
    u64* O = out.atw(it);
    const u64 a0 = A[i * n + k], a1 = A[(nl + i) * n + k];
    const u64 b0 = B[i * n + k], b1 = B[(nl + i) * n + k];
    O[i * n + k] = mul_mod(a0, b0, P);
    u64 lo = 0, hi = 0;
    mac128(lo, hi, a0, b1);
    mac128(lo, hi, a1, b0);
    O[(nl + i) * n + k] = barrett128(lo, hi, P);
    O[(2 * nl + i) * n + k] = mul_mod(a1, b1, P);
}

void tensor_batch(const Dev& d, int B, int l, ItemPtr a, ItemPtr b, ItemPtr out, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, l + 1, B);
    tensor_kernel<<<g, 256, 0, st>>>(d, l, a, b, out);
    note_launch();
}

__global__ void mult_pt_kernel(Dev d, int l, int npoly, ItemPtr ct, ItemPtr pt, ItemPtr out,
                               bool mont) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y % (l + 1), c = blockIdx.y / (l + 1), it = blockIdx.z;
    if (k >= n) return;
    const PrimeConst P = d.pc[i];
    const size_t o = ((size_t)c * (l + 1) + i) * n + k;
    const u64 x = ct.at(it)[o], y = pt.at(it)[(size_t)i * n + k];
    out.atw(it)[o] = mont ? mont_mul(x, y, P.q, P.qinv_neg) : mul_mod(x, y, P);
}

void mult_pt_batch(const Dev& d, int B, int l, int npoly, ItemPtr ct, ItemPtr pt, ItemPtr out,
                   bool pt_mont, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, npoly * (l + 1), B);
    mult_pt_kernel<<<g, 256, 0, st>>>(d, l, npoly, ct, pt, out, pt_mont);
    note_launch();
}

__global__ void add_kernel(Dev d, int l, ItemPtr a, ItemPtr b, ItemPtr out) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y % (l + 1), it = blockIdx.z;
    if (k >= n) return;
    const size_t o = (size_t)blockIdx.y * n + k;
    out.atw(it)[o] = add_mod(a.at(it)[o], b.at(it)[o], d.pc[i].q);
}

void add_batch(const Dev& d, int B, int l, int npoly, ItemPtr a, ItemPtr b, ItemPtr out,
               cudaStream_t st) {
    dim3 g((d.n + 255) / 256, npoly * (l + 1), B);
    add_kernel<<<g, 256, 0, st>>>(d, l, a, b, out);
    note_launch();
}

// Order-free modular sum over items, in two stages so that
// the item loop is split over CTAs: stage 1 writes one partial per chunk of
// items (grid.z = chunks), stage 2 folds the partials into acc.  (One CTA
// column per limb walking all B items serially left the GPU idle at level 0.)
__global__ void accum_partial_kernel(Dev d, int B, int nl, int chunk, ItemPtr src, u64* part,
                                     bool accumulate_into) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int m = blockIdx.y % nl;
    const u64 q = d.pc[m].q;
    const size_t o = (size_t)blockIdx.y * n + k;
    const int b0 = blockIdx.z * chunk, b1 = min(B, b0 + chunk);
    u64* dst = part + (size_t)blockIdx.z * gridDim.y * n + o;
    u64 s = accumulate_into ? *dst : 0ull;
    for (int b = b0; b < b1; b++) s = add_mod(s, __ldg(src.at(b) + o), q);
    *dst = s;
}

__global__ void accum_fold_kernel(Dev d, int nl, int nchunks, const u64* part, u64* acc) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int m = blockIdx.y % nl;
    const u64 q = d.pc[m].q;
    const size_t o = (size_t)blockIdx.y * n + k, stride = (size_t)gridDim.y * n;
    u64 s = acc[o];
    for (int c = 0; c < nchunks; c++) s = add_mod(s, part[c * stride + o], q);
    acc[o] = s;
}

void accumulate(const Dev& d, int B, int nl, int npoly, ItemPtr src, u64* acc, cudaStream_t st) {
    if (B <= 0) return;
    const int limbs = npoly * nl;
    const int cols = (int)((d.n + 255) / 256) * limbs;
    // enough CTAs for ~8 per SM, chunks of >= 16 items
    int nchunks = std::max(1, std::min((B + 15) / 16, (148 * 8 + cols - 1) / cols));
    const int chunk = (B + nchunks - 1) / nchunks;
    nchunks = (B + chunk - 1) / chunk;
    u64* part = nullptr;
    if (cudaMallocAsync((void**)&part, (size_t)nchunks * limbs * d.n * sizeof(u64), st) != cudaSuccess) {
        cudaGetLastError();
        part = nullptr;
    }
    if (!part) {                                   // no scratch: one chunk straight into acc
        accum_partial_kernel<<<dim3((d.n + 255) / 256, limbs, 1), 256, 0, st>>>(d, B, nl, B, src, acc, true);
        note_launch();
        return;
    }
    accum_partial_kernel<<<dim3((d.n + 255) / 256, limbs, nchunks), 256, 0, st>>>(d, B, nl, chunk, src, part,
                                                                                  false);
    accum_fold_kernel<<<dim3((d.n + 255) / 256, limbs), 256, 0, st>>>(d, nl, nchunks, part, acc);
    note_launch(2);
    cudaFreeAsync(part, st);
}

__global__ void mont_kernel(Dev d, u64* buf, size_t total, PrimeMap pm, bool inverse) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total) return;
    const int limb = (int)((idx / d.n) % pm.nl);
    const PrimeConst P = d.pc[pm.p[limb]];
    buf[idx] = mont_mul(buf[idx], inverse ? 1ull : P.r2_mod, P.q, P.qinv_neg);
}

void to_montgomery(const Dev& d, u64* buf, size_t nlimb_total, const PrimeMap& pm, bool inverse,
                   cudaStream_t st) {
    size_t total = nlimb_total * d.n;
    if (!total) return;
    mont_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(d, buf, total, pm, inverse);
    note_launch();
}

__global__ void signed_kernel(Dev d, const long long* coeffs, int nl, PrimeMap pm, u64* out) {
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d.n) return;
    const int l = blockIdx.y;
    const PrimeConst P = d.pc[pm.p[l]];
    const long long c = coeffs[k];
    u64 r;
    if (c >= 0) {
        r = reduce64((u64)c, P);
    } else {
        u64 t = reduce64((u64)(-(c + 1)) + 1ull, P);
        r = t ? P.q - t : 0ull;
    }
    out[(size_t)l * d.n + k] = r;
}

void signed_to_limbs(const Dev& d, const long long* coeffs, int nl, const PrimeMap& pm, u64* out,
                     cudaStream_t st) {
    dim3 g((d.n + 255) / 256, nl);
    signed_kernel<<<g, 256, 0, st>>>(d, coeffs, nl, pm, out);
    note_launch();
}

// key layout [2][L+1][L+2][n]; ntt_e [L+1][L+2][n]; target/sk [L+2][n]; f [(L+1)*(L+1)]
__global__ void ksk_kernel(Dev d, u64* key, const u64* ntt_e, const u64* target, const u64* sk,
                           const ulonglong2* f) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int m = blockIdx.y, i = blockIdx.z, L = d.L;
    const PrimeConst P = d.pc[m];
    const size_t o = ((size_t)i * (L + 2) + m) * n + k;
    u64 acc = ntt_e[o];
    if (m <= L) {
        ulonglong2 w = f[i * (L + 1) + m];
        acc = add_mod(acc, shoup(target[(size_t)m * n + k], w.x, w.y, P.q), P.q);
    }
    const u64* a = key + (size_t)(L + 1) * (L + 2) * n;
    acc = sub_mod(acc, mul_mod(a[o], sk[(size_t)m * n + k], P), P.q);
    key[o] = acc;
}

void ksk_combine(const Dev& d, u64* key, const u64* ntt_e, const u64* target, const u64* sk,
                 const ulonglong2* f, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, d.L + 2, d.L + 1);
    ksk_kernel<<<g, 256, 0, st>>>(d, key, ntt_e, target, sk, f);
    note_launch();
}

__global__ void enc_kernel(Dev d, int nl, const u64* v, const u64* pkb, const u64* pka,
                           const u64* e0, const u64* e1, const u64* pt, u64* ct) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = blockIdx.y;
    const PrimeConst P = d.pc[i];
    const size_t o = (size_t)i * n + k;
    const u64 vv = v[o];
    u64 c0 = add_mod(mul_mod(vv, pkb[o], P), e0[o], P.q);
    ct[o] = add_mod(c0, pt[o], P.q);
    ct[(size_t)nl * n + o] = add_mod(mul_mod(vv, pka[o], P), e1[o], P.q);
}

void encrypt_combine(const Dev& d, int nl, const u64* v, const u64* pkb, const u64* pka,
                     const u64* e0, const u64* e1, const u64* pt, u64* ct, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, nl);
    enc_kernel<<<g, 256, 0, st>>>(d, nl, v, pkb, pka, e0, e1, pt, ct);
    note_launch();
}

__global__ void dec_kernel(Dev d, int nl, const u64* ct, const u64* sk, u64* pt) {
    const u32 n = d.n;
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = blockIdx.y;
    const PrimeConst P = d.pc[i];
    const size_t o = (size_t)i * n + k;
    pt[o] = add_mod(ct[o], mul_mod(ct[(size_t)nl * n + o], sk[o], P), P.q);
}

void decrypt_combine(const Dev& d, int nl, const u64* ct, const u64* sk, u64* pt, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, nl);
    dec_kernel<<<g, 256, 0, st>>>(d, nl, ct, sk, pt);
    note_launch();
}

__global__ void seam_kernel(int op, size_t count, const u64* a, const u64* b, u64* out,
                            PrimeConst P, u64 s, u64 s_sh, u64 q_src) {
    const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const u64 q = P.q;
    switch (op) {
        case SEAM_ADD: out[k] = add_mod(a[k], b[k], q); break;
        case SEAM_SUB: out[k] = sub_mod(a[k], b[k], q); break;
        case SEAM_NEG: out[k] = a[k] ? q - a[k] : 0ull; break;
        case SEAM_MUL: out[k] = mul_mod(a[k], b[k], P); break;
        case SEAM_SCALAR: out[k] = shoup(a[k], s, s_sh, q); break;
        case SEAM_FMA: out[k] = add_mod(out[k], mul_mod(a[k], b[k], P), q); break;
        case SEAM_EXTEND: out[k] = lift_mod(a[k], q_src, P); break;
    }
}

void seam_op(int op, size_t count, const u64* a, const u64* b, u64* out, PrimeConst P, u64 s,
             u64 q_src, cudaStream_t st) {
    if (!count) return;
    s %= P.q;
    u64 s_sh = (u64)(((unsigned __int128)s << 64) / P.q);
    seam_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(op, count, a, b, out, P, s, s_sh,
                                                                 q_src);
    note_launch();
}

}  // namespace hs

namespace hs {
__global__ void reduce_kernel(Dev d, u64* data, int nl) {
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d.n) return;
    const PrimeConst P = d.pc[blockIdx.y % nl];
    const size_t o = (size_t)blockIdx.y * d.n + k;
    data[o] = reduce64(data[o], P);
}
void reduce_mod(const Dev& d, u64* data, int npoly, int nl, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, npoly * nl);
    reduce_kernel<<<g, 256, 0, st>>>(d, data, nl);
    note_launch();
}
}  // namespace hs
