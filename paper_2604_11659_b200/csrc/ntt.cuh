// Batched negacyclic NTT / INTT for RNS limbs, sm_100a.
//
// Transform definition (bit-exact with the reference _fast.pyx:44-100):
//   forward  = Cooley-Tukey, stage s = 0..log n-1 (m = 2^s, t = n/2m),
//              butterfly (v[j], v[j+t]) with twiddle roots[m + (j >> (log n - s))],
//              roots[k] = psi^brev(k); natural order in, bit-reversed out.
//   inverse  = Gentleman-Sande stages in reverse order with iroots, then * n^-1.
// Any schedule of the same butterflies that canonicalises its output gives
// identical residues, so the device is free to tile, fuse and reduce lazily.
//
// Tiling: a pass covers a contiguous range of stages [s0, s0+LOGG).  Those
// stages only mix indices that differ in bits [log n - s0 - LOGG, log n - s0),
// so the limb splits into independent groups of G = 2^LOGG elements.  One CTA
// owns H x G x C elements: H consecutive "hi" values (bits above the range)
// and C consecutive "lo" columns (bits below it).  n <= 2^11 runs as one pass
// (whole limb per CTA); larger limbs run as two passes (strided column pass +
// contiguous row pass), in place in the destination buffer.
//
// Two engines share the butterfly helpers:
//  * PassEngine (ntt_pass_kernel): radix-16 register rounds, 16 elements per
//    thread, the first/last round talking to global memory directly when that
//    is coalesced, one padded shared-memory exchange per round boundary.
//  * the radix-8 shared-memory rounds (ntt_round*), kept for the fused
//    ModUp + key inner-product kernel (ops.cu) whose 128-bit accumulators
//    leave no registers for 16 elements per thread.
//
// A "Job" functor supplies, per batch entry (blockIdx.y): prime(), the
// first-pass load(), the last-pass store(), and scratch() -- the limb buffer
// used in place between passes.  Fusions (basis lift on load, key-switch /
// rescale epilogues on store) are expressed as Job types in ops.cu.
#pragma once
#include <type_traits>

#include "hs_internal.cuh"

namespace hs {

constexpr int NTT_TILE = 2048;      // elements per CTA tile (16 KiB + padding)

// ======================================================= modular helpers
// x - m if x >= m (x, m < 2^63): sign test on the difference.
HS_DEV u64 csub_s(u64 x, u64 m) {
    const u64 d = x - m;
    return (long long)d < 0 ? x : d;
}

HS_DEV u64 mulhi_ex(u64 x, u64 y) { return __umul64hi(x, y); }

// hi64(x*y) minus 0, 1 or 2: drops the low x0*y0 product and the low halves
// of the two cross products (each dropped part is < one unit of 2^64).
HS_DEV u64 mulhi_apx(u64 x, u64 y) {
    const u32 x0 = (u32)x, x1 = (u32)(x >> 32), y0 = (u32)y, y1 = (u32)(y >> 32);
    const u64 r = (u64)x1 * y1 + __umulhi(x1, y0);
    return r + __umulhi(x0, y1);
}

// Shoup products x*w mod q given w_sh = floor(w 2^64 / q), any x < 2^64:
// exact quotient estimate -> [0, 2q); approximate -> [0, 4q).
// x*w - Q*q is formed as x*w + Q*(2^64 - q) (nq) so the chain is pure IMADs.
HS_DEV u64 shoup_ex(u64 x, u64 w, u64 w_sh, u64 nq) { return x * w + mulhi_ex(x, w_sh) * nq; }

#ifndef NTT_SHOUP_CC
#define NTT_SHOUP_CC 1
#endif
// Approximate-quotient Shoup product in 11 IMADs (all on the FMA pipe; the
// 64-bit accumulations use IMAD.WIDE with a unit multiplier so no register
// pair has to be assembled with MOVs):
//   Q = x1 s1 + hi(x1 s0) + hi(x0 s1)               (Q in [Q_exact - 2, Q_exact])
//   r = lo64(x w + Q nq)                              (r in [0, 4q))
HS_DEV u64 shoup_ax(u64 x, u64 w, u64 w_sh, u64 nq) {
    u64 r;
    asm("{\n\t"
        ".reg .u32 x0, x1, w0, w1, s0, s1, n0, n1, a, b, q0, q1, t0, t1;\n\t"
        ".reg .u64 Q, T;\n\t"
        "mov.b64 {x0, x1}, %1;\n\t"
        "mov.b64 {w0, w1}, %2;\n\t"
        "mov.b64 {s0, s1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\t"
#if NTT_SHOUP_CC == 2
        // as below, with x1 s1 as mul.lo + mul.hi (no IMAD.WIDE for Q)
        "mul.lo.u32 q0, x1, s1;\n\t"
        "mul.hi.u32 q1, x1, s1;\n\t"
        "mad.hi.cc.u32 q0, x1, s0, q0;\n\t"
        "addc.u32 q1, q1, 0;\n\t"
        "mad.hi.cc.u32 q0, x0, s1, q0;\n\t"
        "addc.u32 q1, q1, 0;\n\t"
#elif NTT_SHOUP_CC
        // Q = x1 s1 + hi(x1 s0) + hi(x0 s1): the two high halves added into
        // the low word with carry (mad.hi.cc + addc): no zero-extended 64-bit
        // addends, so no register moves on the FMA pipe
        "mul.wide.u32 Q, x1, s1;\n\t"
        "mov.b64 {q0, q1}, Q;\n\t"
        "mad.hi.cc.u32 q0, x1, s0, q0;\n\t"
        "addc.u32 q1, q1, 0;\n\t"
        "mad.hi.cc.u32 q0, x0, s1, q0;\n\t"
        "addc.u32 q1, q1, 0;\n\t"
#else
        "mul.hi.u32 a, x1, s0;\n\t"
        "mul.hi.u32 b, x0, s1;\n\t"
        "mul.wide.u32 Q, x1, s1;\n\t"
        "mad.wide.u32 Q, a, 1, Q;\n\t"
        "mad.wide.u32 Q, b, 1, Q;\n\t"
        "mov.b64 {q0, q1}, Q;\n\t"
#endif
        "mul.wide.u32 T, x0, w0;\n\t"
        "mad.wide.u32 T, q0, n0, T;\n\t"
        "mov.b64 {t0, t1}, T;\n\t"
        "mad.lo.u32 t1, x0, w1, t1;\n\t"
        "mad.lo.u32 t1, x1, w0, t1;\n\t"
        "mad.lo.u32 t1, q0, n1, t1;\n\t"
        "mad.lo.u32 t1, q1, n0, t1;\n\t"
        "mov.b64 %0, {t0, t1};\n\t"
        "}"
        : "=l"(r)
        : "l"(x), "l"(w), "l"(w_sh), "l"(nq));
    return r;
}

// t mod q up to a small multiple: [0, 4q) for any t < 2^64 (approximate
// Barrett quotient with floor(2^64 / q)).
HS_DEV u64 reduce64_lazy(u64 t, const PrimeConst& P) { return t - mulhi_apx(t, P.m64) * P.q; }

// Centred lift of v mod q_src into q_dst = P.q, left in [0, 4 q_dst) (a
// forward NTT's first-pass loader may return < 4q): the magnitude reduced
// with the approximate Barrett quotient, negatives as 4q - t.
HS_DEV u64 lift_lazy(u64 v, u64 q_src, const PrimeConst& P) {
    const bool neg = v > (q_src >> 1);
    const u64 t = reduce64_lazy(neg ? q_src - v : v, P);
    return (neg && t) ? (P.two_q << 1) - t : t;
}

// ======================================================= radix-8 smem rounds
constexpr int NTT_EPT = 8;          // elements per thread
constexpr int NTT_THREADS = NTT_TILE / NTT_EPT;

// Shared-memory index with one pad word per 8.
HS_DEV u32 spad(u32 i) { return i + (i >> 3); }

// One register round: local stages [A, A+R) of a tile with H rows, G = 2^LOGG
// group elements and C columns, read from and written back to shared memory.
template <bool FWD, int LOGG, int H, int C, int A, int R>
__device__ __forceinline__ void ntt_round(u64* sm, const ulonglong2* __restrict__ tw, u32 hi0,
                                          int s0, u64 q, u64 two_q) {
    constexpr int G = 1 << LOGG;
    constexpr int TILE = H * G * C;
    constexpr int T = TILE / NTT_EPT;
    constexpr int NU = 1 << R;
    constexpr int UPT = NTT_EPT / NU;
    constexpr int LOWB = LOGG - A - R;
    constexpr int S = (1 << LOWB) * C;
    static_assert(S % 8 == 0 || (S == 1 && R == 3), "round schedule must keep smem affine");
    constexpr int PS = S % 8 == 0 ? S + S / 8 : 1;
    const u64 nq = 0ull - q;
#pragma unroll
    for (int k = 0; k < UPT; k++) {
        const u32 U = threadIdx.x + k * T;
        const u32 c = U % C;
        const u32 rest = U / C;
        const u32 go = rest % (G >> R);
        const u32 h = rest / (G >> R);
        const u32 go_high = go >> LOWB;
        const u32 go_low = go & ((1u << LOWB) - 1);
        const u32 gbase = (go_high << (LOWB + R)) | go_low;
        const u32 hi = hi0 + h;
        const u32 base = spad((h * G + gbase) * C + c);
        u64 v[NU];
#pragma unroll
        for (int e = 0; e < NU; e++) v[e] = sm[base + e * PS];
#pragma unroll
        for (int jj = 0; jj < R; jj++) {
            const int j = FWD ? jj : R - 1 - jj;
            const int ls = A + j;
            const ulonglong2* __restrict__ twb = tw + ((1u << (s0 + ls)) + (hi << ls) + (go_high << j));
            const int bit = 1 << (R - 1 - j);
#pragma unroll
            for (int e = 0; e < NU; e++) {
                if (e & bit) continue;
                const ulonglong2 w = twb[e >> (R - j)];
                if (FWD) {
                    const u64 x = csub_s(v[e], two_q);
                    const u64 t = shoup_ex(v[e + bit], w.x, w.y, nq);
                    v[e] = x + t;
                    v[e + bit] = x - t + two_q;
                } else {
                    const u64 x = v[e], y = v[e + bit];
                    v[e] = csub_s(x + y, two_q);
                    v[e + bit] = shoup_ex(x - y + two_q, w.x, w.y, nq);
                }
            }
        }
#pragma unroll
        for (int e = 0; e < NU; e++) sm[base + e * PS] = v[e];
    }
}

// Round schedule: radix-8 rounds, the remainder (LOGG mod 3) as the
// second-to-last round, so the last (lowest-bit) round is always radix 8.
template <int LOGG>
struct RoundPlan {
    static constexpr int F = LOGG / 3, REM = LOGG % 3;
    static constexpr int count() { return F + (REM ? 1 : 0); }
    static constexpr int start(int r) {
        return REM == 0 ? 3 * r : (r < F - 1 ? 3 * r : (r == F - 1 ? 3 * (F - 1) : LOGG - 3));
    }
    static constexpr int width(int r) { return REM == 0 ? 3 : (r == F - 1 ? REM : 3); }
};

template <int LOGG, int H, int C, int RI>
__device__ __forceinline__ void ntt_rounds_fwd_from(u64* sm, const ulonglong2* tw, u32 hi0, int s0,
                                                    u64 q, u64 two_q) {
    if constexpr (RI < RoundPlan<LOGG>::count()) {
        ntt_round<true, LOGG, H, C, RoundPlan<LOGG>::start(RI), RoundPlan<LOGG>::width(RI)>(
            sm, tw, hi0, s0, q, two_q);
        __syncthreads();
        ntt_rounds_fwd_from<LOGG, H, C, RI + 1>(sm, tw, hi0, s0, q, two_q);
    }
}

// Forward stages [s0, s0+LOGG) of a tile held in shared memory (inputs < 4q,
// outputs in [0, 4q)).
template <int LOGG, int H, int C>
__device__ __forceinline__ void ntt_rounds_fwd(u64* sm, const ulonglong2* tw, u32 hi0, int s0, u64 q,
                                               u64 two_q) {
    ntt_rounds_fwd_from<LOGG, H, C, 0>(sm, tw, hi0, s0, q, two_q);
}

// ======================================================= radix-16 engine
// A pass of LOGG stages is split into register rounds of <= 4 stages (<= 3
// when EPT = 8).  Each thread holds EPT elements; in round r it owns
// EPT / 2^R "units" -- the 2^R elements that differ only in the round's bits
// -- and performs all their butterflies in registers.
#ifndef NTT_EPT_BIG
#define NTT_EPT_BIG 16
#endif
constexpr int NTT_EPT16 = NTT_EPT_BIG;   // elements per thread of the two-pass kernels (A/B knob)

template <int LOGG, int EPT>
struct Plan {
    static constexpr int MAXR = EPT >= 16 ? 4 : 3;
    static constexpr int count() { return LOGG <= MAXR ? 1 : (LOGG + MAXR - 1) / MAXR; }
    static constexpr int width(int r) { return LOGG / count() + (r < LOGG % count() ? 1 : 0); }
    static constexpr int start(int r) {
        int a = 0;
        for (int i = 0; i < r; i++) a += width(i);
        return a;
    }
};

// Padded shared-memory index (one pad word per 16 u64): with the unit
// mappings below, 16 consecutive lanes hit 16 distinct 8-byte bank pairs.
HS_DEV u32 spad16(u32 i) { return i + (i >> 4); }

template <int LOGG, int H, int C, int EPT, int A, int R>
struct RoundMap {
    static constexpr int G = 1 << LOGG;
    static constexpr int TILE = H * G * C;
    static constexpr int T = TILE / EPT;
    static constexpr int RR = R;
    static constexpr int AA = A;
    static constexpr int NU = 1 << R;
    static constexpr int UPT = EPT / NU;
    static constexpr int LOWB = LOGG - A - R;
    static constexpr int S = (1 << LOWB) * C;          // tile-index stride of a unit
    // Unit elements differ only in tile-index bits that are zero in the unit
    // base, so their padded offsets are compile-time constants.
    static constexpr u32 off(int e) { return (u32)(e * S + ((e * S) >> 4)); }
    // Consecutive threads touch runs of >= 4 consecutive global elements.
    static constexpr bool direct = C >= 4 || LOWB >= 2;
    struct Unit {
        u32 base;    // tile index of element 0
        u32 h;       // row within the tile
        u32 g;       // group index of element 0
        u32 c;       // column
        u32 gh;      // group bits above the round
    };
    HS_DEV static Unit unit(u32 U) {
        Unit u;
        u.c = U % C;
        const u32 rest = U / C;
        const u32 go = rest % (G >> R);
        u.h = rest / (G >> R);
        u.gh = go >> LOWB;
        u.g = (u.gh << (LOWB + R)) | (go & ((1u << LOWB) - 1u));
        u.base = (u.h * G + u.g) * C + u.c;
        return u;
    }
};

// Butterflies of one unit (2^R values in v[]).  Twiddle of local stage j,
// element e: tw[(Y << j) + (e >> (R - j))] with Y = ((2^s0 + hi) << A) + gh,
// i.e. roots[m + block] of the reference loop (_fast.pyx:55-66).
// Forward values grow lazily (all primes are < 2^60, so 16q < 2^64): with
// inputs in [0, 4q) and t = approximate Shoup product in [0, 4q), a stage
// maps bound b to b + 4q, so stages 0-2 need no reduction (4q -> 16q); from
// stage 3 on, every other stage first reduces the upper input by 8q
// (16q -> 12q -> 16q ...).  GS = global index of the stage.
HS_DEV constexpr bool fwd_reduce_at(int gs) { return gs >= 3 && ((gs - 3) & 1) == 0; }

template <bool FWD, int R, int GS>
HS_DEV void unit_butterflies(u64* v, const ulonglong2* __restrict__ tw, u32 Y, u64 nq, u64 two_q,
                             u64 four_q) {
    constexpr int NU = 1 << R;
#pragma unroll
    for (int jj = 0; jj < R; jj++) {
        const int j = FWD ? jj : R - 1 - jj;
        const ulonglong2* __restrict__ twp = tw + (Y << j);
        const int bit = 1 << (R - 1 - j);
#pragma unroll
        for (int e = 0; e < NU; e++) {
            if (e & bit) continue;
            const ulonglong2 w = twp[e >> (R - j)];
            if (FWD) {
                const u64 x = fwd_reduce_at(GS + jj) ? csub_s(v[e], four_q << 1) : v[e];   // < 12q
                const u64 t = shoup_ax(v[e + bit], w.x, w.y, nq);          // [0, 4q)
                v[e] = x + t;
                v[e + bit] = x - t + four_q;
            } else {
                const u64 x = v[e], y = v[e + bit];                      // [0, 4q)
                v[e] = csub_s(x + y, four_q);
                v[e + bit] = shoup_ax(x - y + four_q, w.x, w.y, nq);       // [0, 4q)
            }
        }
    }
}

// ---- NTT butterflies on the FP64 pipe (primes q <= 2^50 + 2^40, PC_F64);
// forward (Cooley-Tukey) here, inverse (Gentleman-Sande) in unit_butterflies_f64_inv
// The Shoup products above are 64-bit multiplies (IMAD.WIDE / IMAD.HI) that
// keep the FMA-heavy pipe ~80% busy; B200 also has a full-rate FP64 pipe, and
// for ~50-bit primes a residue is an exact double.  Values are signed
// integers held in doubles; every operation below is exact:
//   rint(y), |y| < 2^51:   FMA against 1.5*2^52 then subtract it (the sum stays
//                          in [2^52, 2^53), where the spacing of doubles is 1)
//   t = a*w mod q (lazy):  hi = RN(a w), lo = a w - hi (FMA, exact: TwoProduct),
//                          Q = rint(a * RN(w/q)), t = (hi - Q q) + lo (FMA then
//                          add; both results are integers below 2^53, hence
//                          exact), so t = a w - Q q.
//   |Q - a w/q| <= 1/2 + |a| 2^-53  =>  |t| <= (1/2 + k |a|/q) q, k = q 2^-53.
// Bounds (k <= 0.1252): the first pass reduces its inputs to |x| <= q/2; the
// unmultiplied input x is reduced to |x| <= q/2 at every odd global stage, so
// after a reducing stage B_r = 1 + k B_f and after a free one B_f = B_r + 1/2
// + k B_r (in units of q): the fixed point B_f = 1.89q bounds every value,
// and every multiplied |a| < 1.89q (1 + 2^-10) 2^50 < 2^51 keeps rint exact.
// The last pass reduces to [-q/2, q/2] and returns [q/2, 3q/2] as u64.
// Passes hand raw doubles to each other.  Any other prime (the 60-bit first
// and auxiliary primes) stays on the integer path.
HS_DEV constexpr bool f64_reduce_at(int gs) { return gs & 1; }
#ifndef HS_NTT_F64_INV
#define HS_NTT_F64_INV 1           // inverse NTTs on the FP64 pipe too
#endif
constexpr double kF64Magic = 6755399441055744.0;   // 1.5 * 2^52

HS_DEV double f64_rint_mul(double a, double b) {
    return __dsub_rn(__fma_rn(a, b, kF64Magic), kF64Magic);   // rint(a b), |a b| < 2^51
}
HS_DEV double f64_reduce(double x, double q, double qinv) {
    return __fma_rn(-f64_rint_mul(x, qinv), q, x);             // x - q rint(x / q), |.| <= q/2 + tiny
}
HS_DEV double f64_mulmod(double a, double w, double wq, double q) {
    const double hi = __dmul_rn(a, w);
    const double lo = __fma_rn(a, w, -hi);
    const double Q = f64_rint_mul(a, wq);
    return __dadd_rn(__fma_rn(-Q, q, hi), lo);
}

template <int R, int GS>
HS_DEV void unit_butterflies_f64(u64* v, const double2* __restrict__ tw, u32 Y, double q, double qinv) {
    constexpr int NU = 1 << R;
#pragma unroll
    for (int j = 0; j < R; j++) {
        const double2* __restrict__ twp = tw + (Y << j);
        const int bit = 1 << (R - 1 - j);
#pragma unroll
        for (int e = 0; e < NU; e++) {
            if (e & bit) continue;
            const double2 w = twp[e >> (R - j)];
            double x = __longlong_as_double((long long)v[e]);
            if (f64_reduce_at(GS + j)) x = f64_reduce(x, q, qinv);
            const double t = f64_mulmod(__longlong_as_double((long long)v[e + bit]), w.x, w.y, q);
            v[e] = (u64)__double_as_longlong(__dadd_rn(x, t));
            v[e + bit] = (u64)__double_as_longlong(__dsub_rn(x, t));
        }
    }
}

// Inverse (Gentleman-Sande) butterflies on the FP64 pipe: x' = rint-reduce(x + y)
// (|x'| <= q/2 + tiny), y' = (x - y) w mod q (lazy).  Every value stays below
// B = 1/2 + k 2B, i.e. 0.67q (k <= 0.1252), and |x - y| <= 1.34q keeps the
// rint argument below 2^51.
template <int R>
HS_DEV void unit_butterflies_f64_inv(u64* v, const double2* __restrict__ tw, u32 Y, double q, double qinv) {
    constexpr int NU = 1 << R;
#pragma unroll
    for (int jj = 0; jj < R; jj++) {
        const int j = R - 1 - jj;
        const double2* __restrict__ twp = tw + (Y << j);
        const int bit = 1 << (R - 1 - j);
#pragma unroll
        for (int e = 0; e < NU; e++) {
            if (e & bit) continue;
            const double2 w = twp[e >> (R - j)];
            const double x = __longlong_as_double((long long)v[e]);
            const double y = __longlong_as_double((long long)v[e + bit]);
            v[e] = (u64)__double_as_longlong(f64_reduce(__dadd_rn(x, y), q, qinv));
            v[e + bit] = (u64)__double_as_longlong(f64_mulmod(__dsub_rn(x, y), w.x, w.y, q));
        }
    }
}

// u64 in [0, 4q) -> reduced double bits, |x| <= q/2 (first pass)
HS_DEV u64 f64_enter(u64 u, double q, double qinv) {
    return (u64)__double_as_longlong(f64_reduce(__ull2double_rn(u), q, qinv));
}
// double bits, |x| < 2^52.5 -> u64 in [q/2, 3q/2] (last pass):
// x - q rint(x/q) + q + 2^52 lies in [2^52, 2^53), whose mantissa is the value
HS_DEV u64 f64_leave(u64 bits, double q, double qinv, double q_plus_2p52) {
    const double r = __dadd_rn(f64_reduce(__longlong_as_double((long long)bits), q, qinv), q_plus_2p52);
    return (u64)__double_as_longlong(r) & 0x000FFFFFFFFFFFFFull;
}

// Job interface: `typename Job::Ctx ctx = job.make(jb)` is evaluated once per
// CTA (pointer-table lookups, index decoding), then prime(ctx),
// load(ctx, j, P), scratch(ctx), store(ctx, j, v, P) per element.  load()
// returns [0, q) (forward loads may return < 4q); store() receives
// [0, 4q) in both directions.  Internal invariants: forward (Harvey) values
// stay below 16q (fwd_reduce_at; forward loads must return < 4q, passes hand
// raw values to the next pass), approximate Shoup in [0, 4q); inverse values
// stay in [0, 4q).
// Unroll factor of the staged (coalesced, one element per step) load/store
// loops: these inline the job's loader/epilogue, so full unrolling of 16
// copies of a heavy epilogue costs instruction-cache misses.
#ifndef NTT_IO_UNROLL
#define NTT_IO_UNROLL 8            // A/B at cfg2: 16 -> 174.0 ms, 4 -> 167.5, 2 -> 171.0 (6 CTAs/SM); at 8 CTAs/SM: 2 -> 121.4, 4 -> 121.0, 8 -> 120.0
#endif
constexpr int kIoUnroll = NTT_IO_UNROLL;   // (#pragma arguments are not macro-expanded)
// 1: rounds with two units per thread run them as a rolled loop (one copy of
// the butterfly code + register swaps).
#ifndef NTT_ROLL_UNITS
#define NTT_ROLL_UNITS 0
#endif
// 1: a pass whose loader is the job's (FIRST) always stages its tile through
// shared memory (rolled loop: smaller code) instead of loading directly.
#ifndef NTT_STAGED_FIRST
#define NTT_STAGED_FIRST 0
#endif

// Shared-memory exchange buffers per CTA: 2 = double-buffered (one barrier
// per exchange), 1 = single buffer (an extra barrier before each reuse).
#ifndef NTT_NBUF
#define NTT_NBUF 1             // A/B cfg2|cfg3s: 2 -> 125.0|892 ms, 1 -> 123.0|856, 1 + 8 CTAs/SM -> 120.5|850
#endif

// LOGN (log2 ring degree) and S0 (first stage of the pass) are template
// parameters so every index shift/mask below is a compile-time constant.
template <bool FWD, bool FIRST, bool LAST, int LOGG, int H, int C, int EPT, int LOGN, int S0, class Job>
struct PassEngine {
    static constexpr int LO_BITS = LOGN - S0 - LOGG;   // bits below the pass's range
    using PL = Plan<LOGG, EPT>;
    static constexpr int G = 1 << LOGG;
    static constexpr int TILE = H * G * C;
    static constexpr int T = TILE / EPT;
    static constexpr int NR = PL::count();
    static constexpr int SMW = TILE + TILE / 16;       // padded words per buffer
    template <int r>
    using RM = RoundMap<LOGG, H, C, EPT, PL::start(r), PL::width(r)>;
    static constexpr int RFIRST = FWD ? 0 : NR - 1;
    static constexpr int RLAST = FWD ? NR - 1 : 0;

    struct Env {
        typename Job::Ctx jc;
        PrimeConst P;
        const ulonglong2* __restrict__ tw;
        const double2* __restrict__ twd;   // FP64 roots of the pass's direction (f64)
        u32 t, hi0, lo0;
        u64 nq, four_q;
        bool f64;                          // butterflies on the FP64 pipe (PC_F64)
        double qd, qinvd;
        HS_DEV u32 gidx(u32 h, u32 g, u32 c) const {
            return ((hi0 + h) << (LOGN - S0)) | (g << LO_BITS) | (lo0 + c);
        }
    };

    HS_DEV static u64 in(const Job& job, const Env& E, u32 j) {
        if constexpr (FIRST) return job.load(E.jc, j, E.P);
        else return job.scratch(E.jc)[j];
    }
    HS_DEV static void out(const Job& job, const Env& E, u32 j, u64 v) {
        if constexpr (LAST) {
            if (FWD) v = csub_s(csub_s(v, E.four_q << 1), E.four_q);   // [0, 16q) -> [0, 4q)
            job.store(E.jc, j, v, E.P);
        } else {
            job.scratch(E.jc)[j] = v;
        }
    }

    template <int r>
    HS_DEV static void gather(const u64* buf, u64* v, const Env& E) {
        using M = RM<r>;
#pragma unroll
        for (int k = 0; k < M::UPT; k++) {
            const auto u = M::unit(E.t + k * T);
            const u64* p = buf + spad16(u.base);
#pragma unroll
            for (int e = 0; e < M::NU; e++) v[k * M::NU + e] = p[M::off(e)];
        }
    }
    template <int r>
    HS_DEV static void scatter(u64* buf, const u64* v, const Env& E) {
        using M = RM<r>;
#pragma unroll
        for (int k = 0; k < M::UPT; k++) {
            const auto u = M::unit(E.t + k * T);
            u64* p = buf + spad16(u.base);
#pragma unroll
            for (int e = 0; e < M::NU; e++) p[M::off(e)] = v[k * M::NU + e];
        }
    }
    template <int r>
    HS_DEV static void compute(u64* v, const Env& E) {
        using M = RM<r>;
        if constexpr (NTT_ROLL_UNITS && M::UPT == 2) {
            // two units of NU: one copy of the butterfly code, the halves
            // swapped between iterations (code size over a few moves)
#pragma unroll 1
            for (int k = 0; k < 2; k++) {
                const auto u = M::unit(E.t + k * T);
                const u32 Y = (((1u << S0) + E.hi0 + u.h) << M::AA) + u.gh;
                if (E.f64) {
                    if constexpr (FWD) unit_butterflies_f64<M::RR, S0 + M::AA>(v, E.twd, Y, E.qd, E.qinvd);
                    else unit_butterflies_f64_inv<M::RR>(v, E.twd, Y, E.qd, E.qinvd);
                } else
                    unit_butterflies<FWD, M::RR, S0 + M::AA>(v, E.tw, Y, E.nq, E.P.two_q, E.four_q);
#pragma unroll
                for (int e = 0; e < M::NU; e++) {
                    const u64 x = v[e];
                    v[e] = v[M::NU + e];
                    v[M::NU + e] = x;
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < M::UPT; k++) {
                const auto u = M::unit(E.t + k * T);
                const u32 Y = (((1u << S0) + E.hi0 + u.h) << M::AA) + u.gh;
                if (E.f64) {
                    if constexpr (FWD) unit_butterflies_f64<M::RR, S0 + M::AA>(v + k * M::NU, E.twd, Y, E.qd, E.qinvd);
                    else unit_butterflies_f64_inv<M::RR>(v + k * M::NU, E.twd, Y, E.qd, E.qinvd);
                } else
                    unit_butterflies<FWD, M::RR, S0 + M::AA>(v + k * M::NU, E.tw, Y, E.nq, E.P.two_q, E.four_q);
            }
        }
    }
    // FP64 path: enter after the first pass's load, leave before the last
    // pass's store (passes in between exchange raw doubles)
    HS_DEV static void f64_in(u64* v, const Env& E) {
        if constexpr (FIRST) {
            if (E.f64) {
#pragma unroll
                for (int k = 0; k < EPT; k++) v[k] = f64_enter(v[k], E.qd, E.qinvd);
            }
        }
    }
    HS_DEV static void f64_out(u64* v, const Env& E) {
        if constexpr (LAST) {
            if (E.f64) {
                const double k = E.qd + 4503599627370496.0;   // q + 2^52
#pragma unroll
                for (int i = 0; i < EPT; i++) v[i] = f64_leave(v[i], E.qd, E.qinvd, k);
            }
        }
    }

    // rounds after the first, in execution order (I = 1 .. NR-1)
    template <int I>
    HS_DEV static void rest(u64* sm, u64* v, const Env& E) {
        if constexpr (I < NR) {
            constexpr int rp = FWD ? I - 1 : NR - I;        // previous round
            constexpr int r = FWD ? I : NR - 1 - I;
            u64* buf = sm + (NTT_NBUF == 2 ? (I & 1) * SMW : 0);
            if constexpr (NTT_NBUF == 1) __syncthreads();   // previous readers of the buffer
            scatter<rp>(buf, v, E);
            __syncthreads();
            gather<r>(buf, v, E);
            compute<r>(v, E);
            rest<I + 1>(sm, v, E);
        }
    }

    HS_DEV static void run(u64* sm, const Env& E, const Job& job) {
        u64 v[EPT];
        using MF = RM<RFIRST>;
        using ML = RM<RLAST>;

        // ---- load
        if constexpr (MF::direct && !(FIRST && NTT_STAGED_FIRST)) {
            constexpr u32 gstride = 1u << (MF::LOWB + LO_BITS);
#pragma unroll
            for (int k = 0; k < MF::UPT; k++) {
                const auto u = MF::unit(E.t + k * T);
                const u32 j0 = E.gidx(u.h, u.g, u.c);
#pragma unroll
                for (int e = 0; e < MF::NU; e++) v[k * MF::NU + e] = in(job, E, j0 + e * gstride);
            }
        } else {
            u64* buf = sm;                // "exchange 0": exchange I uses buffer I & 1
#pragma unroll kIoUnroll
            for (int k = 0; k < EPT; k++) {
                const u32 i = E.t + k * T;
                buf[spad16(i)] = in(job, E, E.gidx(i / (G * C), (i / C) % G, i % C));
            }
            __syncthreads();
            gather<RFIRST>(buf, v, E);
        }
        f64_in(v, E);
        compute<RFIRST>(v, E);
        rest<1>(sm, v, E);
        f64_out(v, E);
        // ---- store
        if constexpr (ML::direct) {
            constexpr u32 gstride = 1u << (ML::LOWB + LO_BITS);
#pragma unroll
            for (int k = 0; k < ML::UPT; k++) {
                const auto u = ML::unit(E.t + k * T);
                const u32 j0 = E.gidx(u.h, u.g, u.c);
#pragma unroll
                for (int e = 0; e < ML::NU; e++) out(job, E, j0 + e * gstride, v[k * ML::NU + e]);
            }
        } else {
            u64* buf = sm + (NTT_NBUF == 2 ? (NR & 1) * SMW : 0);   // not written by the last exchange
            if constexpr (NTT_NBUF == 1) __syncthreads();
            scatter<RLAST>(buf, v, E);
            __syncthreads();
#pragma unroll kIoUnroll
            for (int k = 0; k < EPT; k++) {
                const u32 i = E.t + k * T;
                out(job, E, E.gidx(i / (G * C), (i / C) % G, i % C), buf[spad16(i)]);
            }
        }
    }
};

#ifndef NTT_MINB
#define NTT_MINB 8            // CTAs/SM for 16 elements per thread (128 threads; 64 registers)
#endif
#ifndef NTT_MINB8
#define NTT_MINB8 4           // for 8 elements per thread (256 threads)
#endif
template <bool FWD, bool FIRST, bool LAST, int LOGG, int H, int C, int EPT, int LOGN, int S0, class Job>
__global__ void __launch_bounds__(((H << LOGG) * C) / EPT, EPT >= 16 ? NTT_MINB : NTT_MINB8)
ntt_pass_kernel(Dev d, Job job, int jbase) {
    using PE = PassEngine<FWD, FIRST, LAST, LOGG, H, C, EPT, LOGN, S0, Job>;
    __shared__ u64 sm[NTT_NBUF * PE::SMW];
    typename PE::Env E;
    const int jb = jbase + (int)blockIdx.y;
    E.jc = job.make(jb);
    const int p = job.prime(E.jc);
    E.P = d.pc[p];
    E.tw = (FWD ? d.tw : d.itw) + ((size_t)p << LOGN);

    constexpr u32 ncolblk = (1u << PE::LO_BITS) / C;
    E.hi0 = (blockIdx.x / ncolblk) * H;
    E.lo0 = (blockIdx.x % ncolblk) * C;
    E.t = threadIdx.x;
    E.nq = 0ull - E.P.q;
    E.four_q = E.P.two_q << 1;
    E.f64 = (E.P.pad & PC_F64) && (FWD || HS_NTT_F64_INV);
    E.twd = (FWD ? d.twd : d.itwd) + ((size_t)p << LOGN);
    E.qd = (double)E.P.q;
    E.qinvd = __drcp_rn(E.qd);
    // One code path for every prime: a lazy forward variant (no upper-input
    // reduction for sub-2^56 primes) saved ~5 instructions per butterfly but
    // doubled the kernel's code, and instruction-cache misses cost more than
    // that (A/B on B200: 194.9 vs 206.7 ms per cfg2 matmul).
    PE::run(sm, E, job);
}

// Single-pass variant for small limbs (whole limb in one CTA, 8 per thread).
template <bool FWD, int LOGN, class Job>
void launch_ntt_single(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    dim3 grid(1, njobs);
    constexpr int EPT = LOGN >= 3 ? 8 : (1 << LOGN);
    constexpr int threads = (1 << LOGN) / EPT;
    ntt_pass_kernel<FWD, true, true, LOGN, 1, 1, EPT, LOGN, 0, Job><<<grid, threads, 0, st>>>(d, job, jbase);
    note_launch();
}

// Elements per thread of a job's column pass (A) and row pass (B): 16 unless
// the job declares kEptA / kEptB = 8 (256 threads).  No job does: per-kernel
// A/B at cfg2 favoured 8 for a few loader/epilogue-heavy passes (-3.7% of
// kernel time) but the same choice cost 45% at N = 2^16, L = 24.
template <class J, class = void>
struct EptA { static constexpr int value = NTT_EPT16; };
template <class J>
struct EptA<J, std::void_t<decltype(J::kEptA)>> { static constexpr int value = J::kEptA; };
template <class J, class = void>
struct EptB { static constexpr int value = NTT_EPT16; };
template <class J>
struct EptB<J, std::void_t<decltype(J::kEptB)>> { static constexpr int value = J::kEptB; };

// Two-pass variant: pass A covers stages [0, LA) over strided columns, pass B
// covers [LA, log n) over contiguous rows.  Forward runs A then B; inverse
// runs B then A.
template <bool FWD, int LA, int LB, class Job>
void launch_ntt_two(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    constexpr int CA = NTT_TILE >> LA;   // columns per tile in pass A
    constexpr int HB = NTT_TILE >> LB;   // rows per tile in pass B
    constexpr int EA = EptA<Job>::value, EB = EptB<Job>::value;
    const u32 n = 1u << (LA + LB);
    dim3 grid(n / NTT_TILE, njobs);
    note_launch(2);
    if constexpr (FWD) {
        ntt_pass_kernel<true, true, false, LA, 1, CA, EA, LA + LB, 0, Job>
            <<<grid, NTT_TILE / EA, 0, st>>>(d, job, jbase);
        ntt_pass_kernel<true, false, true, LB, HB, 1, EB, LA + LB, LA, Job>
            <<<grid, NTT_TILE / EB, 0, st>>>(d, job, jbase);
    } else {
        ntt_pass_kernel<false, true, false, LB, HB, 1, EB, LA + LB, LA, Job>
            <<<grid, NTT_TILE / EB, 0, st>>>(d, job, jbase);
        ntt_pass_kernel<false, false, true, LA, 1, CA, EA, LA + LB, 0, Job>
            <<<grid, NTT_TILE / EA, 0, st>>>(d, job, jbase);
    }
}

template <bool FWD, class Job>
void launch_ntt_chunk(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    switch (d.log_n) {
        case 3: launch_ntt_single<FWD, 3>(d, job, jbase, njobs, st); break;
        case 4: launch_ntt_single<FWD, 4>(d, job, jbase, njobs, st); break;
        case 5: launch_ntt_single<FWD, 5>(d, job, jbase, njobs, st); break;
        case 6: launch_ntt_single<FWD, 6>(d, job, jbase, njobs, st); break;
        case 7: launch_ntt_single<FWD, 7>(d, job, jbase, njobs, st); break;
        case 8: launch_ntt_single<FWD, 8>(d, job, jbase, njobs, st); break;
        case 9: launch_ntt_single<FWD, 9>(d, job, jbase, njobs, st); break;
        case 10: launch_ntt_single<FWD, 10>(d, job, jbase, njobs, st); break;
        case 11: launch_ntt_single<FWD, 11>(d, job, jbase, njobs, st); break;
        case 12: launch_ntt_two<FWD, 6, 6>(d, job, jbase, njobs, st); break;
        case 13: launch_ntt_two<FWD, 6, 7>(d, job, jbase, njobs, st); break;
        case 14: launch_ntt_two<FWD, 7, 7>(d, job, jbase, njobs, st); break;
        case 15: launch_ntt_two<FWD, 7, 8>(d, job, jbase, njobs, st); break;
        case 16: launch_ntt_two<FWD, 8, 8>(d, job, jbase, njobs, st); break;
        case 17: launch_ntt_two<FWD, 8, 9>(d, job, jbase, njobs, st); break;
        default: break;   // rejected at context creation
    }
}

// Batched launch over njobs limbs (grid.y is limited to 65535 per launch).
template <bool FWD, class Job>
void launch_ntt(const Dev& d, const Job& job, int njobs, cudaStream_t st) {
    for (int base = 0; base < njobs; base += 65535) {
        int cnt = njobs - base < 65535 ? njobs - base : 65535;
        launch_ntt_chunk<FWD>(d, job, base, cnt, st);
    }
}

}  // namespace hs
