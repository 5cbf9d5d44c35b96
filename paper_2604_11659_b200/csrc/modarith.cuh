// 64-bit modular arithmetic for RNS limbs on sm_100a integer pipes.
//
// All chain/aux primes are < 2^60 (params.py:185-198 of the reference), so
// lazy representatives in [0, 4q) fit comfortably in 64 bits.  Every kernel
// canonicalises to [0, q) before a value leaves the device op, which is what
// makes the results bit-identical to the reference's canonical residues no
// matter which reduction algorithm produced them.
#pragma once
#include <cstdint>

typedef uint64_t u64;
typedef unsigned int u32;

#define HS_DEV __device__ __forceinline__

// Per-prime constants, computed on the host (csrc/context.cu).
struct PrimeConst {
    u64 q;
    u64 two_q;
    u64 mu64;        // floor(2^(63+k) / q), k = bitlen(q): one-umulhi Barrett
    u64 qinv_neg;    // -q^{-1} mod 2^64 (Montgomery)
    u64 r_mod;       // 2^64 mod q
    u64 r2_mod;      // 2^128 mod q  (to enter Montgomery form)
    u64 n_inv, n_inv_sh;
    u64 m64;         // floor(2^64 / q): generic 64-bit Barrett (reduce64)
    u64 r_sh;        // floor(r_mod 2^64 / q): Shoup companion of 2^64 mod q
    u32 k;           // bitlen(q)
    u32 pad;         // flags: PC_F64 = NTT butterflies on the FP64 pipe (q <= 2^50 + 2^40)
};
#define PC_F64 1u

HS_DEV u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// x - m if x >= m.  Every value the kernels reduce is < 8q < 2^63 (all
// primes < 2^60), so the sign of x - m decides (one compare fewer than an
// unsigned 64-bit >=).
HS_DEV u64 csub(u64 x, u64 m) {
    const u64 d = x - m;
    return (long long)d < 0 ? x : d;
}

// Shoup product, w_sh = floor(w*2^64/q).  Any x < 2^64; result in [0, 2q).
HS_DEV u64 shoup_lazy(u64 x, u64 w, u64 w_sh, u64 q) {
    u64 hi = mulhi64(x, w_sh);
    return x * w - hi * q;
}
HS_DEV u64 shoup(u64 x, u64 w, u64 w_sh, u64 q) { return csub(shoup_lazy(x, w, w_sh, q), q); }

// Barrett product a*b mod q for a, b < q (both variable).
// q1 = floor(x / 2^(k-1)) < 2^(k+1); quotient estimate umulhi(q1, mu64) is
// at most 3 below floor(x/q), so r < 4q < 2^62 and 3 conditional subtracts
// give the canonical residue.
HS_DEV u64 mul_mod(u64 a, u64 b, const PrimeConst& P) {
    u64 lo = a * b, hi = mulhi64(a, b);
    u64 q1 = (hi << (65 - P.k)) | (lo >> (P.k - 1));
    u64 qt = mulhi64(q1, P.mu64);
    u64 r = lo - qt * P.q;
    r = csub(r, P.two_q);
    return csub(r, P.q);
}

// Montgomery product a * b' * 2^-64 mod q, a < q, b' < q.  When b' = b*2^64
// mod q (keys and masks are stored that way on the device) the result is the
// plain product a*b mod q, canonical.
HS_DEV u64 mont_mul(u64 a, u64 b, u64 q, u64 qinv_neg) {
    u64 lo = a * b, hi = mulhi64(a, b);
    u64 m = lo * qinv_neg;
    u64 r = hi + mulhi64(m, q) + (lo != 0ull);
    return csub(r, q);
}

// Lazy Montgomery (result in [0, 2q)).
HS_DEV u64 mont_mul_lazy(u64 a, u64 b, u64 q, u64 qinv_neg) {
    u64 lo = a * b, hi = mulhi64(a, b);
    u64 m = lo * qinv_neg;
    return hi + mulhi64(m, q) + (lo != 0ull);
}

HS_DEV u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
HS_DEV u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// t mod q for any t < 2^64: quotient estimate is at most 1 low.
HS_DEV u64 reduce64(u64 t, const PrimeConst& P) {
    u64 r = t - mulhi64(t, P.m64) * P.q;
    return csub(r, P.q);
}

// Centred lift of a residue mod q_src into q_dst (reference _fast.pyx:175-192):
// v > q_src>>1 stands for the negative integer v - q_src.  Zero maps to zero.
HS_DEV u64 lift_mod(u64 v, u64 q_src, const PrimeConst& D) {
    bool neg = v > (q_src >> 1);
    u64 t = reduce64(neg ? q_src - v : v, D);
    return (neg && t) ? D.q - t : t;
}

// Same lift when the caller knows q_src/2 < q_dst (no reduction needed):
// the magnitude of the centred value already is a residue mod q_dst.
HS_DEV u64 lift_mod_small(u64 v, u64 q_src, u64 q_dst) {
    const bool neg = v > (q_src >> 1);
    const u64 t = neg ? q_src - v : v;
    return (neg && t) ? q_dst - t : t;
}

// Dispatch on a CTA-uniform flag.
#ifndef HS_LIFT_ONEPATH
#define HS_LIFT_ONEPATH 1        // A/B at cfg2: 167.6 -> 156.3 ms (instruction cache)
#endif
HS_DEV u64 lift_mod_sel(u64 v, u64 q_src, const PrimeConst& D, bool small) {
#if HS_LIFT_ONEPATH
    (void)small;                     // one code path (smaller inlined loaders)
    return lift_mod(v, q_src, D);
#else
    return small ? lift_mod_small(v, q_src, D.q) : lift_mod(v, q_src, D);
#endif
}
