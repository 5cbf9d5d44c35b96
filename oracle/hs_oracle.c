/*
 * hs_oracle.c -- CPU ORACLE for the encrypted SpMSpM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file restates, in plain C, the reference
 * package's arithmetic for the CSR/C encrypted matmul path so the CUDA
 * product path can be checked bit-for-bit against it.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load the library built from it.  The product path never calls it.
 *
 * Every function cites the reference location it restates
 * (paths relative to /root/reference/pkg/src/hespmm/).
 *
 * Pinning: tests/test_oracle_golden.py checks these functions against golden
 * vectors produced by the real reference (tests/golden/make_golden.py).
 *
 * Layout conventions (shared with the CUDA library):
 *   limb      = uint64[n], canonical residues in [0, q)
 *   RNS poly  = [limbs][n], limb i over chain prime q_i (aux prime last)
 *   ct@l      = [npoly][l+1][n] (npoly = 2, or 3 after mult_ct)
 *   KSK       = b[L+1 digits][L+2 moduli][n] followed by a[..][..][n]
 *               (moduli q_0..q_L then the aux prime, context.py:150-174)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef unsigned __int128 u128;

/* ------------------------------------------------------------ scalar math */

static u64 or_powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = (u64)(((u128)r * b) % q);
        b = (u64)(((u128)b * b) % q);
        e >>= 1;
    }
    return r;
}

static u64 or_invmod(u64 a, u64 q) { return or_powmod(a % q, q - 2, q); } /* q prime */

static unsigned or_bitrev(unsigned x, int bits) {
    unsigned y = 0;
    for (int i = 0; i < bits; i++) { y = (y << 1) | (x & 1); x >>= 1; }
    return y;
}

static int or_bitlen(u64 q) { return 64 - __builtin_clzll(q); }

/* Shoup product, w_sh = floor(w*2^64/q), x < q  (_kernels/_fast.pyx:21-27) */
static inline u64 shoup(u64 x, u64 w, u64 w_sh, u64 q) {
    u64 hi = (u64)(((u128)x * w_sh) >> 64);
    u64 r = x * w - hi * q;
    return r >= q ? r - q : r;
}

/* Barrett product with mu = floor(2^(2k)/q), k = bitlen(q) (_fast.pyx:30-37,
 * params.py:97-98).  Result canonical. */
static inline u64 barrett(u64 a, u64 b, u64 q, u64 mu, int k) {
    u128 x = (u128)a * b;
    u64 q1 = (u64)(x >> (k - 1));
    u64 q2 = (u64)(((u128)q1 * mu) >> (k + 1));
    u64 r = (u64)x - q2 * q;
    while (r >= q) r -= q;
    return r;
}

static u64 or_mu(u64 q) {
    int k = or_bitlen(q);
    /* floor(2^(2k)/q); 2k <= 124 so u128 holds it */
    return (u64)(((u128)1 << (2 * k)) / q);
}

/* ------------------------------------------------------------ NTT tables */

/* find_primitive_root(q, 2n): first g in [2,1000) whose g^((q-1)/2n) has
 * order exactly 2n (params.py:75-84).  Returns 0 if none. */
u64 or_find_psi(u64 q, u64 n) {
    u64 order = 2 * n;
    if ((q - 1) % order) return 0;
    u64 e = (q - 1) / order;
    for (u64 g = 2; g < 1000; g++) {
        u64 psi = or_powmod(g, e, q);
        if (or_powmod(psi, order / 2, q) == q - 1) return psi;
    }
    return 0;
}

/* PrimeTables (params.py:87-107): roots[i] = psi^bitrev(i), iroots = inverse,
 * *_sh = floor(r*2^64/q), n_inv.  Returns 0 on success. */
int or_tables(u64 q, unsigned n, u64 *roots, u64 *roots_sh, u64 *iroots,
              u64 *iroots_sh, u64 *n_inv) {
    u64 psi = or_find_psi(q, n);
    if (!psi) return -1;
    int bits = __builtin_ctz(n);
    for (unsigned i = 0; i < n; i++) {
        u64 r = or_powmod(psi, or_bitrev(i, bits), q);
        u64 ir = or_invmod(r, q);
        roots[i] = r;
        iroots[i] = ir;
        roots_sh[i] = (u64)(((u128)r << 64) / q);
        iroots_sh[i] = (u64)(((u128)ir << 64) / q);
    }
    *n_inv = or_invmod(n, q);
    return 0;
}

/* ------------------------------------------------------- the 9 limb kernels
 * (_kernels/__init__.py:20-28; _fast.pyx:44-192; _py.py:26-102) */

/* Forward negacyclic CT NTT, natural in, bit-reversed out (_fast.pyx:44-67) */
void or_ntt(u64 *v, unsigned n, u64 q, const u64 *rt, const u64 *rt_sh) {
    unsigned t = n;
    for (unsigned m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (unsigned i = 0; i < m; i++) {
            u64 w = rt[m + i], wsh = rt_sh[m + i];
            unsigned base = 2 * i * t;
            for (unsigned j = base; j < base + t; j++) {
                u64 x = v[j];
                u64 y = shoup(v[j + t], w, wsh, q);
                u64 s = x + y;
                v[j] = s >= q ? s - q : s;
                v[j + t] = x >= y ? x - y : x + q - y;
            }
        }
    }
}

/* Inverse GS NTT then Shoup by n^-1 (_fast.pyx:70-100) */
void or_intt(u64 *v, unsigned n, u64 q, const u64 *irt, const u64 *irt_sh,
             u64 n_inv) {
    unsigned t = 1;
    for (unsigned m = n >> 1; m >= 1; m >>= 1) {
        for (unsigned i = 0; i < m; i++) {
            u64 w = irt[m + i], wsh = irt_sh[m + i];
            unsigned base = 2 * i * t;
            for (unsigned j = base; j < base + t; j++) {
                u64 x = v[j], y = v[j + t];
                u64 s = x + y;
                v[j] = s >= q ? s - q : s;
                v[j + t] = shoup(x >= y ? x - y : x + q - y, w, wsh, q);
            }
        }
        t <<= 1;
    }
    u64 ninv_sh = (u64)(((u128)n_inv << 64) / q);
    for (unsigned j = 0; j < n; j++) v[j] = shoup(v[j], n_inv, ninv_sh, q);
}

void or_add_mod(const u64 *a, const u64 *b, u64 *r, unsigned n, u64 q) {
    for (unsigned j = 0; j < n; j++) { u64 s = a[j] + b[j]; r[j] = s >= q ? s - q : s; }
}
void or_sub_mod(const u64 *a, const u64 *b, u64 *r, unsigned n, u64 q) {
    for (unsigned j = 0; j < n; j++) r[j] = a[j] >= b[j] ? a[j] - b[j] : a[j] + q - b[j];
}
void or_neg_mod(const u64 *a, u64 *r, unsigned n, u64 q) {
    for (unsigned j = 0; j < n; j++) r[j] = a[j] ? q - a[j] : 0;
}
void or_mul_mod(const u64 *a, const u64 *b, u64 *r, unsigned n, u64 q, u64 mu) {
    int k = or_bitlen(q);
    for (unsigned j = 0; j < n; j++) r[j] = barrett(a[j], b[j], q, mu, k);
}
void or_scalar_mul_mod(const u64 *a, u64 s, u64 *r, unsigned n, u64 q) {
    s %= q;
    u64 ssh = (u64)(((u128)s << 64) / q);
    for (unsigned j = 0; j < n; j++) r[j] = shoup(a[j], s, ssh, q);
}
/* in place acc = (acc + a*b) mod q (_fast.pyx:162-172) */
void or_fma_mod(u64 *acc, const u64 *a, const u64 *b, unsigned n, u64 q, u64 mu) {
    int k = or_bitlen(q);
    for (unsigned j = 0; j < n; j++) {
        u64 s = acc[j] + barrett(a[j], b[j], q, mu, k);
        acc[j] = s >= q ? s - q : s;
    }
}
/* centred lift q_src -> q_dst (_fast.pyx:175-192): v > q_src>>1 is negative */
void or_extend_mod(const u64 *a, u64 *r, unsigned n, u64 q_src, u64 q_dst) {
    u64 half = q_src >> 1;
    for (unsigned j = 0; j < n; j++) {
        u64 v = a[j];
        if (v > half) {
            v = (q_src - v) % q_dst;
            r[j] = v ? q_dst - v : 0;
        } else {
            r[j] = v % q_dst;
        }
    }
}

/* ------------------------------------------------------------ CKKS context
 * Restates the precomputation of CkksContext.__init__ (context.py:31-58). */

typedef struct {
    unsigned n, L;            /* ring degree, levels (chain has L+1 primes) */
    u64 *primes;              /* L+2: chain then aux */
    u64 *mu;                  /* Barrett mu per prime */
    u64 *roots, *roots_sh, *iroots, *iroots_sh;  /* (L+2)*n */
    u64 *n_inv;               /* L+2 */
    u64 *digit_factor;        /* L+1: (Q_L/q_i)^-1 mod q_i       (context.py:44) */
    u64 *aux_inv;             /* L+1: p^-1 mod q_m               (context.py:49) */
    u64 *qlast_inv;           /* (L+1)*(L+1): [lvl][i] q_lvl^-1 mod q_i (:50-53) */
} or_ctx;

void or_ctx_destroy(or_ctx *c) {
    if (!c) return;
    free(c->primes); free(c->mu); free(c->roots); free(c->roots_sh);
    free(c->iroots); free(c->iroots_sh); free(c->n_inv);
    free(c->digit_factor); free(c->aux_inv); free(c->qlast_inv);
    free(c);
}

or_ctx *or_ctx_create(unsigned n, unsigned L, const u64 *chain, u64 aux) {
    or_ctx *c = (or_ctx *)calloc(1, sizeof(or_ctx));
    unsigned P = L + 2;
    c->n = n; c->L = L;
    c->primes = malloc(P * sizeof(u64));
    c->mu = malloc(P * sizeof(u64));
    c->roots = malloc((size_t)P * n * sizeof(u64));
    c->roots_sh = malloc((size_t)P * n * sizeof(u64));
    c->iroots = malloc((size_t)P * n * sizeof(u64));
    c->iroots_sh = malloc((size_t)P * n * sizeof(u64));
    c->n_inv = malloc(P * sizeof(u64));
    c->digit_factor = malloc((L + 1) * sizeof(u64));
    c->aux_inv = malloc((L + 1) * sizeof(u64));
    c->qlast_inv = calloc((size_t)(L + 1) * (L + 1), sizeof(u64));
    for (unsigned i = 0; i <= L; i++) c->primes[i] = chain[i];
    c->primes[L + 1] = aux;
    for (unsigned p = 0; p < P; p++) {
        u64 q = c->primes[p];
        c->mu[p] = or_mu(q);
        if (or_tables(q, n, c->roots + (size_t)p * n, c->roots_sh + (size_t)p * n,
                      c->iroots + (size_t)p * n, c->iroots_sh + (size_t)p * n,
                      &c->n_inv[p])) {
            or_ctx_destroy(c);
            return NULL;
        }
    }
    /* (Q_L/q_i) mod q_i = prod_{j != i} q_j mod q_i over the FULL chain */
    for (unsigned i = 0; i <= L; i++) {
        u64 qi = chain[i], prod = 1;
        for (unsigned j = 0; j <= L; j++)
            if (j != i) prod = (u64)(((u128)prod * (chain[j] % qi)) % qi);
        c->digit_factor[i] = or_invmod(prod, qi);
        c->aux_inv[i] = or_invmod(aux % qi, qi);
    }
    for (unsigned lvl = 0; lvl <= L; lvl++)
        for (unsigned i = 0; i < lvl; i++)
            c->qlast_inv[lvl * (L + 1) + i] = or_invmod(chain[lvl] % chain[i], chain[i]);
    return c;
}

/* accessors so the Python side can read the derived constants */
u64 or_ctx_digit_factor(const or_ctx *c, unsigned i) { return c->digit_factor[i]; }
u64 or_ctx_aux_inv(const or_ctx *c, unsigned i) { return c->aux_inv[i]; }
u64 or_ctx_qlast_inv(const or_ctx *c, unsigned lvl, unsigned i) {
    return c->qlast_inv[lvl * (c->L + 1) + i];
}
const u64 *or_ctx_roots(const or_ctx *c, unsigned p) { return c->roots + (size_t)p * c->n; }
const u64 *or_ctx_roots_sh(const or_ctx *c, unsigned p) { return c->roots_sh + (size_t)p * c->n; }
const u64 *or_ctx_iroots(const or_ctx *c, unsigned p) { return c->iroots + (size_t)p * c->n; }
const u64 *or_ctx_iroots_sh(const or_ctx *c, unsigned p) { return c->iroots_sh + (size_t)p * c->n; }
u64 or_ctx_n_inv(const or_ctx *c, unsigned p) { return c->n_inv[p]; }
u64 or_ctx_mu(const or_ctx *c, unsigned p) { return c->mu[p]; }

/* prime index p: 0..L chain, L+1 aux */
void or_ctx_ntt(const or_ctx *c, u64 *v, unsigned p) {
    or_ntt(v, c->n, c->primes[p], c->roots + (size_t)p * c->n, c->roots_sh + (size_t)p * c->n);
}
void or_ctx_intt(const or_ctx *c, u64 *v, unsigned p) {
    or_intt(v, c->n, c->primes[p], c->iroots + (size_t)p * c->n,
            c->iroots_sh + (size_t)p * c->n, c->n_inv[p]);
}

/* ------------------------------------------------------- evaluation ops */

#define LIMB(base, idx, n) ((base) + (size_t)(idx) * (n))

/* _key_switch (context.py:462-498): digits[(l+1)][n] coefficient-domain,
 * ksk = b[(L+1)][(L+2)][n] then a[...]; out_b/out_a [(l+1)][n]. */
void or_key_switch(const or_ctx *c, const u64 *digits, const u64 *ksk, unsigned level,
                   u64 *out_b, u64 *out_a) {
    unsigned n = c->n, L = c->L, nl = level + 1;
    size_t dig_stride = (size_t)(L + 2) * n;          /* one digit of b */
    const u64 *kb = ksk, *ka = ksk + (size_t)(L + 1) * dig_stride;
    u64 *acc_b = calloc((size_t)(nl + 1) * n, sizeof(u64));
    u64 *acc_a = calloc((size_t)(nl + 1) * n, sizeof(u64));
    u64 *ext = malloc((size_t)n * sizeof(u64));
    for (unsigned i = 0; i < nl; i++) {
        u64 qi = c->primes[i];
        for (unsigned m = 0; m <= nl; m++) {
            unsigned pm = m < nl ? m : L + 1;           /* prime index == kidx */
            u64 qm = c->primes[pm];
            if (m == i) memcpy(ext, LIMB(digits, i, n), n * sizeof(u64));
            else or_extend_mod(LIMB(digits, i, n), ext, n, qi, qm);
            or_ctx_ntt(c, ext, pm);
            or_fma_mod(LIMB(acc_b, m, n), ext, kb + i * dig_stride + (size_t)pm * n, n, qm, c->mu[pm]);
            or_fma_mod(LIMB(acc_a, m, n), ext, ka + i * dig_stride + (size_t)pm * n, n, qm, c->mu[pm]);
        }
    }
    u64 aux = c->primes[L + 1];
    u64 *auxc = malloc((size_t)n * sizeof(u64));
    for (int which = 0; which < 2; which++) {
        u64 *acc = which ? acc_a : acc_b;
        u64 *out = which ? out_a : out_b;
        memcpy(auxc, LIMB(acc, nl, n), n * sizeof(u64));
        or_ctx_intt(c, auxc, L + 1);
        for (unsigned m = 0; m < nl; m++) {
            u64 q = c->primes[m];
            or_extend_mod(auxc, ext, n, aux, q);
            or_ctx_ntt(c, ext, m);
            or_sub_mod(LIMB(acc, m, n), ext, ext, n, q);
            or_scalar_mul_mod(ext, c->aux_inv[m], LIMB(out, m, n), n, q);
        }
    }
    free(acc_b); free(acc_a); free(ext); free(auxc);
}

/* eval_add (context.py:321-332) on degree-1 cts at `level` */
void or_eval_add(const or_ctx *c, const u64 *a, const u64 *b, u64 *out, unsigned level) {
    unsigned n = c->n, nl = level + 1;
    for (unsigned p = 0; p < 2; p++)
        for (unsigned i = 0; i < nl; i++)
            or_add_mod(LIMB(a, p * nl + i, n), LIMB(b, p * nl + i, n),
                       LIMB(out, p * nl + i, n), n, c->primes[i]);
}

/* eval_mult_ct (context.py:334-351): out = [3][nl][n] */
void or_eval_mult_ct(const or_ctx *c, const u64 *a, const u64 *b, u64 *out, unsigned level) {
    unsigned n = c->n, nl = level + 1;
    u64 *tmp = malloc((size_t)n * sizeof(u64));
    for (unsigned i = 0; i < nl; i++) {
        u64 q = c->primes[i], mu = c->mu[i];
        const u64 *a0 = LIMB(a, i, n), *a1 = LIMB(a, nl + i, n);
        const u64 *b0 = LIMB(b, i, n), *b1 = LIMB(b, nl + i, n);
        or_mul_mod(a0, b0, LIMB(out, i, n), n, q, mu);
        or_mul_mod(a0, b1, LIMB(out, nl + i, n), n, q, mu);
        or_mul_mod(a1, b0, tmp, n, q, mu);
        or_add_mod(LIMB(out, nl + i, n), tmp, LIMB(out, nl + i, n), n, q);
        or_mul_mod(a1, b1, LIMB(out, 2 * nl + i, n), n, q, mu);
    }
    free(tmp);
}

/* eval_mult_pt (context.py:353-361): ct [npoly][nl][n] x pt [nl][n] */
void or_eval_mult_pt(const or_ctx *c, const u64 *ct, const u64 *pt, u64 *out,
                     unsigned npoly, unsigned level) {
    unsigned n = c->n, nl = level + 1;
    for (unsigned p = 0; p < npoly; p++)
        for (unsigned i = 0; i < nl; i++)
            or_mul_mod(LIMB(ct, p * nl + i, n), LIMB(pt, i, n), LIMB(out, p * nl + i, n),
                       n, c->primes[i], c->mu[i]);
}

/* _digits_from_ntt (context.py:454-460) */
static void or_digits_from_ntt(const or_ctx *c, const u64 *limbs, unsigned level, u64 *digits) {
    unsigned n = c->n;
    for (unsigned i = 0; i <= level; i++) {
        or_scalar_mul_mod(LIMB(limbs, i, n), c->digit_factor[i], LIMB(digits, i, n), n,
                          c->primes[i]);
        or_ctx_intt(c, LIMB(digits, i, n), i);
    }
}

/* relinearize (context.py:363-380): ct3 [3][nl][n] -> out [2][nl][n] */
void or_relinearize(const or_ctx *c, const u64 *ct3, const u64 *relin, u64 *out, unsigned level) {
    unsigned n = c->n, nl = level + 1;
    u64 *digits = malloc((size_t)nl * n * sizeof(u64));
    u64 *kb = malloc((size_t)nl * n * sizeof(u64));
    u64 *ka = malloc((size_t)nl * n * sizeof(u64));
    or_digits_from_ntt(c, LIMB(ct3, 2 * nl, n), level, digits);
    or_key_switch(c, digits, relin, level, kb, ka);
    for (unsigned i = 0; i < nl; i++) {
        or_add_mod(LIMB(ct3, i, n), LIMB(kb, i, n), LIMB(out, i, n), n, c->primes[i]);
        or_add_mod(LIMB(ct3, nl + i, n), LIMB(ka, i, n), LIMB(out, nl + i, n), n, c->primes[i]);
    }
    free(digits); free(kb); free(ka);
}

/* rescale (context.py:382-399): ct [npoly][nl][n] -> out [npoly][nl-1][n] */
int or_rescale(const or_ctx *c, const u64 *ct, u64 *out, unsigned npoly, unsigned level) {
    if (level == 0) return -1;
    unsigned n = c->n, nl = level + 1, L = c->L;
    u64 ql = c->primes[level];
    u64 *last = malloc((size_t)n * sizeof(u64));
    u64 *delta = malloc((size_t)n * sizeof(u64));
    for (unsigned p = 0; p < npoly; p++) {
        memcpy(last, LIMB(ct, p * nl + level, n), n * sizeof(u64));
        or_ctx_intt(c, last, level);
        for (unsigned i = 0; i < level; i++) {
            u64 q = c->primes[i];
            or_extend_mod(last, delta, n, ql, q);
            or_ctx_ntt(c, delta, i);
            or_sub_mod(LIMB(ct, p * nl + i, n), delta, delta, n, q);
            or_scalar_mul_mod(delta, c->qlast_inv[level * (L + 1) + i],
                              LIMB(out, p * level + i, n), n, q);
        }
    }
    free(last); free(delta);
    return 0;
}

/* _perm_tables (context.py:429-445) for g = 5^r mod 2n */
static void or_perm_tables(unsigned n, u64 g, unsigned *src, unsigned char *neg) {
    for (unsigned i = 0; i < n; i++) {
        u64 t = ((u64)i * g) % (2 * (u64)n);
        if (t < n) { src[t] = i; neg[t] = 0; }
        else { src[t - n] = i; neg[t - n] = 1; }
    }
}

/* _apply_perm (context.py:447-452): zero residues are never flipped */
static void or_apply_perm(const u64 *in, u64 *out, unsigned n, const unsigned *src,
                          const unsigned char *neg, u64 q) {
    for (unsigned k = 0; k < n; k++) {
        u64 v = in[src[k]];
        out[k] = (neg[k] && v) ? q - v : v;
    }
}

/* eval_rotate (context.py:401-425) for a NORMALISED step r in [1, slots).
 * ct [2][nl][n] -> out [2][nl][n]. gk = Galois KSK for r. */
void or_eval_rotate(const or_ctx *c, const u64 *ct, unsigned r, const u64 *gk, u64 *out,
                    unsigned level) {
    unsigned n = c->n, nl = level + 1;
    u64 g = or_powmod(5, r, 2 * (u64)n);
    unsigned *src = malloc(n * sizeof(unsigned));
    unsigned char *neg = malloc(n);
    or_perm_tables(n, g, src, neg);
    u64 *tmp = malloc((size_t)n * sizeof(u64));
    u64 *new0 = malloc((size_t)nl * n * sizeof(u64));
    u64 *digits = calloc((size_t)nl * n, sizeof(u64));      /* filled below (calloc: no -Wmaybe-uninitialized) */
    u64 *kb = malloc((size_t)nl * n * sizeof(u64));
    for (unsigned i = 0; i < nl; i++) {
        u64 q = c->primes[i];
        memcpy(tmp, LIMB(ct, i, n), n * sizeof(u64));
        or_ctx_intt(c, tmp, i);
        or_apply_perm(tmp, LIMB(new0, i, n), n, src, neg, q);
        or_ctx_ntt(c, LIMB(new0, i, n), i);
        memcpy(tmp, LIMB(ct, nl + i, n), n * sizeof(u64));
        or_ctx_intt(c, tmp, i);
        or_apply_perm(tmp, LIMB(digits, i, n), n, src, neg, q);
        or_scalar_mul_mod(LIMB(digits, i, n), c->digit_factor[i], LIMB(digits, i, n), n, q);
    }
    or_key_switch(c, digits, gk, level, kb, LIMB(out, nl, n));
    for (unsigned i = 0; i < nl; i++)
        or_add_mod(LIMB(new0, i, n), LIMB(kb, i, n), LIMB(out, i, n), n, c->primes[i]);
    free(src); free(neg); free(tmp); free(new0); free(digits); free(kb);
}

/* ------------------------------------------------------------- the runner
 * Algorithm 1/2: _run_schedule (engine.py:136-164) + fhe_spmspm_step
 * (engine.py:99-133), over an explicit pair list (i, j, a_pos, b_pos) as
 * produced by pair_schedule (encmat.py:208-229).
 *
 * Inputs: ct_a, ct_b at level L ([2][L+1][n]); masks[p] = mask plaintext for
 * pair p (level L-1, [L][n]); relin = relin KSK; galois[r] = KSK for the
 * normalised step r (NULL when absent), table length slots.
 * Output: acc [2][L-1][n] = modular sum of all pair contributions.  The sum
 * is order-free (modular addition is associative and commutative), so pairs
 * may be distributed over threads; each per-pair contribution follows the
 * reference op sequence exactly, with no deduplication.
 *
 * Returns 0 ok, -2 missing Galois key (KeyMissingError, context.py:408-410),
 * -3 level too small.  *npairs_done receives the number of contributions.
 */
static unsigned or_norm_step(long long s, unsigned slots) {
    long long r = s % (long long)slots;
    if (r < 0) r += slots;
    return (unsigned)r;
}

int or_spmspm(const or_ctx *c, const u64 *ct_a, const u64 *ct_b, const long long *pairs,
              long long npairs, unsigned dim, const u64 *const *masks, const u64 *relin,
              const u64 *const *galois, u64 *acc_out, int nthreads) {
    unsigned n = c->n, L = c->L, slots = n / 2;
    if (L < 2) return -3;
    size_t ct_l = (size_t)2 * (L + 1) * n;
    size_t out_sz = (size_t)2 * (L - 1) * n;
    /* key presence check up front (the reference raises on first use) */
    for (long long p = 0; p < npairs; p++) {
        long long ap = pairs[4 * p + 2], bp = pairs[4 * p + 3];
        long long i = pairs[4 * p], j = pairs[4 * p + 1];
        if (ap != bp) {
            unsigned r = or_norm_step(ap > bp ? ap - bp : bp - ap, slots);
            if (r && !galois[r]) return -2;
        }
        long long mn = ap < bp ? ap : bp;
        unsigned r2 = or_norm_step(mn - (i * dim + j), slots);
        if (mn - (i * (long long)dim + j) != 0 && r2 && !galois[r2]) return -2;
    }
    memset(acc_out, 0, out_sz * sizeof(u64));
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel
    {
        u64 *acc = calloc(out_sz, sizeof(u64));
        u64 *va = malloc(ct_l * sizeof(u64));
        u64 *vb = malloc(ct_l * sizeof(u64));
        u64 *t3 = malloc((size_t)3 * (L + 1) * n * sizeof(u64));
        u64 *t2 = malloc(ct_l * sizeof(u64));
        u64 *u2 = malloc(ct_l * sizeof(u64));
#pragma omp for schedule(dynamic, 1)
        for (long long p = 0; p < npairs; p++) {
            long long i = pairs[4 * p], j = pairs[4 * p + 1];
            long long ap = pairs[4 * p + 2], bp = pairs[4 * p + 3];
            const u64 *pa = ct_a, *pb = ct_b;
            long long mn;
            if (ap < bp) {
                unsigned r = or_norm_step(bp - ap, slots);
                if (r) { or_eval_rotate(c, ct_b, r, galois[r], vb, L); pb = vb; }
                mn = ap;
            } else if (bp < ap) {
                unsigned r = or_norm_step(ap - bp, slots);
                if (r) { or_eval_rotate(c, ct_a, r, galois[r], va, L); pa = va; }
                mn = bp;
            } else {
                mn = ap;
            }
            or_eval_mult_ct(c, pa, pb, t3, L);                 /* ct@L deg 2 */
            or_relinearize(c, t3, relin, t2, L);               /* ct@L */
            or_rescale(c, t2, u2, 2, L);                       /* ct@L-1 */
            or_eval_mult_pt(c, u2, masks[p], t2, 2, L - 1);    /* ct@L-1 */
            or_rescale(c, t2, u2, 2, L - 1);                   /* ct@L-2 */
            long long rot = mn - (i * (long long)dim + j);
            const u64 *contrib = u2;
            if (rot != 0) {
                unsigned r = or_norm_step(rot, slots);
                if (r) { or_eval_rotate(c, u2, r, galois[r], t2, L - 2); contrib = t2; }
            }
            for (unsigned pp = 0; pp < 2; pp++)
                for (unsigned l = 0; l + 1 < L; l++)
                    or_add_mod(acc + ((size_t)pp * (L - 1) + l) * n,
                               contrib + ((size_t)pp * (L - 1) + l) * n,
                               acc + ((size_t)pp * (L - 1) + l) * n, n, c->primes[l]);
        }
#pragma omp critical
        {
            for (unsigned pp = 0; pp < 2; pp++)
                for (unsigned l = 0; l + 1 < L; l++)
                    or_add_mod(acc_out + ((size_t)pp * (L - 1) + l) * n,
                               acc + ((size_t)pp * (L - 1) + l) * n,
                               acc_out + ((size_t)pp * (L - 1) + l) * n, n, c->primes[l]);
        }
        free(acc); free(va); free(vb); free(t3); free(t2); free(u2);
    }
    return 0;
}

/* Decrypt (context.py:303-313): pt[i] = c0[i] + c1[i]*s[i] ; sk_ntt [L+1][n] */
void or_decrypt(const or_ctx *c, const u64 *ct, const u64 *sk_ntt, u64 *pt, unsigned level) {
    unsigned n = c->n, nl = level + 1;
    u64 *tmp = malloc((size_t)n * sizeof(u64));
    for (unsigned i = 0; i < nl; i++) {
        or_mul_mod(LIMB(ct, nl + i, n), LIMB(sk_ntt, i, n), tmp, n, c->primes[i], c->mu[i]);
        or_add_mod(LIMB(ct, i, n), tmp, LIMB(pt, i, n), n, c->primes[i]);
    }
    free(tmp);
}
