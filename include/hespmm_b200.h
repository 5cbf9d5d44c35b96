/*
 * hespmm_b200.h -- C-ABI of libhespmm_b200.so, the B200 (sm_100a) engine
 * behind the encrypted SpMSpM hot path of the reference package `hespmm`.
 *
 * Plain C: pointers, sizes and status codes only (no torch / CUDA types in
 * the signatures; `void* stream` is a cudaStream_t, NULL = legacy default).
 * Reference paths are relative to /root/reference/pkg/src/hespmm/.
 *
 * Data layout (device memory, canonical residues in [0, q)):
 *   limb          uint64[n]
 *   ct at level l [npoly][l+1][n]   npoly = 2 (3 after mult_ct)
 *   plaintext     [l+1][n]
 *   key           [2][L+1][L+2][n]  b then a; digit i, modulus m over
 *                                   q_0..q_L then the aux prime
 *                                   (ckks/types.py:53-62, context.py:150-174)
 * Prime index p: 0..L = chain q_0..q_L, L+1 = aux prime.
 *
 * Threading: one context per device; calls are asynchronous on `stream` and
 * not re-entrant per context (the reference evaluator is single-threaded,
 * ckks/context.py:26-29).  Errors: every call returns hs_status; the message
 * of the last failure on the calling thread is hs_last_error().  Status
 * codes map onto the reference's exception types (errors.py:4-17).
 */
#ifndef HESPMM_B200_H
#define HESPMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HS_OK = 0,
    HS_PARAMETER_ERROR = 1,   /* errors.ParameterError */
    HS_CAPACITY_ERROR = 2,    /* errors.CapacityError  */
    HS_KEY_MISSING = 3,       /* errors.KeyMissingError */
    HS_EVAL_ERROR = 4,        /* errors.EvalError */
    HS_CUDA_ERROR = 5,
    HS_OUT_OF_MEMORY = 6
} hs_status;

typedef struct hs_ctx hs_ctx;

/* Logical operation counts of one matmul, identical to the reference
 * OpCounter (engine.py:29-58), plus the physical work actually executed
 * after alignment-rotation deduplication. */
typedef struct {
    int64_t ct_ct_mults, pt_mults, rotations, relins, relin_noops, rescales, adds;
    int64_t alignment_rotations, accumulation_rotations;
    int64_t pairs;                 /* pairs executed by this shard */
    int64_t physical_alignment;    /* distinct (operand, step) rotations executed */
    int64_t has_result;            /* 0 when the schedule is empty (engine.py:162-164) */
    double plan_ms;                /* host planning time inside the call */
    int64_t ranges;                /* pair ranges run (> 1 when the aligned operands exceed HBM) */
} hs_counters;

const char* hs_last_error(void);
const char* hs_version(void);
/* Total kernels launched by this library since load (benchmark evidence). */
int64_t hs_launch_count(void);

/* Measurement hooks for bench.py's roofline line (no reference counterpart).
 * hs_probe_arm(mask): every later launch of an armed kernel class (bit k of
 * mask arms kind k: 1 = the ModUp NTT passes of the key switch, 2 = the key
 * inner product, 3 = one device key-generation call; 0 = off) records a
 * CUDA event pair on its own launching
 * stream; arming clears the record.  hs_probe_read(kind, out4) synchronises
 * on those events and returns {launches, total ms, algorithmic DRAM bytes,
 * integer work (butterflies resp. 64x64-bit MACs)} of that kind.
 * hs_int_peak(q, out4, stream): integer-pipe peaks measured on this GPU:
 * {NTT butterflies/s (the engine's butterfly, register-resident, prime q),
 *  mad.wide.u32/s, 32-bit add instructions/s, SMs}. */
hs_status hs_probe_arm(int32_t mask);
hs_status hs_probe_read(int32_t kind, double* out4);
hs_status hs_int_peak(uint64_t q, double* out4, void* stream);
/* hs_f64_peak(q, out4, stream): the FP64-pipe forward butterflies used for
 * primes q <= 2^50 + 2^40, measured the same way: {butterflies/s, DFMA/s, 0, SMs}. */
hs_status hs_f64_peak(uint64_t q, double* out4, void* stream);

/* ---------------------------------------------------------------- context
 * Replaces CkksContext.__init__ precomputation (ckks/context.py:31-58) and
 * PrimeTables (ckks/params.py:87-112): NTT twiddles (psi = first g in
 * [2,1000) of exact order 2n, bit-reversed powers, Shoup companions), digit
 * factors, ModDown and rescale constants, all uploaded to `device`. */
hs_status hs_ctx_create(hs_ctx** out, int device, uint32_t ring_degree, uint32_t levels,
                        const uint64_t* modulus_chain /* levels+1 */, uint64_t aux_prime);
void hs_ctx_destroy(hs_ctx* ctx);
/* Host copies of the tables for prime index p (each n entries); any may be NULL. */
hs_status hs_ctx_tables(const hs_ctx* ctx, uint32_t p, uint64_t* roots, uint64_t* roots_sh,
                        uint64_t* iroots, uint64_t* iroots_sh, uint64_t* n_inv, uint64_t* mu);

/* ------------------------------------------------------------------- keys
 * Key switching keys live inside the context (device, standard form).
 * kind 0 = relinearisation key (KeyBundle.relin), kind 1 = Galois key for
 * normalised step `step` in [1, slots) (KeyBundle.galois[step]). */
hs_status hs_key_upload(hs_ctx* ctx, int kind, uint32_t step, const uint64_t* key, int key_on_host,
                        void* stream);
/* Device key generation (context.py:150-174 `_make_ksk`, arithmetic only; the
 * numpy-stream draws are made on the host): a = uniform limbs [L+1][L+2][n],
 * e = Gaussian coefficients [L+1][n] (int64), target/sk = NTT limbs [L+2][n];
 * all device pointers.  b = NTT(e) + [m<=L] p(Q_L/q_i) target - a sk. */
hs_status hs_key_generate(hs_ctx* ctx, int kind, uint32_t step, const uint64_t* a,
                          const int64_t* e, const uint64_t* target, const uint64_t* sk,
                          void* stream);
/* ---- on-device Galois key generation (keygen.cu), bit-exact with
 * gen_galois_keys (context.py:176-200): each key's numpy stream
 * default_rng(SeedSequence((seed, 0x90, r))) is replayed on the GPU
 * (PCG64 XSL-RR, Lemire bounded uint64, ziggurat normal). */
/* numpy's ziggurat tables as compiled into the installed numpy (host pointers). */
hs_status hs_keygen_set_tables(hs_ctx* ctx, const double* wi, const double* fi, const uint64_t* ki);
/* Secret key in NTT form over all L+2 primes (device pointer, copied). */
hs_status hs_keygen_set_secret(hs_ctx* ctx, const uint64_t* sk_ntt, void* stream);
/* pcg_states: per step {state_hi, state_lo, inc_hi, inc_lo} of the numpy PCG64
 * *before* its first draw (host array).  generate_galois: make the keys now
 * into the key store; register: make them on demand inside the runner (keys
 * that do not fit in HBM, e.g. 8.8 TB at N=2^16, L=24). */
hs_status hs_key_generate_galois(hs_ctx* ctx, const uint32_t* steps, const uint64_t* pcg_states,
                                 int32_t nsteps, void* stream);
hs_status hs_keygen_register(hs_ctx* ctx, const uint32_t* steps, const uint64_t* pcg_states,
                             int32_t nsteps);
/* Raw draws only (testing): a [K][L+1][L+2][n] uniform limbs, e [K][L+1][n] int64 (device). */
hs_status hs_keygen_streams(hs_ctx* ctx, const uint64_t* pcg_states, int32_t nkeys, uint64_t* a_out,
                            int64_t* e_out, void* stream);
int64_t hs_keys_generated(const hs_ctx* ctx);
/* Standard-form copy [2][L+1][L+2][n] into device buffer `out`. */
/* A key switching key straight from a reference HESP container record
 * (ckks/serial.py:48-66: u32 digits, per digit the b and a polys, each a u32
 * count and count x (u32 size, 8n bytes)) already copied to the device as
 * raw bytes (4-byte aligned): one gather kernel writes the key -- no host
 * unpacking of the per-limb records. */
hs_status hs_key_upload_hesp(hs_ctx* ctx, int kind, uint32_t step, const uint8_t* record, int64_t record_bytes,
                             void* stream);
hs_status hs_key_download(hs_ctx* ctx, int kind, uint32_t step, uint64_t* out, void* stream);
int hs_key_has(const hs_ctx* ctx, int kind, uint32_t step);
hs_status hs_key_drop(hs_ctx* ctx, int kind, uint32_t step);
int64_t hs_key_count(const hs_ctx* ctx);

/* ------------------------------------------------------------ limb kernels
 * Batched forms of the reference kernel seam (_kernels/__init__.py:20-28).
 * hs_ntt: `nitems` items of `nlimbs` limbs each; limb k of an item uses
 * prime index prime_first + k.  In place.  inverse=1 -> intt (incl. n^-1). */
hs_status hs_ntt(hs_ctx* ctx, uint64_t* data, int32_t nitems, int32_t nlimbs, int32_t prime_first,
                 int32_t inverse, void* stream);
/* coeffs (int64, n, device) -> NTT limbs over primes prime_first.. (coeffs mod q then NTT,
 * context.py:80-95) */
hs_status hs_signed_to_ntt(hs_ctx* ctx, const int64_t* coeffs, int32_t nlimbs, int32_t prime_first,
                           uint64_t* out, void* stream);
/* Per-limb seam op with an explicit prime q (any NTT-friendly q < 2^61):
 * op 0 add, 1 sub, 2 neg, 3 mul (Barrett), 4 scalar (Shoup by s), 5 fma
 * (out += a*b, in place), 6 extend (centred lift q_src -> q).  `count` elements. */
hs_status hs_seam_op(int32_t op, uint64_t count, const uint64_t* a, const uint64_t* b, uint64_t* out,
                     uint64_t q, uint64_t s, uint64_t q_src, void* stream);
/* Single-limb NTT with caller tables (roots/roots_sh or iroots/iroots_sh,
 * device pointers, n entries), the literal seam signature of _fast.ntt/intt. */
hs_status hs_seam_ntt(uint64_t* a, uint32_t n, uint64_t q, const uint64_t* roots,
                      const uint64_t* roots_sh, uint64_t n_inv, int32_t inverse, void* stream);

/* -------------------------------------------------------- CKKS primitives
 * Device-pointer forms of CkksContext.eval_* (context.py:321-425).  All ct
 * buffers compact at the given level; outputs must not alias inputs. */
hs_status hs_eval_add(hs_ctx* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out,
                      uint32_t level, void* stream);
hs_status hs_eval_mult_ct(hs_ctx* ctx, const uint64_t* a, const uint64_t* b, uint64_t* out3,
                          uint32_t level, void* stream);
/* pt in standard form (pt_mont=0) or Montgomery form (pt_mont=1) */
hs_status hs_eval_mult_pt(hs_ctx* ctx, const uint64_t* ct, const uint64_t* pt, uint64_t* out,
                          uint32_t npoly, uint32_t level, int32_t pt_mont, void* stream);
hs_status hs_relinearize(hs_ctx* ctx, const uint64_t* ct3, uint64_t* out, uint32_t level,
                         void* stream);
hs_status hs_rescale(hs_ctx* ctx, const uint64_t* ct, uint64_t* out, uint32_t npoly, uint32_t level,
                     void* stream);
/* step: normalised rotation amount in [1, slots); KeyMissing if no key */
hs_status hs_eval_rotate(hs_ctx* ctx, const uint64_t* ct, uint64_t* out, uint32_t level,
                         uint32_t step, void* stream);
/* Hoisted rotations of one ct by `nsteps` normalised steps: outs[k] receives step k. */
hs_status hs_eval_rotate_hoisted(hs_ctx* ctx, const uint64_t* ct, uint64_t* const* outs,
                                 const uint32_t* steps, int32_t nsteps, uint32_t level, void* stream);
/* Public-key encryption arithmetic (context.py:281-301): v/e0/e1 signed coeffs (device, n). */
hs_status hs_encrypt(hs_ctx* ctx, const int64_t* v, const int64_t* e0, const int64_t* e1,
                     const uint64_t* pk_b, const uint64_t* pk_a, const uint64_t* pt,
                     uint32_t level, uint64_t* ct, void* stream);
/* pt[i] = c0[i] + c1[i] s[i] (context.py:303-313) */
hs_status hs_decrypt(hs_ctx* ctx, const uint64_t* ct, const uint64_t* sk, uint32_t level,
                     uint64_t* pt, void* stream);
/* Exact centred CRT lift of nl coefficient-domain limbs [nl][n] (device) to
 * float64 (device, n): Garner + big-integer centring + round-half-even, the
 * doubles bit-equal to the reference's big-int decode (context.py:244-279). */
hs_status hs_crt_decode(hs_ctx* ctx, const uint64_t* coeff, int32_t nlimbs, double* out, void* stream);
/* Convert limbs to / from Montgomery form in place (masks are kept that way). */
hs_status hs_to_montgomery(hs_ctx* ctx, uint64_t* data, int32_t nitems, int32_t nlimbs,
                           int32_t prime_first, int32_t inverse, void* stream);

/* --------------------------------------------------------------- planner
 * pair_schedule for CSR x CSC (encmat.py:150-186, 208-221): two-pointer
 * intersection per output cell, row-major (i, j) order.  Writes up to
 * `cap` (i, j, a_pos, b_pos) rows into `pairs` (host) and returns the
 * total count via *npairs (call with cap=0 to size). */
hs_status hs_plan_csr_csc(int32_t dim, const int64_t* offsets_a, const int64_t* indices_a,
                          const int64_t* offsets_b, const int64_t* indices_b, int64_t* pairs,
                          int64_t cap, int64_t* npairs);

/* ---------------------------------------------------------------- runner
 * The drop-in for spmm_csr_csc / _run_schedule (engine.py:136-184):
 * plan (in the timed region, like the reference) + execute all pairs on the
 * device.  ct_a/ct_b: [2][L+1][n] at level L (device).  masks: host array
 * of `nmasks` device pointers, masks[pos] = mask plaintext for slot `pos`
 * at level L-1 in Montgomery form (engine.MaskCache).  out: [2][L-1][n]
 * device buffer receiving the modular sum of this shard's contributions
 * (zero when the shard has no pairs).  Sharding: pairs sorted by
 * accumulation step are split into `shard_count` contiguous ranges; this
 * call executes range `shard_index` (logical counters still describe the
 * whole matmul).  Result is bit-identical to the reference for any sharding
 * once the shards are summed mod q. */
hs_status hs_spmspm_csr_csc(hs_ctx* ctx, int32_t dim, const int64_t* offsets_a,
                            const int64_t* indices_a, const int64_t* offsets_b,
                            const int64_t* indices_b, const uint64_t* ct_a, const uint64_t* ct_b,
                            const uint64_t* const* masks, int64_t nmasks, uint64_t* out,
                            hs_counters* counters, int32_t shard_index, int32_t shard_count,
                            void* stream);
/* Same executor over an explicit pair list (VCSR/C and the naive runners,
 * engine.py:187-225 -- they differ from CSR/C only in their schedule). */
hs_status hs_spmspm_pairs(hs_ctx* ctx, int32_t dim, const int64_t* pairs, int64_t npairs,
                          const uint64_t* ct_a, const uint64_t* ct_b,
                          const uint64_t* const* masks, int64_t nmasks, uint64_t* out,
                          hs_counters* counters, int32_t shard_index, int32_t shard_count,
                          void* stream);
/* Several operand products accumulated into one or more outputs in ONE
 * schedule (multi-ciphertext tiling, beyond the reference's one-ciphertext
 * capacity, encmat.py:131-133): output block C[I][J] = sum_K A[I][K] B[K][J]
 * for every block at once.  pairs are (i, j, a_pos, b_pos, k, o) rows: k
 * indexes cts_a[k] / cts_b[k], o the output outs[o].  All pairs are
 * scheduled together (sorted by accumulation step across products and
 * outputs), so a Galois key is generated once per step for the whole tiled
 * product and alignment rotations are deduplicated per (operand, step).
 * Logical counters: the products' counts plus the joining adds (adds =
 * pairs - outputs with a pair). */
hs_status hs_spmspm_multi(hs_ctx* ctx, int32_t dim, const int64_t* pairs, int64_t npairs,
                          const uint64_t* const* cts_a, const uint64_t* const* cts_b, int32_t nproducts,
                          const uint64_t* const* masks, int64_t nmasks, uint64_t* const* outs, int32_t noutputs,
                          hs_counters* counters, int32_t shard_index, int32_t shard_count, void* stream);

/* Alignment rotations shared across ranks (multi-GPU, dist.py).  The CSR/C
 * runner rotates the higher-positioned operand of a pair by |a_pos - b_pos|
 * (engine.py:136-160); each distinct (operand, step) is one hoisted rotation
 * of ct_a (operand 0) or ct_b (operand 1) at level L.
 * hs_align_compute: those rotations for count (operand, normalised step)
 * entries into outs[k] (device buffers [2][L+1][n]); Galois keys resident or
 * lazily registered.  hs_align_provide: hand the runner aligned operands
 * another rank computed (device pointers, valid until hs_align_clear); the
 * runner then uses them instead of computing those rotations. */
hs_status hs_align_compute(hs_ctx* ctx, const uint64_t* ct_a, const uint64_t* ct_b, const int32_t* operand,
                           const uint32_t* steps, int64_t count, uint64_t* const* outs, void* stream);
hs_status hs_align_provide(hs_ctx* ctx, const int32_t* operand, const uint32_t* steps,
                           const uint64_t* const* cts, int64_t count);
void hs_align_clear(hs_ctx* ctx);
/* Final modular reduction after an integer SUM collective of shard results
 * (shard_count * q < 2^63, so an int64 NCCL sum is exact). */
hs_status hs_reduce_mod(hs_ctx* ctx, uint64_t* data, int32_t npoly, int32_t nlimbs, void* stream);
/* Tuning knob: device bytes the runner may use for per-batch work buffers. */
void hs_set_batch_bytes(hs_ctx* ctx, uint64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* HESPMM_B200_H */
