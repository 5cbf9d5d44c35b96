// On-device Galois key generation, bit-exact with the reference's
// gen_galois_keys (ckks/context.py:176-200 -> _make_ksk :150-174).
//
// The reference draws every key from its own numpy stream
//   rng = default_rng(SeedSequence(entropy=(seed, 0x90, r)))     (PCG64)
// in this order, per digit i = 0..L:
//   (L+2) x rng.integers(0, q_m, n, uint64)   -- Lemire bounded ints, 64-bit
//   rng.normal(0, 3.2, n) -> rint -> int64     -- ziggurat (256 layers)
// and assembles b[i][m] = NTT(e_i mod q_m) + [m<=L] p(Q_L/q_i) sk(X^g) - a[i][m] sk.
//
// Here one CTA replays one key's stream in order, 1024 positions per chunk:
// every thread advances its own PCG64 state by 1024 per chunk (precomputed
// LCG jump constants), raw outputs go to a two-chunk shared-memory ring, and
// the block consumes them segment by segment:
//   uniform: accept iff low64(x*q) >= (2^64 - q) mod q (Lemire's rejection
//            rule), value = high64(x*q); block scan assigns output indices;
//   normal:  ziggurat fast path in parallel (rabs < ki[idx]); the token parse
//            (slow tokens consume 2 draws, tail tokens 1+2k) is walked by one
//            thread over a fast-path bitmap; block scan assigns indices.
// The SeedSequence -> PCG64 state and the ziggurat tables (read from the
// installed numpy binary and validated against numpy on the host) are inputs.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "ops.cuh"

namespace hs {

constexpr int RNG_T = 512;              // threads per key CTA
constexpr int RNG_E = 8;                // draws per thread per chunk (positions t + k*RNG_T)
constexpr int RNG_CH = RNG_T * RNG_E;   // positions per chunk
constexpr int RNG_W = RNG_T / 32;       // warps
constexpr int UNI_E = 32;               // digit-window kernels: draws per thread per tile
constexpr int UNI_TILE = RNG_T * UNI_E; // positions per tile (16384)
constexpr int UNI_TW = UNI_TILE / 32;   // bitmap words per tile (512)
static_assert(UNI_E == 32, "pk_uni_flags keeps draw e's bitmap words in lane e");

struct U128 {
    u64 hi, lo;
};

HS_DEV U128 mul128(U128 a, U128 b) {    // mod 2^128
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}
HS_DEV U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}
HS_DEV u64 xsl_rr(U128 s) {
    const u64 x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct ZigTables {
    double wi[256];
    double fi[256];
    u64 ki[256];
};

struct RngJump {                          // for t = 0..RNG_CH: A_t = M^t, S_t = sum_{k<t} M^k
    U128 A[RNG_CH + 1];
    U128 S[RNG_CH + 1];
    U128 PA[64];                          // A_{2^j}
    U128 PS[64];                          // S_{2^j}
    U128 TA[1024];                        // A_{t * UNI_TILE}: digit-window tiles (t < 1024)
    U128 TS[1024];                        // S_{t * UNI_TILE}
};

struct KeyStream {
    u64 state_hi, state_lo, inc_hi, inc_lo;   // numpy PCG64 state before the first draw
};

struct KeygenArgs {
    const KeyStream* streams;              // [K]
    u64* const* a_out;                     // [K] -> [L+1][L+2][n] (a half of the key)
    long long* e_out;                      // [K][L+1][n]
    const RngJump* jump;
    const ZigTables* zig;
    const PrimeConst* pc;                  // chain then aux
    const u64* thr;                        // [L+2] Lemire thresholds (2^64 - q) mod q
    int L;
    u32 n;
};

// Set bits [lo, hi) of a shared bitmap.
HS_DEV void set_bit_range(unsigned* bm, u32 lo, u32 hi) {
    while (lo < hi) {
        const u32 w = lo >> 5, b = lo & 31;
        const u32 take = min(32u - b, hi - lo);
        const unsigned mask = take == 32 ? 0xffffffffu : (((1u << take) - 1u) << b);
        bm[w] |= mask;
        lo += take;
    }
}

constexpr double ZIG_R = 3.6541528853610088;
constexpr double ZIG_INV_R = 0.27366123732975828;

HS_DEV double next_double_of(u64 raw) { return (double)(raw >> 11) * (1.0 / 9007199254740992.0); }

// Exclusive scan of the per-(k, warp) ballot counts of a chunk in stream
// order (k-major, then warp, then lane).  cnt[] in/out; returns the total.
HS_DEV u32 chunk_scan(u32* cnt, u32* s_total) {
    __syncthreads();
    if (threadIdx.x < 32) {
        const u32 lane = threadIdx.x;
        constexpr int PER = RNG_E * RNG_W / 32;    // entries per lane
        u32 v[PER > 0 ? PER : 1];
        u32 sum = 0;
#pragma unroll
        for (int k = 0; k < PER; k++) {
            v[k] = cnt[lane * PER + k];
            sum += v[k];
        }
        u32 inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (u32)o) inc += t;
        }
        u32 run = inc - sum;
#pragma unroll
        for (int k = 0; k < PER; k++) {
            cnt[lane * PER + k] = run;
            run += v[k];
        }
        if (lane == 31) *s_total = inc;
    }
    __syncthreads();
    return *s_total;
}

// One CTA per key; thread t owns chunk positions t + k*RNG_T (k < RNG_E), so
// shared-memory traffic is conflict free and stream order is k-major.
__global__ void __launch_bounds__(RNG_T) keygen_stream_kernel(KeygenArgs A) {
    extern __shared__ u64 dyn[];
    u64* raw0 = dyn;                                   // [2][RNG_CH] ring
    double* xval = (double*)(dyn + 2 * RNG_CH);        // [RNG_CH]
    __shared__ unsigned fastbits[RNG_CH / 32];
    __shared__ unsigned emitbits[RNG_CH / 32];
    __shared__ u32 cnt[RNG_E * RNG_W];
    __shared__ u32 s_total;
    __shared__ long long s_cursor;        // absolute stream position of the consumer
    __shared__ u32 s_count;               // outputs produced in the current segment
    __shared__ int s_seg;                 // segment index over the whole key
    __shared__ u32 s_end;

    const int key = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int L = A.L;
    const u32 n = A.n;
    const int segs_per_digit = L + 3;     // (L+2) uniform + 1 normal
    const int nseg = (L + 1) * segs_per_digit;
    const KeyStream ks = A.streams[key];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);       // stride within chunk
    const U128 ACH = A.jump->A[RNG_CH], CCH = mul128(A.jump->S[RNG_CH], inc);  // chunk to chunk
    // state whose output is position t of the next chunk to generate
    U128 st = add128(mul128(A.jump->A[t + 1], U128{ks.state_hi, ks.state_lo}),
                     mul128(A.jump->S[t + 1], inc));
    u64* a_key = A.a_out[key];
    long long* e_key = A.e_out + (size_t)key * (L + 1) * n;

    auto generate = [&](u64* buf) {
        U128 s = st;
#pragma unroll
        for (int k = 0; k < RNG_E; k++) {
            buf[k * RNG_T + t] = xsl_rr(s);
            s = add128(mul128(s, AT), CT);
        }
        st = add128(mul128(st, ACH), CCH);
    };
    generate(raw0);
    generate(raw0 + RNG_CH);
    if (t == 0) {
        s_cursor = 0;
        s_count = 0;
        s_seg = 0;
    }
    __syncthreads();

    long long chunk_base = 0;
    int cur = 0;
    while (true) {
        u64* raw = raw0 + cur * RNG_CH;
        u64* nxt = raw0 + (cur ^ 1) * RNG_CH;
        while (true) {
            const int seg = s_seg;
            if (seg >= nseg) break;
            const long long cursor = s_cursor;
            if (cursor >= chunk_base + RNG_CH) break;
            const int digit = seg / segs_per_digit;
            const int sidx = seg % segs_per_digit;
            const u32 count0 = s_count;
            if (sidx < L + 2) {
                // ---- uniform: integers(0, q, n), Lemire (accept iff lo >= (2^64-q) mod q)
                const u64 q = A.pc[sidx].q;
                const u64 thr = A.thr[sidx];
                u64 val[RNG_E];
                unsigned ball[RNG_E];
#pragma unroll
                for (int k = 0; k < RNG_E; k++) {
                    const u32 i = k * RNG_T + t;
                    const u64 x = raw[i];
                    const bool acc = chunk_base + i >= cursor && x * q >= thr;
                    val[k] = __umul64hi(x, q);
                    ball[k] = __ballot_sync(0xffffffffu, acc);
                    if (lane == 0) cnt[k * RNG_W + warp] = __popc(ball[k]);
                }
                const u32 total = chunk_scan(cnt, &s_total);
                u64* dst = a_key + ((size_t)digit * (L + 2) + sidx) * n;
#pragma unroll
                for (int k = 0; k < RNG_E; k++) {
                    if (!((ball[k] >> lane) & 1u)) continue;
                    const u32 idx = count0 + cnt[k * RNG_W + warp] + __popc(ball[k] & lt);
                    if (idx < n) dst[idx] = val[k];
                    if (idx == n - 1) s_end = k * RNG_T + t + 1;
                }
                __syncthreads();
                if (t == 0) {
                    if (count0 + total >= n) {
                        s_cursor = chunk_base + s_end;
                        s_count = 0;
                        s_seg = seg + 1;
                    } else {
                        s_cursor = chunk_base + RNG_CH;
                        s_count = count0 + total;
                    }
                }
                __syncthreads();
            } else {
                // ---- normal: 0 + 3.2 * standard_normal (ziggurat), rint -> int64
#pragma unroll
                for (int k = 0; k < RNG_E; k++) {
                    const u32 i = k * RNG_T + t;
                    const u64 r = raw[i];
                    const int zi = (int)(r & 0xff);
                    const u64 r8 = r >> 8;
                    const u64 rabs = (r8 >> 1) & 0x000fffffffffffffull;
                    double x = (double)rabs * A.zig->wi[zi];
                    if (r8 & 1) x = -x;
                    xval[i] = x;
                    const unsigned fb = __ballot_sync(0xffffffffu, rabs < A.zig->ki[zi]);
                    if (lane == 0) {
                        fastbits[i >> 5] = fb;
                        emitbits[i >> 5] = 0u;
                    }
                }
                __syncthreads();
                if (t == 0) {
                    // token walk over [cursor, chunk end): fast tokens are 1 draw;
                    // slow tokens consume the following draw(s), maybe from the next chunk
                    long long c = cursor;
                    u32 cntv = count0;
                    const long long cend = chunk_base + RNG_CH;
                    bool done = false;
                    auto draw_at = [&](long long pos) -> u64 {
                        const long long rp = pos - chunk_base;
                        return rp < RNG_CH ? raw[rp] : nxt[rp - RNG_CH];
                    };
                    while (c < cend && !done) {
                        const u32 rel = (u32)(c - chunk_base);
                        u32 s = RNG_CH;
                        for (u32 w = rel >> 5; w < RNG_CH / 32; w++) {
                            unsigned bits = ~fastbits[w];
                            if (w == (rel >> 5)) bits &= ~((1u << (rel & 31)) - 1u);
                            if (bits) {
                                s = (w << 5) + __ffs(bits) - 1;
                                break;
                            }
                        }
                        u32 run = s - rel;
                        if (cntv + run >= n) {
                            run = n - cntv;
                            done = true;
                        }
                        set_bit_range(emitbits, rel, rel + run);
                        cntv += run;
                        c += run;
                        if (done || s >= RNG_CH) break;
                        const u64 rs = raw[s];
                        const int zs = (int)(rs & 0xff);
                        const u64 rabs_s = ((rs >> 8) >> 1) & 0x000fffffffffffffull;
                        if (zs != 0) {
                            const double xs = xval[s];
                            const double u = next_double_of(draw_at(c + 1));
                            if ((A.zig->fi[zs - 1] - A.zig->fi[zs]) * u + A.zig->fi[zs] < exp(-0.5 * xs * xs)) {
                                emitbits[s >> 5] |= 1u << (s & 31);
                                if (++cntv >= n) done = true;
                            }
                            c += 2;
                        } else {
                            long long pos = c + 1;
                            double v;
                            while (true) {
                                const double xx = -ZIG_INV_R * log1p(-next_double_of(draw_at(pos)));
                                const double yy = -log1p(-next_double_of(draw_at(pos + 1)));
                                pos += 2;
                                if (yy + yy > xx * xx) {
                                    v = ((rabs_s >> 8) & 1) ? -(ZIG_R + xx) : ZIG_R + xx;
                                    break;
                                }
                            }
                            xval[s] = v;
                            emitbits[s >> 5] |= 1u << (s & 31);
                            if (++cntv >= n) done = true;
                            c = pos;
                        }
                    }
                    s_cursor = c;
                    s_end = done ? 1u : 0u;
                }
                __syncthreads();
                unsigned ball[RNG_E];
#pragma unroll
                for (int k = 0; k < RNG_E; k++) {
                    const u32 i = k * RNG_T + t;
                    ball[k] = __ballot_sync(0xffffffffu, (emitbits[i >> 5] >> (i & 31)) & 1u);
                    if (lane == 0) cnt[k * RNG_W + warp] = __popc(ball[k]);
                }
                chunk_scan(cnt, &s_total);
                long long* dst = e_key + (size_t)digit * n;
#pragma unroll
                for (int k = 0; k < RNG_E; k++) {
                    if (!((ball[k] >> lane) & 1u)) continue;
                    const u32 i = k * RNG_T + t;
                    const u32 idx = count0 + cnt[k * RNG_W + warp] + __popc(ball[k] & lt);
                    dst[idx] = (long long)rint(0.0 + 3.2 * xval[i]);
                }
                __syncthreads();
                if (t == 0) {
                    if (s_end) {
                        s_count = 0;
                        s_seg = seg + 1;
                    } else {
                        s_count = count0 + s_total;
                    }
                }
                __syncthreads();
            }
        }
        if (s_seg >= nseg) break;
        // ring advance: chunk c+1 becomes current, generate chunk c+2 in place of c
        __syncthreads();
        generate(raw);
        cur ^= 1;
        chunk_base += RNG_CH;
        __syncthreads();
    }
}

// Assemble b[i][m] in place: on entry b holds NTT(e_i mod q_m); adds
// f[i][m] * sk(X^g)_m (m <= L; sk(X^g) = NTT-domain automorphism of sk,
// SURVEY P2) and subtracts a[i][m] * sk_m.
__global__ void ksk_galois_kernel(Dev d, u64* const* keys, const u32* gal, const u64* sk,
                                  const ulonglong2* f) {
    const u32 n = d.n;
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int m = blockIdx.y % (d.L + 2), i = blockIdx.y / (d.L + 2), kk = blockIdx.z;
    const int L = d.L;
    const PrimeConst P = d.pc[m];
    u64* key = keys[kk];
    const size_t o = ((size_t)i * (L + 2) + m) * n + j;
    u64 acc = key[o];
    if (m <= L) {
        const u32 src = __brev(j) >> (32 - d.log_n);
        const u32 e = (u32)((((u64)(2 * src + 1)) * gal[kk]) & ((2ull << d.log_n) - 1));
        const u32 pj = __brev((e - 1) >> 1) >> (32 - d.log_n);
        const ulonglong2 w = f[i * (L + 1) + m];
        acc = add_mod(acc, shoup(sk[(size_t)m * n + pj], w.x, w.y, P.q), P.q);
    }
    const u64* a = key + (size_t)(L + 1) * (L + 2) * n;
    acc = sub_mod(acc, mul_mod(a[o], sk[(size_t)m * n + j], P), P.q);
    key[o] = acc;
}

void keygen_streams(const Dev& d, int K, const void* streams, u64* const* a_out, long long* e_out,
                    const void* jump, const void* zig, const u64* thr, cudaStream_t st) {
    KeygenArgs A{(const KeyStream*)streams, a_out, e_out, (const RngJump*)jump, (const ZigTables*)zig,
                 d.pc, thr, d.L, d.n};
    constexpr size_t smem = (size_t)3 * RNG_CH * sizeof(u64);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(keygen_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    keygen_stream_kernel<<<K, RNG_T, smem, st>>>(A);
    note_launch();
}

// ====================================================== grid-parallel streams
// The serial kernel above gives each key one SM.  Here all keys of a batch
// advance through their streams in lockstep, one segment (one integers() or
// normal() call) per pair of launches, and each segment is spread over
// W / RNG_CH CTAs per key: a CTA jumps its key's PCG64 to its tile (binary
// composition of power-of-two LCG jumps), generates the tile's draws, and
// acceptance counts / ranks come from per-tile counts and block scans.  The
// normal segment's token parse (fast tokens 1 draw, slow 2, tail 1+2k) is a
// one-warp walk over the fast-path bitmap, skipping 32 fast draws per step.

struct ParArgs {
    const KeyStream* streams;
    const RngJump* jump;
    const ZigTables* zig;
    const PrimeConst* pc;
    const u64* thr;
    u64* raw;              // [K][W] window draws
    u32* cnt;              // [K][NT] per-tile counts (exclusive prefix after scan)
    unsigned* fastb;       // [K][W/32]
    unsigned* emitb;       // [K][W/32]
    double* tailx;         // [K][W] values of tail tokens (sparse)
    u32* tlen;             // [K][W] draws consumed by a tail token (sparse, 0 = window too short)
    u64* pos_in;           // [K] segment start
    u64* pos_out;          // [K] next segment start
    u64* const* a_out;     // [K] a half of each key
    long long* e_out;      // [K][L+1][n]
    int* err;              // window overflow
    int L, W, NT;
    u32 n;
};

// State producing the draw at absolute position P + t + 1 ... : thread 0 jumps
// the key's start state by P (power-of-two compositions), threads fan out.
HS_DEV U128 tile_state(const ParArgs& A, const KeyStream& ks, u64 P, U128* s_x) {
    const U128 inc{ks.inc_hi, ks.inc_lo};
    if (threadIdx.x < 32) {
        // jumps by 2^j commute: lane l composes the set bits l and l+32 of P,
        // then a butterfly reduction composes the 32 affine maps x -> Ax + B
        const u32 l = threadIdx.x;
        U128 Am{0, 1}, Bm{0, 0};
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const u32 j = l + 32u * h;
            if ((P >> j) & 1ull) {
                const U128 Aj = A.jump->PA[j], Bj = mul128(A.jump->PS[j], inc);
                Bm = add128(mul128(Aj, Bm), Bj);
                Am = mul128(Aj, Am);
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            U128 Ao, Bo;
            Ao.hi = __shfl_xor_sync(0xffffffffu, Am.hi, o);
            Ao.lo = __shfl_xor_sync(0xffffffffu, Am.lo, o);
            Bo.hi = __shfl_xor_sync(0xffffffffu, Bm.hi, o);
            Bo.lo = __shfl_xor_sync(0xffffffffu, Bm.lo, o);
            Bm = add128(mul128(Ao, Bm), Bo);
            Am = mul128(Ao, Am);
        }
        if (l == 0) *s_x = add128(mul128(Am, U128{ks.state_hi, ks.state_lo}), Bm);
    }
    __syncthreads();
    const U128 x = *s_x;
    return add128(mul128(A.jump->A[threadIdx.x + 1], x), mul128(A.jump->S[threadIdx.x + 1], inc));
}

// Generate the tile's draws; uniform mode counts Lemire accepts for bound
// pc[sidx], normal mode writes the fast-path bitmap.
__global__ void __launch_bounds__(RNG_T) pk_gen_kernel(ParArgs A, int normal, int sidx) {
    __shared__ U128 s_x;
    __shared__ u32 s_cnt[RNG_W];
    const int k = blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    const u64 base = A.pos_in[k] + (u64)tile * RNG_CH;
    U128 s = tile_state(A, ks, base, &s_x);
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);
    u64* raw = A.raw + (size_t)k * A.W + (size_t)tile * RNG_CH;
    u32 c = 0;
    const u64 q = A.pc[sidx].q, thr = A.thr[sidx];
#pragma unroll
    for (int e = 0; e < RNG_E; e++) {
        const u32 i = e * RNG_T + t;
        const u64 x = xsl_rr(s);
        s = add128(mul128(s, AT), CT);
        raw[i] = x;
        if (normal) {
            const u64 r8 = x >> 8;
            const u64 rabs = (r8 >> 1) & 0x000fffffffffffffull;
            const unsigned fb = __ballot_sync(0xffffffffu, rabs < A.zig->ki[x & 0xff]);
            if (lane == 0) A.fastb[(size_t)k * (A.W / 32) + ((size_t)tile * RNG_CH + i) / 32] = fb;
        } else {
            c += __popc(__ballot_sync(0xffffffffu, x * q >= thr));
        }
    }
    if (!normal) {
        if (lane == 0) s_cnt[warp] = c;
        __syncthreads();
        if (t == 0) {
            u32 tot = 0;
            for (int w = 0; w < RNG_W; w++) tot += s_cnt[w];
            A.cnt[(size_t)k * A.NT + tile] = tot;
        }
    }
}

// Uniform segment in one launch (decoupled look-back): each tile generates
// its draws, publishes its Lemire accept count (tagged with the launch
// sequence number), sums its predecessors' counts and writes its accepted
// values at their stream ranks.  Tiles that may lie past the segment end
// look back first and skip generation when the segment is already complete.
HS_DEV void publish(unsigned long long* f, u32 seq, u32 v) {
    const unsigned long long x = ((unsigned long long)seq << 32) | v;
    // the flag word carries the count itself: relaxed ordering suffices
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(f), "l"(x) : "memory");
}
HS_DEV u32 look_back(const unsigned long long* fl, int tile, u32 seq) {
    u32 sum = 0;
    for (int j = (int)(threadIdx.x & 31); j < tile; j += 32) {
        unsigned long long x;
        do {
            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(fl + j) : "memory");
        } while ((u32)(x >> 32) != seq);
        sum += (u32)x;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    return sum;
}

__global__ void __launch_bounds__(RNG_T) pk_uniform_fused(ParArgs A, int digit, int sidx,
                                                          unsigned long long* flags, u32 seq) {
    __shared__ U128 s_x;
    __shared__ u32 cnt[RNG_E * RNG_W];
    __shared__ u32 s_total, s_prefix;
    const int k = blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const u32 n = A.n;
    unsigned long long* fl = flags + (size_t)k * A.NT;
    const bool spec = (u64)tile * RNG_CH >= n;
    if (spec) {
        if (warp == 0) {
            const u32 p = look_back(fl, tile, seq);
            if (lane == 0) s_prefix = p;
        }
        __syncthreads();
        if (s_prefix >= n) {
            if (t == 0) publish(fl + tile, seq, 0u);
            return;
        }
    }
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    U128 s = tile_state(A, ks, A.pos_in[k] + (u64)tile * RNG_CH, &s_x);
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);
    const u64 q = A.pc[sidx].q, thr = A.thr[sidx];
    u64 val[RNG_E];
    unsigned ball[RNG_E];
#pragma unroll
    for (int e = 0; e < RNG_E; e++) {
        const u64 x = xsl_rr(s);
        s = add128(mul128(s, AT), CT);
        val[e] = __umul64hi(x, q);
        ball[e] = __ballot_sync(0xffffffffu, x * q >= thr);
        if (lane == 0) cnt[e * RNG_W + warp] = __popc(ball[e]);
    }
    const u32 total = chunk_scan(cnt, &s_total);
    if (t == 0) publish(fl + tile, seq, total);
    if (!spec) {
        if (warp == 0) {
            const u32 p = look_back(fl, tile, seq);
            if (lane == 0) s_prefix = p;
        }
        __syncthreads();
    }
    const u32 prefix = s_prefix;
    if (t == 0 && tile == A.NT - 1 && prefix + total < n) *A.err = 1;
    if (prefix >= n) return;
    u64* dst = A.a_out[k] + ((size_t)digit * (A.L + 2) + sidx) * n;
#pragma unroll
    for (int e = 0; e < RNG_E; e++) {
        if (!((ball[e] >> lane) & 1u)) continue;
        const u32 idx = prefix + cnt[e * RNG_W + warp] + __popc(ball[e] & lt);
        if (idx < n) dst[idx] = val[e];
        if (idx == n - 1) A.pos_out[k] = A.pos_in[k] + (u64)tile * RNG_CH + e * RNG_T + t + 1;
    }
}


// All L+2 uniform segments of one digit in ONE cooperative launch: CTA
// (tile, key) stays resident and walks the segments in order.  A segment's
// start position is published by the CTA that wrote its predecessor's n-th
// value (tagged word: tag << 40 | position); within a segment the tiles use
// the same decoupled look-back as pk_uniform_fused.  Flags and start words
// have one slot per (key, segment[, tile]): tiles past a segment's end can lag
// arbitrarily far behind without their slots being overwritten.  Saves ~L+1
// launches per digit and the launch-to-launch drain (dominant at K ~ 20).
#ifndef KG_PERSIST_MINB
#define KG_PERSIST_MINB 3      // (A/B: 3 -> 1.16 ms/key vs 2 -> 1.26 at K=23) co-resident CTAs per SM (keys per cooperative launch = that x 148 / tiles)
#endif
HS_DEV unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long x;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}

__global__ void __launch_bounds__(RNG_T, KG_PERSIST_MINB) pk_uniform_persist(ParArgs A, int digit, int kbase,
                                                            unsigned long long* flags,
                                                            unsigned long long* segpos, u32 seq0) {
    __shared__ U128 s_x;
    __shared__ u32 cnt[RNG_E * RNG_W];
    __shared__ u32 s_total, s_prefix;
    __shared__ u64 s_pos;
    const int k = kbase + (int)blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const u32 n = A.n;
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);
    const int nseg = A.L + 2;
    unsigned long long* sp = segpos + (size_t)k * nseg;       // [nseg] start words
    const bool spec = (u64)tile * RNG_CH >= n;
    for (int m = 0; m < nseg; m++) {
        const u32 seq = seq0 + (u32)m;
        unsigned long long* fl = flags + ((size_t)k * nseg + m) * A.NT;
        if (t == 0) {
            u64 p;
            if (m == 0) {
                p = A.pos_in[k];
            } else {
                unsigned long long x;
                do {
                    x = ld_relaxed(sp + m);
                } while ((u32)(x >> 40) != seq);
                p = x & ((1ull << 40) - 1ull);
            }
            s_pos = p;
        }
        __syncthreads();
        const u64 pos = s_pos;
        bool skip = false;
        if (spec) {
            if (warp == 0) {
                const u32 pf = look_back(fl, tile, seq);
                if (lane == 0) s_prefix = pf;
            }
            __syncthreads();
            skip = s_prefix >= n;
            if (skip && t == 0) publish(fl + tile, seq, 0u);
        }
        if (!skip) {
            U128 st = tile_state(A, ks, pos + (u64)tile * RNG_CH, &s_x);
            const u64 q = A.pc[m].q, thr = A.thr[m];
            u64 val[RNG_E];
            unsigned ball[RNG_E];
#pragma unroll
            for (int e = 0; e < RNG_E; e++) {
                const u64 x = xsl_rr(st);
                st = add128(mul128(st, AT), CT);
                val[e] = __umul64hi(x, q);
                ball[e] = __ballot_sync(0xffffffffu, x * q >= thr);
                if (lane == 0) cnt[e * RNG_W + warp] = __popc(ball[e]);
            }
            const u32 total = chunk_scan(cnt, &s_total);
            if (t == 0) publish(fl + tile, seq, total);
            if (!spec) {
                if (warp == 0) {
                    const u32 pf = look_back(fl, tile, seq);
                    if (lane == 0) s_prefix = pf;
                }
                __syncthreads();
            }
            const u32 prefix = s_prefix;
            if (t == 0 && tile == A.NT - 1 && prefix + total < n) *A.err = 1;
            if (prefix < n) {
                u64* dst = A.a_out[k] + ((size_t)digit * (A.L + 2) + m) * n;
#pragma unroll
                for (int e = 0; e < RNG_E; e++) {
                    if (!((ball[e] >> lane) & 1u)) continue;
                    const u32 idx = prefix + cnt[e * RNG_W + warp] + __popc(ball[e] & lt);
                    if (idx < n) dst[idx] = val[e];
                    if (idx == n - 1) {
                        const u64 next = pos + (u64)tile * RNG_CH + e * RNG_T + t + 1;
                        if (m + 1 < nseg) {
                            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sp + m + 1),
                                         "l"(((unsigned long long)(seq + 1) << 40) | next)
                                         : "memory");
                        } else {
                            A.pos_out[k] = next;
                        }
                    }
                }
            }
        }
        __syncthreads();            // shared state is reused by the next segment
    }
}

// Normal segment token parse, one CTA per key, everything in shared memory:
//  1. every non-fast position s is evaluated as if it started a token:
//     layer zs != 0 -> accept bit from the exp test with draw s+1 (2 draws);
//     zs == 0 (tail) -> value and length 1 + 2k of the log1p loop;
//  2. warp 0 walks the token chain: 32 bitmap words per ballot to find the
//     next slow position, counting the fast tokens in between; only slow
//     token starts are visited one by one (about 1 in 80 positions);
//  3. emit bits = (fast & not consumed) | accepted slow starts, up to the
//     n-th emission; per-tile exclusive prefix counts for pk_normal_write.
constexpr int NW_T = 512;

// Clear bits [lo, hi) of a shared bitmap (one warp).
HS_DEV void clear_bits(unsigned* bmp, u32 lo, u32 hi, u32 lane) {
    if (lo >= hi) return;
    for (u32 w = (lo >> 5) + lane; w <= ((hi - 1) >> 5); w += 32) {
        const u32 b0 = max(lo, w << 5) - (w << 5), b1 = min(hi, (w + 1) << 5) - (w << 5);
        const unsigned m = (b1 - b0 == 32u) ? 0xffffffffu : (((1u << (b1 - b0)) - 1u) << b0);
        bmp[w] &= ~m;
    }
}

// Walk the token chain from token start c while c < stop (one warp): fast
// positions are single-draw tokens; a slow position s starts a token of 2
// draws (tail: tl[s]).  Marks slow starts in sb and consumed draws in cb;
// returns the first token start >= stop.  A token running past the window
// sets trunc to its start and ends the walk (returns W).
HS_DEV u32 walk_chain(u32 c, u32 stop, const unsigned* fb, const unsigned* tb, unsigned* sb,
                      unsigned* cb, const u32* tl, u32 W, u32 lane, u32& trunc) {
    while (c < stop) {
        const u32 w0 = c >> 5;
        const u32 w = w0 + lane;
        unsigned x = 0u;
        if ((w << 5) < stop) {
            x = ~fb[w];
            if (lane == 0) x &= ~((1u << (c & 31)) - 1u);
            const u32 top = stop - (w << 5);
            if (top < 32u) x &= (1u << top) - 1u;
        }
        const unsigned ball = __ballot_sync(0xffffffffu, x != 0u);
        if (ball == 0u) {
            c = min((w0 + 32u) << 5, stop);
            continue;
        }
        const int f = __ffs(ball) - 1;
        const unsigned xf = __shfl_sync(0xffffffffu, x, f);
        const u32 s = ((w0 + (u32)f) << 5) + (u32)(__ffs(xf) - 1);
        const unsigned bit = 1u << (s & 31);
        const u32 len = (tb[s >> 5] & bit) ? tl[s] : 2u;
        if (len == 0 || s + len > W) {       // token runs past the window: chain truncated at s
            trunc = s;
            return W;
        }
        if (lane == 0) {            // neighbouring pieces may share a word: atomics
            atomicOr(&sb[s >> 5], bit);
            for (u32 p = s + 1; p < s + len; p++) atomicOr(&cb[p >> 5], 1u << (p & 31));
        }
        __syncwarp();
        c = s + len;
    }
    return c;
}

__global__ void __launch_bounds__(NW_T) pk_normal_walk2(ParArgs A) {
    extern __shared__ unsigned bm[];
    const int k = blockIdx.x;
    const int words = A.W / 32;
    unsigned* fb = bm;                 // fast-path bits
    unsigned* ab = bm + words;         // slow token would emit (layer test / tail)
    unsigned* tb = bm + 2 * words;     // slow token is a tail
    unsigned* cb = bm + 3 * words;     // consumed as a uniform by a token start
    unsigned* sb = bm + 4 * words;     // slow token starts
    __shared__ int s_err;
    __shared__ u32 s_tile[64];
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const u32 n = A.n;
    const u32 W = (u32)A.W;
    const unsigned* gfb = A.fastb + (size_t)k * words;
    const u64* raw = A.raw + (size_t)k * A.W;
    double* tx = A.tailx + (size_t)k * A.W;
    u32* tl = A.tlen + (size_t)k * A.W;
    for (int w = t; w < words; w += NW_T) {
        fb[w] = gfb[w];
        cb[w] = 0u;
        sb[w] = 0u;
    }
    if (t == 0) s_err = 0;
    __syncthreads();
    // ---- 1. speculative evaluation of every slow position
    for (int w = t; w < words; w += NW_T) {
        unsigned slow = ~fb[w], acc = 0u, tail = 0u;
        while (slow) {
            const int b = __ffs(slow) - 1;
            slow &= slow - 1u;
            const u32 s = (u32)w * 32u + (u32)b;
            const u64 rs = raw[s];
            const int zs = (int)(rs & 0xff);
            const u64 rabs = ((rs >> 8) >> 1) & 0x000fffffffffffffull;
            if (zs != 0) {
                if (s + 1 >= W) continue;                     // cannot be decided: walk errors out
                double xs = (double)rabs * A.zig->wi[zs];
                if ((rs >> 8) & 1) xs = -xs;
                const double u = next_double_of(raw[s + 1]);
                if ((A.zig->fi[zs - 1] - A.zig->fi[zs]) * u + A.zig->fi[zs] < exp(-0.5 * xs * xs))
                    acc |= 1u << b;
            } else {
                tail |= 1u << b;
                acc |= 1u << b;
                u32 pos = s + 1, len = 0;
                while (pos + 1 < W) {
                    const double xx = -ZIG_INV_R * log1p(-next_double_of(raw[pos]));
                    const double yy = -log1p(-next_double_of(raw[pos + 1]));
                    pos += 2;
                    if (yy + yy > xx * xx) {
                        tx[s] = ((rabs >> 8) & 1) ? -(ZIG_R + xx) : ZIG_R + xx;
                        len = pos - s;
                        break;
                    }
                }
                tl[s] = len;
            }
        }
        ab[w] = acc;
        tb[w] = tail;
    }
    __syncthreads();
    // ---- 2. token chain: speculative walks of 16 pieces, then serial fix-ups
    // (a piece's entry is its first position unless the previous piece's last
    // token spills over it; chains re-synchronise within a token or two).
    // A token running past the window end truncates the chain there; the
    // segment is valid only if its n-th emission comes before that point.
    constexpr int NWARP = NW_T / 32;
    __shared__ u32 s_exit[NWARP], s_trunc[NWARP];
    __shared__ u32 s_chain_trunc;
    const u32 pw = ((u32)words + NWARP - 1) / NWARP;          // words per piece
    {
        const u32 ps = min(warp * pw, (u32)words) << 5, pe = min((warp + 1) * pw, (u32)words) << 5;
        u32 tr = W;
        const u32 x = walk_chain(ps, pe, fb, tb, sb, cb, tl, W, lane, tr);
        if (lane == 0) {
            s_exit[warp] = x;
            s_trunc[warp] = tr;
        }
    }
    __syncthreads();
    if (warp == 0) {
        u32 actual = s_exit[0], ctr = s_trunc[0];
        bool dirty = false;                  // a re-walk cleared marks inside piece i
        for (int i = 1; i < NWARP && ctr == W; i++) {
            const u32 ps = min((u32)i * pw, (u32)words) << 5, pe = min((u32)(i + 1) * pw, (u32)words) << 5;
            if (ps >= pe) continue;
            if (actual == ps && !dirty) {
                actual = s_exit[i];
                ctr = s_trunc[i];
                continue;
            }
            // misprediction: drop piece i's speculative marks, re-walk from `actual`
            const u32 spec_end = max(s_exit[i], actual);
            clear_bits(sb, ps, spec_end, lane);
            clear_bits(cb, actual, spec_end, lane);
            __syncwarp();
            actual = walk_chain(actual, pe, fb, tb, sb, cb, tl, W, lane, ctr);
            dirty = spec_end > pe;
        }
        if (lane == 0) s_chain_trunc = ctr;
    }
    __syncthreads();
    // ---- 3. emissions = (fast & not consumed) | emitting slow starts; the
    // segment ends after the n-th emission
    constexpr int WPTH = 12;                                // words per thread in the scan (W <= 196608)
    __shared__ u32 s_wsum[NW_T / 32];
    __shared__ u32 s_pos;
    u32 pop[WPTH], tsum = 0;
#pragma unroll
    for (int q = 0; q < WPTH; q++) {
        const u32 w = t * WPTH + q;
        pop[q] = w < (u32)words ? __popc((fb[w] & ~cb[w]) | (ab[w] & sb[w])) : 0u;
        tsum += pop[q];
    }
    u32 inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (u32)o) inc += v;
    }
    if (lane == 31) s_wsum[warp] = inc;
    if (t == 0) s_pos = 0xffffffffu;
    __syncthreads();
    u32 before = inc - tsum;
    for (int w = 0; w < (int)warp; w++) before += s_wsum[w];
    if (!s_err && before < n && before + tsum >= n) {
        u32 need = n - before;                              // 1-based rank within this thread's words
#pragma unroll
        for (int q = 0; q < WPTH; q++) {
            if (need > pop[q]) {
                need -= pop[q];
                continue;
            }
            const u32 w = t * WPTH + q;
            unsigned e = (fb[w] & ~cb[w]) | (ab[w] & sb[w]);
            for (u32 r = 1; r < need; r++) e &= e - 1u;
            s_pos = (w << 5) + (u32)(__ffs(e) - 1);
            break;
        }
    }
    __syncthreads();
    if (s_err || s_pos >= s_chain_trunc) {
        if (t == 0) {
            *A.err = 1;
            A.pos_out[k] = A.pos_in[k];
        }
        return;
    }
    const u32 last = s_pos;                                 // position of the n-th emission
    const unsigned lbit = 1u << (last & 31);
    const u32 end = (sb[last >> 5] & lbit) ? last + ((tb[last >> 5] & lbit) ? tl[last] : 2u) : last + 1u;
    unsigned* eb = A.emitb + (size_t)k * words;
    constexpr int WPT = RNG_CH / 32;       // words per tile
    const int NT = A.NT;
    for (int tile = warp; tile < NT; tile += NW_T / 32) {
        u32 sum = 0;
        for (int w = tile * WPT + lane; w < (tile + 1) * WPT; w += 32) {
            unsigned e = (fb[w] & ~cb[w]) | (ab[w] & sb[w]);
            const u32 base = (u32)w << 5;
            if (base > last) e = 0u;
            else if (last - base < 31u) e &= (2u << (last - base)) - 1u;
            eb[w] = e;
            sum += __popc(e);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) s_tile[tile] = sum;
    }
    __syncthreads();
    if (t == 0) {
        u32 run = 0;
        for (int tile = 0; tile < NT; tile++) {
            A.cnt[(size_t)k * NT + tile] = run;
            run += s_tile[tile];
        }
        A.pos_out[k] = A.pos_in[k] + end;
    }
}

// Normal segment: write e values (0 + 3.2 z, rint) of emitted tokens.
__global__ void __launch_bounds__(RNG_T) pk_normal_write(ParArgs A, int digit) {
    __shared__ u32 cnt[RNG_E * RNG_W];
    __shared__ u32 s_total;
    const int k = blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const u32 n = A.n;
    const u32 prefix = A.cnt[(size_t)k * A.NT + tile];
    if (prefix >= n) return;
    const unsigned* eb = A.emitb + (size_t)k * (A.W / 32) + (size_t)tile * (RNG_CH / 32);
    const u64* raw = A.raw + (size_t)k * A.W + (size_t)tile * RNG_CH;
    const double* tx = A.tailx + (size_t)k * A.W + (size_t)tile * RNG_CH;
    unsigned ball[RNG_E];
#pragma unroll
    for (int e = 0; e < RNG_E; e++) {
        const u32 i = e * RNG_T + t;
        ball[e] = __ballot_sync(0xffffffffu, (eb[i >> 5] >> (i & 31)) & 1u);
        if (lane == 0) cnt[e * RNG_W + warp] = __popc(ball[e]);
    }
    chunk_scan(cnt, &s_total);
    long long* dst = A.e_out + ((size_t)k * (A.L + 1) + digit) * n;
#pragma unroll
    for (int e = 0; e < RNG_E; e++) {
        if (!((ball[e] >> lane) & 1u)) continue;
        const u32 i = e * RNG_T + t;
        const u32 idx = prefix + cnt[e * RNG_W + warp] + __popc(ball[e] & lt);
        if (idx >= n) continue;
        const u64 r = raw[i];
        const int zi = (int)(r & 0xff);
        const u64 rabs = ((r >> 8) >> 1) & 0x000fffffffffffffull;
        double x;
        if (zi == 0 && rabs >= A.zig->ki[0]) {
            x = tx[i];                                   // tail token value
        } else {
            x = (double)rabs * A.zig->wi[zi];
            if ((r >> 8) & 1) x = -x;
        }
        dst[idx] = (long long)rint(0.0 + 3.2 * x);
    }
}

// ============================================ digit-window uniform segments
// The L+2 uniform segments of one digit (integers(0, q_m, n) for m = 0..L+1)
// resolved WITHOUT a sequential chain of segment launches.  Rejections are
// rare (p < q/2^64), so position r of the digit's stream (relative to the
// digit start) lies in segment z = r / n ("zone") or z - 1:
//  0. pk_uni_start (one warp per key): PCG64 state at the digit start (binary
//     composition of power-of-two jumps); every tile then jumps from it with
//     one affine map from a table (TA/TS, tiles of UNI_TILE draws);
//  1. pk_uni_flags (all tiles, all keys): generate every draw of the window
//     once, store two accept bitmaps -- under q_z (hi) and under q_{z-1}
//     (lo) -- and per-tile popcounts;
//  2. pk_uni_bounds (one warp per key): segment starts S_1..S_{L+2} in order
//     (S_{m+1} = one past the n-th q_m-accept from S_m: hi bits up to the end
//     of zone m, then lo bits of zone m+1), from tile counts + a few words;
//  3. pk_uni_emit (all tiles): effective accept bits (hi if r >= S_z, else lo)
//     from the bitmaps, tile totals chained by decoupled look-back, then the
//     draws regenerated once more for their values; accepted draws land at
//     their rank in the digit's flat [L+2][n] block of the a half (segment m's
//     n values are exactly ranks m*n .. m*n+n-1).
// If the cumulative rejections of a digit reach n (tiny rings) or the window
// is too short, *err is set and the caller replays serially (exact either way).
struct UniArgs {
    unsigned* hib;          // [K][WU/32]
    unsigned* lob;          // [K][WU/32]
    u32* chi;               // [K][NTU]
    u32* seg;               // [K][L+3] segment starts relative to the digit start
    U128* s0;               // [K] PCG64 state at the digit start
    unsigned long long* flags;   // [K][NTU] look-back flags of pk_uni_emit
    u32 WU, NTU;
    int log_n;
};

__global__ void __launch_bounds__(32) pk_uni_start(ParArgs A, UniArgs U) {
    const int k = blockIdx.x;
    const u32 l = threadIdx.x;
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    const u64 P = A.pos_in[k];
    U128 Am{0, 1}, Bm{0, 0};
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const u32 j = l + 32u * h;
        if ((P >> j) & 1ull) {
            const U128 Aj = A.jump->PA[j], Bj = mul128(A.jump->PS[j], inc);
            Bm = add128(mul128(Aj, Bm), Bj);
            Am = mul128(Aj, Am);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        U128 Ao, Bo;
        Ao.hi = __shfl_xor_sync(0xffffffffu, Am.hi, o);
        Ao.lo = __shfl_xor_sync(0xffffffffu, Am.lo, o);
        Bo.hi = __shfl_xor_sync(0xffffffffu, Bm.hi, o);
        Bo.lo = __shfl_xor_sync(0xffffffffu, Bm.lo, o);
        Bm = add128(mul128(Ao, Bm), Bo);
        Am = mul128(Ao, Am);
    }
    if (l == 0) U.s0[k] = add128(mul128(Am, U128{ks.state_hi, ks.state_lo}), Bm);
}

// State whose output is the draw at window position tile*UNI_TILE + t.
HS_DEV U128 uni_thread_state(const ParArgs& A, const UniArgs& U, int k, int tile, const U128& inc) {
    const U128 s0 = U.s0[k];
    const U128 T = add128(mul128(A.jump->TA[tile], s0), mul128(A.jump->TS[tile], inc));
    return add128(mul128(A.jump->A[threadIdx.x + 1], T), mul128(A.jump->S[threadIdx.x + 1], inc));
}

// ZU: every tile lies inside one zone (n >= UNI_TILE): the two candidate
// moduli and thresholds are CTA constants; otherwise they are looked up per
// position from shared memory.
template <bool ZU>
__global__ void __launch_bounds__(RNG_T) pk_uni_flags(ParArgs A, UniArgs U) {
    __shared__ u32 s_h[RNG_W];
    __shared__ u64 s_q[66], s_t[66];
    const int k = blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int L = A.L;
    if (!ZU) {
        for (int m = t; m <= L + 1; m += RNG_T) {
            s_q[m] = A.pc[m].q;
            s_t[m] = A.thr[m];
        }
        __syncthreads();
    }
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    U128 s = uni_thread_state(A, U, k, tile, inc);
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);
    const int zt = (int)(((u32)tile * UNI_TILE) >> U.log_n);      // the tile's zone (ZU)
    const bool hv = zt <= L + 1, lv = zt >= 1 && zt <= L + 2;
    const u64 qh = hv ? __ldg(&A.pc[zt].q) : 0ull, th = hv ? __ldg(A.thr + zt) : 0ull;
    const u64 ql = lv ? __ldg(&A.pc[zt - 1].q) : 0ull, tl = lv ? __ldg(A.thr + zt - 1) : 0ull;
    unsigned myh = 0u, myl = 0u;                                 // lane e keeps the words of draw e
    u32 ch = 0;
#pragma unroll 4
    for (int e = 0; e < UNI_E; e++) {
        const u64 x = xsl_rr(s);
        s = add128(mul128(s, AT), CT);
        bool hi, lo;
        if (ZU) {
            hi = hv && x * qh >= th;
            lo = lv && x * ql >= tl;
        } else {
            const u32 r = (u32)tile * UNI_TILE + e * RNG_T + t;
            const int z = (int)(r >> U.log_n);
            hi = z <= L + 1 && x * s_q[z] >= s_t[z];
            lo = z >= 1 && z <= L + 2 && x * s_q[z - 1] >= s_t[z - 1];
        }
        const unsigned bh = __ballot_sync(0xffffffffu, hi), bl = __ballot_sync(0xffffffffu, lo);
        ch += __popc(bh);
        if (lane == (u32)e) {
            myh = bh;
            myl = bl;
        }
    }
    // word of draw e (positions e*RNG_T + warp*32 ...) = tile word e*RNG_W + warp
    unsigned* hib = U.hib + (size_t)k * (U.WU / 32) + (size_t)tile * UNI_TW;
    unsigned* lob = U.lob + (size_t)k * (U.WU / 32) + (size_t)tile * UNI_TW;
    hib[lane * RNG_W + warp] = myh;
    lob[lane * RNG_W + warp] = myl;
    if (lane == 0) s_h[warp] = ch;
    __syncthreads();
    if (t == 0) {
        u32 a = 0;
        for (int w = 0; w < RNG_W; w++) a += s_h[w];
        U.chi[(size_t)k * U.NTU + tile] = a;
    }
}

// Set bits of bm in positions [a, b) (one warp; all lanes get the sum).
HS_DEV u32 warp_count_words(const unsigned* bm, u32 a, u32 b, u32 lane) {
    u32 c = 0;
    if (a < b) {
        for (u32 w = (a >> 5) + lane; w <= ((b - 1) >> 5); w += 32) {
            unsigned x = bm[w];
            const u32 base = w << 5;
            if (base < a) x &= ~((1u << (a - base)) - 1u);
            if (b - base < 32u) x &= (1u << (b - base)) - 1u;
            c += __popc(x);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    return c;
}

// Set bits in [a, b): whole tiles from the per-tile counts, the rest by words.
HS_DEV u32 warp_count_range(const unsigned* bm, const u32* tc, u32 a, u32 b, u32 lane) {
    const u32 t0 = (a + UNI_TILE - 1) / UNI_TILE, t1 = b / UNI_TILE;
    if (t0 >= t1) return warp_count_words(bm, a, b, lane);
    u32 c = 0;
    for (u32 tt = t0 + lane; tt < t1; tt += 32) c += tc[tt];
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    return c + warp_count_words(bm, a, t0 * UNI_TILE, lane) + warp_count_words(bm, t1 * UNI_TILE, b, lane);
}

// Position of the need-th (1-based) set bit at or after `from` (< limit), or
// limit if there is none.  `from` is a word boundary.
HS_DEV u32 warp_select(const unsigned* bm, u32 from, u32 need, u32 limit, u32 lane) {
    for (u32 w0 = from >> 5; (w0 << 5) < limit; w0 += 32) {
        const u32 w = w0 + lane;
        const unsigned x = (w << 5) < limit ? bm[w] : 0u;
        const u32 c = __popc(x);
        u32 inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (u32)o) inc += v;
        }
        const unsigned hit = __ballot_sync(0xffffffffu, inc >= need);
        if (hit) {
            const int f = __ffs(hit) - 1;
            const u32 before = __shfl_sync(0xffffffffu, inc - c, f);
            unsigned xf = __shfl_sync(0xffffffffu, x, f);
            for (u32 r = 1; r < need - before; r++) xf &= xf - 1u;
            return ((w0 + (u32)f) << 5) + (u32)(__ffs(xf) - 1);
        }
        need -= __shfl_sync(0xffffffffu, inc, 31);
    }
    return limit;
}

// Segment starts of one key's digit window.  Fast path (n >= UNI_TILE, so
// tiles align with zones): zone totals of the hi bits come from the per-tile
// counts, and the first 32 words of every zone's hi and lo bitmaps are
// prefetched into shared memory in one parallel pass, so the serial chain
// over the L+2 segments only touches shared memory (segment starts lie within
// 1024 positions of their zone start unless a digit has > 1024 rejections,
// which falls back to the global-memory walk).
constexpr int UB_W = 32;                      // prefetched words per zone
__global__ void __launch_bounds__(32) pk_uni_bounds(ParArgs A, UniArgs U) {
    __shared__ unsigned sh[66][UB_W], sl[66][UB_W];
    __shared__ u32 ztot[66];
    const int k = blockIdx.x;
    const u32 lane = threadIdx.x;
    const int L = A.L;
    const u32 n = A.n;
    const unsigned* hib = U.hib + (size_t)k * (U.WU / 32);
    const unsigned* lob = U.lob + (size_t)k * (U.WU / 32);
    const u32* chi = U.chi + (size_t)k * U.NTU;
    u32* S = U.seg + (size_t)k * (L + 3);
    const bool fast = n >= (u32)UNI_TILE;
    if (fast) {
        // all loads independent: unrolled so many are in flight at once
        const u32 tpz = n / UNI_TILE;                          // tiles per zone
        const int nz = L + 3;
        if (lane < (u32)nz) ztot[lane] = 0u;
        if (lane + 32 < (u32)nz) ztot[lane + 32] = 0u;
        __syncwarp();
#pragma unroll 8
        for (int m = 0; m < nz; m++) {
            const u32 w0 = (u32)m * (n / 32);
            const bool in = (w0 + lane) * 32u < U.WU;
            sh[m][lane] = in ? hib[w0 + lane] : 0u;
            sl[m][lane] = in ? lob[w0 + lane] : 0u;
        }
        for (u32 tt = lane; tt < (u32)nz * tpz && tt < U.NTU; tt += 32) atomicAdd(&ztot[tt / tpz], chi[tt]);
        __syncwarp();
    }
    u32 s = 0;
    bool bad = false;
    if (lane == 0) S[0] = 0;
    for (int m = 0; m <= L + 1 && !bad; m++) {
        const u32 z0 = (u32)m * n, z1 = z0 + n;                // zone m = [z0, z1)
        u32 a1;
        if (fast && s - z0 < UB_W * 32u) {
            // hi bits in [s, z1) = zone total - hi bits in [z0, s)
            const u32 off = s - z0;
            unsigned x = sh[m][lane];
            const u32 b0 = lane * 32u;
            if (off <= b0) x = 0u;
            else if (off - b0 < 32u) x &= (1u << (off - b0)) - 1u;
            u32 c = __popc(x);
#pragma unroll
            for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            a1 = ztot[m] - c;
        } else {
            a1 = warp_count_range(hib, chi, s, z1, lane);
        }
        u32 nx = z1;
        if (a1 < n) {
            const u32 need = n - a1;
            u32 p = U.WU;
            bool found = false;
            if (fast && m + 1 <= L + 2) {
                const unsigned x = sl[m + 1][lane];
                const u32 c = __popc(x);
                u32 inc = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const u32 v = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= (u32)o) inc += v;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, inc >= need);
                if (hit) {
                    const int f = __ffs(hit) - 1;
                    const u32 before = __shfl_sync(0xffffffffu, inc - c, f);
                    unsigned xf = __shfl_sync(0xffffffffu, x, f);
                    for (u32 r = 1; r < need - before; r++) xf &= xf - 1u;
                    p = z1 + (u32)f * 32u + (u32)(__ffs(xf) - 1);
                    found = true;
                }
            }
            if (!found) p = warp_select(lob, z1, need, U.WU, lane);
            nx = p + 1;
            // the next segment must start inside zone m+1 (fewer than n
            // cumulative rejections) and inside the window
            if (p >= U.WU || nx - z1 >= n) bad = true;
        }
        s = nx;
        if (lane == 0) S[m + 1] = s;
    }
    if (lane == 0) {
        if (bad) {
            *A.err = 1;
            A.pos_out[k] = A.pos_in[k];
        } else {
            A.pos_out[k] = A.pos_in[k] + s;
        }
    }
}

__global__ void __launch_bounds__(RNG_T) pk_uni_emit(ParArgs A, UniArgs U, int digit, u32 seq) {
    __shared__ unsigned s_eff[UNI_TW];
    __shared__ u32 s_pre[UNI_TW];
    __shared__ u32 s_wsum[RNG_W];
    __shared__ u32 s_prefix;
    __shared__ u32 s_seg[66];
    const int k = blockIdx.y, tile = blockIdx.x;
    const u32 t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int L = A.L;
    const u32 n = A.n;
    unsigned long long* fl = U.flags + (size_t)k * U.NTU;
    for (int m = t; m <= L + 2; m += RNG_T) s_seg[m] = U.seg[(size_t)k * (L + 3) + m];
    __syncthreads();
    const u32 end = s_seg[L + 2];
    const u32 base = (u32)tile * UNI_TILE;
    if (base >= end) {
        if (t == 0) publish(fl + tile, seq, 0u);
        return;
    }
    // ---- effective accept bits of this tile (one word per thread: UNI_TW == RNG_T)
    {
        const u32 w = t;
        const u32 p0 = base + 32u * w;                         // first position of the word
        const int z = (int)(p0 >> U.log_n);                    // one zone per word (n >= 64)
        const size_t gw = (size_t)k * (U.WU / 32) + (size_t)tile * UNI_TW + w;
        const unsigned hi = U.hib[gw], lo = U.lob[gw];
        const u32 sz = z <= L + 1 ? s_seg[z] : end;            // positions >= sz are in segment z
        unsigned m_hi;                                          // word bits at positions >= sz
        if (sz <= p0) m_hi = 0xffffffffu;
        else if (sz >= p0 + 32u) m_hi = 0u;
        else m_hi = ~((1u << (sz - p0)) - 1u);
        unsigned e = (z <= L + 1 ? (hi & m_hi) : 0u) | (z >= 1 ? (lo & ~m_hi) : 0u);
        if (p0 >= end) e = 0u;
        else if (end - p0 < 32u) e &= (1u << (end - p0)) - 1u;
        s_eff[w] = e;
        // exclusive scan of word popcounts over the tile
        const u32 c = __popc(e);
        u32 inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (u32)o) inc += v;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        u32 before = 0;
        for (u32 j = 0; j < warp; j++) before += s_wsum[j];
        s_pre[w] = before + inc - c;
        if (t == RNG_T - 1) {
            publish(fl + tile, seq, before + inc);
        }
    }
    if (warp == 0) {
        const u32 p = look_back(fl, tile, seq);
        if (lane == 0) s_prefix = p;
    }
    __syncthreads();
    const u32 prefix = s_prefix;
    const u32 lim = (u32)(L + 2) * n;
    u64* dst = A.a_out[k] + (size_t)digit * (L + 2) * n;
    const KeyStream ks = A.streams[k];
    const U128 inc{ks.inc_hi, ks.inc_lo};
    U128 s = uni_thread_state(A, U, k, tile, inc);
    const U128 AT = A.jump->A[RNG_T], CT = mul128(A.jump->S[RNG_T], inc);
    // candidate moduli of the tile's zone (exact when the tile lies in one zone)
    const int zt = (int)(base >> U.log_n);
    const bool one_zone = ((base + UNI_TILE - 1) >> U.log_n) == (u32)zt;
    const u64 qh = zt <= L + 1 ? __ldg(&A.pc[zt].q) : 0ull, ql = zt >= 1 ? __ldg(&A.pc[zt - 1].q) : 0ull;
    const u32 szt = zt <= L + 1 ? s_seg[zt] : end;
#pragma unroll 4
    for (int e = 0; e < UNI_E; e++) {
        const u64 x = xsl_rr(s);
        s = add128(mul128(s, AT), CT);
        const u32 w = e * RNG_W + warp;
        const unsigned eb = s_eff[w];
        if (!((eb >> lane) & 1u)) continue;
        const u32 r = base + e * RNG_T + t;
        u64 q;
        if (one_zone) {
            q = r >= szt ? qh : ql;
        } else {
            const int z = (int)(r >> U.log_n);
            q = __ldg(&A.pc[(z <= L + 1 && r >= s_seg[z]) ? z : z - 1].q);
        }
        const u32 idx = prefix + s_pre[w] + __popc(eb & lt);
        if (idx < lim) dst[idx] = __umul64hi(x, q);
    }
}

static u32 uni_window(u32 n, int L) {
    const size_t w = (size_t)(L + 2) * n + std::max<size_t>(n / 2, 4096);
    return (u32)((w + UNI_TILE - 1) / UNI_TILE * UNI_TILE);      // <= 1024 tiles (L <= 62, n <= 2^17)
}

static size_t uni_scratch_bytes(int K, u32 n, int L) {
    const size_t WU = uni_window(n, L), NTU = WU / UNI_TILE;
    return (size_t)K * (WU / 32 * 4 * 2 + NTU * 4 + (size_t)(L + 3) * 4 + 16 + NTU * 8) + 512;
}

size_t keygen_par_window(u32 n) {
    const size_t w = (size_t)n + n / 16 + 8192;
    return (w + RNG_CH - 1) / RNG_CH * RNG_CH;
}

static size_t keygen_par_scratch_core(int K, u32 n) {
    const size_t W = keygen_par_window(n), NT = W / RNG_CH;
    return (size_t)K * (W * 8 + W * 8 + W * 4 + W / 32 * 4 * 2 + NT * 4 + NT * 8) + (size_t)K * 16;
}

// flags [K][L+2][NT] and start words [K][L+2] of the persistent uniform kernel
// (L+2 <= 64 primes bounds the size; the layout only needs K, n and L).
static size_t keygen_persist_scratch(int K, u32 n) {
    const size_t W = keygen_par_window(n), NT = W / RNG_CH;
    return (size_t)K * 64 * (NT + 1) * 8;
}

size_t keygen_par_scratch_bytes(int K, u32 n, int L) {
    return keygen_par_scratch_core(K, n) + keygen_persist_scratch(K, n) + uni_scratch_bytes(K, n, L) + 256;
}

// Replays K key streams in lockstep.  Returns false (nothing guaranteed) if
// a window overflowed; the caller then falls back to the serial kernel.
void keygen_streams_parallel(const Dev& d, int K, const void* streams, u64* const* a_out,
                             long long* e_out, const void* jump, const void* zig, const u64* thr,
                             void* scratch, int* err, cudaStream_t st) {
    const int W = (int)keygen_par_window(d.n), NT = W / RNG_CH;
    char* p = (char*)scratch;
    ParArgs A{};
    A.streams = (const KeyStream*)streams;
    A.jump = (const RngJump*)jump;
    A.zig = (const ZigTables*)zig;
    A.pc = d.pc;
    A.thr = thr;
    A.raw = (u64*)p;
    p += (size_t)K * W * 8;
    A.tailx = (double*)p;
    p += (size_t)K * W * 8;
    A.tlen = (u32*)p;
    p += (size_t)K * W * 4;
    A.fastb = (unsigned*)p;
    p += (size_t)K * (W / 32) * 4;
    A.emitb = (unsigned*)p;
    p += (size_t)K * (W / 32) * 4;
    A.cnt = (u32*)p;
    p += (size_t)K * NT * 4;
    p = (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);     // K * NT may be odd
    u64* pos[2] = {(u64*)p, (u64*)p + K};
    p += (size_t)2 * K * 8;
    unsigned long long* flags = (unsigned long long*)p;     // [K][NT] look-back flags
    cudaMemsetAsync(flags, 0, (size_t)K * NT * 8, st);
    p += (size_t)K * NT * 8;
    const int nseg = d.L + 2;
    unsigned long long* pflags = (unsigned long long*)p;    // [K][L+2][NT] persistent look-back
    p += (size_t)K * nseg * NT * 8;
    unsigned long long* segpos = (unsigned long long*)p;    // [K][L+2] published segment starts
    cudaMemsetAsync(pflags, 0, (size_t)K * nseg * (NT + 1) * 8, st);
    p += keygen_persist_scratch(K, d.n) - (size_t)K * nseg * NT * 8;
    p = (char*)(((uintptr_t)p + 255) & ~(uintptr_t)255);
    // digit-window uniform path (HS_KEYGEN_PERSIST=1: the persistent chain, A/B)
    static const bool persist_only = getenv("HS_KEYGEN_PERSIST") != nullptr;
    const bool uni = !persist_only && d.n >= 64 && uni_window(d.n, d.L) / UNI_TILE <= 1024;
    UniArgs U{};
    U.WU = uni_window(d.n, d.L);
    U.NTU = U.WU / UNI_TILE;
    U.log_n = d.log_n;
    U.hib = (unsigned*)p;
    p += (size_t)K * (U.WU / 32) * 4;
    U.lob = (unsigned*)p;
    p += (size_t)K * (U.WU / 32) * 4;
    U.chi = (u32*)p;
    p += (size_t)K * U.NTU * 4;
    U.seg = (u32*)p;
    p += (size_t)K * (d.L + 3) * 4;
    p = (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    U.s0 = (U128*)p;
    p += (size_t)K * sizeof(U128);
    U.flags = (unsigned long long*)p;
    if (uni) cudaMemsetAsync(U.flags, 0, (size_t)K * U.NTU * 8, st);
    u32 seq = 0;
    // keys per cooperative launch of the persistent uniform kernel (all its
    // CTAs must be co-resident); 0 = use one launch per segment
    static int coresident = -1;          // CTAs of pk_uniform_persist that fit at once
    if (coresident < 0) {
        int dev = 0, nsm = 0, per = 0, coop = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pk_uniform_persist, RNG_T, 0);
        coresident = (coop && !getenv("HS_KEYGEN_NO_PERSIST")) ? per * nsm : 0;
    }
    const int kgroup = coresident / NT;
    u32 useq = 0;
    cudaMemsetAsync(pos[0], 0, (size_t)K * sizeof(u64), st);
    A.a_out = a_out;
    A.e_out = e_out;
    A.err = err;
    A.L = d.L;
    A.W = W;
    A.NT = NT;
    A.n = d.n;
    int cur = 0;
    const dim3 grid(NT, K);
    const size_t walk_smem = (size_t)5 * (W / 32) * sizeof(unsigned);
    cudaFuncSetAttribute(pk_normal_walk2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)walk_smem);
    for (int digit = 0; digit <= d.L; digit++) {
        if (uni) {
            A.pos_in = pos[cur];
            A.pos_out = pos[cur ^ 1];
            const dim3 gu(U.NTU, K);
            pk_uni_start<<<K, 32, 0, st>>>(A, U);
            if (d.n >= (u32)UNI_TILE) pk_uni_flags<true><<<gu, RNG_T, 0, st>>>(A, U);
            else pk_uni_flags<false><<<gu, RNG_T, 0, st>>>(A, U);
            pk_uni_bounds<<<K, 32, 0, st>>>(A, U);
            pk_uni_emit<<<gu, RNG_T, 0, st>>>(A, U, digit, ++useq);
            note_launch(4);
            cur ^= 1;
        } else if (kgroup > 0) {
            A.pos_in = pos[cur];
            A.pos_out = pos[cur ^ 1];
            const u32 seq0 = seq + 1;
            for (int k0 = 0; k0 < K; k0 += kgroup) {
                const int kc = std::min(kgroup, K - k0);
                int dg = digit, kb = k0;
                u32 s0 = seq0;
                void* args[] = {&A, &dg, &kb, &pflags, &segpos, &s0};
                cudaLaunchCooperativeKernel((void*)pk_uniform_persist, dim3(NT, kc), dim3(RNG_T), args, 0, st);
                note_launch();
            }
            seq += d.L + 2;
            cur ^= 1;
        } else {
            for (int m = 0; m < d.L + 2; m++) {
                A.pos_in = pos[cur];
                A.pos_out = pos[cur ^ 1];
                pk_uniform_fused<<<grid, RNG_T, 0, st>>>(A, digit, m, flags, ++seq);
                note_launch();
                cur ^= 1;
            }
        }
        A.pos_in = pos[cur];
        A.pos_out = pos[cur ^ 1];
        pk_gen_kernel<<<grid, RNG_T, 0, st>>>(A, 1, 0);
        pk_normal_walk2<<<K, NW_T, walk_smem, st>>>(A);
        pk_normal_write<<<grid, RNG_T, 0, st>>>(A, digit);
        note_launch(3);
        cur ^= 1;
    }
}

void ksk_galois_combine(const Dev& d, int K, u64* const* keys, const u32* gal, const u64* sk,
                        const ulonglong2* f, cudaStream_t st) {
    dim3 g((d.n + 255) / 256, (d.L + 1) * (d.L + 2), K);
    ksk_galois_kernel<<<g, 256, 0, st>>>(d, keys, gal, sk, f);
    note_launch();
}

// b half of each key: b[i][m] = e_i mod q_m (signed coefficients)
__global__ void e_to_limbs_kernel(Dev d, const long long* e, u64* const* keys) {
    const u32 n = d.n;
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int m = blockIdx.y % (d.L + 2), i = blockIdx.y / (d.L + 2), kk = blockIdx.z;
    const PrimeConst P = d.pc[m];
    const long long c = e[((size_t)kk * (d.L + 1) + i) * n + j];
    u64 r;
    if (c >= 0) {
        r = reduce64((u64)c, P);
    } else {
        const u64 tt = reduce64((u64)(-(c + 1)) + 1ull, P);
        r = tt ? P.q - tt : 0ull;
    }
    keys[kk][((size_t)i * (d.L + 2) + m) * n + j] = r;
}

__global__ void mont_keys_kernel(Dev d, u64* const* keys) {
    const u32 n = d.n;
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int limb = blockIdx.y, m = limb % (d.L + 2);
    const PrimeConst P = d.pc[m];
    u64* p = keys[blockIdx.z] + (size_t)limb * n + j;
    *p = mont_mul(*p, P.r2_mod, P.q, P.qinv_neg);
}

// Forward NTT over the b halves of a key list (limb jb of key jb / per).
struct JobKeyB {
    u64* const* keys;
    int per, L;
    u32 n;
    struct Ctx {
        u64* limb;
        int p;
    };
    HS_DEV Ctx make(int jb) const {
        return Ctx{keys[jb / per] + (size_t)(jb % per) * n, (jb % per) % (L + 2)};
    }
    HS_DEV int prime(const Ctx& c) const { return c.p; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst&) const { return c.limb[j]; }
    HS_DEV u64* scratch(const Ctx& c) const { return c.limb; }
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        c.limb[j] = csub(csub(v, P.two_q), P.q);
    }
};

// Fully fused key assembly: one forward NTT per (key, digit i, modulus m)
// whose loader reduces e_i mod q_m and whose epilogue forms
//   b = NTT(e_i) + [m<=L] f_im sk(X^g)_m - a_im sk_m
// (keys are kept in standard form; a is left as drawn).
struct JobKeyFused {
    u64* const* keys;
    const long long* e;          // [K][L+1][n]
    const u32* gal;
    const u64* sk;               // [L+2][n] then Shoup companions [L+2][n]
    const u64* skp;              // [K][L+1][n] sk(X^g) per key (NTT-domain automorphism)
    const ulonglong2* f;         // [(L+1)^2]
    int per, L;
    Dev d;
    struct Ctx {
        u64* b;
        u64* a;
        const long long* e;
        const u64* skm;
        const u64* skpm;
        ulonglong2 f;
        int m;
    };
    HS_DEV Ctx make(int jb) const {
        // job order (key, modulus, digit): sk_m, its companion and sk(X^g)_m
        // stay in L2 across the L+1 digits, e_i across the moduli of a key
        const int kk = jb / per, r = jb % per;
        const int m = r / (L + 1), i = r % (L + 1);
        const int limb = i * (L + 2) + m;
        u64* key = keys[kk];
        const size_t half = (size_t)per * d.n;
        return Ctx{key + (size_t)limb * d.n, key + half + (size_t)limb * d.n,
                   e + ((size_t)kk * (L + 1) + i) * d.n, sk + (size_t)m * d.n,
                   skp + ((size_t)kk * (L + 1) + (m <= L ? m : 0)) * d.n,
                   m <= L ? f[i * (L + 1) + m] : make_ulonglong2(0, 0), m};
    }
    HS_DEV int prime(const Ctx& c) const { return c.m; }
    HS_DEV u64 load(const Ctx& c, u32 j, const PrimeConst& P) const {
        const long long v = __ldg(c.e + j);
        const bool neg = v < 0;                               // |v| mod q, then negate: one path
        u64 t = neg ? (u64)(-(v + 1)) + 1ull : (u64)v;
        // e = rint(3.2 x) of a ziggurat normal: |e| < 64 << q in practice
        // (the tail's x stays below ~14); the reduction is a never-taken branch
        if (t >= P.q) t = reduce64(t, P);
        return (neg && t) ? P.q - t : t;
    }
    HS_DEV u64* scratch(const Ctx& c) const { return c.b; }
    // b = NTT(e) + f sk(X^g) - a sk, with f = p (Q_L / q_i) mod q_m nonzero only
    // for m == i (a warp-uniform branch), reduced once at the end:
    // v in [0, 4q), a sk in [0, 2q) -> v + 2q - a sk in (0, 6q), + f sk' < 8q
    HS_DEV void store(const Ctx& c, u32 j, u64 v, const PrimeConst& P) const {
        const u64 ask = shoup_lazy(__ldg(c.a + j), __ldg(c.skm + j), __ldg(c.skm + (size_t)(L + 2) * d.n + j), P.q);
        u64 r = v + P.two_q - ask;
        if (c.f.x) r += shoup_lazy(__ldg(c.skpm + j), c.f.x, c.f.y, P.q);
        r = csub(r, P.two_q << 1);
        r = csub(r, P.two_q);
        c.b[j] = csub(r, P.q);
    }
};

__global__ void shoup_companion_kernel(Dev d, const u64* v, u64* sh) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d.n) return;
    const int m = blockIdx.y;
    const size_t o = (size_t)m * d.n + j;
    sh[o] = (u64)(((unsigned __int128)v[o] << 64) / d.pc[m].q);
}

// sh[m][j] = floor(v[m][j] 2^64 / q_m) for nl limbs of moduli 0..nl-1.
void shoup_companions(const Dev& d, const u64* v, u64* sh, int nl, cudaStream_t st) {
    shoup_companion_kernel<<<dim3((d.n + 255) / 256, nl), 256, 0, st>>>(d, v, sh);
    note_launch();
}

// skp[k][m][j] = sk[m][perm_g(j)]: the automorphism of the secret for key k,
// gathered once per (key, modulus) instead of once per key limb.
__global__ void sk_perm_kernel(Dev d, const u32* gal, const u64* sk, u64* skp) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d.n) return;
    const int m = blockIdx.y, k = blockIdx.z;
    const u32 br = __brev(j) >> (32 - d.log_n);
    const u32 ex = (u32)((((u64)(2 * br + 1)) * gal[k]) & ((2ull << d.log_n) - 1));
    const u32 pj = __brev((ex - 1) >> 1) >> (32 - d.log_n);
    skp[((size_t)k * (d.L + 1) + m) * d.n + j] = sk[(size_t)m * d.n + pj];
}

size_t keygen_assemble_scratch_bytes(int K, const Dev& d) { return (size_t)K * (d.L + 1) * d.n * sizeof(u64); }

void keygen_assemble(const Dev& d, int K, u64* const* keys, const long long* e, const u32* gal,
                     const u64* sk, const ulonglong2* f, u64* skp, cudaStream_t st) {
    const int per = (d.L + 1) * (d.L + 2);
    sk_perm_kernel<<<dim3((d.n + 255) / 256, d.L + 1, K), 256, 0, st>>>(d, gal, sk, skp);
    note_launch();
    launch_ntt<true>(d, JobKeyFused{keys, e, gal, sk, skp, f, per, d.L, d}, K * per, st);
}

size_t rng_jump_bytes() { return sizeof(RngJump); }
size_t zig_tables_bytes() { return sizeof(ZigTables); }

}  // namespace hs

// ====================================================================== host

using namespace hs;
typedef unsigned __int128 u128h;

namespace {

const u128h PCG_MULT = ((u128h)2549297995355413924ULL << 64) + 4865540595714422341ULL;

hs_status ensure_keygen_tables(hs_ctx* c) {
    if (c->d_jump) return HS_OK;
    const int L = c->L;
    RngJump* J = new RngJump();
    u128h a = 1, s = 0;
    for (int t = 0; t <= RNG_CH; t++) {
        J->A[t] = U128{(u64)(a >> 64), (u64)a};
        J->S[t] = U128{(u64)(s >> 64), (u64)s};
        s += a;
        a *= PCG_MULT;
    }
    {   // power-of-two jumps: (A,S)_{2^(j+1)} = (A^2, S + A S)
        u128h pa = PCG_MULT, ps = 1;
        for (int j = 0; j < 64; j++) {
            J->PA[j] = U128{(u64)(pa >> 64), (u64)pa};
            J->PS[j] = U128{(u64)(ps >> 64), (u64)ps};
            ps = ps + pa * ps;
            pa = pa * pa;
        }
    }
    {   // digit-window tile jumps: (TA, TS)_{t+1} = (TA_t A_U, TS_t + TA_t S_U), U = UNI_TILE = 2^14
        static_assert(UNI_TILE == 1 << 14, "UNI_TILE is a power of two");
        const u128h au = ((u128h)J->PA[14].hi << 64) | J->PA[14].lo;
        const u128h su = ((u128h)J->PS[14].hi << 64) | J->PS[14].lo;
        u128h ta = 1, ts = 0;
        for (int t = 0; t < 1024; t++) {
            J->TA[t] = U128{(u64)(ta >> 64), (u64)ta};
            J->TS[t] = U128{(u64)(ts >> 64), (u64)ts};
            ts = ts + ta * su;
            ta = ta * au;
        }
    }
    std::vector<u64> thr(L + 2);
    for (int p = 0; p < L + 2; p++) {
        const u64 q = c->primes[p];
        thr[p] = (u64)((((u128h)1 << 64) - q) % q);
    }
    std::vector<ulonglong2> f((size_t)(L + 1) * (L + 1));
    for (int i = 0; i <= L; i++)
        for (int m = 0; m <= L; m++) {
            const u64 qm = c->primes[m];
            u64 v = c->primes[L + 1] % qm;
            for (int j = 0; j <= L; j++)
                if (j != i) v = (u64)((u128h)v * (c->primes[j] % qm) % qm);
            f[(size_t)i * (L + 1) + m] = make_ulonglong2(v, (u64)(((u128h)v << 64) / qm));
        }
    cudaError_t e = cudaMalloc(&c->d_jump, sizeof(RngJump));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_jump, J, sizeof(RngJump), cudaMemcpyHostToDevice);
    delete J;
    if (e == cudaSuccess) e = cudaMalloc((void**)&c->d_thr, thr.size() * sizeof(u64));
    if (e == cudaSuccess) e = cudaMemcpy(c->d_thr, thr.data(), thr.size() * sizeof(u64), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc((void**)&c->d_kskf, f.size() * sizeof(ulonglong2));
    if (e == cudaSuccess)
        e = cudaMemcpy(c->d_kskf, f.data(), f.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        set_error(std::string("keygen tables: ") + cudaGetErrorString(e));
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}

u64 powmod_u(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = (u64)((u128h)r * b % q);
        b = (u64)((u128h)b * b % q);
        e >>= 1;
    }
    return r;
}

}  // namespace

namespace hs {

hs_status keygen_check(hs_ctx* c) {
    if (!c->d_kg_err) return HS_OK;
    int err = 0;
    HS_CUDA(cudaMemcpy(&err, c->d_kg_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
        cudaMemset(c->d_kg_err, 0, sizeof(int));
        set_error("device key stream exceeded its window (rerun with HS_KEYGEN_SERIAL=1)");
        return HS_EVAL_ERROR;
    }
    return HS_OK;
}

// Generate keys for `steps` (PCG64 start states `streams`) into `dests`
// (each a [2][L+1][L+2][n] buffer).  Used eagerly (hs_key_generate_galois)
// and lazily by the runner for keys it was told how to make.
hs_status generate_galois_keys(hs_ctx* c, const std::vector<u32>& steps,
                               const std::vector<hs_ctx::Stream>& streams,
                               const std::vector<u64*>& dests, cudaStream_t st) {
    if (!c->d_zig || !c->d_sk) {
        set_error("device key generation needs hs_keygen_set_tables and hs_keygen_set_secret");
        return HS_PARAMETER_ERROR;
    }
    hs_status s = ensure_keygen_tables(c);
    if (s != HS_OK) return s;
    const int L = c->L;
    const u32 n = c->n;
    const size_t half = (size_t)(L + 1) * (L + 2) * n;
    static const long kb_env = getenv("HS_KEYGEN_BATCH") ? atol(getenv("HS_KEYGEN_BATCH")) : 0;
    const int KB = (int)std::max<size_t>(1, kb_env > 0 ? (size_t)kb_env : c->keygen_batch);
    long long* e = nullptr;
    u64** d_keys = nullptr;
    u64** d_aout = nullptr;
    u32* d_gal = nullptr;
    hs_ctx::Stream* d_streams = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&e, (size_t)KB * (L + 1) * n * sizeof(long long), st));
    HS_CUDA(cudaMallocAsync((void**)&d_keys, KB * sizeof(u64*), st));
    HS_CUDA(cudaMallocAsync((void**)&d_aout, KB * sizeof(u64*), st));
    HS_CUDA(cudaMallocAsync((void**)&d_gal, KB * sizeof(u32), st));
    HS_CUDA(cudaMallocAsync((void**)&d_streams, KB * sizeof(hs_ctx::Stream), st));
    u64* skp = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&skp, keygen_assemble_scratch_bytes(KB, c->dev), st));
    static const bool serial = getenv("HS_KEYGEN_SERIAL") != nullptr;
    void* par_scratch = nullptr;
    if (!serial) {
        if (!c->d_kg_err) {
            HS_CUDA(cudaMalloc((void**)&c->d_kg_err, sizeof(int)));
            HS_CUDA(cudaMemset(c->d_kg_err, 0, sizeof(int)));
        }
        // room for KG_LANES sub-chunk slices, each 256-byte aligned
        HS_CUDA(cudaMallocAsync(&par_scratch, keygen_par_scratch_bytes(KB, c->n, c->L) + hs_ctx::KG_LANES * 512, st));
    }
    // in-step timer (bench.py): the whole generation of these keys on its stream;
    // bytes = the keys written, work = keys
    ProbeScope probe(PROBE_KEYGEN, st, (double)steps.size() * c->key_bytes(), (double)steps.size());
    for (size_t k0 = 0; k0 < steps.size(); k0 += KB) {
        const int K = (int)std::min<size_t>(KB, steps.size() - k0);
        std::vector<u64*> keys(K), aout(K);
        std::vector<u32> gal(K);
        for (int k = 0; k < K; k++) {
            keys[k] = dests[k0 + k];
            aout[k] = dests[k0 + k] + half;
            gal[k] = (u32)powmod_u(5, steps[k0 + k], 2ull * n);
        }
        HS_CUDA(cudaMemcpyAsync(d_keys, keys.data(), K * sizeof(u64*), cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(d_aout, aout.data(), K * sizeof(u64*), cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(d_gal, gal.data(), K * sizeof(u32), cudaMemcpyHostToDevice, st));
        HS_CUDA(cudaMemcpyAsync(d_streams, streams.data() + k0, K * sizeof(hs_ctx::Stream),
                                cudaMemcpyHostToDevice, st));
        if (par_scratch) {
            // split the chunk over concurrent chains: each chain's launches are
            // latency-bound (small grids, serial segment chain), so chains overlap
            static const int lanes_env = getenv("HS_KEYGEN_LANES") ? atoi(getenv("HS_KEYGEN_LANES")) : 0;
            const int lanes = lanes_env > 0 ? std::min(lanes_env, (int)hs_ctx::KG_LANES) : 1;   // A/B: 1 lane fastest at K=12..23
            const int S = std::min(K, lanes);
            if (!c->kg_stream[0]) {
                for (int j = 0; j < hs_ctx::KG_LANES; j++)
                    HS_CUDA(cudaStreamCreateWithFlags(&c->kg_stream[j], cudaStreamNonBlocking));
                for (int j = 0; j <= hs_ctx::KG_LANES; j++)
                    HS_CUDA(cudaEventCreateWithFlags(&c->kg_event[j], cudaEventDisableTiming));
            }
            HS_CUDA(cudaEventRecord(c->kg_event[hs_ctx::KG_LANES], st));
            size_t soff = 0;
            for (int j = 0; j < S; j++) {
                const int ka = K * j / S, kc = K * (j + 1) / S - ka;
                cudaStream_t sj = c->kg_stream[j];
                HS_CUDA(cudaStreamWaitEvent(sj, c->kg_event[hs_ctx::KG_LANES], 0));
                keygen_streams_parallel(c->dev, kc, d_streams + ka, d_aout + ka, e + (size_t)ka * (L + 1) * n,
                                        c->d_jump, c->d_zig, c->d_thr, (char*)par_scratch + soff,
                                        c->d_kg_err, sj);
                soff += (keygen_par_scratch_bytes(kc, c->n, c->L) + 255) & ~(size_t)255;
                keygen_assemble(c->dev, kc, d_keys + ka, e + (size_t)ka * (L + 1) * n, d_gal + ka, c->d_sk,
                                c->d_kskf, skp + (size_t)ka * (L + 1) * n, sj);
                HS_CUDA(cudaEventRecord(c->kg_event[j], sj));
            }
            for (int j = 0; j < S; j++) HS_CUDA(cudaStreamWaitEvent(st, c->kg_event[j], 0));
        } else {
            keygen_streams(c->dev, K, d_streams, d_aout, e, c->d_jump, c->d_zig, c->d_thr, st);
            keygen_assemble(c->dev, K, d_keys, e, d_gal, c->d_sk, c->d_kskf, skp, st);
        }
        // pageable host staging is copied at call time; device arrays are stream-ordered
        c->keys_generated += K;
    }
    if (par_scratch) cudaFreeAsync(par_scratch, st);
    cudaFreeAsync(e, st);
    cudaFreeAsync(d_keys, st);
    cudaFreeAsync(d_aout, st);
    cudaFreeAsync(d_gal, st);
    cudaFreeAsync(d_streams, st);
    cudaFreeAsync(skp, st);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        set_error(std::string("keygen launch failed: ") + cudaGetErrorString(err));
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}

}  // namespace hs

extern "C" {

hs_status hs_keygen_set_tables(hs_ctx* c, const double* wi, const double* fi, const uint64_t* ki) {
    ZigTables z;
    memcpy(z.wi, wi, sizeof(z.wi));
    memcpy(z.fi, fi, sizeof(z.fi));
    memcpy(z.ki, ki, sizeof(z.ki));
    if (!c->d_zig) HS_CUDA(cudaMalloc(&c->d_zig, sizeof(ZigTables)));
    HS_CUDA(cudaMemcpy(c->d_zig, &z, sizeof(z), cudaMemcpyHostToDevice));
    return HS_OK;
}

hs_status hs_keygen_set_secret(hs_ctx* c, const uint64_t* sk_ntt, void* stream) {
    const size_t bytes = (size_t)(c->L + 2) * c->n * sizeof(u64);
    if (!c->d_sk) HS_CUDA(cudaMalloc((void**)&c->d_sk, 2 * bytes));     // values, then Shoup companions
    HS_CUDA(cudaMemcpyAsync(c->d_sk, sk_ntt, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    shoup_companions(c->dev, c->d_sk, c->d_sk + (size_t)(c->L + 2) * c->n, c->L + 2, (cudaStream_t)stream);
    return HS_OK;
}

hs_status hs_keygen_register(hs_ctx* c, const uint32_t* steps, const uint64_t* states, int32_t nsteps) {
    for (int k = 0; k < nsteps; k++) {
        if (steps[k] == 0 || steps[k] >= c->n / 2) {
            set_error("rotation step " + std::to_string(steps[k]) + " out of range");
            return HS_PARAMETER_ERROR;
        }
        c->lazy[steps[k]] = hs_ctx::Stream{states[4 * k], states[4 * k + 1], states[4 * k + 2],
                                           states[4 * k + 3]};
    }
    return HS_OK;
}

hs_status hs_key_generate_galois_impl(hs_ctx* c, const uint32_t* steps, const uint64_t* states,
                                      int32_t nsteps, void* stream);

hs_status hs_key_generate_galois(hs_ctx* c, const uint32_t* steps, const uint64_t* states, int32_t nsteps,
                                 void* stream) {
    hs_status s = hs_key_generate_galois_impl(c, steps, states, nsteps, stream);
    if (s != HS_OK) return s;
    HS_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return keygen_check(c);
}

hs_status hs_key_generate_galois_impl(hs_ctx* c, const uint32_t* steps, const uint64_t* states,
                                      int32_t nsteps, void* stream) {
    std::vector<u32> st(steps, steps + nsteps);
    std::vector<hs_ctx::Stream> ss(nsteps);
    std::vector<u64*> dests(nsteps);
    for (int k = 0; k < nsteps; k++) {
        if (steps[k] == 0 || steps[k] >= c->n / 2) {
            set_error("rotation step " + std::to_string(steps[k]) + " out of range");
            return HS_PARAMETER_ERROR;
        }
        ss[k] = hs_ctx::Stream{states[4 * k], states[4 * k + 1], states[4 * k + 2], states[4 * k + 3]};
        auto it = c->galois.find(steps[k]);
        if (it == c->galois.end()) {
            KeyBuf kb;
            HS_CUDA(cudaMalloc((void**)&kb.d, c->key_bytes()));
            it = c->galois.emplace(steps[k], kb).first;
        }
        dests[k] = it->second.d;
    }
    return generate_galois_keys(c, st, ss, dests, (cudaStream_t)stream);
}

hs_status hs_keygen_streams(hs_ctx* c, const uint64_t* states, int32_t nkeys, uint64_t* a_out,
                            int64_t* e_out, void* stream) {
    if (!c->d_zig) {
        set_error("hs_keygen_set_tables first");
        return HS_PARAMETER_ERROR;
    }
    hs_status s = ensure_keygen_tables(c);
    if (s != HS_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t half = (size_t)(c->L + 1) * (c->L + 2) * c->n;
    std::vector<u64*> aout(nkeys);
    for (int k = 0; k < nkeys; k++) aout[k] = a_out + k * half;
    u64** d_aout = nullptr;
    void* d_streams = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&d_aout, nkeys * sizeof(u64*), st));
    HS_CUDA(cudaMallocAsync(&d_streams, nkeys * 4 * sizeof(u64), st));
    HS_CUDA(cudaMemcpyAsync(d_aout, aout.data(), nkeys * sizeof(u64*), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_streams, states, nkeys * 4 * sizeof(u64), cudaMemcpyHostToDevice, st));
    // the production (grid-parallel) path; the serial replay if a window overflowed
    if (!c->d_kg_err) {
        HS_CUDA(cudaMalloc((void**)&c->d_kg_err, sizeof(int)));
        HS_CUDA(cudaMemset(c->d_kg_err, 0, sizeof(int)));
    }
    void* scratch = nullptr;
    HS_CUDA(cudaMallocAsync(&scratch, keygen_par_scratch_bytes(nkeys, c->n, c->L), st));
    keygen_streams_parallel(c->dev, nkeys, d_streams, d_aout, (long long*)e_out, c->d_jump, c->d_zig,
                            c->d_thr, scratch, c->d_kg_err, st);
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(scratch, st);
    int err = 0;
    HS_CUDA(cudaMemcpy(&err, c->d_kg_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
        HS_CUDA(cudaMemset(c->d_kg_err, 0, sizeof(int)));
        keygen_streams(c->dev, nkeys, d_streams, d_aout, (long long*)e_out, c->d_jump, c->d_zig, c->d_thr, st);
    }
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(d_aout, st);
    cudaFreeAsync(d_streams, st);
    return HS_OK;
}

}  // extern "C"

extern "C" int64_t hs_keys_generated(const hs_ctx* c) { return c->keys_generated; }
