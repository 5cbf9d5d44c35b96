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
// stages H x G x C elements in shared memory: H consecutive "hi" values
// (bits above the range) and C consecutive "lo" columns (bits below it).
// n <= 2^11 runs as one pass (whole limb per CTA); larger limbs run as two
// passes (strided column pass + contiguous row pass), in place in the
// destination buffer.  Values stay lazy between stages: [0,4q) forward
// (Harvey), [0,2q) inverse; Shoup products with precomputed twiddle pairs.
//
// A "Job" functor supplies, per batch entry (blockIdx.y): prime(), the
// first-pass load(), the last-pass store(), and scratch() -- the limb buffer
// used in place between passes.  Fusions (basis lift on load, key-switch /
// rescale epilogues on store) are expressed as Job types in ops.cu.
#pragma once
#include "hs_internal.cuh"

namespace hs {

constexpr int NTT_TILE = 2048;      // elements per CTA tile (16 KiB smem + padding)
constexpr int NTT_EPT = 8;          // elements per thread (radix-8 register rounds)
constexpr int NTT_THREADS = NTT_TILE / NTT_EPT;

// Shared-memory index with one pad word per 8 (keeps the stride-8 accesses of
// the lowest-bit round at the 2-wavefront minimum).
HS_DEV u32 spad(u32 i) { return i + (i >> 3); }

// One register round: local stages [A, A+R) of a tile with H rows, G = 2^LOGG
// group elements and C columns.  A "unit" is the 2^R elements that differ in
// the round's bits (smem stride S = 2^LOWB * C); each thread owns 8 / 2^R
// units.  The round schedule (ntt_rounds_*) keeps LOWB = 0 or LOWB >= 3, so
// the padded smem index of a unit's elements is affine: base + e * PS.
template <bool FWD, bool LZ, int LOGG, int H, int C, int A, int R>
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
        if (FWD) {
#pragma unroll
            for (int j = 0; j < R; j++) {
                const int ls = A + j;
                const ulonglong2* __restrict__ twb = tw + ((1u << (s0 + ls)) + (hi << ls) + (go_high << j));
#pragma unroll
                for (int e = 0; e < NU; e++) {
                    const int bit = 1 << (R - 1 - j);
                    if (e & bit) continue;
                    const ulonglong2 w = twb[e >> (R - j)];
                    const u64 x = LZ ? v[e] : csub(v[e], two_q);
                    const u64 t = shoup_lazy(v[e + bit], w.x, w.y, q);
                    v[e] = x + t;
                    v[e + bit] = x - t + two_q;
                }
            }
        } else {
#pragma unroll
            for (int j = R - 1; j >= 0; j--) {
                const int ls = A + j;
                const ulonglong2* __restrict__ twb = tw + ((1u << (s0 + ls)) + (hi << ls) + (go_high << j));
#pragma unroll
                for (int e = 0; e < NU; e++) {
                    const int bit = 1 << (R - 1 - j);
                    if (e & bit) continue;
                    const ulonglong2 w = twb[e >> (R - j)];
                    const u64 x = v[e], y = v[e + bit];
                    v[e] = csub(x + y, two_q);
                    v[e + bit] = shoup_lazy(x - y + two_q, w.x, w.y, q);
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
    // start stage and width of round number r (0-based, forward order)
    static constexpr int count() { return F + (REM ? 1 : 0); }
    static constexpr int start(int r) {
        return REM == 0 ? 3 * r : (r < F - 1 ? 3 * r : (r == F - 1 ? 3 * (F - 1) : LOGG - 3));
    }
    static constexpr int width(int r) { return REM == 0 ? 3 : (r == F - 1 ? REM : 3); }
};

template <int LOGG, int H, int C, bool LZ, int RI>
__device__ __forceinline__ void ntt_rounds_fwd_from(u64* sm, const ulonglong2* tw, u32 hi0, int s0,
                                                    u64 q, u64 two_q) {
    if constexpr (RI < RoundPlan<LOGG>::count()) {
        ntt_round<true, LZ, LOGG, H, C, RoundPlan<LOGG>::start(RI), RoundPlan<LOGG>::width(RI)>(
            sm, tw, hi0, s0, q, two_q);
        __syncthreads();
        ntt_rounds_fwd_from<LOGG, H, C, LZ, RI + 1>(sm, tw, hi0, s0, q, two_q);
    }
}

template <int LOGG, int H, int C, int RI>
__device__ __forceinline__ void ntt_rounds_inv_from(u64* sm, const ulonglong2* tw, u32 hi0, int s0,
                                                    u64 q, u64 two_q) {
    if constexpr (RI >= 0) {
        ntt_round<false, false, LOGG, H, C, RoundPlan<LOGG>::start(RI), RoundPlan<LOGG>::width(RI)>(
            sm, tw, hi0, s0, q, two_q);
        __syncthreads();
        ntt_rounds_inv_from<LOGG, H, C, RI - 1>(sm, tw, hi0, s0, q, two_q);
    }
}

// LZ: skip the per-butterfly reduction of the upper input (values grow by
// < 2q per stage; only for primes with fwd_lazy_ok()).
template <int LOGG, int H, int C, bool LZ = false>
__device__ __forceinline__ void ntt_rounds_fwd(u64* sm, const ulonglong2* tw, u32 hi0, int s0, u64 q,
                                               u64 two_q) {
    ntt_rounds_fwd_from<LOGG, H, C, LZ, 0>(sm, tw, hi0, s0, q, two_q);
}

// Forward passes may run fully lazy when every intermediate stays below
// 2^64: inputs < 4q, each of <= 17 stages adds < 2q, so < 38q < 2^64 for
// q < 2^58 (the ~50-bit chain primes; the 60-bit q_0 and aux keep Harvey's
// per-butterfly reduction).  Lazy outputs are brought to [0, 2q) with
// reduce64_lazy before a job's store() sees them.
HS_DEV bool fwd_lazy_ok(const PrimeConst& P) { return P.q < (1ull << 58); }
HS_DEV u64 reduce64_lazy(u64 t, const PrimeConst& P) { return t - mulhi64(t, P.m64) * P.q; }

template <int LOGG, int H, int C>
__device__ __forceinline__ void ntt_rounds_inv(u64* sm, const ulonglong2* tw, u32 hi0, int s0, u64 q,
                                               u64 two_q) {
    ntt_rounds_inv_from<LOGG, H, C, RoundPlan<LOGG>::count() - 1>(sm, tw, hi0, s0, q, two_q);
}

// Job interface: `typename Job::Ctx ctx = job.make(jb)` is evaluated once per
// CTA (pointer-table lookups, index decoding), then prime(ctx),
// load(ctx, j, P), scratch(ctx), store(ctx, j, v, P) per element.
template <bool FWD, bool FIRST, bool LAST, int LOGG, int H, int C, class Job>
__global__ void __launch_bounds__(NTT_THREADS)
ntt_pass_kernel(Dev d, Job job, int s0, int jbase) {
    constexpr int G = 1 << LOGG;
    constexpr int TILE = H * G * C;
    constexpr int T = TILE / NTT_EPT;
    __shared__ u64 sm[TILE + TILE / 8];

    const int log_n = d.log_n;
    const int lo_bits = log_n - s0 - LOGG;
    const int jb = jbase + (int)blockIdx.y;
    const typename Job::Ctx jc = job.make(jb);
    const int p = job.prime(jc);
    const PrimeConst P = d.pc[p];
    const ulonglong2* __restrict__ tw = (FWD ? d.tw : d.itw) + (size_t)p * d.n;

    const u32 ncolblk = (1u << lo_bits) / C;
    const u32 hi0 = (blockIdx.x / ncolblk) * H;
    const u32 lo0 = (blockIdx.x % ncolblk) * C;

    // element e = t + k*T of the tile sits at global index j0 + k*jstep
    auto gidx = [&](u32 e) -> u32 {
        u32 c = e % C, g = (e / C) % G, h = e / (C * G);
        return ((hi0 + h) << (log_n - s0)) | (g << lo_bits) | (lo0 + c);
    };
    const u32 t = threadIdx.x;
    const u32 j0 = gidx(t);
    const u32 jstep = NTT_EPT > 1 ? gidx(t + T) - j0 : 0;

    if (FIRST) {
#pragma unroll
        for (int k = 0; k < NTT_EPT; k++) sm[spad(t + k * T)] = job.load(jc, j0 + k * jstep, P);
    } else {
        const u64* __restrict__ src = job.scratch(jc);
#pragma unroll
        for (int k = 0; k < NTT_EPT; k++) sm[spad(t + k * T)] = src[j0 + k * jstep];
    }
    __syncthreads();
    const bool lz = FWD && fwd_lazy_ok(P);
    if (FWD) {
        if (lz) ntt_rounds_fwd<LOGG, H, C, true>(sm, tw, hi0, s0, P.q, P.two_q);
        else ntt_rounds_fwd<LOGG, H, C, false>(sm, tw, hi0, s0, P.q, P.two_q);
    } else {
        ntt_rounds_inv<LOGG, H, C>(sm, tw, hi0, s0, P.q, P.two_q);
    }

    if (LAST) {
#pragma unroll
        for (int k = 0; k < NTT_EPT; k++) {
            u64 v = sm[spad(t + k * T)];
            if (FWD && lz) v = reduce64_lazy(v, P);
            job.store(jc, j0 + k * jstep, v, P);
        }
    } else {
        u64* __restrict__ dst = job.scratch(jc);
#pragma unroll
        for (int k = 0; k < NTT_EPT; k++) dst[j0 + k * jstep] = sm[spad(t + k * T)];
    }
}

// Single-pass variant for small limbs (whole limb in one CTA).
template <bool FWD, int LOGN, class Job>
void launch_ntt_single(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    dim3 grid(1, njobs);
    const int threads = (1 << LOGN) / NTT_EPT;
    ntt_pass_kernel<FWD, true, true, LOGN, 1, 1, Job><<<grid, threads, 0, st>>>(d, job, 0, jbase);
    note_launch();
}

// Two-pass variant: pass A covers stages [0, LA) over strided columns, pass B
// covers [LA, log n) over contiguous rows.  Forward runs A then B; inverse
// runs B then A.
template <bool FWD, int LA, int LB, class Job>
void launch_ntt_two(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    constexpr int CA = NTT_TILE >> LA;   // columns per tile in pass A
    constexpr int HB = NTT_TILE >> LB;   // rows per tile in pass B
    const u32 n = 1u << (LA + LB);
    dim3 grid(n / NTT_TILE, njobs);
    note_launch(2);
    if constexpr (FWD) {
        ntt_pass_kernel<true, true, false, LA, 1, CA, Job><<<grid, NTT_THREADS, 0, st>>>(d, job, 0, jbase);
        ntt_pass_kernel<true, false, true, LB, HB, 1, Job><<<grid, NTT_THREADS, 0, st>>>(d, job, LA, jbase);
    } else {
        ntt_pass_kernel<false, true, false, LB, HB, 1, Job><<<grid, NTT_THREADS, 0, st>>>(d, job, LA, jbase);
        ntt_pass_kernel<false, false, true, LA, 1, CA, Job><<<grid, NTT_THREADS, 0, st>>>(d, job, 0, jbase);
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
