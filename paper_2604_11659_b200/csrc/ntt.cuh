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
// the round's bits; each thread owns 8 / 2^R units, 8 elements in registers.
template <bool FWD, int LOGG, int H, int C, int A, int R>
__device__ __forceinline__ void ntt_round(u64* sm, const ulonglong2* __restrict__ tw, u32 hi0,
                                          int s0, u64 q, u64 two_q) {
    constexpr int G = 1 << LOGG;
    constexpr int TILE = H * G * C;
    constexpr int T = TILE / NTT_EPT;
    constexpr int NU = 1 << R;
    constexpr int UPT = NTT_EPT / NU;
    constexpr int LOWB = LOGG - A - R;
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
        u64 v[NU];
#pragma unroll
        for (int e = 0; e < NU; e++) v[e] = sm[spad((h * G + (gbase | ((u32)e << LOWB))) * C + c)];
        if (FWD) {
#pragma unroll
            for (int j = 0; j < R; j++) {
                const int ls = A + j;
                const u32 base = (1u << (s0 + ls)) + (hi << ls) + (go_high << j);
                constexpr int dummy = 0;
                (void)dummy;
#pragma unroll
                for (int e = 0; e < NU; e++) {
                    const int bit = 1 << (R - 1 - j);
                    if (e & bit) continue;
                    const ulonglong2 w = tw[base + (e >> (R - j))];
                    u64 x = csub(v[e], two_q);
                    const u64 t = shoup_lazy(v[e + bit], w.x, w.y, q);
                    v[e] = x + t;
                    v[e + bit] = x - t + two_q;
                }
            }
        } else {
#pragma unroll
            for (int j = R - 1; j >= 0; j--) {
                const int ls = A + j;
                const u32 base = (1u << (s0 + ls)) + (hi << ls) + (go_high << j);
#pragma unroll
                for (int e = 0; e < NU; e++) {
                    const int bit = 1 << (R - 1 - j);
                    if (e & bit) continue;
                    const ulonglong2 w = tw[base + (e >> (R - j))];
                    const u64 x = v[e], y = v[e + bit];
                    v[e] = csub(x + y, two_q);
                    v[e + bit] = shoup_lazy(x - y + two_q, w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int e = 0; e < NU; e++) sm[spad((h * G + (gbase | ((u32)e << LOWB))) * C + c)] = v[e];
    }
}

template <int LOGG, int H, int C, int A>
__device__ __forceinline__ void ntt_rounds_fwd(u64* sm, const ulonglong2* tw, u32 hi0, int s0,
                                               u64 q, u64 two_q) {
    if constexpr (A < LOGG) {
        constexpr int R = (LOGG - A) < 3 ? (LOGG - A) : 3;
        ntt_round<true, LOGG, H, C, A, R>(sm, tw, hi0, s0, q, two_q);
        __syncthreads();
        ntt_rounds_fwd<LOGG, H, C, A + R>(sm, tw, hi0, s0, q, two_q);
    }
}

template <int LOGG, int H, int C, int TOP>
__device__ __forceinline__ void ntt_rounds_inv(u64* sm, const ulonglong2* tw, u32 hi0, int s0,
                                               u64 q, u64 two_q) {
    if constexpr (TOP > 0) {
        constexpr int R = TOP < 3 ? TOP : 3;
        ntt_round<false, LOGG, H, C, TOP - R, R>(sm, tw, hi0, s0, q, two_q);
        __syncthreads();
        ntt_rounds_inv<LOGG, H, C, TOP - R>(sm, tw, hi0, s0, q, two_q);
    }
}

template <bool FWD, bool FIRST, bool LAST, int LOGG, int H, int C, class Job>
__global__ void __launch_bounds__(NTT_THREADS)
ntt_pass_kernel(Dev d, Job job, int s0, int jbase) {
    constexpr int G = 1 << LOGG;
    constexpr int TILE = H * G * C;
    __shared__ u64 sm[TILE + TILE / 8];

    const int log_n = d.log_n;
    const int s1 = s0 + LOGG;
    const int lo_bits = log_n - s1;
    const int jb = jbase + (int)blockIdx.y;
    const int p = job.prime(jb);
    const PrimeConst P = d.pc[p];
    const ulonglong2* __restrict__ tw = (FWD ? d.tw : d.itw) + (size_t)p * d.n;

    const u32 ncolblk = (1u << lo_bits) / C;
    const u32 hi0 = (blockIdx.x / ncolblk) * H;
    const u32 lo0 = (blockIdx.x % ncolblk) * C;

    auto gidx = [&](u32 e) -> u32 {
        u32 c = e % C, g = (e / C) % G, h = e / (C * G);
        return ((hi0 + h) << (log_n - s0)) | (g << lo_bits) | (lo0 + c);
    };

    if (FIRST) {
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) sm[spad(e)] = job.load(jb, gidx(e), P);
    } else {
        const u64* __restrict__ src = job.scratch(jb);
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) sm[spad(e)] = src[gidx(e)];
    }
    __syncthreads();
    if (FWD) ntt_rounds_fwd<LOGG, H, C, 0>(sm, tw, hi0, s0, P.q, P.two_q);
    else ntt_rounds_inv<LOGG, H, C, LOGG>(sm, tw, hi0, s0, P.q, P.two_q);

    if (LAST) {
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) job.store(jb, gidx(e), sm[spad(e)], P);
    } else {
        u64* __restrict__ dst = job.scratch(jb);
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) dst[gidx(e)] = sm[spad(e)];
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
