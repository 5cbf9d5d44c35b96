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

constexpr int NTT_TILE = 2048;      // elements per CTA tile (16 KiB smem)
constexpr int NTT_THREADS = 256;    // 4 butterflies per thread per stage

template <bool FWD, bool FIRST, bool LAST, int LOGG, int H, int C, class Job>
__global__ void __launch_bounds__(NTT_THREADS)
ntt_pass_kernel(Dev d, Job job, int s0, int jbase) {
    constexpr int G = 1 << LOGG;
    constexpr int TILE = H * G * C;
    constexpr int NB = TILE / 2;     // butterflies per stage
    __shared__ u64 sm[TILE];

    const int log_n = d.log_n;
    const int s1 = s0 + LOGG;
    const int lo_bits = log_n - s1;
    const int jb = jbase + (int)blockIdx.y;
    const int p = job.prime(jb);
    const PrimeConst P = d.pc[p];
    const u64 q = P.q, two_q = P.two_q;
    const ulonglong2* __restrict__ tw = (FWD ? d.tw : d.itw) + (size_t)p * d.n;

    const u32 ncolblk = (1u << lo_bits) / C;
    const u32 hi0 = (blockIdx.x / ncolblk) * H;
    const u32 lo0 = (blockIdx.x % ncolblk) * C;

    auto gidx = [&](u32 e) -> u32 {
        u32 c = e % C, g = (e / C) % G, h = e / (C * G);
        return ((hi0 + h) << (log_n - s0)) | (g << lo_bits) | (lo0 + c);
    };

    if (FIRST) {
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) sm[e] = job.load(jb, gidx(e), P);
    } else {
        const u64* __restrict__ src = job.scratch(jb);
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) sm[e] = src[gidx(e)];
    }
    __syncthreads();

#pragma unroll 1
    for (int st = 0; st < LOGG; st++) {
        const int ls = FWD ? st : LOGG - 1 - st;     // local stage
        const int s = s0 + ls;                        // global stage
        const u32 lhalf = LOGG - 1 - ls;              // log2(half)
        const u32 half = 1u << lhalf;
        for (u32 u = threadIdx.x; u < NB; u += blockDim.x) {
            const u32 c = u % C;
            const u32 rest = u / C;
            const u32 b = rest % (G / 2);
            const u32 h = rest / (G / 2);
            const u32 blk = b >> lhalf, off = b & (half - 1);
            const u32 g0 = (blk << (lhalf + 1)) + off;
            const u32 i0 = (h * G + g0) * C + c;
            const u32 i1 = i0 + half * C;
            const ulonglong2 w = tw[(1u << s) + ((hi0 + h) << ls) + blk];
            u64 x = sm[i0], y = sm[i1];
            if (FWD) {
                x = csub(x, two_q);
                const u64 t = shoup_lazy(y, w.x, w.y, q);
                sm[i0] = x + t;
                sm[i1] = x - t + two_q;
            } else {
                sm[i0] = csub(x + y, two_q);
                sm[i1] = shoup_lazy(x - y + two_q, w.x, w.y, q);
            }
        }
        __syncthreads();
    }

    if (LAST) {
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) job.store(jb, gidx(e), sm[e], P);
    } else {
        u64* __restrict__ dst = job.scratch(jb);
        for (u32 e = threadIdx.x; e < TILE; e += blockDim.x) dst[gidx(e)] = sm[e];
    }
}

// Single-pass variant for small limbs (whole limb in one CTA).
template <bool FWD, int LOGN, class Job>
void launch_ntt_single(const Dev& d, const Job& job, int jbase, int njobs, cudaStream_t st) {
    dim3 grid(1, njobs);
    int threads = (1 << LOGN) / 2 < NTT_THREADS ? (1 << LOGN) / 2 : NTT_THREADS;
    if (threads < 1) threads = 1;
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
    if (FWD) {
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
