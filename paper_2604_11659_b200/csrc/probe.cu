// Measurement support for bench.py's roofline line (not part of the
// reference interface):
//  * hs_probe_arm / hs_probe_read: the in-step kernel timer of ops.cuh
//    (CUDA events recorded on each armed launch's own stream);
//  * hs_int_peak: integer-pipe peak microbenchmarks on this GPU -- the
//    denominator of the INT-pipe fraction the BASELINE asks for:
//      - butterflies/s of the NTT engine's own forward butterfly
//        (unit_butterflies, approximate-quotient Shoup, lazy reduction
//        schedule) on register-resident data, radix-16 units, full occupancy;
//      - IMAD/s (mad.wide.u32 chains, FMA pipe) and IADD3/s (ALU pipe);
//  * hs_f64_peak: the same for the FP64-pipe butterflies (ntt.cuh
//    unit_butterflies_f64) and DFMA/s.
#include <vector>

#include "ops.cuh"

namespace hs {

namespace {

constexpr int PK_T = 128;          // threads per CTA (the NTT engine's CTA size)
constexpr int PK_MINB = 8;         // CTAs per SM (the NTT engine's occupancy)

// Radix-16 forward butterflies on 16 register values, ITER rounds of 4
// stages; twiddles from shared memory as in the engine.
template <int MINB>
__global__ void __launch_bounds__(PK_T, MINB) bfly_peak_kernel(PrimeConst P, const ulonglong2* tw_g,
                                                               int iters, u64* sink) {
    __shared__ ulonglong2 tw[64];
    if (threadIdx.x < 64) tw[threadIdx.x] = tw_g[threadIdx.x];
    __syncthreads();
    u64 v[16];
#pragma unroll
    for (int e = 0; e < 16; e++) v[e] = ((u64)threadIdx.x << 20) + e + blockIdx.x;   // < q (q > 2^40)
    const u64 nq = 0ull - P.q, four_q = P.two_q << 1;
    const u32 Y = 1u + (threadIdx.x & 1u);
#pragma unroll 1
    for (int it = 0; it < iters; it++) {
        // stage indices 3..6: the lazy schedule reduces at 3 and 5 (as in a pass)
        // (the schedule keeps every value < 16q across repeated rounds)
        unit_butterflies<true, 4, 3>(v, tw, Y, nq, P.two_q, four_q);
    }
    u64 acc = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) acc ^= v[e];
    if (acc == 0x123456789abcdefull) sink[0] = acc;    // never true in practice; keeps the work live
}

// The FP64-pipe forward butterflies (unit_butterflies_f64, ~50-bit primes)
// on 16 register values, same shape as bfly_peak_kernel.
template <int MINB>
__global__ void __launch_bounds__(PK_T, MINB) bfly_f64_peak_kernel(double q, double qinv, const double2* tw_g,
                                                                   int iters, u64* sink) {
    __shared__ double2 tw[64];
    if (threadIdx.x < 64) tw[threadIdx.x] = tw_g[threadIdx.x];
    __syncthreads();
    u64 v[16];
#pragma unroll
    for (int e = 0; e < 16; e++)
        v[e] = (u64)__double_as_longlong((double)(((int)threadIdx.x << 12) + e - (int)blockIdx.x));
    const u32 Y = 1u + (threadIdx.x & 1u);
#pragma unroll 1
    for (int it = 0; it < iters; it++) unit_butterflies_f64<4, 3>(v, tw, Y, q, qinv);   // reduces at 3 and 5
    u64 acc = 0;
#pragma unroll
    for (int e = 0; e < 16; e++) acc ^= v[e];
    if (acc == 0x123456789abcdefull) sink[0] = acc;
}

// 8 independent DFMA chains per thread (FP64 pipe).
__global__ void __launch_bounds__(PK_T, PK_MINB) dfma_peak_kernel(int iters, u64* sink) {
    double a[8];
    const double m = 0.999999 + threadIdx.x * 1e-12, c = 1e-9;
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = __fma_rn(a[k], m, c);
    }
    double x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x += a[k];
    if (x == 1234.5) sink[0] = 1;
}

// 8 independent mad.wide.u32 chains per thread (FMA pipe).
__global__ void __launch_bounds__(PK_T, PK_MINB) imad_peak_kernel(int iters, u64* sink) {
    u64 a[8];
    u32 m = 0x9e3779b9u + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++)
            asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(m), "r"((u32)k + 3u));
    }
    u64 x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x ^= a[k];
    if (x == 0x123456789abcdefull) sink[0] = x;
}

// 8 independent 3-input add chains per thread (IADD3, ALU pipe).
__global__ void __launch_bounds__(PK_T, PK_MINB) iadd_peak_kernel(int iters, u64* sink) {
    u32 a[8];
    const u32 b = threadIdx.x * 7u + 1u, c = blockIdx.x | 1u;
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
    }
    u32 x = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) x ^= a[k];
    if (x == 0x12345678u) sink[0] = x;
}

}  // namespace
}  // namespace hs

using namespace hs;

namespace hs {
// defined in ops.cu
void probe_arm(int mask);
int probe_read(int kind, double* out4);
}  // namespace hs

extern "C" {

hs_status hs_probe_arm(int32_t mask) {
    if (mask < 0 || mask >= (1 << PROBE_KINDS)) {
        set_error("probe mask out of range");
        return HS_PARAMETER_ERROR;
    }
    probe_arm(mask);
    return HS_OK;
}

hs_status hs_probe_read(int32_t kind, double* out4) {
    if (probe_read(kind, out4)) {
        set_error("probe: CUDA event query failed");
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}

// out[0] = butterflies/s, out[1] = IMAD (mad.wide.u32)/s, out[2] = 32-bit adds/s,
// out[3] = SM count used; q = the prime the butterfly probe runs under.
hs_status hs_int_peak(uint64_t q, double* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const PrimeConst P = make_prime_const(q, 1u << 16);
    std::vector<ulonglong2> tw(64);
    u64 w = 3;
    for (int k = 0; k < 64; k++) {
        w = (u64)((unsigned __int128)w * 0x9e3779b97f4a7c15ull % q);
        tw[k] = make_ulonglong2(w, (u64)(((unsigned __int128)w << 64) / q));
    }
    ulonglong2* d_tw = nullptr;
    u64* d_sink = nullptr;
    HS_CUDA(cudaMalloc(&d_tw, 64 * sizeof(ulonglong2)));
    HS_CUDA(cudaMalloc(&d_sink, 8));
    HS_CUDA(cudaMemcpy(d_tw, tw.data(), 64 * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    const int grid = nsm * PK_MINB * 4;            // 4 waves of resident CTAs
    cudaEvent_t e0, e1;
    HS_CUDA(cudaEventCreate(&e0));
    HS_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto launch) -> double {
        launch();                                    // warm-up
        cudaEventRecord(e0, st);
        for (int r = 0; r < 3; r++) launch();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 3.0;
    };
    const int ib = 512, ii = 4096;
    // the butterfly probe at the engine's 8 CTAs/SM (64-register cap: the
    // compiler spills a little) and at 4 CTAs/SM (no cap pressure); best of both
    const double ms_b8 = timed([&] { bfly_peak_kernel<8><<<grid, PK_T, 0, st>>>(P, d_tw, ib, d_sink); });
    const double ms_b4 = timed([&] { bfly_peak_kernel<4><<<grid, PK_T, 0, st>>>(P, d_tw, ib, d_sink); });
    const double ms_b = ms_b8 < ms_b4 ? ms_b8 : ms_b4;
    const double ms_m = timed([&] { imad_peak_kernel<<<grid, PK_T, 0, st>>>(ii, d_sink); });
    const double ms_a = timed([&] { iadd_peak_kernel<<<grid, PK_T, 0, st>>>(ii, d_sink); });
    note_launch(16);
    const double threads = (double)grid * PK_T;
    out[0] = threads * ib * 32.0 / (ms_b * 1e-3);    // 4 stages x 8 butterflies per round
    out[1] = threads * ii * 8.0 / (ms_m * 1e-3);
    out[2] = threads * ii * 16.0 / (ms_a * 1e-3);
    out[3] = nsm;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_tw);
    cudaFree(d_sink);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("int peak probe failed: ") + cudaGetErrorString(e));
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}

// out[0] = FP64-path butterflies/s (prime q, which must be <= 2^50 + 2^40),
// out[1] = DFMA/s, out[2] = 0, out[3] = SM count.
hs_status hs_f64_peak(uint64_t q, double* out, void* stream) {
    if (q > (1ull << 50) + (1ull << 40)) {
        set_error("hs_f64_peak: the FP64 butterflies need q <= 2^50 + 2^40");
        return HS_PARAMETER_ERROR;
    }
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    std::vector<double2> tw(64);
    u64 w = 3;
    for (int k = 0; k < 64; k++) {
        w = (u64)((unsigned __int128)w * 0x9e3779b97f4a7c15ull % q);
        tw[k] = make_double2((double)w, (double)w / (double)q);
    }
    double2* d_tw = nullptr;
    u64* d_sink = nullptr;
    HS_CUDA(cudaMalloc(&d_tw, 64 * sizeof(double2)));
    HS_CUDA(cudaMalloc(&d_sink, 8));
    HS_CUDA(cudaMemcpy(d_tw, tw.data(), 64 * sizeof(double2), cudaMemcpyHostToDevice));
    const int grid = nsm * PK_MINB * 4;
    cudaEvent_t e0, e1;
    HS_CUDA(cudaEventCreate(&e0));
    HS_CUDA(cudaEventCreate(&e1));
    auto timed = [&](auto launch) -> double {
        launch();
        cudaEventRecord(e0, st);
        for (int r = 0; r < 3; r++) launch();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / 3.0;
    };
    const int ib = 512, ii = 4096;
    const double qd = (double)q, qinv = 1.0 / qd;
    const double ms_b8 = timed([&] { bfly_f64_peak_kernel<8><<<grid, PK_T, 0, st>>>(qd, qinv, d_tw, ib, d_sink); });
    const double ms_b4 = timed([&] { bfly_f64_peak_kernel<4><<<grid, PK_T, 0, st>>>(qd, qinv, d_tw, ib, d_sink); });
    const double ms_b = ms_b8 < ms_b4 ? ms_b8 : ms_b4;
    const double ms_f = timed([&] { dfma_peak_kernel<<<grid, PK_T, 0, st>>>(ii, d_sink); });
    note_launch(12);
    const double threads = (double)grid * PK_T;
    out[0] = threads * ib * 32.0 / (ms_b * 1e-3);
    out[1] = threads * ii * 8.0 / (ms_f * 1e-3);
    out[2] = 0.0;
    out[3] = nsm;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d_tw);
    cudaFree(d_sink);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("f64 peak probe failed: ") + cudaGetErrorString(e));
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}

}  // extern "C"
