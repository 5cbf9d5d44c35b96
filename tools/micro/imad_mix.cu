// Which pipe takes IMAD.HI / IMAD (lo) next to IMAD.WIDE (fmaheavy)?  Mixed
// independent chains: if a pair (WIDE + X) runs at the WIDE-alone rate, X
// issued to the other FMA pipe.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void mix_k(int it, uint64_t* out) {
    uint64_t a[4]; uint32_t b[4];
    const uint32_t m = 0x9e3779b9u + threadIdx.x;
    for (int k = 0; k < 4; k++) { a[k] = threadIdx.x + k; b[k] = threadIdx.x * 3 + k; }
    for (int i = 0; i < it; i++) {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (MODE != 3) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(m), "r"((uint32_t)k + 3u));
            if (MODE == 1 || MODE == 3) asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(b[k]) : "r"(m), "r"((uint32_t)k + 5u));
            if (MODE == 2) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(b[k]) : "r"(m), "r"((uint32_t)k + 5u));
        }
    }
    uint64_t t = 0; for (int k = 0; k < 4; k++) t ^= a[k] ^ b[k];
    if (t == 12345) out[0] = t;
}
template <int MODE> void run(const char* name, int sms) {
    uint64_t* d; cudaMalloc(&d, 8);
    const int grid = sms * 16, thr = 256, it = 4096;
    mix_k<MODE><<<grid, thr>>>(it, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) mix_k<MODE><<<grid, thr>>>(it, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double groups = 3.0 * grid * thr * it * 4;     // (k, iteration) groups
    printf("%-14s %6.1f groups/clk/SM\n", name, groups / (ms * 1e-3) / (sms * clk * 1e3));
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("wide", sms); run<1>("wide+hi", sms); run<2>("wide+lo", sms); run<3>("hi", sms);
    return 0;
}
