// Throughput probe: DFMA, I2F.F64.U64, F2I.U64.F64, IMAD.WIDE, IMAD.HI on this GPU
// (decides whether FP64 can take work off the integer fmaheavy pipe).
#include <cstdio>
#include <cstdint>
__global__ void dfma_k(int it, double* out) {
    double a[8];
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    const double b = 1.0000001, c = 0.5;
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
    double s = 0; for (int k = 0; k < 8; k++) s += a[k];
    if (s == 1.2345) out[0] = s;
}
__global__ void i2f_k(int it, double* out) {
    uint64_t x[8]; double s[8];
    for (int k = 0; k < 8; k++) { x[k] = threadIdx.x * 977ull + k; s[k] = 0; }
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) { s[k] += (double)x[k]; x[k] += 3; }
    double t = 0; for (int k = 0; k < 8; k++) t += s[k];
    if (t == 1.2345) out[0] = t;
}
__global__ void f2i_k(int it, double* out) {
    double x[8]; uint64_t s[8];
    for (int k = 0; k < 8; k++) { x[k] = threadIdx.x * 977.0 + k; s[k] = 0; }
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) { s[k] += (uint64_t)x[k]; x[k] += 3.0; }
    uint64_t t = 0; for (int k = 0; k < 8; k++) t += s[k];
    if (t == 12345) out[0] = t;
}
__global__ void wide_k(int it, double* out) {
    uint64_t a[8]; uint32_t m = 0x9e3779b9u + threadIdx.x;
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a[k]) : "r"(m), "r"((uint32_t)k + 3u));
    uint64_t t = 0; for (int k = 0; k < 8; k++) t ^= a[k];
    if (t == 12345) out[0] = t;
}
__global__ void hi_k(int it, double* out) {
    uint32_t a[8]; uint32_t m = 0x9e3779b9u + threadIdx.x;
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(a[k]) : "r"(m), "r"((uint32_t)k + 3u));
    uint32_t t = 0; for (int k = 0; k < 8; k++) t ^= a[k];
    if (t == 12345) out[0] = t;
}
__global__ void lo_k(int it, double* out) {
    uint32_t a[8]; uint32_t m = 0x9e3779b9u + threadIdx.x;
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x + k;
    for (int i = 0; i < it; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a[k]) : "r"(m), "r"((uint32_t)k + 3u));
    uint32_t t = 0; for (int k = 0; k < 8; k++) t ^= a[k];
    if (t == 12345) out[0] = t;
}
template <class F> void run(const char* name, F f, int sms) {
    double* d; cudaMalloc(&d, 8);
    const int grid = sms * 16, thr = 256, it = 2048;
    f<<<grid, thr>>>(it, d);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; r++) f<<<grid, thr>>>(it, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 3.0 * grid * thr * it * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-8s %8.2f T ops/s  = %6.1f ops/clk/SM (at %d MHz)\n", name, ops / (ms * 1e-3) / 1e12,
           ops / (ms * 1e-3) / (sms * clk * 1e3), clk / 1000);
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("dfma", dfma_k, sms); run("i2f.f64", i2f_k, sms); run("f2i.u64", f2i_k, sms);
    run("imad.wd", wide_k, sms); run("imad.hi", hi_k, sms); run("imad.lo", lo_k, sms);
    return 0;
}
