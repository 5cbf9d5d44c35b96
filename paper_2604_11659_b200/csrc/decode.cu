// Exact centred CRT lift of RNS coefficients to float64 on the device
// (host I/O).  The reference decodes with Python big
// integers (hespmm/ckks/context.py:244-279: x = sum_i x_i M_i (M_i^-1 mod
// q_i) mod Q, centred, then float(x)) -- ~0.5 s at N = 2^16 on one core.
//
// Here one thread per coefficient:
//   1. Garner: mixed-radix digits v_i < q_i with x = v_0 + v_1 q_0 + ... ,
//      v_i = (((x_i - v_0) c_0i - v_1) c_1i - ...) with c_ji = q_j^-1 mod q_i;
//   2. X = sum v_i prod_{j<i} q_j as a little-endian array of 64-bit words
//      (Horner from the top: X = X q_i + v_i);
//   3. centre: X > (Q-1)/2  ->  -(Q - X)  (Q odd, so "> Q//2" in the reference);
//   4. float(X) correctly rounded to nearest-even: the top 64 bits with the
//      OR of every lower bit folded into bit 0 (sticky), converted with
//      __ull2double_rn and scaled by an exact power of two.
// Python's float(int) also rounds half to even, so the doubles are bit-equal
// (checked against the golden decoded digests and the host big-int path).
#include "ops.cuh"

namespace hs {

constexpr int CRT_MAXW = 64;       // 64-bit words of Q (63 limbs of < 61 bits fit 60 words)
constexpr int CRT_MAXL = 64;       // limbs (hs_ctx_create accepts L <= 62: 63 limbs)

struct CrtArgs {
    const u64* coeff;              // [nl][n] coefficient domain, canonical
    const u64* q;                  // [nl]
    const ulonglong2* c;           // [nl][nl] Shoup pairs c[j][i] = q_j^-1 mod q_i (j < i)
    const u64* Q;                  // [W] words of Q = prod q_i
    const u64* Qh;                 // [W] words of (Q - 1) / 2
    double* out;                   // [n]
    int nl, W;
    u32 n;
};

__global__ void __launch_bounds__(128) crt_decode_kernel(CrtArgs A) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= A.n) return;
    const int nl = A.nl, W = A.W;
    u64 v[CRT_MAXL];
    for (int i = 0; i < nl; i++) {
        const u64 qi = A.q[i];
        u64 t = A.coeff[(size_t)i * A.n + j];
        for (int k = 0; k < i; k++) {
            const ulonglong2 c = A.c[k * nl + i];
            const u64 vk = v[k] >= qi ? v[k] % qi : v[k];
            const u64 d = t >= vk ? t - vk : t + qi - vk;
            t = shoup(d, c.x, c.y, qi);
        }
        v[i] = t;
    }
    // X = v_{nl-1}; X = X q_i + v_i for i = nl-2 .. 0
    u64 X[CRT_MAXW];
    for (int w = 0; w < W; w++) X[w] = 0;
    X[0] = v[nl - 1];
    int used = 1;
    for (int i = nl - 2; i >= 0; i--) {
        const u64 qi = A.q[i];
        u64 carry = v[i];
        for (int w = 0; w < used; w++) {
            const unsigned __int128 p = (unsigned __int128)X[w] * qi + carry;
            X[w] = (u64)p;
            carry = (u64)(p >> 64);
        }
        if (carry && used < W) X[used++] = carry;
    }
    // centre against (Q-1)/2
    bool gt = false;
    for (int w = W - 1; w >= 0; w--) {
        if (X[w] != A.Qh[w]) {
            gt = X[w] > A.Qh[w];
            break;
        }
    }
    bool neg = false;
    if (gt) {                      // X = Q - X
        neg = true;
        u64 borrow = 0;
        for (int w = 0; w < W; w++) {
            const u64 a = A.Q[w], b = X[w];
            const u64 d = a - b - borrow;
            borrow = (a < b || (a == b && borrow)) ? 1ull : 0ull;
            X[w] = d;
        }
    }
    // correctly rounded conversion: the top 64 bits, sticky-ORed into bit 0,
    // rounded once by the hardware, times 2^(64 top - lz) (exact)
    int top = W - 1;
    while (top > 0 && X[top] == 0) top--;
    double r;
    if (top == 0) {
        r = __ull2double_rn(X[0]);
    } else {
        const int lz = __clzll(X[top]);
        const u64 hi = lz ? (X[top] << lz) | (X[top - 1] >> (64 - lz)) : X[top];
        bool sticky = lz ? (X[top - 1] << lz) != 0 : X[top - 1] != 0;
        for (int w = top - 2; w >= 0 && !sticky; w--) sticky = X[w] != 0;
        r = ldexp(__ull2double_rn(hi | (sticky ? 1ull : 0ull)), 64 * top - lz);
    }
    A.out[j] = neg ? -r : r;
}

}  // namespace hs

using namespace hs;
typedef unsigned __int128 u128h;

extern "C" hs_status hs_crt_decode(hs_ctx* c, const uint64_t* coeff, int32_t nl, double* out,
                                   void* stream) {
    if (nl < 1 || nl > CRT_MAXL || nl > (int)c->primes.size() - 1) {
        set_error("crt decode: limb count out of range");
        return HS_PARAMETER_ERROR;
    }
    // host tables: Garner constants, Q and (Q-1)/2 as 64-bit words
    std::vector<u64> q(c->primes.begin(), c->primes.begin() + nl);
    std::vector<ulonglong2> cc((size_t)nl * nl, make_ulonglong2(0, 0));
    for (int i = 0; i < nl; i++)
        for (int k = 0; k < i; k++) {
            const u64 qi = q[i], qk = q[k] % qi;
            // inverse by Fermat (qi prime)
            u64 r = 1, b = qk, e = qi - 2;
            while (e) {
                if (e & 1) r = (u64)((u128h)r * b % qi);
                b = (u64)((u128h)b * b % qi);
                e >>= 1;
            }
            cc[(size_t)k * nl + i] = make_ulonglong2(r, (u64)(((u128h)r << 64) / qi));
        }
    std::vector<u64> Q(CRT_MAXW, 0);
    Q[0] = 1;
    int W = 1;
    for (int i = 0; i < nl; i++) {
        u64 carry = 0;
        for (int w = 0; w < W; w++) {
            const u128h p = (u128h)Q[w] * q[i] + carry;
            Q[w] = (u64)p;
            carry = (u64)(p >> 64);
        }
        if (carry) Q[W++] = carry;
    }
    std::vector<u64> Qh(W);                              // (Q - 1) / 2: Q is odd
    {
        u64 carry = 0;
        for (int w = W - 1; w >= 0; w--) {
            const u64 word = w == 0 ? Q[0] & ~1ull : Q[w];
            Qh[w] = (word >> 1) | (carry << 63);
            carry = word & 1ull;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    u64* d_q = nullptr;
    ulonglong2* d_c = nullptr;
    u64* d_Q = nullptr;
    HS_CUDA(cudaMallocAsync((void**)&d_q, nl * sizeof(u64), st));
    HS_CUDA(cudaMallocAsync((void**)&d_c, cc.size() * sizeof(ulonglong2), st));
    HS_CUDA(cudaMallocAsync((void**)&d_Q, 2 * W * sizeof(u64), st));
    HS_CUDA(cudaMemcpyAsync(d_q, q.data(), nl * sizeof(u64), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_c, cc.data(), cc.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_Q, Q.data(), W * sizeof(u64), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_Q + W, Qh.data(), W * sizeof(u64), cudaMemcpyHostToDevice, st));
    CrtArgs A{coeff, d_q, d_c, d_Q, d_Q + W, out, nl, W, c->n};
    crt_decode_kernel<<<(c->n + 127) / 128, 128, 0, st>>>(A);
    note_launch();
    HS_CUDA(cudaStreamSynchronize(st));                 // pageable host tables above
    cudaFreeAsync(d_q, st);
    cudaFreeAsync(d_c, st);
    cudaFreeAsync(d_Q, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("crt decode: ") + cudaGetErrorString(e));
        return HS_CUDA_ERROR;
    }
    return HS_OK;
}
