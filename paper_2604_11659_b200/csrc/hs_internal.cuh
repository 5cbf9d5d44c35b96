// Internal declarations shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hespmm_b200.h"
#include "modarith.cuh"

namespace hs {

// Kernel-side view of a context (passed by value).
struct Dev {
    u32 n;
    int log_n;
    int L;                       // chain has L+1 primes; aux prime index L+1
    u64 aux_q;                   // the key-switch auxiliary prime p
    const PrimeConst* pc;        // [L+2]
    const ulonglong2* tw;        // [(L+2) * n] {w, floor(w 2^64 / q)} forward roots
    const ulonglong2* itw;       // inverse roots
    const double2* twd;          // [(L+2) * n] {w, RN(w / q)} forward roots as doubles
                                 // (primes with PrimeConst::pad & PC_F64; ntt.cuh FP64 butterflies)
    const double2* itwd;         // inverse roots as doubles
    const ulonglong2* df;        // [L+1] digit factor (Q_L/q_i)^-1 mod q_i, Shoup pair
    const ulonglong2* dfR;       // [L+1] the same times 2^64 mod q_i
    const ulonglong2* auxinv;    // [L+1] p^-1 mod q_m
    const ulonglong2* qlinv;     // [(L+1)*(L+1)] q_lvl^-1 mod q_i at [lvl*(L+1)+i]
};

void set_error(const std::string& msg);

// Number of kernels this library has launched (for the bench's gpu_launches).
void note_launch(int count = 1);

struct KeyBuf {
    u64* d = nullptr;            // [2][L+1][L+2][n], standard form
};

}  // namespace hs

// Opaque context type of the C-ABI.
struct hs_ctx {
    int device = 0;
    hs::Dev dev{};
    u32 n = 0;
    int log_n = 0;
    int L = 0;
    std::vector<u64> primes;                 // chain then aux
    std::vector<PrimeConst> pc;              // host copy
    std::vector<u64> df, auxinv;             // host copies (plain values)
    std::vector<u64> qlinv;                  // [(L+1)*(L+1)]
    void* d_blob = nullptr;                  // one allocation for all tables
    // on-device Galois key generation (keygen.cu)
    void* d_jump = nullptr;                  // PCG64 LCG jump constants
    void* d_zig = nullptr;                   // numpy ziggurat tables
    u64* d_thr = nullptr;                    // Lemire thresholds per prime
    u64* d_sk = nullptr;                     // secret key, NTT form [L+2][n]
    ulonglong2* d_kskf = nullptr;            // p (Q_L/q_i) mod q_m, Shoup pairs [(L+1)^2]
    struct Stream { u64 s_hi, s_lo, i_hi, i_lo; };
    std::unordered_map<u32, Stream> lazy;    // registered steps generated on demand
    // aligned operands computed elsewhere (another rank), key = operand * n/2 + step
    std::unordered_map<u64, const u64*> ext_align;
    size_t keygen_batch = 64;                // keys generated per launch (per-launch latency amortised)
    int64_t keys_generated = 0;
    int* d_kg_err = nullptr;                 // set if a keygen stream window overflowed
    // Buffers of the runner's generated-key pool, kept across calls (cudaMalloc
    // of tens of GB per call dominated and varied the step time); contents
    // are NOT reused across calls -- every call regenerates the keys it uses.
    std::vector<u64*> kpool_buf;
    std::vector<cudaEvent_t> kpool_gen_ev, kpool_use_ev;
    cudaStream_t kpool_side = nullptr;
    static constexpr int KG_LANES = 4;       // concurrent key-generation chains
    cudaStream_t kg_stream[KG_LANES] = {};   // (latency-bound launches overlap across chains)
    cudaEvent_t kg_event[KG_LANES + 1] = {};
    hs::KeyBuf relin;
    size_t batch_bytes = (size_t)6 << 30;   // runner work-buffer budget
    std::unordered_map<u32, hs::KeyBuf> galois;   // normalised step -> key
    size_t key_bytes() const { return (size_t)2 * (L + 1) * (L + 2) * n * sizeof(u64); }
};

#define HS_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t e_ = (call);                                               \
        if (e_ != cudaSuccess) {                                               \
            hs::set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                          " at " __FILE__ ":" + std::to_string(__LINE__));      \
            return e_ == cudaErrorMemoryAllocation ? HS_OUT_OF_MEMORY           \
                                                   : HS_CUDA_ERROR;            \
        }                                                                      \
    } while (0)

namespace hs {
// Generate Galois keys on the device into `dests` ([2][L+1][L+2][n] each).
// Raises HS_EVAL_ERROR if any device key stream ran out of its window.
hs_status keygen_check(hs_ctx* c);
hs_status generate_galois_keys(hs_ctx* c, const std::vector<u32>& steps,
                               const std::vector<hs_ctx::Stream>& streams,
                               const std::vector<u64*>& dests, cudaStream_t st);
}  // namespace hs
