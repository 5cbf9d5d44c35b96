// The encrypted SpMSpM runner: CSR x CSC planner + batched device executor.
//
// Replaces the reference's timed region `spmm_csr_csc` -> `_run_schedule`
// -> `fhe_spmspm_step` (engine.py:99-184; encmat.py:150-221).  The reference
// walks pairs one at a time; here the pair list is planned on the host and
// executed in phases, each a handful of batched kernel launches:
//
//   1. alignment  distinct (operand, step) rotations only, hoisted: one
//                 decompose+ModUp per source operand, then per step the
//                 automorphism-gathered key inner product + ModDown.
//   2. pairs      per batch of B pairs: mult_ct fused into relinearisation
//                 (tensor computed on the fly in the digit loader and the
//                 ModDown epilogue), rescale fused with the mask multiply,
//                 second rescale, accumulation rotation (pairs sorted by
//                 step so equal keys are adjacent), modular accumulation.
//
// Bit-exactness of this re-ordering: each pair's
// contribution is computed exactly as the reference computes it, and the
// final modular sum is order-free.
#include <algorithm>
#include <chrono>
#include <numeric>
#include <unordered_map>

#include "../../include/hespmm_b200.h"
#include "ops.cuh"

using namespace hs;
typedef unsigned __int128 u128;

namespace {

struct PlanPair {
    int64_t i, j, ap, bp;
    int32_t k = 0;         // operand product (hs_spmspm_multi): operands cta[k], ctb[k]
    int32_t o = 0;         // output ciphertext (hs_spmspm_multi): outs[o]
};

u32 norm_step(int64_t s, u32 slots) {
    int64_t r = s % (int64_t)slots;
    if (r < 0) r += slots;
    return (u32)r;
}

u64 powmod_h(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = (u64)((u128)r * b % q);
        b = (u64)((u128)b * b % q);
        e >>= 1;
    }
    return r;
}

// Two-pointer intersection per output cell (encmat.py:170-186).
template <class Emit>
void merge_pairs(int dim, const int64_t* oa, const int64_t* ia, const int64_t* ob, const int64_t* ib,
                 Emit emit) {
    for (int i = 0; i < dim; i++) {
        const int64_t a0 = oa[i], a1 = oa[i + 1];
        if (a0 == a1) continue;
        for (int j = 0; j < dim; j++) {
            int64_t x = a0, y = ob[j];
            const int64_t y1 = ob[j + 1];
            while (x < a1 && y < y1) {
                const int64_t c = ia[x], r = ib[y];
                if (c == r) {
                    emit(PlanPair{i, j, x, y});
                    x++;
                    y++;
                } else if (c < r) {
                    x++;
                } else {
                    y++;
                }
            }
        }
    }
}

struct DeviceArena {
    cudaStream_t st;
    std::vector<void*> ptrs;
    bool failed = false;
    template <class T>
    T* get(size_t count) {
        void* p = nullptr;
        if (count == 0) count = 1;
        if (cudaMallocAsync(&p, count * sizeof(T), st) != cudaSuccess) {
            failed = true;
            return nullptr;
        }
        ptrs.push_back(p);
        return (T*)p;
    }
    ~DeviceArena() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

// Galois keys for a set of steps: resident keys from the context store, or
// keys generated on the device on demand (steps registered with
// hs_keygen_register).  Generated keys live in a fixed pool of `cap` key
// buffers; generation runs on a side stream so the next batch's keys are
// produced while the current batch computes (events order reuse).
// HS_KEYGEN_NO_PREFETCH=1: generate each batch's keys only when it needs
// them (A/B knob for the side-stream overlap).
static bool prefetch_on() {
    static const bool off = getenv("HS_KEYGEN_NO_PREFETCH") != nullptr;
    return !off;
}

struct KeyProvider {
    hs_ctx* c;
    cudaStream_t st;
    cudaStream_t side = nullptr;
    std::vector<u64*> buf;
    std::vector<int64_t> tag, last;
    std::vector<cudaEvent_t> gen_ev, use_ev;
    int64_t clock = 0;

    ~KeyProvider() {
        // buffers, events and the side stream belong to the context (reused)
        if (side) cudaStreamSynchronize(side);
    }
    bool resident(u32 r) const { return c->galois.count(r) != 0; }
    int slot_of(u32 r) const {
        for (size_t k = 0; k < tag.size(); k++)
            if (tag[k] == (int64_t)r) return (int)k;
        return -1;
    }
    bool needs_generation(u32 r) const { return !resident(r) && slot_of(r) < 0; }
    hs_status init(int cap) {
        if (!buf.empty() || cap <= 0) return HS_OK;
        if (!c->kpool_side) HS_CUDA(cudaStreamCreateWithFlags(&c->kpool_side, cudaStreamNonBlocking));
        side = c->kpool_side;
        while ((int)c->kpool_buf.size() < cap) {
            u64* b = nullptr;
            cudaEvent_t g, u;
            HS_CUDA(cudaMalloc((void**)&b, c->key_bytes()));
            HS_CUDA(cudaEventCreateWithFlags(&g, cudaEventDisableTiming));
            HS_CUDA(cudaEventCreateWithFlags(&u, cudaEventDisableTiming));
            c->kpool_buf.push_back(b);
            c->kpool_gen_ev.push_back(g);
            c->kpool_use_ev.push_back(u);
        }
        buf.assign(c->kpool_buf.begin(), c->kpool_buf.begin() + cap);
        gen_ev.assign(c->kpool_gen_ev.begin(), c->kpool_gen_ev.begin() + cap);
        use_ev.assign(c->kpool_use_ev.begin(), c->kpool_use_ev.begin() + cap);
        tag.assign(cap, -1);                 // contents are regenerated every call
        last.assign(cap, 0);
        for (int k = 0; k < cap; k++) HS_CUDA(cudaEventRecord(use_ev[k], st));
        return HS_OK;
    }
    // Start generating the missing keys of `steps` on the side stream, never
    // evicting keys of `protect`.
    hs_status prefetch(const std::vector<u32>& steps, const std::vector<u32>& protect) {
        std::vector<u32> gen;
        std::vector<hs_ctx::Stream> ss;
        std::vector<u64*> dst;
        std::vector<int> slots;
        for (u32 r : steps) {
            if (!needs_generation(r) || std::find(gen.begin(), gen.end(), r) != gen.end()) continue;
            auto lz = c->lazy.find(r);
            if (lz == c->lazy.end()) {
                set_error("missing Galois key for step " + std::to_string(r));
                return HS_KEY_MISSING;
            }
            int victim = -1;
            for (int k = 0; k < (int)buf.size(); k++) {
                const bool keep = tag[k] >= 0 &&
                                  (std::find(protect.begin(), protect.end(), (u32)tag[k]) != protect.end() ||
                                   std::find(steps.begin(), steps.end(), (u32)tag[k]) != steps.end());
                if (keep || std::find(slots.begin(), slots.end(), k) != slots.end()) continue;
                if (victim < 0 || tag[k] < 0 || (tag[victim] >= 0 && last[k] < last[victim])) victim = k;
                if (tag[victim] < 0) break;
            }
            if (victim < 0) {
                set_error("Galois key pool exhausted");
                return HS_OUT_OF_MEMORY;
            }
            HS_CUDA(cudaStreamWaitEvent(side, use_ev[victim], 0));
            tag[victim] = r;
            last[victim] = ++clock;
            gen.push_back(r);
            ss.push_back(lz->second);
            dst.push_back(buf[victim]);
            slots.push_back(victim);
        }
        if (gen.empty()) return HS_OK;
        hs_status s = generate_galois_keys(c, gen, ss, dst, side);
        if (s != HS_OK) return s;
        for (int k : slots) HS_CUDA(cudaEventRecord(gen_ev[k], side));
        return HS_OK;
    }
    hs_status acquire(const std::vector<u32>& steps, std::vector<const u64*>& out) {
        hs_status s = prefetch(steps, steps);
        if (s != HS_OK) return s;
        out.resize(steps.size());
        for (size_t k = 0; k < steps.size(); k++) {
            auto it = c->galois.find(steps[k]);
            if (it != c->galois.end()) {
                out[k] = it->second.d;
                continue;
            }
            const int sl = slot_of(steps[k]);
            HS_CUDA(cudaStreamWaitEvent(st, gen_ev[sl], 0));
            last[sl] = ++clock;
            out[k] = buf[sl];
        }
        return HS_OK;
    }
    hs_status release(const std::vector<u32>& steps) {
        for (u32 r : steps) {
            const int sl = slot_of(r);
            if (sl >= 0) HS_CUDA(cudaEventRecord(use_ev[sl], st));
        }
        return HS_OK;
    }
};

// Hoisted alignment rotations: todo[k] = (source operand 0|1, normalised
// step) rotated at level L into outs[k]; per source one decomposition + ModUp
// per chunk of steps (chunks bounded by the work budget and, for generated
// keys, by the key pool).
static hs_status compute_alignments(hs_ctx* c, const std::vector<const u64*>& operands,
                                    const std::vector<std::pair<int, u32>>& todo,
                                    const std::vector<u64*>& outs_all, KeyProvider& KP, DeviceArena& A,
                                    size_t budget, int64_t max_gen, cudaStream_t st) {
    // Chunks of distinct STEPS across all source operands: each chunk's keys
    // are acquired once and serve every operand rotated by those steps (at
    // cfg3, 2,963 rotations share 1,544 steps: per-operand chunks generated
    // 1,419 of those keys twice).
    const int L = c->L;
    const u32 n = c->n;
    const Dev& d = c->dev;
    const int R = (int)todo.size();
    if (!R) return HS_OK;
    std::vector<u32> steps;                                  // distinct, first-use order
    {
        std::unordered_map<u32, int> seen;
        for (const auto& al : todo)
            if (seen.emplace(al.second, 0).second) steps.push_back(al.second);
    }
    const size_t base_e = ks_hoisted_scratch_elems(0, L, n);
    const size_t per_e = ks_hoisted_scratch_elems(1, L, n) - base_e;
    int64_t rmax = budget / 8 > base_e ? (int64_t)((budget / 8 - base_e) / per_e) : 1;
    rmax = std::max<int64_t>(1, std::min<int64_t>(rmax, (int64_t)steps.size()));
    bool any_gen = false;
    for (u32 r : steps) any_gen |= !KP.resident(r);
    if (any_gen) rmax = std::min<int64_t>(rmax, max_gen);
    u64* scratch = A.get<u64>(ks_hoisted_scratch_elems((int)rmax, L, n));
    u32* d_gal = A.get<u32>(R);
    const u64** d_keys = A.get<const u64*>(R);
    const u64** d_outs = A.get<const u64*>(R);
    if (A.failed) {
        set_error("out of device memory (alignment)");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    std::vector<u32> hgal(R);
    std::vector<const u64*> hkeys(R), houts(R);
    int used = 0;                                            // entries of the device arrays filled
    const int nchunks = (int)((steps.size() + rmax - 1) / rmax);
    for (int ci = 0; ci < nchunks; ci++) {
        const size_t s0 = (size_t)ci * rmax, s1 = std::min(steps.size(), s0 + (size_t)rmax);
        std::vector<u32> chunk(steps.begin() + s0, steps.begin() + s1);
        std::unordered_map<u32, int> kidx;
        for (size_t k = 0; k < chunk.size(); k++) kidx[chunk[k]] = (int)k;
        std::vector<const u64*> kp;
        hs_status ks_ = KP.acquire(chunk, kp);
        if (ks_ != HS_OK) return ks_;
        if (any_gen && ci + 1 < nchunks && prefetch_on()) {   // next chunk's keys while this one computes
            const size_t n0 = s1, n1 = std::min(steps.size(), s1 + (size_t)rmax);
            ks_ = KP.prefetch(std::vector<u32>(steps.begin() + n0, steps.begin() + n1), chunk);
            if (ks_ != HS_OK) return ks_;
        }
        for (int src = 0; src < (int)operands.size(); src++) {
            const int r0 = used;
            for (int k = 0; k < R; k++) {
                const auto& al = todo[k];
                if (al.first != src) continue;
                auto it = kidx.find(al.second);
                if (it == kidx.end()) continue;
                hgal[used] = (u32)powmod_h(5, al.second, 2ull * n);
                hkeys[used] = kp[it->second];
                houts[used] = outs_all[k];
                used++;
            }
            const int rc = used - r0;
            if (!rc) continue;
            HS_CUDA(cudaMemcpyAsync(d_gal + r0, hgal.data() + r0, rc * sizeof(u32), cudaMemcpyHostToDevice, st));
            HS_CUDA(cudaMemcpyAsync(d_keys + r0, hkeys.data() + r0, rc * sizeof(u64*), cudaMemcpyHostToDevice,
                                    st));
            HS_CUDA(cudaMemcpyAsync(d_outs + r0, houts.data() + r0, rc * sizeof(u64*), cudaMemcpyHostToDevice,
                                    st));
            rotate_hoisted(d, rc, L, operands[src], d_gal + r0, d_keys + r0, table(d_outs + r0), scratch, st);
        }
        KP.release(chunk);
    }
    return HS_OK;
}

// Operand product k of a pair: ct_a = cta[k], ct_b = ctb[k] (one product for
// the plain runner; the products of one tiled output block otherwise).
// Alignment rotations are deduplicated per (operand, step), operand id 2k+src.
hs_status run_pairs(hs_ctx* c, int dim, const std::vector<PlanPair>& pairs,
                    const std::vector<const u64*>& cta, const std::vector<const u64*>& ctb,
                    const u64* const* masks, int64_t nmasks, const std::vector<u64*>& outs,
                    hs_counters* cnt, int shard, int nshard, cudaStream_t st,
                    std::chrono::steady_clock::time_point t_start) {
    const int L = c->L;
    const u32 n = c->n, slots = n / 2;
    const Dev& d = c->dev;
    hs_counters C{};
    if (L < 2) {
        set_error("insufficient depth: need at least 2 levels");
        return (hs_status)HS_EVAL_ERROR;
    }
    if (nshard < 1 || shard < 0 || shard >= nshard) {
        set_error("bad shard index/count");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    const int64_t np = (int64_t)pairs.size();

    // ---- plan: per pair sources, mask, accumulation key (logical counts over all pairs)
    std::vector<int32_t> ia(np), ib(np);
    std::vector<u32> accr(np);
    std::vector<int64_t> mpos(np);
    std::unordered_map<u64, int32_t> align_idx;      // key = src * slots + r
    std::vector<std::pair<int, u32>> align_list;     // (src, r)
    auto galois_key = [&](int64_t raw, u32 r) -> const u64* {
        auto it = c->galois.find(r);
        if (it != c->galois.end()) return it->second.d;
        if (c->lazy.count(r)) return (const u64*)1;     // generated on demand
        set_error("missing Galois key for step " + std::to_string(raw));
        return nullptr;
    };
    if (!c->relin.d && np) {
        set_error("no relinearization key in bundle");
        return (hs_status)HS_KEY_MISSING;
    }
    // operand ids for the alignment deduplication: ct_a 0, ct_b 1 for one
    // product (the ids hs_align_provide uses); with several products the
    // distinct ciphertexts (A[I][K] serves every J), so a block operand is
    // rotated by a step once for the whole tiled product
    std::vector<const u64*> operands;
    std::vector<int> opid_a(cta.size()), opid_b(cta.size());
    {
        auto id_of = [&](const u64* ptr) {
            if (cta.size() > 1)
                for (size_t k = 0; k < operands.size(); k++)
                    if (operands[k] == ptr) return (int)k;
            operands.push_back(ptr);
            return (int)operands.size() - 1;
        };
        for (size_t k = 0; k < cta.size(); k++) {
            opid_a[k] = id_of(cta[k]);
            opid_b[k] = id_of(ctb[k]);
        }
    }
    for (int64_t p = 0; p < np; p++) {
        const PlanPair& q = pairs[p];
        if (q.k < 0 || q.k >= (int32_t)cta.size() || q.o < 0 || q.o >= (int32_t)outs.size()) {
            set_error("pair operand product / output index out of range");
            return (hs_status)HS_PARAMETER_ERROR;
        }
        int64_t mn;
        ia[p] = 0;
        ib[p] = 1;
        if (q.ap != q.bp) {
            const bool rot_b = q.ap < q.bp;                   // the higher-positioned operand rotates
            const int src = rot_b ? opid_b[q.k] : opid_a[q.k];
            const int64_t raw = q.ap < q.bp ? q.bp - q.ap : q.ap - q.bp;
            const u32 r = norm_step(raw, slots);
            C.rotations++;
            C.alignment_rotations++;
            if (r) {
                if (!galois_key(raw, r)) return (hs_status)HS_KEY_MISSING;
                const u64 key = (u64)src * slots + r;
                auto it = align_idx.find(key);
                int32_t idx;
                if (it == align_idx.end()) {
                    idx = 2 + (int32_t)align_list.size();
                    align_idx.emplace(key, idx);
                    align_list.push_back({src, r});
                } else {
                    idx = it->second;
                }
                (rot_b ? ib[p] : ia[p]) = idx;
            }
            mn = std::min(q.ap, q.bp);
        } else {
            mn = q.ap;
        }
        const int64_t rot = mn - (q.i * dim + q.j);
        accr[p] = 0;
        if (rot != 0) {
            C.rotations++;
            C.accumulation_rotations++;
            const u32 r = norm_step(rot, slots);
            if (r && !galois_key(rot, r)) return (hs_status)HS_KEY_MISSING;
            accr[p] = r;
        }
        if (mn < 0 || mn >= nmasks || !masks[mn]) {
            set_error("mask for slot " + std::to_string(mn) + " not prewarmed");
            return (hs_status)HS_EVAL_ERROR;
        }
        mpos[p] = mn;
    }
    C.ct_ct_mults = C.pt_mults = C.relins = C.relin_noops = np;
    C.rescales = 2 * np;
    {
        // one accumulator per output: adds = pairs - (outputs with a pair)
        std::vector<char> has(outs.size(), 0);
        int64_t nonempty = 0;
        for (const PlanPair& q : pairs)
            if (!has[q.o]) {
                has[q.o] = 1;
                nonempty++;
            }
        C.adds = np - nonempty;
    }
    C.has_result = np > 0;

    // ---- shard: pairs sorted by accumulation step, contiguous ranges
    std::vector<int64_t> order(np);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
        return accr[x] != accr[y] ? accr[x] < accr[y] : pairs[x].o < pairs[y].o;
    });
    const int64_t lo = np * shard / nshard, hi = np * (shard + 1) / nshard;
    const int64_t P = hi - lo;
    C.pairs = P;

    const auto t_plan = std::chrono::steady_clock::now();
    C.plan_ms = std::chrono::duration<double, std::milli>(t_plan - t_start).count();

    const size_t ctL = (size_t)2 * (L + 1) * n;           // ct at level L
    const size_t ctL2 = (size_t)2 * (L - 1) * n;          // ct at level L-2
    for (u64* o : outs) HS_CUDA(cudaMemsetAsync(o, 0, ctL2 * sizeof(u64), st));
    if (P == 0) {
        *cnt = C;
        return (hs_status)HS_OK;
    }
    const size_t budget = c->batch_bytes;
    // generated keys per chunk/batch: the key pool holds two such sets (the
    // one in use and the one being prefetched), bounded by twice the budget
    const int64_t max_gen = std::max<int64_t>(1, (int64_t)(budget / c->key_bytes()));

    // The aligned operands of a range live in HBM for the whole range (one
    // ct at level L each: 25 MiB at N=2^16, L=24; 72 MiB at 2^17, L=35).
    // When all of them do not fit next to the batch work and the key pool,
    // the step-sorted pair list runs in consecutive ranges whose aligned
    // operands fit (their alignments recomputed per range; the output is
    // one modular sum either way).
    int64_t amax = INT64_MAX;
    {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            // memory the stream-ordered pool holds but does not use (freed by
            // the previous call's DeviceArena) is available to this one
            int dev = 0;
            cudaMemPool_t mpool;
            unsigned long long reserved = 0, used = 0;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&mpool, dev) == cudaSuccess &&
                cudaMemPoolGetAttribute(mpool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
                cudaMemPoolGetAttribute(mpool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
                reserved > used)
                free_b += (size_t)(reserved - used);
            const size_t pool = c->kpool_buf.size() >= (size_t)(2 * max_gen) ? 0
                              : (size_t)(2 * max_gen) * c->key_bytes();
            const size_t reserve = budget + budget / 4 + pool + ((size_t)2 << 30);
            amax = free_b > reserve ? (int64_t)((free_b - reserve) / (ctL * sizeof(u64))) : 1;
            amax = std::max<int64_t>(1, amax);
        }
        static const long long cap_env = getenv("HS_ALIGN_MAX") ? atoll(getenv("HS_ALIGN_MAX")) : 0;
        if (cap_env > 0) amax = std::min<int64_t>(amax, cap_env);        // A/B and tests: force ranges
    }
    std::vector<int64_t> cuts{lo};
    {
        std::vector<char> seen(2 + align_list.size(), 0);
        int64_t cnt_a = 0;
        for (int64_t t = lo; t < hi; t++) {
            int64_t add = 0;
            for (int32_t idx : {ia[order[t]], ib[order[t]]})
                if (idx >= 2 && !seen[idx] && !c->ext_align.count((u64)align_list[idx - 2].first * slots +
                                                                   align_list[idx - 2].second))
                    add++;
            if (cnt_a + add > amax && t > cuts.back()) {
                cuts.push_back(t);
                std::fill(seen.begin(), seen.end(), 0);
                cnt_a = 0;
                add = 0;
                for (int32_t idx : {ia[order[t]], ib[order[t]]})
                    if (idx >= 2 && !c->ext_align.count((u64)align_list[idx - 2].first * slots +
                                                        align_list[idx - 2].second))
                        add++;
            }
            for (int32_t idx : {ia[order[t]], ib[order[t]]})
                if (idx >= 2) seen[idx] = 1;
            cnt_a += add;
        }
        cuts.push_back(hi);
    }
    C.physical_alignment = 0;
    bool lazy_used = false;

    // one range of the step-sorted pairs: its alignments, then its pair batches
    auto run_range = [&](const int64_t lo, const int64_t hi) -> hs_status {
    const int64_t P = hi - lo;
    std::vector<char> seen(2 + align_list.size(), 0);
    std::vector<int32_t> need;
    for (int64_t t = lo; t < hi; t++) {
        for (int32_t idx : {ia[order[t]], ib[order[t]]})
            if (idx >= 2 && !seen[idx]) {
                seen[idx] = 1;
                need.push_back(idx);
            }
    }
    DeviceArena A{st};
    KeyProvider KP{c, st};

    // ---- phase 1: hoisted alignment rotations (those another rank computed
    // and handed over with hs_align_provide are used as they are)
    std::vector<const u64*> align_ptr(2 + align_list.size(), nullptr);
    std::vector<std::pair<int, u32>> todo;
    std::vector<u64*> todo_out;
    size_t n_local = 0;
    for (int32_t idx : need) {
        const auto& al = align_list[idx - 2];
        auto it = c->ext_align.find((u64)al.first * slots + al.second);
        if (it != c->ext_align.end()) align_ptr[idx] = it->second;
        else n_local++;
    }
    u64* aligned = A.get<u64>(n_local * ctL);
    if (A.failed) {
        set_error("out of device memory for aligned operands");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    for (int32_t idx : need) {
        if (align_ptr[idx]) continue;
        u64* o = aligned + todo.size() * ctL;
        align_ptr[idx] = o;
        todo.push_back(align_list[idx - 2]);
        todo_out.push_back(o);
    }
    C.physical_alignment += (int64_t)todo.size();
    bool lazy_needed = false;
    for (const auto& al : todo) lazy_needed |= !c->galois.count(al.second);
    for (int64_t t = lo; t < hi && !lazy_needed; t++)
        lazy_needed |= accr[order[t]] && !c->galois.count(accr[order[t]]);
    if (lazy_needed) {
        hs_status ks_ = KP.init((int)(2 * max_gen));
        if (ks_ != HS_OK) return ks_;
    }
    {
        // the alignment scratch lives in its own arena, released before the
        // pair batches allocate theirs (stream-ordered frees)
        DeviceArena A1{st};
        hs_status s_ = compute_alignments(c, operands, todo, todo_out, KP, A1, budget, max_gen, st);
        if (s_ != HS_OK) return s_;
    }

    // ---- phase 2: pair batches
    const size_t per_pair = ks_scratch_elems(1, L, n) +
                            (size_t)n * (2 * (L + 1) + 2 * L + 4 * (L - 1) + 2);
    int64_t B = std::max<int64_t>(1, std::min<int64_t>((int64_t)(budget / 8 / per_pair), P));
    B = std::min<int64_t>(B, 8192);
    // batches over the step-sorted range: up to B pairs and at most max_gen
    // distinct non-resident keys
    std::vector<int64_t> bstart;
    std::vector<std::vector<u32>> bsteps_all;
    for (int64_t s = 0, bnext; s < P; s = bnext) {
        std::vector<u32> bsteps;
        int64_t ngen = 0;
        bnext = s;
        while (bnext < P && bnext - s < B) {
            const u32 r = accr[order[lo + bnext]];
            if (r && (bsteps.empty() || bsteps.back() != r)) {
                const bool lazy = !KP.resident(r);
                if (lazy && ngen + 1 > max_gen && bnext > s) break;
                bsteps.push_back(r);
                ngen += lazy;
            }
            bnext++;
        }
        bstart.push_back(s);
        bsteps_all.push_back(bsteps);
    }
    bstart.push_back(P);
    // several outputs (tiled blocks): within a batch, items of one output
    // are made contiguous (then by step), so each output's accumulation runs
    // once per batch while the batch's keys serve every output
    if (outs.size() > 1)
        for (size_t bi = 0; bi + 1 < bstart.size(); bi++)
            std::stable_sort(order.begin() + lo + bstart[bi], order.begin() + lo + bstart[bi + 1],
                             [&](int64_t x, int64_t y) {
                                 return pairs[x].o != pairs[y].o ? pairs[x].o < pairs[y].o : accr[x] < accr[y];
                             });
    std::vector<const u64*> hA(P), hB(P), hM(P), hK(P);
    std::vector<u32> hG(P), hR(P);
    std::vector<int32_t> hO(P);
    for (int64_t t = 0; t < P; t++) {
        const int64_t p = order[lo + t];
        hA[t] = ia[p] >= 2 ? align_ptr[ia[p]] : cta[pairs[p].k];
        hB[t] = ib[p] >= 2 ? align_ptr[ib[p]] : ctb[pairs[p].k];
        hM[t] = masks[mpos[p]];
        hG[t] = accr[p] ? (u32)powmod_h(5, accr[p], 2ull * n) : 0u;
        hR[t] = accr[p];
        hO[t] = pairs[p].o;
    }
    const u64** dA = A.get<const u64*>(P);
    const u64** dB = A.get<const u64*>(P);
    const u64** dM = A.get<const u64*>(P);
    const u64** dK = A.get<const u64*>(P);
    const u64** dR = A.get<const u64*>(B);
    u32* dG = A.get<u32>(P);
    u64* ks = A.get<u64>(ks_scratch_elems((int)B, L, n));
    u64* Rb = A.get<u64>((size_t)B * 2 * (L + 1) * n);
    u64* Mb = A.get<u64>((size_t)B * 2 * L * n);
    u64* Cb = A.get<u64>((size_t)B * ctL2);
    u64* Fb = A.get<u64>((size_t)B * ctL2);
    u64* Tb = A.get<u64>((size_t)B * 2 * n);
    if (A.failed) {
        set_error("out of device memory (pair batch)");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    std::vector<const u64*> relin_rep(B, c->relin.d);
    HS_CUDA(cudaMemcpyAsync(dA, hA.data(), P * sizeof(u64*), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(dB, hB.data(), P * sizeof(u64*), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(dM, hM.data(), P * sizeof(u64*), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(dG, hG.data(), P * sizeof(u32), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(dR, relin_rep.data(), B * sizeof(u64*), cudaMemcpyHostToDevice, st));

    // key runs of each batch's rotated items (rotate_accumulate_grouped):
    // group starts relative to the run's first rotated item, and head flags;
    // host arrays stay alive (and distinct per run) for the async copies
    static const bool no_group = getenv("HS_NO_GROUP_ROT") != nullptr;   // A/B knob
    std::vector<int> hGS(2 * P + 2);
    std::vector<unsigned char> hHead(P);
    int* dGS = A.get<int>(2 * P + 2);
    unsigned char* dHead = A.get<unsigned char>(P);
    if (A.failed) {
        set_error("out of device memory (group tables)");
        return (hs_status)HS_OUT_OF_MEMORY;
    }
    for (size_t bi = 0; bi + 1 < bstart.size(); bi++) {
        const int64_t s = bstart[bi], bnext = bstart[bi + 1];
        const std::vector<u32>& bsteps = bsteps_all[bi];
        const int bn = (int)(bnext - s);
        std::vector<const u64*> bkeys;
        hs_status ks_ = KP.acquire(bsteps, bkeys);
        if (ks_ != HS_OK) return ks_;
        if (lazy_needed && bi + 2 < bstart.size() && prefetch_on()) {
            ks_ = KP.prefetch(bsteps_all[bi + 1], bsteps);
            if (ks_ != HS_OK) return ks_;
        }
        {
            std::unordered_map<u32, const u64*> kmap;
            for (size_t k = 0; k < bsteps.size(); k++) kmap[bsteps[k]] = bkeys[k];
            for (int64_t t = s; t < bnext; t++) hK[t] = hR[t] ? kmap[hR[t]] : nullptr;
        }
        HS_CUDA(cudaMemcpyAsync(dK + s, hK.data() + s, bn * sizeof(u64*), cudaMemcpyHostToDevice, st));
        // mult_ct + relinearize, level L, then rescale L -> L-1 fused with the
        // mask product (mask in Montgomery form)
        static const bool split_mdr = getenv("HS_SPLIT_MODDOWN_RESCALE") != nullptr;
        if (split_mdr) {
            mult_relin_batch(d, bn, L, table(dA + s), table(dB + s), dR, strided(Rb, (size_t)2 * (L + 1) * n),
                             ks, st);
            rescale_batch(d, bn, L, 2, strided(Rb, (size_t)2 * (L + 1) * n), strided(Mb, (size_t)2 * L * n),
                          table(dM + s), Tb, st);
        } else {
            // ModDown and the first rescale merged (ops.cu JobModDownRescale)
            mult_relin_rescale_batch(d, bn, L, table(dA + s), table(dB + s), dR, table(dM + s),
                                     strided(Rb, (size_t)2 * (L + 1) * n), strided(Mb, (size_t)2 * L * n), ks,
                                     Tb, st);
        }
        // relinearize of a degree-1 ct is a counted no-op (context.py:368-370)
        // rescale L-1 -> L-2
        rescale_batch(d, bn, L - 1, 2, strided(Mb, (size_t)2 * L * n), strided(Cb, ctL2),
                      ItemPtr{nullptr, nullptr, 0}, Tb, st);
        // accumulation per output run of the batch (one run without tiling);
        // step-0 pairs form each run's sorted prefix
        static const bool split_rot = getenv("HS_SPLIT_ROTATE_ACCUM") != nullptr;
        for (int64_t r0 = s; r0 < bnext;) {
            int64_t r1 = r0 + 1;
            while (r1 < bnext && hO[r1] == hO[r0]) r1++;
            u64* out = outs[hO[r0]];
            const int rb = (int)(r0 - s), rn = (int)(r1 - r0);
            int z = 0;
            while (z < rn && hG[r0 + z] == 0) z++;
            accumulate(d, z, L - 1, 2, strided(Cb + (size_t)rb * ctL2, ctL2), out, st);
            bool done = false;
            const int nr = rn - z;
            const int64_t q0 = r0 + z;                     // first rotated item of the run
            int nsteps_run = 0;
            for (int64_t t = q0; t < r1; t++) nsteps_run += (t == q0 || hR[t] != hR[t - 1]);
            if (nr > 0 && !split_rot && !no_group && nsteps_run < nr) {
                // runs of equal steps among the rotated items [q0, r1)
                int* gsh = hGS.data() + q0 + bi;           // distinct slice per run
                int G = 0;
                for (int t = 0, run = 0; t < nr; t++) {
                    // at most 16 items per group: the group's digit sums stay exact in int64
                    const bool h = t == 0 || hR[q0 + t] != hR[q0 + t - 1] || run == 16;
                    run = h ? 1 : run + 1;
                    hHead[q0 + t] = h;
                    if (h) gsh[G++] = t;
                }
                gsh[G] = nr;
                int* dgs = dGS + (gsh - hGS.data());
                HS_CUDA(cudaMemcpyAsync(dgs, gsh, (G + 1) * sizeof(int), cudaMemcpyHostToDevice, st));
                HS_CUDA(cudaMemcpyAsync(dHead + q0, hHead.data() + q0, nr, cudaMemcpyHostToDevice, st));
                done = rotate_accumulate_grouped(d, nr, G, dgs, dHead + q0, L - 2,
                                                 strided(Cb + (size_t)(rb + z) * ctL2, ctL2), dG + q0, dK + q0,
                                                 out, ks, st);
            }
            if (nr > 0 && !done &&
                (split_rot || !rotate_accumulate(d, nr, L - 2, strided(Cb + (size_t)(rb + z) * ctL2, ctL2),
                                                 dG + q0, dK + q0, out, ks, st, nsteps_run))) {
                rotate_batch(d, nr, L - 2, strided(Cb + (size_t)(rb + z) * ctL2, ctL2), dG + q0, dK + q0,
                             strided(Fb + (size_t)(rb + z) * ctL2, ctL2), ks, st);
                accumulate(d, nr, L - 1, 2, strided(Fb + (size_t)(rb + z) * ctL2, ctL2), out, st);
            }
            r0 = r1;
        }
        KP.release(bsteps);
    }
    lazy_used |= lazy_needed;
    return (hs_status)HS_OK;
    };

    C.ranges = (int64_t)cuts.size() - 1;
    for (size_t ci = 0; ci + 1 < cuts.size(); ci++) {
        hs_status s_ = run_range(cuts[ci], cuts[ci + 1]);
        if (s_ != HS_OK) return s_;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
        return (hs_status)HS_CUDA_ERROR;
    }
    if (lazy_used) {              // generated keys must have come from complete streams
        HS_CUDA(cudaStreamSynchronize(st));
        hs_status ks_ = keygen_check(c);
        if (ks_ != HS_OK) return ks_;
    }
    *cnt = C;
    return (hs_status)HS_OK;
}

}  // namespace

extern "C" {

hs_status hs_plan_csr_csc(int32_t dim, const int64_t* oa, const int64_t* ia, const int64_t* ob,
                          const int64_t* ib, int64_t* pairs, int64_t cap, int64_t* npairs) {
    int64_t cntp = 0;
    merge_pairs(dim, oa, ia, ob, ib, [&](const PlanPair& p) {
        if (cntp < cap) {
            pairs[4 * cntp] = p.i;
            pairs[4 * cntp + 1] = p.j;
            pairs[4 * cntp + 2] = p.ap;
            pairs[4 * cntp + 3] = p.bp;
        }
        cntp++;
    });
    *npairs = cntp;
    return (hs_status)HS_OK;
}

hs_status hs_spmspm_csr_csc(hs_ctx* c, int32_t dim, const int64_t* oa, const int64_t* ia,
                            const int64_t* ob, const int64_t* ib, const uint64_t* ct_a,
                            const uint64_t* ct_b, const uint64_t* const* masks, int64_t nmasks,
                            uint64_t* out, hs_counters* counters, int32_t shard, int32_t nshard,
                            void* stream) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<PlanPair> pairs;
    merge_pairs(dim, oa, ia, ob, ib, [&](const PlanPair& p) { pairs.push_back(p); });
    return run_pairs(c, dim, pairs, {ct_a}, {ct_b}, masks, nmasks, std::vector<u64*>{out}, counters, shard,
                     nshard, (cudaStream_t)stream, t0);
}

hs_status hs_spmspm_pairs(hs_ctx* c, int32_t dim, const int64_t* pl, int64_t np, const uint64_t* ct_a,
                          const uint64_t* ct_b, const uint64_t* const* masks, int64_t nmasks,
                          uint64_t* out, hs_counters* counters, int32_t shard, int32_t nshard,
                          void* stream) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<PlanPair> pairs(np);
    for (int64_t p = 0; p < np; p++) pairs[p] = PlanPair{pl[4 * p], pl[4 * p + 1], pl[4 * p + 2], pl[4 * p + 3]};
    return run_pairs(c, dim, pairs, {ct_a}, {ct_b}, masks, nmasks, std::vector<u64*>{out}, counters, shard,
                     nshard, (cudaStream_t)stream, t0);
}

hs_status hs_spmspm_multi(hs_ctx* c, int32_t dim, const int64_t* pl, int64_t np, const uint64_t* const* cts_a,
                          const uint64_t* const* cts_b, int32_t nprod, const uint64_t* const* masks,
                          int64_t nmasks, uint64_t* const* outs, int32_t nout, hs_counters* counters,
                          int32_t shard, int32_t nshard, void* stream) {
    const auto t0 = std::chrono::steady_clock::now();
    if (nprod < 1 || nout < 1) {
        set_error("hs_spmspm_multi: no operand products or outputs");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    std::vector<PlanPair> pairs(np);
    for (int64_t p = 0; p < np; p++)
        pairs[p] = PlanPair{pl[6 * p], pl[6 * p + 1], pl[6 * p + 2], pl[6 * p + 3], (int32_t)pl[6 * p + 4],
                            (int32_t)pl[6 * p + 5]};
    return run_pairs(c, dim, pairs, std::vector<const u64*>(cts_a, cts_a + nprod),
                     std::vector<const u64*>(cts_b, cts_b + nprod), masks, nmasks,
                     std::vector<u64*>(outs, outs + nout), counters, shard, nshard, (cudaStream_t)stream, t0);
}

hs_status hs_reduce_mod(hs_ctx* c, uint64_t* data, int32_t npoly, int32_t nlimbs, void* stream) {
    if (nlimbs < 1 || nlimbs > c->L + 1) {
        set_error("bad limb count");
        return (hs_status)HS_PARAMETER_ERROR;
    }
    reduce_mod(c->dev, data, npoly, nlimbs, (cudaStream_t)stream);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
        return (hs_status)HS_CUDA_ERROR;
    }
    return (hs_status)HS_OK;
}

void hs_set_batch_bytes(hs_ctx* c, uint64_t bytes) { c->batch_bytes = bytes; }

hs_status hs_align_provide(hs_ctx* c, const int32_t* src, const uint32_t* steps, const uint64_t* const* cts,
                           int64_t count) {
    const u32 slots = c->n / 2;
    for (int64_t k = 0; k < count; k++) {
        if ((src[k] != 0 && src[k] != 1) || steps[k] == 0 || steps[k] >= slots) {
            set_error("hs_align_provide: bad (operand, step)");
            return HS_PARAMETER_ERROR;
        }
        c->ext_align[(u64)src[k] * slots + steps[k]] = cts[k];
    }
    return HS_OK;
}

void hs_align_clear(hs_ctx* c) { c->ext_align.clear(); }

hs_status hs_align_compute(hs_ctx* c, const uint64_t* ct_a, const uint64_t* ct_b, const int32_t* src,
                           const uint32_t* steps, int64_t count, uint64_t* const* outs, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const u32 slots = c->n / 2;
    std::vector<std::pair<int, u32>> todo;
    std::vector<u64*> o(outs, outs + count);
    bool lazy = false;
    for (int64_t k = 0; k < count; k++) {
        if ((src[k] != 0 && src[k] != 1) || steps[k] == 0 || steps[k] >= slots) {
            set_error("hs_align_compute: bad (operand, step)");
            return HS_PARAMETER_ERROR;
        }
        if (!c->galois.count(steps[k])) {
            if (!c->lazy.count(steps[k])) {
                set_error("missing Galois key for step " + std::to_string(steps[k]));
                return HS_KEY_MISSING;
            }
            lazy = true;
        }
        todo.push_back({src[k], steps[k]});
    }
    DeviceArena A{st};
    KeyProvider KP{c, st};
    const int64_t max_gen = std::max<int64_t>(1, (int64_t)(c->batch_bytes / c->key_bytes()));
    if (lazy) {
        hs_status s = KP.init((int)(2 * max_gen));
        if (s != HS_OK) return s;
    }
    hs_status s = compute_alignments(c, {ct_a, ct_b}, todo, o, KP, A, c->batch_bytes, max_gen, st);
    if (s != HS_OK) return s;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(std::string("kernel launch failed: ") + cudaGetErrorString(e));
        return HS_CUDA_ERROR;
    }
    if (lazy) {
        HS_CUDA(cudaStreamSynchronize(st));
        return keygen_check(c);
    }
    return HS_OK;
}

}  // extern "C"
