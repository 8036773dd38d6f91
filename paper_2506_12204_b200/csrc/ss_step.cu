// ss_step.cu — the reference's per-step entry points on the device:
//
//   ss_select_batch  <- extract_top_b / stage_aware_schedule (batching.py:46-88)
//                       and the baselines' selection (engine.py:256-285)
//   ss_evict         <- priority_based_eviction (kvcache.py:137-179) with
//                       should_recompute (kvcache.py:81-134) for every victim
//
// Keys are the reference's key tuples — (urgency rank, remaining seconds,
// arrival, id) or a baseline's shorter tuple, eviction keys negated
// (requests.py:81-97) — as four doubles compared lexicographically with IEEE
// `<` (Python's int/float comparison for |ints| < 2^53), padded with -inf.
// Ties (equal tuples) fall back to the pool position, which is Python's
// stable sorted() / first-minimum min() order.
//
// Selection: a grid-wide pass where every warp keeps a running top-32 of its
// slice (bitonic sort + bitonic merge in registers, warp shuffles), then one
// warp merges the per-warp lists and applies the stage-aware rule. The
// eviction loop walks the eviction order 32 entries at a time: a warp
// inclusive scan of the freed slots of unprotected entries finds the victims
// that bring demand + used under capacity; their decisions are independent,
// one lane each.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <mutex>

#include "ss_costs.cuh"
#include "../../include/semsched_b200.h"

namespace ss {
namespace {

constexpr unsigned FULL = 0xffffffffu;

struct K4 {
    double a, b, c, d;
    int i;  // pool position (tie-break), -1 = empty
};

__device__ __forceinline__ bool lt4(const K4& x, const K4& y) {
    if (x.a < y.a) return true;
    if (y.a < x.a) return false;
    if (x.b < y.b) return true;
    if (y.b < x.b) return false;
    if (x.c < y.c) return true;
    if (y.c < x.c) return false;
    if (x.d < y.d) return true;
    if (y.d < x.d) return false;
    return (unsigned)x.i < (unsigned)y.i;  // -1 (empty) sorts last
}
__device__ __forceinline__ K4 k4inf() {
    K4 k;
    k.a = k.b = k.c = k.d = INFINITY;
    k.i = -1;
    return k;
}
__device__ __forceinline__ K4 k4load(const ss_key4* keys, long long i) {
    K4 k;
    const ss_key4 v = keys[i];
    k.a = v.k[0];
    k.b = v.k[1];
    k.c = v.k[2];
    k.d = v.k[3];
    k.i = (int)i;
    return k;
}
__device__ __forceinline__ K4 k4shfl_xor(const K4& k, int m) {
    K4 r;
    r.a = __shfl_xor_sync(FULL, k.a, m);
    r.b = __shfl_xor_sync(FULL, k.b, m);
    r.c = __shfl_xor_sync(FULL, k.c, m);
    r.d = __shfl_xor_sync(FULL, k.d, m);
    r.i = __shfl_xor_sync(FULL, k.i, m);
    return r;
}
__device__ __forceinline__ K4 k4shfl(const K4& k, int src) {
    K4 r;
    r.a = __shfl_sync(FULL, k.a, src);
    r.b = __shfl_sync(FULL, k.b, src);
    r.c = __shfl_sync(FULL, k.c, src);
    r.d = __shfl_sync(FULL, k.d, src);
    r.i = __shfl_sync(FULL, k.i, src);
    return r;
}
__device__ __forceinline__ bool uni(bool x) { return __all_sync(FULL, x); }

// bitonic sort of one key per lane (ascending if asc)
__device__ __forceinline__ K4 bsort32(K4 x, int lane, bool asc) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const K4 y = k4shfl_xor(x, j);
            const bool up = ((lane & k) == 0) == asc;
            const bool lower = (lane & j) == 0;
            if ((lower == up) ? lt4(y, x) : lt4(x, y)) x = y;
        }
    }
    return x;
}
// S ascending (running top-32); fold in one more key per lane
__device__ __forceinline__ K4 fold32(K4 S, K4 x, int lane) {
    x = bsort32(x, lane, false);  // descending
    if (lt4(x, S)) S = x;         // 32 smallest of both, bitonic
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const K4 y = k4shfl_xor(S, j);
        const bool lower = (lane & j) == 0;
        if (lower ? lt4(y, S) : lt4(S, y)) S = y;
    }
    return S;
}

// ---- selection --------------------------------------------------------------
constexpr int SEL_THREADS = 256;

// every warp: running top-32 (stored keys) of its contiguous slice
__global__ void __launch_bounds__(SEL_THREADS) sel_partial(const ss_key4* stored, long long n, K4* part) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * SEL_THREADS + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * SEL_THREADS) >> 5;
    const long long per = ((n + nw - 1) / nw + 31) & ~31ll;
    const long long lo = warp * per, hi = lo + per < n ? lo + per : n;
    K4 S = k4inf();
    for (long long base = lo; uni(base < hi); base += 32) {
        const long long i = base + lane;
        const K4 x = i < hi ? k4load(stored, i) : k4inf();
        if (!__any_sync(FULL, lt4(x, k4shfl(S, 31)))) continue;
        S = fold32(S, x, lane);
    }
    part[warp * 32 + lane] = S;
}

struct SelArgs {
    const ss_key4* stored;
    const ss_key4* current;
    const uint8_t* pool_dec;
    long long n_pool;
    const K4* part;  // per-warp lists (nullptr: scan the pool directly)
    long long n_part;
    const ss_key4* ongoing;
    const uint8_t* ong_dec;
    int n_ong, b, mode;
    int* out;  // [0] n_cand, [1] n_merged, [2] n_selected, [3] kind, then cand[32], merged[64]
};

__global__ void __launch_bounds__(32) sel_final(const SelArgs A) {
    const int lane = threadIdx.x & 31;
    K4 S = k4inf();
    if (A.part) {
        for (long long base = 0; uni(base < A.n_part); base += 32) {
            const long long i = base + lane;
            const K4 x = i < A.n_part ? A.part[i] : k4inf();
            if (!__any_sync(FULL, lt4(x, k4shfl(S, 31)))) continue;
            S = fold32(S, x, lane);
        }
    } else {
        for (long long base = 0; uni(base < A.n_pool); base += 32) {
            const long long i = base + lane;
            const K4 x = i < A.n_pool ? k4load(A.stored, i) : k4inf();
            if (!__any_sync(FULL, lt4(x, k4shfl(S, 31)))) continue;
            S = fold32(S, x, lane);
        }
    }
    // candidates: the first `want` keys in stored order (heap pops)
    int want = A.b;
    if (A.mode == SS_SELECT_FCFS) want = A.b - A.n_ong;
    if (want < 0) want = 0;
    const long long avail = A.n_pool < 32 ? A.n_pool : 32;
    const int nc = (int)(want < avail ? want : avail);
    int* cand = A.out + 4;
    int* merged = A.out + 4 + 32;
    if (lane < nc) cand[lane] = S.i;
    if (A.mode == SS_SELECT_TOP_B) {
        if (lane == 0) {
            A.out[0] = nc;
            A.out[1] = 0;
            A.out[2] = 0;
            A.out[3] = SS_KIND_DECODE;
        }
        return;
    }
    // pool = candidates + ongoing, current keys, position = pool index
    const int np = nc + A.n_ong;
    if (uni(np == 0)) {  // empty pool: Batch(DECODE, []) (batching.py:67-68)
        if (lane == 0) {
            A.out[0] = 0;
            A.out[1] = 0;
            A.out[2] = 0;
            A.out[3] = SS_KIND_DECODE;
        }
        return;
    }
    K4 ck = k4inf(), ok = k4inf();
    bool cdec = false, odec = false;
    if (lane < nc) {
        ck = k4load(A.current, S.i);
        ck.i = lane;
        cdec = A.pool_dec[S.i] != 0;
    }
    if (lane < A.n_ong) {
        ok = k4load(A.ongoing, lane);
        ok.i = nc + lane;
        odec = A.ong_dec[lane] != 0;
    }
    int kind;
    bool ce, oe;  // member of the merge
    if (A.mode == SS_SELECT_FCFS) {
        // ongoing first in their order, then the popped candidates (engine.py:256-262)
        if (lane < A.n_ong) merged[lane] = nc + lane;
        if (lane < nc) merged[A.n_ong + lane] = lane;
        const bool pre = __any_sync(FULL, (lane < nc && !cdec) || (lane < A.n_ong && !odec));
        if (lane == 0) {
            A.out[0] = nc;
            A.out[1] = np;
            A.out[2] = np;
            A.out[3] = pre ? SS_KIND_PREFILL : SS_KIND_DECODE;
        }
        return;
    }
    if (A.mode == SS_SELECT_STAGE_AWARE) {
        // p* = min(pool, key) (batching.py:70-71)
        K4 m = lt4(ck, ok) ? ck : ok;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const K4 y = k4shfl_xor(m, o);
            if (lt4(y, m)) m = y;
        }
        const int ps = m.i;  // pool position of p*
        const bool ps_dec = uni(ps < nc) ? __shfl_sync(FULL, cdec, ps) : __shfl_sync(FULL, odec, ps - nc);
        kind = ps_dec ? SS_KIND_DECODE : SS_KIND_PREFILL;
        ce = lane < nc && (!ps_dec || cdec);
        oe = lane < A.n_ong;
    } else {  // SJF / HPJF: plain sort of candidates + ongoing (engine.py:270-285)
        ce = lane < nc;
        oe = lane < A.n_ong;
        kind = SS_KIND_DECODE;
    }
    // rank of each member in the merge (stable: pool position breaks ties)
    int rc = 0, ro = 0;
    for (int j = 0; uni(j < 32); j++) {
        const K4 x = k4shfl(ck, j);
        const K4 y = k4shfl(ok, j);
        const bool xe = __shfl_sync(FULL, ce, j), ye = __shfl_sync(FULL, oe, j);
        if (xe && lt4(x, ck)) rc++;
        if (ye && lt4(y, ck)) rc++;
        if (xe && lt4(x, ok)) ro++;
        if (ye && lt4(y, ok)) ro++;
    }
    if (ce) merged[rc] = ck.i;
    if (oe) merged[ro] = ok.i;
    const int nm = __popc(__ballot_sync(FULL, ce)) + __popc(__ballot_sync(FULL, oe));
    const int nsel = nm < A.b ? nm : A.b;
    if (A.mode != SS_SELECT_STAGE_AWARE) {
        // BatchKind from the selected members' stages (engine.py:280-284)
        const bool pre = __any_sync(FULL, (ce && rc < nsel && !cdec) || (oe && ro < nsel && !odec));
        kind = pre ? SS_KIND_PREFILL : SS_KIND_DECODE;
    }
    if (lane == 0) {
        A.out[0] = nc;
        A.out[1] = nm;
        A.out[2] = nsel;
        A.out[3] = kind;
    }
}

// ---- eviction ---------------------------------------------------------------
struct EvArgs {
    const ss_key4* keys;
    const uint32_t *prompt, *prefilled, *decoded, *kv_device, *pred_len;
    const double* f_t;
    const uint8_t* prot;
    long long n, demand, used, cap;
    ss_profile P;
    int dep, select;
    ss_victim* victims;
    int* skipped;
    long long* counts;  // [0] victims, [1] skipped, [2] failed
};

// should_recompute (kvcache.py:81-134) for one victim
__device__ void decide(const EvArgs& A, int idx, ss_victim& v) {
    const long long prompt = A.prompt[idx], pf = A.prefilled[idx], dec = A.decoded[idx];
    const long long kvd = A.kv_device[idx];
    v.index = idx;
    v.f_t_before = A.f_t[idx];
    v.freed_slots = kvd;
    long long pf_new = pf, psaved;
    if (pf > 0 && should_cache_prefill(pf, A.P)) {
        v.action = 0;  // offload
        psaved = pf;
    } else {
        v.action = 1;  // discard
        psaved = 0;
        pf_new = 0;
    }
    long long saved = dec > 0 ? optimal_save_tokens(prompt, dec, A.P) : 0;
    if (v.action == 1 && A.dep) saved = 0;
    v.decode_saved = saved;
    v.decode_discarded = dec - saved;
    v.prefilled = pf_new;
    v.kv_host = psaved + saved;
    v.f_t_after = remaining_time(prompt, A.pred_len[idx], pf_new, saved, psaved + saved, A.P);
    v._pad = 0;
}

__global__ void __launch_bounds__(32) evict_kernel(const EvArgs A) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    long long nv = 0, ns = 0;
    bool failed = false;
    if (!A.select) {
        // should_recompute on every given entry, in the given order
        for (long long base = 0; uni(base < A.n); base += 32) {
            const long long i = base + lane;
            if (i < A.n) {
                ss_victim v;
                decide(A, (int)i, v);
                A.victims[i] = v;
            }
        }
        if (lane == 0) {
            A.counts[0] = A.n;
            A.counts[1] = 0;
            A.counts[2] = 0;
        }
        return;
    }
    long long used = A.used;
    K4 thr;  // last key taken (chunks after the first take keys above it)
    bool have_thr = false;
    long long taken = 0;
    while (uni(A.demand + used > A.cap && taken < A.n)) {
        // next 32 keys of the eviction order
        K4 S = k4inf();
        for (long long base = 0; uni(base < A.n); base += 32) {
            const long long i = base + lane;
            K4 x = i < A.n ? k4load(A.keys, i) : k4inf();
            if (have_thr && !lt4(thr, x)) x = k4inf();
            if (!__any_sync(FULL, lt4(x, k4shfl(S, 31)))) continue;
            S = fold32(S, x, lane);
        }
        const bool valid = S.i >= 0;
        const bool prot = valid && A.prot[S.i];
        const long long fr = (valid && !prot) ? (long long)A.kv_device[S.i] : 0;
        long long inc = fr;  // inclusive scan of freed slots in eviction order
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        const long long exc = inc - fr;
        // an unprotected entry is popped as a victim while the loop condition
        // still holds before it (kvcache.py:157-170)
        const bool victim = valid && !prot && (A.demand + used - exc > A.cap);
        const unsigned vm = __ballot_sync(FULL, victim);
        const int last = vm ? 31 - __clz(vm) : -1;
        const bool done = uni(vm != 0 && A.demand + used - __shfl_sync(FULL, inc, last) <= A.cap);
        // protected entries popped before the last victim (or all, on failure)
        const int nvalid = __popc(__ballot_sync(FULL, valid));
        const int upto = done ? last : nvalid - 1;
        const bool sk = prot && lane <= upto;
        const unsigned sm = __ballot_sync(FULL, sk);
        if (sk) A.skipped[ns + __popc(sm & lt)] = S.i;
        if (victim) {
            ss_victim v;
            decide(A, S.i, v);
            A.victims[nv + __popc(vm & lt)] = v;
        }
        nv += __popc(vm);
        ns += __popc(sm);
        used -= vm ? __shfl_sync(FULL, inc, last) : 0;
        taken += nvalid;
        thr = k4shfl(S, nvalid > 0 ? nvalid - 1 : 0);
        have_thr = true;
        if (done) break;
    }
    failed = A.demand + used > A.cap;
    if (lane == 0) {
        A.counts[0] = nv;
        A.counts[1] = ns;
        A.counts[2] = failed ? 1 : 0;
    }
}

// ---- host staging -------------------------------------------------------------
thread_local char g_err[256];
int fail(int code, const char* msg) {
    strncpy(g_err, msg, sizeof g_err - 1);
    return code;
}

struct Stage {
    std::mutex mu;
    void* buf = nullptr;
    size_t cap = 0;
    int dev = -1;          // device `buf` lives on
    void* host = nullptr;  // pinned bounce buffer (portable across devices)
    size_t hcap = 0;
};
Stage g_sel, g_ev;

size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

int ensure(Stage& s, size_t dev, size_t host) {
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) return fail(SS_ERR_CUDA, "cudaGetDevice");
    if (s.buf && s.dev != cur) {  // the caller moved to another device: release on the old one
        cudaSetDevice(s.dev);
        cudaFree(s.buf);
        cudaSetDevice(cur);
        s.buf = nullptr;
        s.cap = 0;
    }
    s.dev = cur;
    if (s.cap < dev) {
        if (s.buf) cudaFree(s.buf);
        s.buf = nullptr;
        s.cap = 0;
        if (cudaMalloc(&s.buf, dev) != cudaSuccess) return fail(SS_ERR_CUDA, "cudaMalloc (step workspace)");
        s.cap = dev;
    }
    if (s.hcap < host) {
        if (s.host) cudaFreeHost(s.host);
        s.host = nullptr;
        s.hcap = 0;
        if (cudaMallocHost(&s.host, host) != cudaSuccess) return fail(SS_ERR_CUDA, "cudaMallocHost (step staging)");
        s.hcap = host;
    }
    return SS_OK;
}

}  // namespace
}  // namespace ss

extern "C" {

const char* ss_step_last_error(void) { return ss::g_err; }

int ss_select_batch(const ss_key4* stored, const ss_key4* current, const uint8_t* pool_decoding, int64_t n_pool,
                    const ss_key4* ongoing, const uint8_t* ongoing_decoding, int32_t n_ongoing, int32_t b,
                    int32_t mode, int32_t* cand, int32_t* n_cand, int32_t* merged, int32_t* n_merged,
                    int32_t* n_selected, int32_t* kind, void* stream) {
    using namespace ss;
    if (b < 1) return fail(SS_ERR_INVALID_ARG, "batch size must be >= 1");
    if (b > SS_MAX_BATCH || n_ongoing > SS_MAX_BATCH) return fail(SS_ERR_UNSUPPORTED, "b and ongoing are limited to 32");
    if (n_pool < 0 || n_ongoing < 0) return fail(SS_ERR_INVALID_ARG, "negative sizes");
    if (mode < SS_SELECT_TOP_B || mode > SS_SELECT_FCFS) return fail(SS_ERR_INVALID_ARG, "unknown selection mode");
    if ((n_pool > 0 && (!stored || !pool_decoding)) || (n_ongoing > 0 && (!ongoing || !ongoing_decoding)))
        return fail(SS_ERR_INVALID_ARG, "null input");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    if (!current) current = stored;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t np = (size_t)(n_pool > 0 ? n_pool : 1);
    const bool grid = n_pool > 8192;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = grid ? sms * 2 : 0;
    const long long nwarps = (long long)blocks * SEL_THREADS / 32;
    const size_t out_words = 4 + 32 + 64;
    const size_t dev_b = 2 * a16(np * sizeof(ss_key4)) + a16(np) + a16(32 * sizeof(ss_key4)) + a16(32) +
                         a16((size_t)nwarps * 32 * sizeof(K4)) + a16(out_words * 4);
    std::lock_guard<std::mutex> lk(g_sel.mu);
    int rc = ensure(g_sel, dev_b, out_words * 4);
    if (rc) return rc;
    char* p = (char*)g_sel.buf;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += a16(bytes);
        return (void*)r;
    };
    ss_key4* d_st = (ss_key4*)take(np * sizeof(ss_key4));
    ss_key4* d_cur = (ss_key4*)take(np * sizeof(ss_key4));
    uint8_t* d_pd = (uint8_t*)take(np);
    ss_key4* d_on = (ss_key4*)take(32 * sizeof(ss_key4));
    uint8_t* d_od = (uint8_t*)take(32);
    K4* d_part = (K4*)take((size_t)nwarps * 32 * sizeof(K4));
    int* d_out = (int*)take(out_words * 4);
    if (n_pool > 0) {
        cudaMemcpyAsync(d_st, stored, (size_t)n_pool * sizeof(ss_key4), cudaMemcpyHostToDevice, st);
        if (current != stored) cudaMemcpyAsync(d_cur, current, (size_t)n_pool * sizeof(ss_key4), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_pd, pool_decoding, (size_t)n_pool, cudaMemcpyHostToDevice, st);
    }
    if (n_ongoing > 0) {
        cudaMemcpyAsync(d_on, ongoing, (size_t)n_ongoing * sizeof(ss_key4), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_od, ongoing_decoding, (size_t)n_ongoing, cudaMemcpyHostToDevice, st);
    }
    SelArgs a;
    a.stored = d_st;
    a.current = current != stored ? d_cur : d_st;
    a.pool_dec = d_pd;
    a.n_pool = n_pool;
    a.part = nullptr;
    a.n_part = 0;
    a.ongoing = d_on;
    a.ong_dec = d_od;
    a.n_ong = n_ongoing;
    a.b = b;
    a.mode = mode;
    a.out = d_out;
    if (grid) {
        sel_partial<<<blocks, SEL_THREADS, 0, st>>>(d_st, n_pool, d_part);
        a.part = d_part;
        a.n_part = nwarps * 32;
    }
    cudaMemsetAsync(d_out, 0, out_words * 4, st);  // words past the lists are copied back too
    sel_final<<<1, 32, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    cudaMemcpyAsync(g_sel.host, d_out, out_words * 4, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    const int* o = (const int*)g_sel.host;
    if (n_cand) *n_cand = o[0];
    if (n_merged) *n_merged = o[1];
    if (n_selected) *n_selected = o[2];
    if (kind) *kind = o[3];
    if (cand) memcpy(cand, o + 4, sizeof(int) * (size_t)o[0]);
    if (merged) memcpy(merged, o + 4 + 32, sizeof(int) * (size_t)o[1]);
    return SS_OK;
}

int ss_evict(const ss_key4* ev_keys, const uint32_t* prompt, const uint32_t* prefilled, const uint32_t* decoded,
             const uint32_t* kv_device, const uint32_t* pred_len, const double* f_t, const uint8_t* protected_,
             int64_t n, int64_t demand, int64_t used, int64_t capacity, const ss_profile* profile,
             int32_t dependency_rule, int32_t select, ss_victim* victims, int64_t* n_victims, int32_t* skipped,
             int64_t* n_skipped, int32_t* failed, void* stream) {
    using namespace ss;
    if (n < 0 || !profile) return fail(SS_ERR_INVALID_ARG, "bad arguments");
    if (n > 0 && (!prompt || !prefilled || !decoded || !kv_device || !pred_len || !f_t || !victims ||
                  (select && (!ev_keys || !protected_ || !skipped))))
        return fail(SS_ERR_INVALID_ARG, "null input");
    if (n >= (1ll << 31)) return fail(SS_ERR_UNSUPPORTED, "more than 2^31 residents");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t nn = (size_t)(n > 0 ? n : 1);
    const size_t dev_b = a16(nn * sizeof(ss_key4)) + 5 * a16(nn * 4) + a16(nn * 8) + a16(nn) +
                         a16(nn * sizeof(ss_victim)) + a16(nn * 4) + a16(3 * 8);
    std::lock_guard<std::mutex> lk(g_ev.mu);
    int rc = ensure(g_ev, dev_b, 3 * 8);
    if (rc) return rc;
    char* p = (char*)g_ev.buf;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += a16(bytes);
        return (void*)r;
    };
    EvArgs a;
    ss_key4* d_k = (ss_key4*)take(nn * sizeof(ss_key4));
    uint32_t* d_pr = (uint32_t*)take(nn * 4);
    uint32_t* d_pf = (uint32_t*)take(nn * 4);
    uint32_t* d_de = (uint32_t*)take(nn * 4);
    uint32_t* d_kv = (uint32_t*)take(nn * 4);
    uint32_t* d_pl = (uint32_t*)take(nn * 4);
    double* d_ft = (double*)take(nn * 8);
    uint8_t* d_pt = (uint8_t*)take(nn);
    ss_victim* d_v = (ss_victim*)take(nn * sizeof(ss_victim));
    int* d_sk = (int*)take(nn * 4);
    long long* d_c = (long long*)take(3 * 8);
    if (n > 0) {
        if (select) cudaMemcpyAsync(d_k, ev_keys, (size_t)n * sizeof(ss_key4), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_pr, prompt, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_pf, prefilled, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_de, decoded, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_kv, kv_device, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_pl, pred_len, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_ft, f_t, (size_t)n * 8, cudaMemcpyHostToDevice, st);
        if (select) cudaMemcpyAsync(d_pt, protected_, (size_t)n, cudaMemcpyHostToDevice, st);
    }
    a.keys = d_k;
    a.prompt = d_pr;
    a.prefilled = d_pf;
    a.decoded = d_de;
    a.kv_device = d_kv;
    a.pred_len = d_pl;
    a.f_t = d_ft;
    a.prot = d_pt;
    a.n = n;
    a.demand = demand;
    a.used = used;
    a.cap = capacity;
    a.P = *profile;
    a.dep = dependency_rule;
    a.select = select;
    a.victims = d_v;
    a.skipped = d_sk;
    a.counts = d_c;
    evict_kernel<<<1, 32, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    cudaMemcpyAsync(g_ev.host, d_c, 3 * 8, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    const long long* c = (const long long*)g_ev.host;
    if (c[0] > 0) cudaMemcpy(victims, d_v, (size_t)c[0] * sizeof(ss_victim), cudaMemcpyDeviceToHost);
    if (c[1] > 0 && skipped) cudaMemcpy(skipped, d_sk, (size_t)c[1] * 4, cudaMemcpyDeviceToHost);
    if (n_victims) *n_victims = c[0];
    if (n_skipped) *n_skipped = c[1];
    if (failed) *failed = (int)c[2];
    return SS_OK;
}

}  // extern "C"
