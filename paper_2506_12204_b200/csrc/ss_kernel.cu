// ss_kernel.cu — warp-per-trace semantic scheduler for sm_100a.
//
// One warp owns one arrival trace and runs every scheduler round of it
// (the reference's Simulator.run loop, engine.py:202-224) without leaving the
// SM. Traces are independent, so warps pull trace ids from a global counter
// (persistent, load-balanced).
//
// Per-trace state:
//   * dispatch queue = sorted FRONT (64 packed keys, shared memory) + unsorted
//     BACK (HBM) + a sorted RUN (HBM, the bulk admission sorted grid-wide by
//     ss_prepass.cu, consumed from its front); every BACK / RUN key is larger
//     than every FRONT key, so the top-b candidates are FRONT[0..b) and the
//     dual heap of heaps.py:32-237 becomes a merge-by-rank in shared memory.
//     The FRONT is refilled with a warp bitonic top-32 of the BACK merged with
//     the next 32 RUN keys when it runs short.
//   * ongoing batch (engine.py:165): one record per lane, kept sorted by key,
//     stored in shared memory between rounds (keys stay in registers).
//   * resident set (the eviction heap, heaps.py:174-207) is an unsorted HBM
//     list scanned with a warp arg-max only when memory is short.
//   * per-request state is two 16-byte HBM records: static (prompt, true
//     output, predicted length, rank|tie) and dynamic (f_t, decoded, flags).
//
// Packed dispatch key (requests.py:81-91, engine.py:114-123), 96 bits:
//   hi = rank:8 | f_t bits 62..7        lo = f_t bits 6..0 | tie:25
// f_t > 0 for every live request, so its IEEE bits order like the value;
// tie = rank of (arrival, id) inside the trace. The order is total, which
// makes heap shape irrelevant: any exact top-b reproduces the heap's pops.
//
// All float64 arithmetic goes through ss_costs.cuh in the reference's
// association order with explicit round-to-nearest intrinsics (no FMA).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ss_common.cuh"
#include "ss_costs.cuh"
#include "ss_kernel.cuh"

#ifdef SS_EVICT_NOINLINE
#define SS_EVICT_INLINE __device__ __noinline__
#else
#define SS_EVICT_INLINE __device__ __forceinline__
#endif
#ifndef SS_MINB
#define SS_MINB 4  // min resident CTAs per SM requested from ptxas (register cap: 128)
#endif
#ifndef SS_CHUNK_UNROLL
#define SS_CHUNK_UNROLL 1  // unroll of the chunk's member loop
#endif
#ifndef SS_REFILL_AHEAD
#define SS_REFILL_AHEAD 2  // chunks of 32 BACK keys in flight while refill merges one
#endif
#ifndef SS_CHUNK_MIN
#define SS_CHUNK_MIN 4  // shortest static bound for which a stretch runs a lane-per-round chunk
#endif

namespace ss {

constexpr int kChunkUnroll = SS_CHUNK_UNROLL;
#ifndef SS_DQ_PERROUND
#define SS_DQ_PERROUND 0  // stretches behind queued decoding candidates in the per-round kernels too
                          // (measured: config D 91.5 -> 104 ms, its stretches end before they pay)
#endif
constexpr bool kDqPerRound = SS_DQ_PERROUND != 0;
#ifndef SS_CHAIN_STEP
#define SS_CHAIN_STEP 4  // clock-chain rounds per uniform loop step in a chunk (8: 3% slower, code size)
#endif
constexpr int kChainStep = SS_CHAIN_STEP;
constexpr int kRefillAhead = SS_REFILL_AHEAD;

// a request's state as one unit: static record, dynamic record, slot
struct __align__(16) MemS {
    uint4 st;      // prompt, true_out, pred_len, rank << 24 | tie
    double ft;     // \ dynamic record (Dyn)
    uint32_t dec;  //  |
    uint32_t flg;  // /
    uint32_t slot, _pad0, _pad1, _pad2;
};

// trace state touched once per round or less: shared memory, lane 0 writes
struct Cold {
    long long evictions, peak, s_pool, s_granted, s_victims, s_res, logpos, logcap;
    unsigned long long dpend;  // digest terms of the current eviction call
    uint32_t* log;
    long long rbase;  // this trace's sorted RUN in w.S starts at rbase + rpos
    int rpos, bulk;   // RUN cursor; requests admitted in bulk (first round)
    int dense;        // no unservable request: pending index == slot
    int nuns, lost, anomalies, n;
    int dbg;  // SS_DEBUG_ANOM builds: general-path rounds run with anom set
    Key dqk;  // stretch with queued decoding candidates: the best one's key (the last member must stay below it)
};

struct WarpSmem {
    Key F[FCAP];    // sorted queue front
    Key X[64];      // scratch keys (pool ranking: candidates 0..31, ongoing 32..63)
    MemS M[32];     // member hand-off between lanes
    MemS OM[32];    // ongoing records, lane order = key order
    Cold c;
};

__device__ __forceinline__ uint32_t m_prompt(const MemS& m) { return m.st.x; }
__device__ __forceinline__ uint32_t m_tout(const MemS& m) { return m.st.y; }
__device__ __forceinline__ uint32_t m_mid(const MemS& m) { return m.st.z; }
__device__ __forceinline__ uint32_t m_rank(const MemS& m) { return m.st.w >> 24; }
__device__ __forceinline__ uint32_t m_tie(const MemS& m) { return m.st.w & SLOT_MASK; }

__device__ __forceinline__ Key kshfl(const Key& k, int src) {
    Key r;
    r.hi = __shfl_sync(FULL, k.hi, src);
    r.lo = __shfl_sync(FULL, k.lo, src);
    r.aux = __shfl_sync(FULL, k.aux, src);
    return r;
}
__device__ __forceinline__ Key kshfl_down(const Key& k, int d) {
    Key r;
    r.hi = __shfl_down_sync(FULL, k.hi, d);
    r.lo = __shfl_down_sync(FULL, k.lo, d);
    r.aux = __shfl_down_sync(FULL, k.aux, d);
    return r;
}
__device__ __forceinline__ Key kshfl_xor(const Key& k, int m) {
    Key r;
    r.hi = __shfl_xor_sync(FULL, k.hi, m);
    r.lo = __shfl_xor_sync(FULL, k.lo, m);
    r.aux = __shfl_xor_sync(FULL, k.aux, m);
    return r;
}
// A branch on a warp-uniform value that the compiler cannot prove uniform
// (smem / global loads, call results, loop-carried counters) makes ptxas guard
// every later shuffle and vote of the loop with a divergence check (BRA.DIV)
// and an out-of-line collective fallback. Routing such conditions through a
// vote makes them provably uniform: no guards, a third less code.
__device__ __forceinline__ bool uni(bool x) { return __all_sync(0xffffffffu, x); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

template <int POL>
__device__ __forceinline__ Key mem_key(const MemS& m) {
    return make_key<POL>(m_rank(m), m.ft, m_tie(m), m.slot, (m.flg & F_STAGE) == ST_DEC);
}

__device__ __forceinline__ Key* BK(const KArgs& A) { return reinterpret_cast<Key*>(A.w.B); }
__device__ __forceinline__ Key* INS(const KArgs& A) { return reinterpret_cast<Key*>(A.w.ins); }
__device__ __forceinline__ uint4* STA(const KArgs& A) { return reinterpret_cast<uint4*>(A.w.st); }
__device__ __forceinline__ Dyn* DYN(const KArgs& A) { return reinterpret_cast<Dyn*>(A.w.dy); }

__device__ __forceinline__ unsigned long long dbits(double x) {
    return (unsigned long long)__double_as_longlong(x);
}

// --------------------------------------------------------------------------
// trace context: hot, warp-uniform values in registers
// --------------------------------------------------------------------------
struct Trace {
    long long off;
    long long used;
    double clock;
    double next_ready;  // ready time of the next pending request (inf if none)
    int npend, cursor;
    int nF, nB, nR, nO, nins;
    int nRun;  // keys left in the sorted RUN
    int rounds, status;
};

struct Env {
    const KArgs* A;
    WarpSmem* sm;
    int lane;
};

__device__ __forceinline__ void load_mem(const KArgs& A, long long off, uint32_t slot, MemS& m) {
    const long long g = off + slot;
    m.st = STA(A)[g];
    const Dyn d = DYN(A)[g];
    m.ft = d.ft;
    m.dec = d.dec;
    m.flg = d.flg;
    m.slot = slot;
}
__device__ __forceinline__ void store_dyn(const KArgs& A, long long g, double ft, uint32_t dec, uint32_t flg) {
    Dyn d;
    d.ft = ft;
    d.dec = dec;
    d.flg = flg;
    DYN(A)[g] = d;
}
__device__ __forceinline__ uint32_t* FLG(const KArgs& A, long long g) { return &DYN(A)[g].flg; }
// read-modify-write of a request's flags in HBM (copies of one request in other
// lanes may hold stale register values, so never write a lane's copy back)
__device__ __forceinline__ uint32_t flg_update(const KArgs& A, long long g, uint32_t clear, uint32_t set) {
    uint32_t* fp = FLG(A, g);
    const uint32_t f = (*fp & ~clear) | set;
    *fp = f;
    return f;
}

// ---- queue front / back maintenance --------------------------------------

// Insert up to 32 keys (one per lane, `valid`) into the queue (FRONT+BACK).
struct QState {
    long long off;
    int nF, nB;
};
__device__ __noinline__ int2 q_insert32(const KArgs* Ap, WarpSmem* sm, long long off, int nF, int nB, int nRun,
                                        Key key, bool valid) {
    const KArgs& A = *Ap;
    const int lane = threadIdx.x & 31;
    QState T{off, nF, nB};
    const unsigned lt = lanemask_lt();
    Key fmax;
    bool have_f = T.nF > 0;
    if (have_f) fmax = sm->F[T.nF - 1];
    bool toF = valid && ((T.nB == 0 && nRun == 0) || (have_f && klt(key, fmax)));
    bool toB = valid && !toF;
    unsigned bm = __ballot_sync(FULL, toB);
    if (toB) BK(A)[T.off + T.nB + __popc(bm & lt)] = key;
    T.nB += __popc(bm);
    unsigned fm = __ballot_sync(FULL, toF);
    int nI = __popc(fm);
    if (nI == 0) return make_int2(T.nF, T.nB);
    // rank of each insert among inserts
    int ii = __popc(fm & lt);
    if (toF) sm->X[ii] = key;
    __syncwarp();
    int rank_i = 0;
    for (int k = 0; k < nI; k++) {
        Key x = sm->X[k];
        rank_i += klt(x, key) ? 1 : 0;
    }
    // position of each insert in the current FRONT (binary search)
    int lo = 0, hi = T.nF;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const bool below = klt(sm->F[mid], key);  // branch-free step
        lo = below ? mid + 1 : lo;
        hi = below ? hi : mid;
    }
    int pos_i = lo + rank_i;
    // FRONT entries shift by the number of inserts below them
    Key e0, e1;
    bool h0 = lane < T.nF, h1 = lane + 32 < T.nF;
    if (h0) e0 = sm->F[lane];
    if (h1) e1 = sm->F[lane + 32];
    int s0 = 0, s1 = 0;
    for (int k = 0; k < nI; k++) {
        Key x = sm->X[k];
        s0 += (h0 & klt(x, e0)) ? 1 : 0;
        s1 += (h1 & klt(x, e1)) ? 1 : 0;
    }
    int p0 = lane + s0, p1 = lane + 32 + s1;
    int total = T.nF + nI;
    __syncwarp();
    // write back; positions >= FCAP spill to the BACK in order
    if (h0) {
        if (p0 < FCAP) sm->F[p0] = e0;
        else BK(A)[T.off + T.nB + (p0 - FCAP)] = e0;
    }
    if (h1) {
        if (p1 < FCAP) sm->F[p1] = e1;
        else BK(A)[T.off + T.nB + (p1 - FCAP)] = e1;
    }
    if (toF) {
        if (pos_i < FCAP) sm->F[pos_i] = key;
        else BK(A)[T.off + T.nB + (pos_i - FCAP)] = key;
    }
    __syncwarp();
    if (total > FCAP) {
        T.nB += total - FCAP;
        T.nF = FCAP;
    } else {
        T.nF = total;
    }
    return make_int2(T.nF, T.nB);
}

// Remove FRONT entries flagged in `rm` (bit i = FRONT[i]).
__device__ void f_compact(const Env& E, Trace& T, unsigned long long rm) {
    if (uni(rm == 0ull)) return;
    WarpSmem* sm = E.sm;
    const int lane = E.lane;
    const unsigned lt = lanemask_lt();
    bool k0 = lane < T.nF && !((rm >> lane) & 1ull);
    bool k1 = lane + 32 < T.nF && !((rm >> (lane + 32)) & 1ull);
    unsigned b0 = __ballot_sync(FULL, k0), b1 = __ballot_sync(FULL, k1);
    Key e0, e1;
    if (k0) e0 = sm->F[lane];
    if (k1) e1 = sm->F[lane + 32];
    __syncwarp();
    if (k0) sm->F[__popc(b0 & lt)] = e0;
    if (k1) sm->F[__popc(b0) + __popc(b1 & lt)] = e1;
    __syncwarp();
    T.nF = __popc(b0) + __popc(b1);
}

// Bitonic sort of one key per lane; ascending if `asc`.
__device__ __forceinline__ Key bitonic32(Key x, int lane, bool asc) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            Key y = kshfl_xor(x, j);
            bool up = ((lane & k) == 0) == asc;
            bool lower = (lane & j) == 0;
            bool take_min = (lower == up);
            bool ylt = klt(y, x);
            if (take_min ? ylt : klt(x, y)) x = y;
        }
    }
    return x;
}

// Move the 32 smallest keys of BACK + RUN (or all of them) behind the FRONT.
// Returns {nF, nB, keys taken from the RUN}.
__device__ __noinline__ int4 refill(const KArgs* Ap, WarpSmem* sm, long long off, int nF, int nB, const Key* run,
                                    int nRun) {
    const KArgs& A = *Ap;
    const int lane = threadIdx.x & 31;
    QState T{off, nF, nB};
    Key S = kinf();  // running top-32, ascending across lanes
    // the next kRefillAhead chunks' loads are in flight while the current one is merged
    Key xq[kRefillAhead];
#pragma unroll
    for (int d = 0; d < kRefillAhead; d++) xq[d] = 32 * d + lane < T.nB ? BK(A)[T.off + 32 * d + lane] : kinf();
    for (int base = 0; uni(base < T.nB); base += 32) {
        Key x = xq[0];
#pragma unroll
        for (int d = 0; d + 1 < kRefillAhead; d++) xq[d] = xq[d + 1];
        const int in = base + 32 * kRefillAhead + lane;
        xq[kRefillAhead - 1] = in < T.nB ? BK(A)[T.off + in] : kinf();
        Key smax = kshfl(S, 31);
        unsigned qm = __ballot_sync(FULL, klt(x, smax));
        if (!qm) continue;
        if (__popc(qm) <= 6) {
            // few keys beat the running 32nd: insert them one by one (rank by ballot,
            // shift the larger entries up one lane, the largest drops out)
            while (qm) {
                const int src = __ffs(qm) - 1;
                qm &= qm - 1;
                const Key y = kshfl(x, src);
                const int pos = __popc(__ballot_sync(FULL, klt(S, y)));
                Key up;
                up.hi = __shfl_up_sync(FULL, S.hi, 1);
                up.lo = __shfl_up_sync(FULL, S.lo, 1);
                up.aux = __shfl_up_sync(FULL, S.aux, 1);
                if (lane > pos) S = up;
                else if (lane == pos) S = y;
            }
            continue;
        }
        x = bitonic32(x, lane, false);                 // descending
        if (klt(x, S)) S = x;                          // bitonic sequence
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {             // merge ascending
            Key y = kshfl_xor(S, j);
            bool lower = (lane & j) == 0;
            if (lower ? klt(y, S) : klt(S, y)) S = y;
        }
    }
    Key r = kinf();  // the RUN's next 32 keys are its 32 smallest (ascending)
    if (uni(nRun > 0)) {
        if (lane < nRun) r = run[lane];
        Key rr = kshfl(r, 31 - lane);                  // descending
        if (klt(rr, S)) S = rr;                        // 32 smallest of both, bitonic
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            Key y = kshfl_xor(S, j);
            bool lower = (lane & j) == 0;
            if (lower ? klt(y, S) : klt(S, y)) S = y;
        }
    }
    const int avail = T.nB + nRun;
    int K = avail < 32 ? avail : 32;
    if (lane < K) sm->F[T.nF + lane] = S;
    Key thr = kshfl(S, K - 1);
    __syncwarp();
    T.nF += K;
    const int from_run = __popc(__ballot_sync(FULL, lane < nRun && !klt(thr, r)));
    if (uni(K > from_run)) {
        // compact the BACK, dropping the selected keys (all <= thr)
        const unsigned lt = lanemask_lt();
        int w = 0;
        // survivors land at or below their own index, never in the chunks loaded ahead
        Key yq[kRefillAhead];
#pragma unroll
        for (int d = 0; d < kRefillAhead; d++) yq[d] = 32 * d + lane < T.nB ? BK(A)[T.off + 32 * d + lane] : kinf();
        for (int base = 0; uni(base < T.nB); base += 32) {
            int i = base + lane;
            const Key x = yq[0];
#pragma unroll
            for (int d = 0; d + 1 < kRefillAhead; d++) yq[d] = yq[d + 1];
            const int in = base + 32 * kRefillAhead + lane;
            yq[kRefillAhead - 1] = in < T.nB ? BK(A)[T.off + in] : kinf();
            const bool keep = i < T.nB && klt(thr, x);
            unsigned km = __ballot_sync(FULL, keep);
            __syncwarp();
            if (keep) BK(A)[T.off + w + __popc(km & lt)] = x;
            w += __popc(km);
            __syncwarp();
        }
        T.nB = w;
    }
    return make_int4(T.nF, T.nB, from_run, 0);
}

// ---- logging ---------------------------------------------------------------
__device__ __forceinline__ void log_put(const Cold& c, long long pos, uint32_t v) {
    if (c.log && pos < c.logcap) c.log[pos] = v;
}

struct Round {
    unsigned G;                // granted batch positions
    unsigned evmask;           // positions evicted with a recorded decision
    int ndec;                  // recorded decisions this round
    unsigned long long rmF;    // FRONT entries to drop at the rebuild
};

__device__ __forceinline__ void set_status(Trace& T, int st) {
    if (T.status == SS_TRACE_OK) T.status = st;
}

// Index of slot v's live entry in this round's re-queue list, or -1.
__device__ int ins_find(const KArgs& A, const Trace& T, uint32_t v, int lane) {
    for (int base = 0; uni(base < T.nins); base += 32) {
        int i = base + lane;
        bool hit = i < T.nins && (INS(A)[T.off + i].aux & SLOT_MASK) == v;
        unsigned hm = __ballot_sync(FULL, hit);
        if (hm) return base + __ffs(hm) - 1;
    }
    return -1;
}

// heap.delete_by_id for a queued request (heaps.py:67-70): FRONT, BACK or the
// pending re-queue list. Caller updates the flags.
__device__ void q_delete(const Env& E, Trace& T, Round& R, uint32_t v, uint32_t flg) {
    const KArgs& A = *E.A;
    WarpSmem* sm = E.sm;
    const int lane = E.lane;
    if (uni(!(flg & F_Q))) return;
    if (uni(flg & F_INS)) {
        int idx = ins_find(A, T, v, lane);
        if (idx >= 0 && lane == 0) INS(A)[T.off + idx].aux = SLOT_MASK;  // dead entry
        __syncwarp();
        return;
    }
    bool f0 = lane < T.nF && !((R.rmF >> lane) & 1ull) && (sm->F[lane].aux & SLOT_MASK) == v;
    bool f1 = lane + 32 < T.nF && !((R.rmF >> (lane + 32)) & 1ull) && (sm->F[lane + 32].aux & SLOT_MASK) == v;
    unsigned m0 = __ballot_sync(FULL, f0), m1 = __ballot_sync(FULL, f1);
    if (m0 | m1) {
        if (m0) R.rmF |= 1ull << (__ffs(m0) - 1);
        else R.rmF |= 1ull << (32 + __ffs(m1) - 1);
        return;
    }
    int found = -1;
    for (int base = 0; uni(base < T.nB && found < 0); base += 32) {
        int i = base + lane;
        bool hit = i < T.nB && (BK(A)[T.off + i].aux & SLOT_MASK) == v;
        unsigned hm = __ballot_sync(FULL, hit);
        if (hm) found = base + __ffs(hm) - 1;
    }
    if (uni(found >= 0)) {
        if (lane == 0) BK(A)[T.off + found] = BK(A)[T.off + T.nB - 1];
        T.nB -= 1;
    }
    __syncwarp();
}

// Evict one victim for member `kslot` (kvcache.py:160-175): the resident with
// the largest dispatch key that is neither granted this round nor `kslot`.
// Returns false if there is none (AdmissionFailure). Cold path: not inlined.
template <int POL, bool LOGGING>
SS_EVICT_INLINE bool evict_one(const Env& E, Trace& T, Round& R, uint32_t kslot, int m, MemS& mem,
                                       unsigned& vcall) {
    const KArgs& A = *E.A;
    const int lane = E.lane;
    Cold& c = E.sm->c;
    const ss_profile& P = A.P.profile;
    if (uni(*A.w.sel == SS_SEL_NO_EVICT)) {  // the resident list is not kept in this regime
        set_status(T, SS_TRACE_INTERNAL);
        return false;
    }
    Key best;
    bool have = false;
    int best_ri = -1;
    for (int base = 0; uni(base < T.nR); base += 32) {
        int i = base + lane;
        if (i < T.nR) {
            uint32_t s = A.w.R[T.off + i];
            long long g = T.off + s;
            const Dyn d = DYN(A)[g];
            if (!(d.flg & F_GRANT) && s != kslot) {
                const uint32_t w = STA(A)[g].w;
                Key k = make_key<POL>(w >> 24, d.ft, w & SLOT_MASK, s, true);
                if (!have || klt(best, k)) {
                    best = k;
                    have = true;
                    best_ri = i;
                }
            }
        }
    }
    if (!have) best.hi = 0, best.lo = 0, best.aux = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Key ok = kshfl_xor(best, o);
        bool oh = __shfl_xor_sync(FULL, have, o);
        int ori = __shfl_xor_sync(FULL, best_ri, o);
        if (oh && (!have || klt(best, ok))) {
            best = ok;
            have = true;
            best_ri = ori;
        }
    }
    if (uni(!have)) return false;
    const uint32_t v = best.aux & SLOT_MASK;
    const long long gv = T.off + v;
    // ---- should_recompute (kvcache.py:81-134), evaluated redundantly per lane
    MemS vm;
    load_mem(A, T.off, v, vm);
    const uint32_t prompt = m_prompt(vm), dec = vm.dec, flg = vm.flg;
    const double ftb = vm.ft;
    const long long freed = (long long)prompt + dec;
    bool pf = (flg & F_PF) != 0;
    int action;
    long long psaved;
    if (pf && should_cache_prefill(prompt, P)) {
        action = 0;
        psaved = prompt;
    } else {
        action = 1;
        psaved = 0;
        pf = false;
    }
    long long saved = dec > 0 ? optimal_save_tokens(prompt, dec, P) : 0;
    if (action == 1 && A.P.dependency_rule) saved = 0;
    const long long discarded = (long long)dec - saved;
    const double fta = remaining_time(prompt, m_mid(vm), pf ? prompt : 0, saved, psaved + saved, P);
    T.used -= freed;
    const Key nkey = make_key<POL>(m_rank(vm), fta, m_tie(vm), v, false);
    // heap: delete_by_id if queued, then insert with the new key
    int ins_idx = -1;
    if (uni((flg & F_Q) && (flg & F_INS))) ins_idx = ins_find(A, T, v, lane);
    else q_delete(E, T, R, v, flg);
    const uint32_t nflg = (flg & ~(F_STAGE | F_PF)) | ST_WAIT | (pf ? F_PF : 0u) | F_Q | F_INS;
    if (lane == 0) {
        uint32_t last = A.w.R[T.off + T.nR - 1];  // resident list: swap-remove
        A.w.R[T.off + best_ri] = last;
        A.w.rpos[T.off + last] = (uint32_t)best_ri;
        if (ins_idx >= 0) INS(A)[T.off + ins_idx] = nkey;
        else INS(A)[T.off + T.nins] = nkey;
        store_dyn(A, gv, fta, (uint32_t)saved, nflg);
        A.out.req.evictions[gv] += 1u;
        const int d = R.ndec;  // decision record: kept only if the admission succeeds
        if (LOGGING && c.log) {  // compile-time: no log code in the digest-only kernels
            long long p = c.logpos + SS_LOG_HEADER_WORDS + (long long)SS_LOG_DECISION_WORDS * d;
            unsigned long long fb = dbits(ftb), fa = dbits(fta);
            log_put(c, p + 0, v);
            log_put(c, p + 1, (uint32_t)action);
            log_put(c, p + 2, (uint32_t)saved);
            log_put(c, p + 3, (uint32_t)discarded);
            log_put(c, p + 4, (uint32_t)freed);
            log_put(c, p + 5, (uint32_t)fb);
            log_put(c, p + 6, (uint32_t)(fb >> 32));
            log_put(c, p + 7, (uint32_t)fa);
            log_put(c, p + 8, (uint32_t)(fa >> 32));
        }
        if (A.P.flags & SS_FLAG_DIGEST) {
            const unsigned long long r = (unsigned long long)T.rounds;
            c.dpend += ss_decision_term(r, (uint32_t)d, (unsigned long long)v | ((unsigned long long)action << 32),
                                        (unsigned long long)(uint32_t)saved | ((unsigned long long)(uint32_t)discarded << 32),
                                        (unsigned long long)freed, dbits(ftb), dbits(fta));
        }
        c.s_victims += 1;
    }
    if (uni(ins_idx < 0)) T.nins += 1;
    T.nR -= 1;
    R.ndec += 1;
    __syncwarp();
    // every batch copy of the victim is skipped (evicted_ids is by id) and refreshed
    const unsigned bpos = __ballot_sync(FULL, lane < m && mem.slot == v);
    vcall |= bpos;
    if ((bpos >> lane) & 1u) load_mem(A, T.off, v, mem);
    __syncwarp();
    return true;
}

// Does a stale dispatch-queue entry remain? An entry is stale
// when its stored key no longer equals the key of the request's current state,
// the request completed, or it is also an ongoing member; duplicate ongoing
// copies of one request count too. The sorted RUN holds only untouched bulk
// arrivals and is never stale.
template <int POL>
__device__ __noinline__ bool queue_has_stale(const KArgs* Ap, const WarpSmem* sm, long long off, int nF, int nB,
                                             int nO) {
    const KArgs& A = *Ap;
    const int lane = threadIdx.x & 31;
    bool st = false;
    auto check = [&](const Key& k) {
        const uint32_t s = k.aux & SLOT_MASK;
        const long long g = off + s;
        const Dyn d = DYN(A)[g];
        const uint32_t w = STA(A)[g].w;
        const Key cur = make_key<POL>(w >> 24, d.ft, w & SLOT_MASK, s, (d.flg & F_STAGE) == ST_DEC);
        return !keq(cur, k) || cur.aux != k.aux || (d.flg & F_STAGE) == ST_DONE || !(d.flg & F_Q);
    };
    if (lane < nF) st |= check(sm->F[lane]);
    if (lane + 32 < nF) st |= check(sm->F[lane + 32]);
    for (int base = 0; uni(base < nB); base += 32) {
        const int i = base + lane;
        if (i < nB) st |= check(BK(A)[off + i]);
    }
    // duplicate ongoing copies of one request (each executes separately)
    const uint32_t os = lane < nO ? sm->OM[lane].slot : (0x80000000u | (uint32_t)lane);
    const unsigned same = __match_any_sync(FULL, os);
    if (lane < nO) st |= __popc(same) > 1;
    if (lane < nO) st |= (DYN(A)[off + sm->OM[lane].slot].flg & F_Q) != 0;
    return __any_sync(FULL, st);
}


// A general round whose batch holds duplicate copies of one request (stale heap
// entries after a lost eviction decision): the copies execute one
// by one (engine.py:351-421), each seeing the previous copy's effect. Out of
// line: only stale-entry rounds of the evicting kernels come here.
struct DupOut {
    long long used;
    int nR, err;
    bool done;
};
__device__ __noinline__ DupOut progress_dups(const KArgs* Ap, long long off, uint32_t G, double clock, double end,
                                             long long cap, long long used, int nR, MemS mem) {
    const KArgs& A = *Ap;
    const ss_profile& P = A.P.profile;
    const int lane = threadIdx.x & 31;
    bool done = false;
    int err_out = 0;
                    // duplicate copies of a request: execute copies one by one,
                    // each seeing the previous copy's effect
                    unsigned gm = G;
                    while (uni(gm != 0u)) {
                        const int k = __ffs(gm) - 1;
                        gm &= gm - 1;
                        int err = 0, dn = 0, nres = 0;
                        long long alloc = 0, rel = 0;
                        if (lane == k) {
                            const long long g = off + mem.slot;
                            const Dyn d = DYN(A)[g];
                            uint32_t dec = d.dec, fl = d.flg;
                            if ((fl & F_STAGE) == ST_DONE) {
                                err = 1;  // transition(PREFILLING) from COMPLETED
                            } else {
                                if (!(fl & F_FIRST)) {
                                    A.out.req.first_scheduled[g] = clock;
                                    fl |= F_FIRST;
                                }
                                if ((fl & F_STAGE) == ST_DEC) {
                                    alloc = 1;
                                    dec += 1;
                                } else {
                                    const long long pfn = (fl & F_PF) ? (long long)m_prompt(mem) : 0;
                                    alloc = pfn + dec + ((long long)m_prompt(mem) - pfn);
                                    fl = (fl & ~F_STAGE) | ST_DEC | F_PF;
                                    nres = 1;
                                }
                                fl &= ~F_GRANT;
                                double ft;
                                if (dec >= m_tout(mem)) {
                                    dn = 1;
                                    rel = (long long)m_prompt(mem) + dec;
                                    A.out.req.finish_time[g] = end;
                                    ft = 0.0;
                                    fl = (fl & ~F_STAGE) | ST_DONE;
                                } else {
                                    ft = remaining_time(m_prompt(mem), m_mid(mem), m_prompt(mem), dec, 0, P);
                                }
                                store_dyn(A, g, ft, dec, fl);
                            }
                        }
                        err = __shfl_sync(FULL, err, k);
                        dn = __shfl_sync(FULL, dn, k);
                        nres = __shfl_sync(FULL, nres, k);
                        alloc = __shfl_sync(FULL, alloc, k);
                        rel = __shfl_sync(FULL, rel, k);
                        const uint32_t s = __shfl_sync(FULL, mem.slot, k);
                        if (uni(err || alloc > cap - used)) {
                            err_out = 1;
                            break;
                        }
                        used += alloc;
                        if (lane == k) done = dn != 0;
                        if (lane == 0 && nres) {
                            A.w.R[off + nR] = s;
                            A.w.rpos[off + s] = (uint32_t)nR;
                        }
                        if (nres) nR += 1;
                        __syncwarp();
                        if (dn) {
                            if (lane == 0) {
                                const uint32_t ri = A.w.rpos[off + s];
                                const uint32_t last = A.w.R[off + nR - 1];
                                A.w.R[off + ri] = last;
                                A.w.rpos[off + last] = ri;
                            }
                            nR -= 1;
                            used -= rel;
                        }
                        __syncwarp();
                    }
    DupOut o;
    o.used = used;
    o.nR = nR;
    o.err = err_out;
    o.done = done;
    return o;
}


// Merged positions of candidates and ongoing copies while stale heap entries may
// exist: a stable sort of (candidates + ongoing) by current key;
// equal keys are copies of one request, ordered by pool position. Out of line.
__device__ __noinline__ int2 rank_general(WarpSmem* sm, int nc, int nO, unsigned cmask, bool c_elig, bool has_o, Key ck,
                                          Key okey) {
    const int lane = threadIdx.x & 31;
    int cnt_c = 0, cnt_o = 0;
    if (c_elig) sm->X[lane] = ck;
    if (has_o) sm->X[32 + lane] = okey;
    __syncwarp();
    for (int k = 0; uni(k < nc); k++) {
        if (!((cmask >> k) & 1u)) continue;
        Key x = sm->X[k];
        if (c_elig && (klt(x, ck) || (keq(x, ck) && k < lane))) cnt_c++;
        if (has_o && (klt(x, okey) || keq(x, okey))) cnt_o++;
    }
    for (int k = 0; uni(k < nO); k++) {
        Key x = sm->X[32 + k];
        if (c_elig && klt(x, ck)) cnt_c++;
        if (has_o && (klt(x, okey) || (keq(x, okey) && k < lane))) cnt_o++;
    }
    return make_int2(cnt_c, cnt_o);
}


// Push-backs of a general round while stale heap entries may exist (DESIGN.md
// §5): candidates not selected whose stored key is stale are re-queued with
// their current key (heaps.py insert after pop); pushed-back ongoing copies are
// re-queued, and one whose request is still queued is the reference's
// DuplicateRequestError (heaps.py:49-51). Out of line.
struct PushOut {
    unsigned rm;
    int nins, err;
};
__device__ __noinline__ PushOut push_back_stale(const KArgs* Ap, WarpSmem* sm, long long off, int nins, bool has_c,
                                                bool c_sel, Key ck, bool pushed, Key okey) {
    const KArgs& A = *Ap;
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    PushOut o;
    o.err = 0;
    const bool refresh = has_c && !c_sel && !keq(ck, sm->F[lane]);
    const unsigned rm2 = __ballot_sync(FULL, refresh);
    o.rm = rm2;
    if (refresh) {
        const uint32_t s = ck.aux & SLOT_MASK;
        INS(A)[off + nins + __popc(rm2 & lt)] = ck;
        *FLG(A, off + s) = *FLG(A, off + s) | F_INS;
    }
    nins += __popc(rm2);
    __syncwarp();
    unsigned pm = __ballot_sync(FULL, pushed);
    while (pm) {
        const int k = __ffs(pm) - 1;
        pm &= pm - 1;
        const uint32_t s = sm->OM[k].slot;
        const uint32_t f = *FLG(A, off + s);
        if (uni(f & F_Q)) {
            o.err = 1;
            break;
        }
        const Key kk = kshfl(okey, k);
        if (lane == 0) {
            *FLG(A, off + s) = f | F_Q | F_INS;
            INS(A)[off + nins] = kk;
        }
        nins += 1;
        __syncwarp();
    }
    o.nins = nins;
    return o;
}

// ---- SS_DEBUG_TIMING builds: warp-cycles per kernel section -----------------
#ifdef SS_DEBUG_TIMING
constexpr int SS_DBG_SLOTS = 32;  // 16 section cycle counters + 16 event counters
__device__ unsigned long long g_dbg_cycles[SS_DBG_SLOTS];
constexpr int SS_DBG_TRACES = 8192;  // per-trace section cycles of the first traces (debug builds)
__device__ unsigned long long g_dbg_trace[SS_DBG_TRACES][SS_DBG_SLOTS];
#define SS_SECT(s_)                                                   \
    do {                                                              \
        const long long now_ = clock64();                             \
        dbg_acc[dbg_cur] += (unsigned long long)(now_ - dbg_t);       \
        dbg_t = now_;                                                 \
        dbg_cur = (s_);                                               \
    } while (0)
#define SS_DCOUNT(k_, v_) (dbg_acc[16 + (k_)] += (unsigned long long)(v_))
#else
#define SS_SECT(s_) ((void)0)
#define SS_DCOUNT(k_, v_) ((void)0)
#endif
// sections: 0 init/admission/top, 1 fast path per-round body, 2 chunk, 3 general round, 4 outputs,
// 5 stretch entry, 6 stretch round vote, 7 stretch order check; general round: 3 composition,
// 8 KV admission, 9 batch duration, 10 progress, 11 record, 12 ongoing rebuild, 13 queue rebuild,
// 14 eviction calls (counter 4: evict_one calls), 15 queue refill (counter 5)
// counters: 8 chunks, 9 chunk rounds, 10 per-round fast rounds, 11 general rounds

// ---- per-lane member quantities (32-bit: token counts of one request) -------
struct MemQ {
    bool isdec;
    uint32_t pfn, kvh, kvd, imm, est;
};
__device__ __forceinline__ MemQ mem_q(const MemS& m) {
    MemQ q;
    q.isdec = (m.flg & F_STAGE) == ST_DEC;
    q.pfn = (m.flg & F_PF) ? m_prompt(m) : 0u;
    q.kvh = q.isdec ? 0u : q.pfn + m.dec;
    q.kvd = q.isdec ? m_prompt(m) + m.dec : 0u;
    q.imm = q.isdec ? 1u : q.kvh + (m_prompt(m) - q.pfn) + 1u;
    const long long e = (long long)m_prompt(m) + m_mid(m) - q.kvd;
    q.est = e > 0 ? (uint32_t)e : 0u;
    return q;
}

// --------------------------------------------------------------------------
// the kernel
// --------------------------------------------------------------------------
// MODE bit 0: schedule digest, bit 1: per-round log (compile-time so the
// common configuration carries no branches for the features it does not use)
template <int POL, int MODE>
__global__ void __launch_bounds__(32 * WPB, SS_MINB) sched_kernel(const __grid_constant__ KArgs args) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const KArgs& A = args;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem* sm = reinterpret_cast<WarpSmem*>(smem_raw) + wib;
    Cold& c = sm->c;
    Env E{&A, sm, lane};
    const ss_profile& P = A.P.profile;
    const int b = A.P.batch_size;
    const long long cap = A.P.memory_capacity;
    const unsigned lt = lanemask_lt();
    constexpr bool want_digest = (MODE & 1) != 0;
    constexpr bool logging = (MODE & 2) != 0;
    // MODE bit 2: the chunked-stretch variant. Semantic runs launch both variants
    // back to back; the one the prepass did not select (ss_prepass.cu
    // select_kernel: chunks only when the KV budget can never bind) exits at once.
    constexpr bool chunking = (MODE & 4) != 0;
    // MODE bit 3 (with bit 2): no trace can ever evict (select_kernel's footprint rule).
    // The eviction path, the stale-entry (anomaly) handling it can cause and the
    // resident list (eviction candidates) are compiled out: a denser hot loop.
    constexpr bool noev = (MODE & 8) != 0;
    // MODE bit 4: decode_batch_cost "sum" (Neumaier sum of the members' decode steps)
    // compiled in; the other kernels carry only the "max" batch duration
    constexpr bool sum_k = (MODE & 16) != 0;
#ifdef SS_LEAN_TEST  // experiment: timing without the stale-entry machinery (wrong on anomaly traces)
    constexpr bool anom_ok = false;
#else
    constexpr bool anom_ok = !noev;  // stale heap entries can arise (an eviction can lose its decisions)
#endif
    const int sel = *A.w.sel;
    if (POL == SS_POLICY_SEMANTIC &&
        sel != (noev ? SS_SEL_NO_EVICT : (chunking ? SS_SEL_CHUNKED : SS_SEL_PERROUND)))
        return;
    const bool track_res = !noev;
#ifdef SS_DEBUG_TIMING
    unsigned long long dbg_acc[SS_DBG_SLOTS] = {0};
    long long dbg_t = clock64();
    int dbg_cur = 0;
#endif

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(A.w.next_trace, 1);
        t = __shfl_sync(FULL, t, 0);
        if (uni(t >= A.in.n_traces)) break;

#ifdef SS_DEBUG_TIMING
        unsigned long long dbg_snap[SS_DBG_SLOTS];
        for (int i = 0; i < SS_DBG_SLOTS; i++) dbg_snap[i] = dbg_acc[i];
#endif
#ifdef SS_DEBUG_TRACE_TIME
        unsigned long long dbg_t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
#endif
        Trace T;
        T.off = A.in.trace_offsets[t];
        const int n = (int)(A.in.trace_offsets[t + 1] - T.off);
        T.clock = 0.0;
        T.used = 0;
        T.nF = T.nB = T.nR = T.nO = T.nins = 0;
        T.rounds = 0;
        T.status = SS_TRACE_OK;
        bool anom = false;  // a stale heap entry may exist: general (exact) round path
        if (lane == 0) {
            c.evictions = c.s_pool = c.s_granted = c.s_victims = c.s_res = 0;
            c.logpos = 0;
            c.log = nullptr;
            c.logcap = 0;
            if ((A.P.flags & SS_FLAG_ROUND_LOG) && A.out.round_log && A.out.log_offsets) {
                c.log = A.out.round_log + A.out.log_offsets[t];
                c.logcap = A.out.log_offsets[t + 1] - A.out.log_offsets[t];
            }
            c.nuns = c.lost = c.anomalies = c.dbg = 0;
            c.n = n;
        }
        unsigned long long dig = 0ull;
        long long peak = 0;

        // ---- init (engine.py:183-199). Records, f_t and output slots were
        // written grid-wide by the prepass (ss_prepass.cu); here only the
        // pending list when some request is unservable (pre-filter, :193-199)
        T.nRun = 0;
        const int bulkP = A.w.bulkP[t];
        const bool dense = A.w.nuns[t] == 0u;
        int nuns = 0, bulk = 0;
        if (uni(dense)) {
            T.npend = n;  // pending index == slot
            bulk = bulkP;
        } else {
            T.npend = 0;
            for (int base = 0; uni(base < n); base += 32) {
                int i = base + lane;
                bool v = i < n;
                bool serv = v && (long long)A.in.prompt_len[T.off + i] + 1 <= cap;
                unsigned sm_ = __ballot_sync(FULL, serv), um = __ballot_sync(FULL, v && !serv);
                if (serv) A.w.pend[T.off + T.npend + __popc(sm_ & lt)] = (uint32_t)i;
                if (v && !serv) A.out.unservable_slots[T.off + nuns + __popc(um & lt)] = (uint32_t)i;
                bulk += __popc(__ballot_sync(FULL, serv && i < bulkP));
                T.npend += __popc(sm_);
                nuns += __popc(um);
            }
        }
        if (lane == 0) {
            c.nuns = nuns;
            c.dense = dense ? 1 : 0;
            c.bulk = bulkP > 0 ? bulk : 0;
            c.rbase = A.w.eoff[t];
            c.rpos = 0;
        }
        // round cap: params.max_rounds, or automatic (the reference has no guard
        // and can cycle forever under some tight-memory schedules)
        const long long tokens = (long long)A.w.tok[t];
        long long round_cap = A.P.max_rounds > 0 ? A.P.max_rounds : 64 * (tokens + n) + 100000;
        if (round_cap > 0x7fffffffll) round_cap = 0x7fffffffll;
        T.cursor = 0;
        __syncwarp();
        T.next_ready = T.npend > 0 ? A.in.ready_time[T.off + (dense ? 0 : A.w.pend[T.off])] : INFINITY;

        Key okey;  // key of the ongoing record in OM[lane] (lane < nO)

        // ---- the round loop (engine.py:202-224)
        while (uni(T.status == SS_TRACE_OK)) {
            SS_SECT(0);
            // admission of prediction-ready requests (engine.py:204-206)
            const double thr = ss::add(T.clock, 1e-12);
            if (uni(T.next_ready <= thr)) {
                if (uni(T.cursor == 0 && c.bulk > 0)) {
                    // bulk admission: the group is already queued (F_Q set by the
                    // prepass) as this trace's sorted RUN
                    T.cursor = c.bulk;
                    T.nRun = c.bulk;
                }
                const bool dn = c.dense != 0;
                // ready times and admission keys (prepass, k0) of the next 32 pending
                // requests load together; the first one not admitted is the next ready time
                double nr = INFINITY;
                while (uni(T.cursor < T.npend)) {
                    int i = T.cursor + lane;
                    bool v = i < T.npend;
                    uint32_t s = 0;
                    double rdy = INFINITY;
                    Key k;
                    if (v) {
                        s = dn ? (uint32_t)i : A.w.pend[T.off + i];
                        rdy = A.in.ready_time[T.off + s];
                        k = reinterpret_cast<const Key*>(A.w.k0)[T.off + s];
                    }
                    const bool ok = rdy <= thr;
                    unsigned am = __ballot_sync(FULL, ok);
                    int cnt = am == FULL ? 32 : __ffs(~am) - 1;
                    nr = __shfl_sync(FULL, rdy, cnt & 31);
                    if (cnt == 0) break;
                    bool mine = lane < cnt;
                    if (mine) *FLG(A, T.off + s) = ST_WAIT | F_Q;
                    const int2 qs = q_insert32(&A, sm, T.off, T.nF, T.nB, T.nRun, k, mine);
                    T.nF = qs.x;
                    T.nB = qs.y;
                    T.cursor += cnt;
                    if (cnt < 32) break;
                    nr = INFINITY;
                }
                T.next_ready = nr;
            }
            const int live = T.nF + T.nB + T.nO + T.nRun;
            if (uni(live == 0)) {
                if (uni(T.cursor >= T.npend)) break;
                T.clock = T.next_ready;
                continue;
            }
            if (uni(T.nF < b && (T.nB > 0 || T.nRun > 0))) {
                SS_SECT(15);
                SS_DCOUNT(5, 1);
                const int4 qs = refill(&A, sm, T.off, T.nF, T.nB,
                                       reinterpret_cast<const Key*>(A.w.S) + c.rbase + c.rpos, T.nRun);
                T.nF = qs.x;
                T.nB = qs.y;
                T.nRun -= qs.z;
                __syncwarp();
                if (lane == 0) c.rpos += qs.z;
                __syncwarp();
                SS_SECT(0);
            }
            // stale entries are transient: once none is left the trace returns to
            // the exact fast paths (checked every 32 rounds while flagged)
#ifndef SS_NO_ANOM_EXIT
            if (anom_ok && uni(anom && (T.rounds & 31) == 0) &&
                !queue_has_stale<POL>(&A, sm, T.off, T.nF, T.nB, T.nO))
                anom = false;
#endif
            // ---- fast path: a stretch of same-batch decode rounds --------------
            // 99.5% of config-B rounds (96% under config D's tight memory) keep the
            // batch equal to the ongoing set: p* is an ongoing (decoding) request,
            // no queued decoding request is eligible (batching.py:73-88), nobody
            // needs eviction and nobody completes. Such rounds run here with the
            // members in registers, record writes deferred to the stretch's end and
            // the same arithmetic, digest terms and bookkeeping as the general
            // round below (engine.py:288-380), which handles every other round.
            if (POL == SS_POLICY_SEMANTIC && uni((!anom_ok || !anom) && T.nO > 0 && T.nO <= b)) {
                SS_SECT(5);
                const int nc0 = T.nF < b ? T.nF : b;
                const bool cdec = lane < nc0 && (sm->F[lane].aux & DEC_BIT);
                // A queued decoding candidate (a preempted member) is eligible under p*'s
                // stage rule (batching.py:73-88). With a full batch it changes nothing
                // while it ranks after the last member: the merged top-b is the ongoing
                // set and every candidate is pushed back with its unchanged key (a queued
                // request's f_t does not move; the members' only decrease, so this holds
                // for the whole stretch). A completion frees a slot the candidate would
                // take: the stretch ends after that round (dq).
                const unsigned dqm = __ballot_sync(FULL, cdec);
                const bool dq = (chunking || kDqPerRound) && dqm != 0u;  // compile-time false in the per-round kernels
                // (chunked kernels only: under the per-round kernel's heavy eviction such
                // stretches mostly end before their first round, config D 91 -> 116 ms)
                const bool blocks = cdec && !((chunking || kDqPerRound) && T.nO == b && klt(sm->X[32 + (b - 1)], sm->F[lane]));
                SS_DCOUNT(8, dq ? 1 : 0);
#ifdef SS_DEBUG_D
                SS_DCOUNT(12, __any_sync(FULL, blocks) ? 1 : 0);
#endif
                if (!__any_sync(FULL, blocks)) {
                    if (dq) {  // the FRONT is sorted: its first decoding entry is the best one
                        if (lane == 0) c.dqk = sm->F[__ffs(dqm) - 1];
                        __syncwarp();
                    }
                    const Key F0 = T.nF > 0 ? sm->F[0] : kinf();
                    int m = T.nO;
                    bool act = lane < m;
                    MemS mem;
                    if (act) mem = sm->OM[lane];
                    // remaining_time of a decoding member (costs.py:174-191): reload(0)
                    // and prefill(0) are the same constants every round
                    const double z0 = A.z0;  // a kernel-argument operand: no register held
                    constexpr bool sum_mode = sum_k;
                    // per-membership values, recomputed when members complete
                    int left;                 // rounds before the first completion (dec + 1 >= tout)
                    unsigned nmax;            // longest context + 1 (decode step of the batch)
                    long long safe_used;      // per-round kernels: no member evicts while used <= this
                    int evleft;               // chunked kernels: rounds before the first one that evicts
                    unsigned long long gt;    // this lane's grant term (ss_grant_term of its batch position)
                    // round multiplier of the grant terms
                    unsigned long long rmul = ss_round_mul((unsigned long long)T.rounds);
                    auto setup = [&]() {
                        left = __reduce_min_sync(FULL, act ? (int)(m_tout(mem) - mem.dec) - 1 : 0x7fffffff);
                        nmax = __reduce_max_sync(FULL, act ? m_prompt(mem) + mem.dec + 1u : 0u);
                        // KV admission (engine.py:296-327) of an all-decode batch: immediate 1,
                        // exclusive scan = lane, demand = max(est, 1), est non-increasing
                        if (noev) {
                            evleft = 0x7fffffff;  // no eviction possible
                            safe_used = 0x7fffffffffffffffll;
                        } else if (!chunking) {
                            const long long est0 = act ? (long long)m_mid(mem) - (long long)mem.dec : 0;
                            const int maxdem = (int)__reduce_max_sync(FULL, (unsigned)(est0 > 1 ? est0 : 1));
                            safe_used = cap - (long long)maxdem - m;
                        } else {
                            // round j (from now) evicts iff some member i has demand_i(j) + i +
                            // used + j*m > cap, demand_i(j) = max(mid - dec - j, 1) (or 1 when
                            // demand + i > cap). Monotone in j: count the safe rounds by binary
                            // lifting per member, then the minimum over the members.
                            const long long e0 = (long long)m_mid(mem) - (long long)mem.dec;
                            const long long room = cap - T.used;
                            auto evicts = [&](int j) {
                                const long long e = e0 - j;
                                long long dm = e > 1 ? e : 1;
                                if (dm + lane > cap) dm = 1;
                                return dm + lane + (long long)j * m > room;
                            };
                            int safe = 0;
#pragma unroll 1
                            for (int st = 2048; st > 0; st >>= 1)
                                safe += evicts(safe + st - 1) ? 0 : st;
                            evleft = __reduce_min_sync(FULL, act ? safe : 0x7fffffff);
                        }
                        gt = act ? ss_grant_term((uint32_t)lane, mem.slot) : 0ull;
                    };
                    // chunked kernels: one call site (one copy of its code) at the loop top;
                    // per-round kernels call it directly (no extra vote per round)
                    bool need_setup = chunking;
                    if (!chunking) setup();
                    int k = 0;
                    bool dq_exit = false;          // a completion freed a slot a queued decoding candidate takes
                    long long spool = 0, sgr = 0;  // live and granted requests summed over the rounds
                    int live_s = live;
                    for (;;) {
                        SS_SECT(6);
                        if (chunking && uni(need_setup)) {
                            setup();
                            need_setup = false;
                        }
                        // one vote for every exit: a completion, an admission due, p*
                        // queued (no ongoing key below the queue front), round cap / log
                        const bool adm = T.next_ready <= ss::add(T.clock, 1e-12);
                        const bool capx = (T.rounds >= round_cap) | (logging && c.logpos > c.logcap);
                        const bool pdec = act & klt_nb(okey, F0);
                        bool cround = false;  // a member completes in this round
                        if (__all_sync(FULL, (left <= 0) | adm | capx | !pdec)) {
#ifdef SS_DEBUG_TIMING
                            SS_DCOUNT(9, uni(adm) ? 1 : 0);
                            SS_DCOUNT(10, (!uni(adm) && !__any_sync(FULL, pdec)) ? 1 : 0);
                            SS_DCOUNT(11, uni((left <= 0) & !adm & !capx) && __any_sync(FULL, pdec) ? 1 : 0);
#endif
                            // completing members are handled here when that is the only reason
                            if (!uni((left <= 0) & !adm & !capx) || !__any_sync(FULL, pdec)) break;
                            cround = true;
                        }
                        if (!noev && chunking && uni(evleft <= 0)) break;  // this round's admission evicts
                        if (!noev && !chunking && uni(T.used > safe_used)) {
                            long long e = (long long)m_mid(mem) - (long long)mem.dec;
                            long long dem = e > 1 ? e : 1;
                            if (dem + lane > cap) dem = 1;
                            if (__any_sync(FULL, act && dem + lane + T.used > cap)) {
#ifdef SS_DEBUG_D
                                SS_DCOUNT(13, 1);
                                SS_DCOUNT(14, k == 0 ? 1 : 0);
#endif
                                break;  // eviction
                            }
                        }
                        // ---- a chunk of up to 32 rounds, one lane per round ----------
                        // Within a stretch nothing but the clock is a serial chain: round
                        // j's batch duration, the members' keys after j decode steps and
                        // every digest term are closed-form in j. The clock is summed in
                        // the reference's order (one add per round); lane j evaluates
                        // round j. The chunk ends before the first round that the per-round
                        // exit vote would refuse (admission due, p* queued, ongoing order
                        // changed, completion, round cap, memory or log bound).
                        // entry: the static bounds (completion, round cap, memory, log) allow
                        // at least SS_CHUNK_MIN rounds; per-round bounds are lane votes below
                        bool chunk = false;
#ifndef SS_NO_CHUNK
                        if (chunking && !cround && !sum_mode) {
                            chunk = left >= SS_CHUNK_MIN && T.rounds + (SS_CHUNK_MIN - 1) < round_cap &&
                                    evleft >= SS_CHUNK_MIN;
                            if (logging)
                                chunk = chunk && c.logpos + (long long)(SS_CHUNK_MIN - 1) * (SS_LOG_HEADER_WORDS + m) <=
                                                     c.logcap;
                        }
#endif
                        if (!chunking || uni(!chunk)) {  // one round here
                        double part;  // batch_duration (engine.py:126-149) of an all-decode batch
                        SS_SECT(1);
                        SS_DCOUNT(2, 1);
                        if (!sum_mode) {  // a kernel parameter: uniform by construction
                            part = decode_step_time((long long)nmax, 1, P);
                        } else {
                            const double st = act ? decode_step_time((long long)m_prompt(mem) + mem.dec + 1, 1, P) : 0.0;
                            PySum ps;
                            ps.init();
                            for (int q = 0; uni(q < m); q++) ps.push(__shfl_sync(FULL, st, q));
                            part = ps.value();
                        }
                        const double end = ss::add(T.clock, ss::add(0.0, part));
                        // every lane computes; only lanes < m are members
                        mem.dec += 1u;
                        {
                            long long lft = (long long)m_mid(mem) - (long long)mem.dec;
                            if (lft < 1) lft = 1;
                            mem.ft = ss::add(z0, decode_total_time((long long)m_prompt(mem) + mem.dec, lft, P));
                        }
                        unsigned cdm = 0;  // completing lanes (cround only)
                        if (!cround) {
                            T.used += m;
                        } else {
                            // _complete (engine.py:414-421): finish = end, KV released
                            const bool done = act & (mem.dec >= m_tout(mem));
                            cdm = __ballot_sync(FULL, done);
                            const int delta = act ? (done ? 1 - (int)(m_prompt(mem) + mem.dec) : 1) : 0;
                            T.used += (long long)__reduce_add_sync(FULL, delta);
                            if (done) {
                                mem.ft = 0.0;
                                mem.flg = (mem.flg & ~F_STAGE) | ST_DONE;
                                const long long g = T.off + mem.slot;
                                A.out.req.finish_time[g] = end;
                                store_dyn(A, g, mem.ft, mem.dec, mem.flg);
                            }
                        }
                        const int ncd = __popc(cdm);
                        if (want_digest) {
                            const unsigned long long r64 = (unsigned long long)T.rounds;
                            // the members' cached grant terms times this round's multiplier; the
                            // completion terms (completion rounds only); header / memory / time as
                            // one weighted sum (ss_round_fields) in lane 31
                            dig += act ? gt * rmul : 0ull;
                            if (cround) {
                                const bool dn = (cdm >> lane) & 1u;
                                const unsigned long long dx =
                                    (unsigned long long)mem.slot ^
                                    (((r64 << 24) ^ ((unsigned long long)SS_TAG_DONE << 20) ^ (unsigned long long)__popc(cdm & lt)) *
                                     0x9E3779B97F4A7C15ull);
                                dig += dn ? ss_mix64(dx) : 0ull;
                            }
                            if (lane == 31)
                                dig += ss_round_fields(r64, ss_hdr_word(SS_KIND_DECODE, m, ncd, 0), (unsigned long long)T.used,
                                                       dbits(end));
                        }
                        rmul += 2u * SS_DG_ROUND;
                        if (logging) {
                            const long long lp = c.logpos;
                            if (act) log_put(c, lp + SS_LOG_HEADER_WORDS + lane, mem.slot);
                            if ((cdm >> lane) & 1u) log_put(c, lp + SS_LOG_HEADER_WORDS + m + __popc(cdm & lt), mem.slot);
                            __syncwarp();
                            if (lane == 0) {
                                const unsigned long long mu = (unsigned long long)T.used, tb = dbits(end);
                                log_put(c, lp + 0, (uint32_t)SS_KIND_DECODE);
                                log_put(c, lp + 1, (uint32_t)m);
                                log_put(c, lp + 2, (uint32_t)ncd);
                                log_put(c, lp + 3, 0u);
                                log_put(c, lp + 4, (uint32_t)mu);
                                log_put(c, lp + 5, (uint32_t)(mu >> 32));
                                log_put(c, lp + 6, (uint32_t)tb);
                                log_put(c, lp + 7, (uint32_t)(tb >> 32));
                                c.logpos = lp + SS_LOG_HEADER_WORDS + m + ncd;
                            }
                            __syncwarp();
                        }
                        peak = T.used > peak ? T.used : peak;
                        T.clock = end;
                        T.rounds += 1;
                        nmax += 1u;
                        left -= 1;
                        evleft -= 1;
                        k += 1;
                        spool += live_s;
                        sgr += m;
                        if (cround) {
                            // resident list upkeep for the completed (engine.py:414-421)
                            unsigned cm = track_res ? cdm : 0u;
                            if (!track_res) T.nR -= ncd;  // no resident list in the no-eviction kernels
                            __syncwarp();
                            while (cm) {
                                const int q = __ffs(cm) - 1;
                                cm &= cm - 1;
                                const uint32_t s = __shfl_sync(FULL, mem.slot, q);
                                if (track_res && lane == 0) {
                                    const uint32_t ri = A.w.rpos[T.off + s];
                                    const uint32_t last = A.w.R[T.off + T.nR - 1];
                                    A.w.R[T.off + ri] = last;
                                    A.w.rpos[T.off + last] = ri;
                                }
                                T.nR -= 1;
                                __syncwarp();
                            }
                            // ongoing = granted members not completed, in granted order
                            const bool stay = act & !((cdm >> lane) & 1u);
                            const unsigned smk = __ballot_sync(FULL, stay);
                            if (stay) sm->OM[__popc(smk & lt)] = mem;
                            __syncwarp();
                            m = __popc(smk);
                            act = lane < m;
                            if (act) mem = sm->OM[lane];
                            __syncwarp();
                            T.nO = m;
                            live_s -= ncd;
                            if (uni(m == 0)) break;
                            // a queued decoding candidate takes the freed slot next round: leave
                            // after this round's key refresh and order check below
                            dq_exit = dq;
                            if (chunking) need_setup = true;
                            else setup();
                        }
                        }
#ifndef SS_NO_CHUNK
                        else {
                            SS_SECT(2);
                            const int L = left < 32 ? left : 32;
                            if (act) sm->OM[lane] = mem;  // broadcast source of the member loop
                            double* chain = reinterpret_cast<double*>(sm->M);  // round ends (scratch)
                            // batch_duration of round j: decode step at the longest context
                            const double pj =
                                ss::add(0.0, decode_step_time((long long)(nmax + (unsigned)lane), 1, P));
                            double clk = T.clock;
                            // the rounds' durations broadcast from shared memory (one load per round
                            // instead of two shuffles of the double)
                            double* pjs = chain + 32;
                            pjs[lane] = pj;
                            __syncwarp();
                            for (int q0 = 0; uni(q0 < L); q0 += kChainStep) {
#pragma unroll
                                for (int q = 0; q < kChainStep; q++) {
                                    clk = ss::add(clk, pjs[q0 + q]);
                                    if (lane == 0) chain[q0 + q] = clk;
                                }
                            }
                            __syncwarp();
                            const double endj = chain[lane];
                            const double befj = lane == 0 ? T.clock : chain[lane - 1];
                            // state after round j (lane j): every member decoded j + 1 more
                            const uint32_t dj = (uint32_t)lane + 1u;
                            const unsigned long long rj = (unsigned long long)(T.rounds + lane);
                            bool ok = true, pk = true;
                            double pft = 0.0;
                            uint32_t prk = 0, ptie = 0;
                            // Order screen (lane i = member i). While no member's predicted
                            // remainder clamps at 1 (costs.py:186-190), f_t of a decoding member
                            // after j' more steps is T(m0 - j') with T(m) = g1*m*(C + 0.5 - 0.5m)
                            // + g2*m exactly (C = prompt + mid): every member has the same
                            // curvature -g1, so the real gap between two members is linear in
                            // j' and its minimum over the chunk lies at an endpoint; f_t itself
                            // is non-increasing (g1, g2 >= 0). The computed f_t of the first
                            // and last round of the chunk bound every round's order: a gap
                            // above 2^-40 f_t (>= 1000x the evaluation's rounding error)
                            // at both ends keeps every pair in order at every round, and a
                            // member 0 at least that far below the queue front keeps p*
                            // ongoing. Same-rank members with equal (context, remainder)
                            // evolve identically (their tie order stands). Otherwise the
                            // exact per-round loop below decides.
                            int i_lo = 0, i_hi = m - 1;  // members the exact loop evaluates
#ifndef SS_NO_SCREEN
                            if (A.screen) {
                                const int l1 = (int)m_mid(mem) - (int)(mem.dec + (uint32_t)L);
                                const uint32_t n0 = m_prompt(mem) + mem.dec + 1u;
                                const int l0 = l1 + L - 1;
                                const bool lin = l1 >= 1;
                                const double f0 = ss::add(z0, decode_total_time_u32(n0, lin ? (uint32_t)l0 : 1u, P));
                                const double f1 =
                                    ss::add(z0, decode_total_time_u32(n0 + (uint32_t)(L - 1), lin ? (uint32_t)l1 : 1u, P));
                                const double thr = 0x1p-40 * f0;
                                const uint32_t rk = m_rank(mem);
                                const double f0p = __shfl_up_sync(FULL, f0, 1), f1p = __shfl_up_sync(FULL, f1, 1);
                                const uint32_t rkp = __shfl_up_sync(FULL, rk, 1), n0p = __shfl_up_sync(FULL, n0, 1);
                                const int l0p = __shfl_up_sync(FULL, l0, 1);
                                const bool linp = __shfl_up_sync(FULL, lin, 1);
                                bool good;  // lane 0: p* stays ongoing; lane i: pair (i - 1, i) stays in order
                                if (lane == 0) {
                                    // member 0 against the queue front (kinf when empty)
                                    const uint32_t frk = (uint32_t)(F0.hi >> 56);
                                    const double fft = __longlong_as_double(
                                        (long long)(((F0.hi & 0x00FFFFFFFFFFFFFFull) << 7) | (F0.lo >> 25)));
                                    good = (F0.hi == ~0ull) | (rk < frk) | ((rk == frk) & lin & (fft - f0 > thr));
                                } else {
                                    good = (rkp < rk) | ((n0p == n0) & (l0p == l0)) |
                                           (lin & linp & (f0 - f0p > thr) & (f1 - f1p > thr));
                                }
                                // a member past its predicted length (remainder clamped at 1) gains
                                // f_t each round: the last member must then be checked against the
                                // best queued decoding candidate round by round
                                if (dq && lane == m - 1) good &= lin;
                                // only the pairs (and p*) the screen cannot settle run the exact loop
                                const unsigned sus = __ballot_sync(FULL, act & !good);
                                const int s_lo = __ffs(sus) - 1;
                                i_lo = sus ? (s_lo > 0 ? s_lo - 1 : 0) : 1;
                                i_hi = sus ? 31 - __clz(sus) : 0;
                            }
#endif
                            SS_DCOUNT(6, i_hi < i_lo ? 1 : 0);
                            SS_DCOUNT(7, i_hi >= i_lo ? i_hi - i_lo + 1 : 0);
                            // no warp-collective inside: a plain (unrollable) loop
#pragma unroll kChunkUnroll
                            for (int i = i_lo; i <= i_hi; i++) {
                                const uint4 st = sm->OM[i].st;
                                const uint32_t dec = sm->OM[i].dec + dj;
                                int lft = (int)st.z - (int)dec;
                                lft = lft < 1 ? 1 : lft;
                                const double ft = ss::add(z0, decode_total_time_u32(st.x + dec, (uint32_t)lft, P));
                                const uint32_t rk = st.w >> 24, tie = st.w & SLOT_MASK;
                                // key order (rank, f_t, tie) without packing: f_t > 0 orders like its bits
                                if (i == 0) pk = klt_nb(make_key<POL>(rk, ft, tie, 0, true), F0);
                                else if (i > i_lo) ok &= (prk < rk) | ((prk == rk) & ((pft < ft) | ((pft == ft) & (ptie < tie))));
                                if (dq && i == m - 1) ok &= klt_nb(make_key<POL>(rk, ft, tie, 0, true), c.dqk);
                                pft = ft;
                                prk = rk;
                                ptie = tie;
                            }
                            // round j runs iff rounds 0..j-1 left the members sorted with p*
                            // ongoing, no admission is due at its start and no static bound
                            // (completion, round cap, memory safety, log space) stops it
                            const bool adm_j = T.next_ready <= ss::add(befj, 1e-12);
                            bool lim = (lane >= L) | (T.rounds + lane >= round_cap);
                            if (!noev) lim |= lane >= evleft;
                            if (logging) lim |= c.logpos + (long long)lane * (SS_LOG_HEADER_WORDS + m) > c.logcap;
                            const unsigned stop = __ballot_sync(FULL, lim | adm_j) |
                                                  (__ballot_sync(FULL, !(pk & ok)) << 1);
                            const int Lx = stop ? __ffs(stop) - 1 : 32;  // >= 1: round 0 passed the vote
#if defined(SS_DEBUG_TIMING) && !defined(SS_DEBUG_D)
                            {
                                const unsigned s_lim = __ballot_sync(FULL, lim), s_adm = __ballot_sync(FULL, adm_j);
                                SS_DCOUNT(12, Lx == L ? 1 : 0);
                                SS_DCOUNT(13, (Lx < L && ((s_adm >> Lx) & 1u) && !((s_lim >> Lx) & 1u)) ? 1 : 0);
                                SS_DCOUNT(14, (Lx < L && !((s_adm >> Lx) & 1u) && !((s_lim >> Lx) & 1u)) ? 1 : 0);
                            }
#endif
                            SS_DCOUNT(0, 1);
                            SS_DCOUNT(1, Lx);
                            const bool runj = lane < Lx;
                            const long long used_j = T.used + (long long)(lane + 1) * m;
                            if (want_digest) {
                                // ss_round_fields of round j (the header is constant over the chunk);
                                // the grant terms of rounds r0..r0+Lx-1: each member's term times
                                // sum_j ss_round_mul(r0 + j) = SS_DG_ROUND * Lx * (2 r0 + Lx)
                                const unsigned long long cst = SS_DG_HDR * (ss_hdr_word(SS_KIND_DECODE, m, 0, 0) ^ SS_DS_HDR);
                                const unsigned long long v = cst + SS_DG_MEM * ((unsigned long long)used_j ^ SS_DS_MEM) +
                                                             SS_DG_TIME * (dbits(endj) ^ SS_DS_TIME);
                                const unsigned long long gsum =
                                    SS_DG_ROUND * ((unsigned long long)Lx * (2ull * (unsigned long long)T.rounds + (unsigned long long)Lx));
                                dig += (runj ? (2ull * rj + 1ull) * v : 0ull) + (act ? gt * gsum : 0ull);
                            }
                            if (logging) {
                                __syncwarp();
                                const long long lp = c.logpos + (long long)lane * (SS_LOG_HEADER_WORDS + m);
                                if (runj) {
                                    const unsigned long long mu = (unsigned long long)used_j, tb = dbits(endj);
                                    log_put(c, lp + 0, (uint32_t)SS_KIND_DECODE);
                                    log_put(c, lp + 1, (uint32_t)m);
                                    log_put(c, lp + 2, 0u);
                                    log_put(c, lp + 3, 0u);
                                    log_put(c, lp + 4, (uint32_t)mu);
                                    log_put(c, lp + 5, (uint32_t)(mu >> 32));
                                    log_put(c, lp + 6, (uint32_t)tb);
                                    log_put(c, lp + 7, (uint32_t)(tb >> 32));
                                    for (int i = 0; i < m; i++) log_put(c, lp + SS_LOG_HEADER_WORDS + i, sm->OM[i].slot);
                                }
                                __syncwarp();
                                if (lane == 0) c.logpos += (long long)Lx * (SS_LOG_HEADER_WORDS + m);
                                __syncwarp();
                            }
                            T.clock = chain[Lx - 1];
                            __syncwarp();
                            T.used += (long long)Lx * m;
                            peak = T.used > peak ? T.used : peak;
                            T.rounds += Lx;
                            nmax += (unsigned)Lx;
                            left -= Lx;
                            evleft -= Lx;
                            k += Lx;
                            spool += (long long)Lx * live_s;
                            sgr += (long long)Lx * m;
                            rmul += (unsigned long long)Lx * (2u * SS_DG_ROUND);
                            mem.dec += (uint32_t)Lx;
                            long long lft = (long long)m_mid(mem) - (long long)mem.dec;
                            if (lft < 1) lft = 1;
                            mem.ft = ss::add(z0, decode_total_time((long long)m_prompt(mem) + mem.dec, lft, P));
                        }
#endif
                        SS_SECT(7);
                        // the ongoing set stays sorted by key (usually already is)
                        okey = make_key<POL>(m_rank(mem), mem.ft, m_tie(mem), mem.slot, true);
                        Key nx;  // order check needs the next lane's (hi, lo) only
                        nx.hi = __shfl_down_sync(FULL, okey.hi, 1);
                        nx.lo = __shfl_down_sync(FULL, okey.lo, 1);
                        const bool reord = uni(__ballot_sync(FULL, (lane + 1 < m) & klt_nb(nx, okey)) != 0u);
                        if (reord) {
                            if (act) sm->X[32 + lane] = okey;
                            __syncwarp();
                            int r = 0;
                            for (int q = 0; uni(q < m); q++) r += klt(sm->X[32 + q], okey) ? 1 : 0;
                            __syncwarp();
                            if (act) {
                                sm->OM[r] = mem;
                                sm->X[32 + r] = okey;
                            }
                            __syncwarp();
                            if (act) {
                                mem = sm->OM[lane];
                                okey = sm->X[32 + lane];
                            }
                            __syncwarp();
                        }
                        SS_DCOUNT(15, reord ? 1 : 0);
                        if (reord) break;  // positions moved: the next stretch recomputes the grant terms
                        // the next round's batch would take a queued decoding candidate
                        if (dq && (dq_exit || __any_sync(FULL, (lane == m - 1) & !klt_nb(okey, c.dqk)))) break;
                    }
                    if (uni(T.rounds >= round_cap)) set_status(T, SS_TRACE_ROUND_CAP);
                    if (logging && uni(c.logpos > c.logcap)) set_status(T, SS_TRACE_LOG_OVERFLOW);
                    if (uni(k > 0)) {
                        if (act) {
                            store_dyn(A, T.off + mem.slot, mem.ft, mem.dec, mem.flg);
                            sm->OM[lane] = mem;
                            sm->X[32 + lane] = okey;
                        }
                        T.nO = m;
                        if (lane == 0) {
                            c.s_pool += spool;
                            c.s_granted += sgr;
                        }
                        __syncwarp();
                        continue;
                    }
                }
            }
            if (lane == 0) c.s_pool += live;
            SS_SECT(3);
            SS_DCOUNT(3, 1);
#ifdef SS_DEBUG_ANOM
            if (lane == 0) c.dbg += anom ? 1 : 0;
#endif

            // ---- stage-aware composition (batching.py:46-88)
            // candidates popped from the queue: top-b (semantic / SJF / HPJF,
            // batching.py:46-54, engine.py:270-276) or the b - |ongoing| that FCFS
            // adds behind its non-preemptible ongoing members (engine.py:256-262)
            const int cwant = POL == SS_POLICY_FCFS ? b - T.nO : b;
            const int nc = T.nF < cwant ? T.nF : cwant;
            const bool has_c = lane < nc;
            const bool has_o = lane < T.nO;
            Key ck;  // candidate key: stored (fast path) or current (general path)
            if (has_c) {
                ck = sm->F[lane];
                if (anom_ok && anom) {
                    MemS cm;
                    load_mem(A, T.off, ck.aux & SLOT_MASK, cm);
                    ck = mem_key<POL>(cm);
                }
            }
            // p* = min over candidates and ongoing (current keys); the ongoing
            // copies are sorted by key across lanes (their order is unobservable
            // in the reference: equal keys are copies of the same request)
            Key pmin = kinf();
            if (POL != SS_POLICY_SEMANTIC) {
            } else if (!anom_ok || uni(!anom)) {
                if (T.nO > 0) pmin = sm->X[32];
                if (nc > 0 && klt(sm->F[0], pmin)) pmin = sm->F[0];
            } else {
                pmin = has_o ? okey : kinf();
                if (has_c && klt(ck, pmin)) pmin = ck;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    Key x = kshfl_xor(pmin, o);
                    if (klt(x, pmin)) pmin = x;
                }
            }
            // semantic: the stage of p* decides which candidates are eligible;
            // the baselines take every candidate (no stage awareness)
            const bool pstar_prefill = !(pmin.aux & DEC_BIT);
            int kind = pstar_prefill ? SS_KIND_PREFILL : SS_KIND_DECODE;
            const bool c_elig =
                has_c && (POL != SS_POLICY_SEMANTIC || pstar_prefill || (ck.aux & DEC_BIT));
            const unsigned cmask = __ballot_sync(FULL, c_elig);
            int cnt_c = 0, cnt_o = 0;
            if (POL == SS_POLICY_FCFS) {
                // ongoing first in their order, then the popped candidates
                cnt_o = lane;
                cnt_c = T.nO + lane;
            } else if (!anom_ok || uni(!anom)) {
                // both lists sorted: rank = own index + lower_bound in the other
                cnt_o = lane;
                if (cmask) {
                    if (c_elig) {
                        int lo = 0, hi = T.nO;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            const bool below = klt(sm->X[32 + mid], ck);  // branch-free step
                            lo = below ? mid + 1 : lo;
                            hi = below ? hi : mid;
                        }
                        cnt_c = __popc(cmask & lt) + lo;
                    }
                    if (has_o) {
                        int lo = 0, hi = nc;
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            const bool below = klt(sm->F[mid], okey);  // branch-free step
                            lo = below ? mid + 1 : lo;
                            hi = below ? hi : mid;
                        }
                        unsigned below = lo >= 32 ? FULL : ((1u << lo) - 1u);
                        cnt_o += __popc(cmask & below);
                    }
                }
            } else {
                // general: stable sort of (candidates + ongoing) by current key (out of line)
                const int2 cc = rank_general(sm, nc, T.nO, cmask, c_elig, has_o, ck, okey);
                cnt_c = cc.x;
                cnt_o = cc.y;
            }
            const int elig = __popc(cmask) + T.nO;
            const int m = elig < b ? elig : b;
            const bool c_sel = c_elig && cnt_c < m;
            Round R;
            R.G = 0;
            R.evmask = 0;
            R.ndec = 0;
            R.rmF = (unsigned long long)__ballot_sync(FULL, c_sel);
            // batch members -> M[rank]; the common decode round (batch == ongoing
            // in order) reads its records straight from OM
            const bool direct = cmask == 0 && T.nO <= b;
            __syncwarp();
            if (c_sel) {
                MemS cm;
                load_mem(A, T.off, ck.aux & SLOT_MASK, cm);
                if (anom_ok && anom) {  // another copy may have moved the flags: re-read them
                    cm.flg = flg_update(A, T.off + cm.slot, F_Q, 0u);  // popped from the heap for good
                } else {  // distinct requests: the loaded flags are current
                    cm.flg &= ~F_Q;
                    *FLG(A, T.off + cm.slot) = cm.flg;
                }
                sm->M[cnt_c] = cm;
            }
            if (!direct && has_o && cnt_o < m) sm->M[cnt_o] = sm->OM[lane];
            if (anom_ok && uni(anom)) {
                // candidates not selected are pushed back with their current key; a stale
                // stored key is replaced; pushed-back ongoing copies (out of line)
                const PushOut po = push_back_stale(&A, sm, T.off, T.nins, has_c, c_sel, ck, has_o && cnt_o >= m, okey);
                R.rmF |= (unsigned long long)po.rm;
                T.nins = po.nins;
                if (po.err) set_status(T, SS_TRACE_REF_ERROR);
            } else {
                const bool pushed = has_o && cnt_o >= m;
                const unsigned pm = __ballot_sync(FULL, pushed);
                if (pushed) {
                    const MemS& o = sm->OM[lane];
                    *FLG(A, T.off + o.slot) = o.flg | F_Q | F_INS;
                    INS(A)[T.off + T.nins + __popc(pm & lt)] = okey;
                }
                T.nins += __popc(pm);
            }
            __syncwarp();
            if (uni(T.status != SS_TRACE_OK)) {
                T.rounds += 1;  // the raising round counts (oracle / golden convention)
                break;
            }
            MemS mem;
            mem.slot = 0xFFFFFFFFu;
            const bool act = lane < m;
            if (act) {
                mem = direct ? sm->OM[lane] : sm->M[lane];
                if (anom_ok && anom) mem.flg = *FLG(A, T.off + mem.slot);  // queued bit may have moved
            }
            if (POL != SS_POLICY_SEMANTIC) {
                // BatchKind from the selected members' stages (engine.py:263-267, 280-284)
                kind = __ballot_sync(FULL, act && (mem.flg & F_STAGE) != ST_DEC) ? SS_KIND_PREFILL : SS_KIND_DECODE;
            }
            const int nO_start = T.nO;
            const int nuns_start = c.nuns;
            __syncwarp();  // lane 0 updates Cold fields next to nuns below (racecheck)
            // a completed request popped from a stale entry: estimate_kv_size raises
            if (anom_ok && uni(anom) && __ballot_sync(FULL, act && (mem.flg & F_STAGE) == ST_DONE)) {
                set_status(T, SS_TRACE_REF_ERROR);
                T.rounds += 1;
                break;
            }

            // ---- admission with KV budget (engine.py:296-327)
            SS_SECT(8);
            MemQ q = mem_q(mem);
            {
                int excl;
                if (__all_sync(FULL, !act || q.isdec)) {
                    excl = lane;  // every immediate is 1
                } else {
                    const int inc = act ? (int)q.imm : 0;
                    int sc = inc;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        int tt = __shfl_up_sync(FULL, sc, o);
                        if (lane >= o) sc += tt;
                    }
                    excl = sc - inc;
                }
                long long dem = q.est > q.imm ? q.est : q.imm;
                if (dem + excl > cap) dem = q.imm;
                const bool need = act && (dem + excl + T.used > cap);
                const unsigned nm = __ballot_sync(FULL, need);
                const unsigned mmask = m >= 32 ? FULL : ((1u << m) - 1u);
                const int f = nm ? __ffs(nm) - 1 : m;
                R.G = (f >= 32 ? FULL : ((1u << f) - 1u)) & mmask;
                if (anom_ok && uni(anom)) {
                    // grants of still-queued requests (stale heap entry) before f
                    const unsigned qa = __ballot_sync(FULL, ((R.G >> lane) & 1u) && (mem.flg & F_Q));
                    if (qa && lane == 0) c.anomalies += __popc(qa);
                }
                if (noev && nm) set_status(T, SS_TRACE_INTERNAL);  // the footprint rule excludes this
                if (!noev && nm) {
                    if (lane == 0) c.s_res += T.nR;
                    // slow path: one member at a time from the first that must evict
                    long long reserved = __shfl_sync(FULL, excl, f);
                    if ((R.G >> lane) & 1u) flg_update(A, T.off + mem.slot, 0u, F_GRANT);
                    __syncwarp();
                    if (act) mem.flg = *FLG(A, T.off + mem.slot);
                    for (int k = f; uni(k < m && T.status == SS_TRACE_OK); k++) {
                        if ((R.evmask >> k) & 1u) continue;
                        q = mem_q(mem);
                        const long long imm_k = __shfl_sync(FULL, q.imm, k);
                        const long long est_k = __shfl_sync(FULL, q.est, k);
                        const long long kvd_k = __shfl_sync(FULL, q.kvd, k);
                        const uint32_t slot_k = __shfl_sync(FULL, mem.slot, k);
                        long long dem_k = est_k > imm_k ? est_k : imm_k;
                        if (dem_k + reserved > cap) dem_k = imm_k;
                        const long long demand = dem_k + reserved;
                        const int d0 = R.ndec;
                        unsigned vcall = 0;
                        if (lane == 0) c.dpend = 0ull;
                        __syncwarp();
                        bool ok = true;
                        SS_SECT(14);
                        while (uni(demand + T.used > cap)) {
                            SS_DCOUNT(4, 1);
                            if (uni(!evict_one<POL, logging>(E, T, R, slot_k, m, mem, vcall))) {
                                ok = false;
                                break;
                            }
                        }
                        SS_SECT(8);
                        const uint32_t flg_k = __shfl_sync(FULL, mem.flg, k);
                        if (uni(!ok)) {
                            // AdmissionFailure: evictions stand, their records are lost
                            if (lane == 0) c.lost += R.ndec - d0;
                            R.ndec = d0;
                            if (uni(kvd_k + imm_k > cap)) {
                                // _mark_unservable (engine.py:402-412)
                                q_delete(E, T, R, slot_k, flg_k);
                                const bool isdec_k = (flg_k & F_STAGE) == ST_DEC;
                                const int un = c.nuns;
                                __syncwarp();
                                if (lane == k) {
                                    const long long g = T.off + mem.slot;
                                    if (isdec_k) {
                                        uint32_t ri = A.w.rpos[g];
                                        uint32_t last = A.w.R[T.off + T.nR - 1];
                                        A.w.R[T.off + ri] = last;
                                        A.w.rpos[T.off + last] = ri;
                                    }
                                    flg_update(A, g, F_STAGE | F_Q | F_INS | F_GRANT, ST_UNS | (isdec_k ? F_UDEC : 0u));
                                    A.out.unservable_slots[T.off + un] = mem.slot;
                                    c.nuns = un + 1;
                                }
                                if (isdec_k) T.nR -= 1;
                                T.used -= kvd_k;
                                __syncwarp();
                                // every batch copy of it sees the new state
                                if (act && mem.slot == slot_k) mem.flg = *FLG(A, T.off + slot_k);
                            } else if (uni(!(flg_k & F_Q))) {
                                if (lane == k) {
                                    const Key kk = make_key<POL>(m_rank(mem), mem.ft, m_tie(mem), mem.slot, q.isdec);
                                    flg_update(A, T.off + mem.slot, 0u, F_Q | F_INS);
                                    INS(A)[T.off + T.nins] = kk;
                                }
                                T.nins += 1;
                                __syncwarp();
                                if (act && mem.slot == slot_k) mem.flg = *FLG(A, T.off + slot_k);
                            }
                            __syncwarp();
                            continue;
                        }
                        // success: commit this call's decisions
                        R.evmask |= vcall;
                        if (lane == 0) dig += c.dpend;
                        if (uni(flg_k & F_Q)) {
                            // granted while it still has a heap entry (a victim whose
                            // decision was lost): the reference keeps that stale entry
                            if (lane == 0) c.anomalies += 1;
                            anom = true;
                        }
                        R.G |= 1u << k;
                        reserved += imm_k;
                        if (lane == k) flg_update(A, T.off + mem.slot, 0u, F_GRANT);
                        __syncwarp();
                        if (act && mem.slot == slot_k) mem.flg = *FLG(A, T.off + slot_k);
                    }
                }
            }
            if (uni(T.status != SS_TRACE_OK)) break;
            if (anom_ok && uni(anom)) {
                // copies of one request must agree before duration and execution
                __syncwarp();
                if (act) {
                    const Dyn d = DYN(A)[T.off + mem.slot];
                    mem.ft = d.ft;
                    mem.dec = d.dec;
                    mem.flg = d.flg;
                }
            }
            const bool g_act = (R.G >> lane) & 1u;
            const int ng = __popc(R.G);
            const unsigned long long r64 = (unsigned long long)T.rounds;
            if (lane == 0) {
                c.evictions += R.ndec;
                c.s_granted += ng;
            }

            if (uni(ng == 0)) {
                // nothing granted (engine.py:329-344): clock does not advance
                T.nO = 0;
                if (want_digest && lane == 0)  // header / memory / time
                    dig += ss_round_fields(r64, ss_hdr_word(SS_KIND_NONE, 0, 0, R.ndec), (unsigned long long)T.used,
                                           dbits(T.clock));
                if (R.ndec > 0 && lane == 0) {
                    if (T.used > peak) peak = T.used;
                    if (logging && c.log) {
                        const unsigned long long mu = (unsigned long long)T.used, tb = dbits(T.clock);
                        log_put(c, c.logpos + 0, SS_KIND_NONE);
                        log_put(c, c.logpos + 1, 0);
                        log_put(c, c.logpos + 2, 0);
                        log_put(c, c.logpos + 3, (uint32_t)R.ndec);
                        log_put(c, c.logpos + 4, (uint32_t)mu);
                        log_put(c, c.logpos + 5, (uint32_t)(mu >> 32));
                        log_put(c, c.logpos + 6, (uint32_t)tb);
                        log_put(c, c.logpos + 7, (uint32_t)(tb >> 32));
                        c.logpos += SS_LOG_HEADER_WORDS + (long long)SS_LOG_DECISION_WORDS * R.ndec;
                    }
                }
                T.rounds += 1;
                __syncwarp();
                if (R.ndec == 0 && c.nuns == nuns_start && nO_start == 0) set_status(T, SS_TRACE_LIVELOCK);
            } else {
                // ---- batch_duration (engine.py:126-149) over granted copies
                SS_SECT(9);
                q = mem_q(mem);
                double total = 0.0;
                const unsigned pre = __ballot_sync(FULL, g_act && !q.isdec);
                if (pre) {
                    const double rl = reload_time(q.kvh, P);
                    const double pft = prefill_time((long long)m_prompt(mem) - q.pfn, P);
                    for (int k = 0; uni(k < m); k++) {
                        const double a = __shfl_sync(FULL, rl, k), c2 = __shfl_sync(FULL, pft, k);
                        if ((pre >> k) & 1u) {
                            total = ss::add(total, a);
                            total = ss::add(total, c2);
                        }
                    }
                }
                const unsigned dm = __ballot_sync(FULL, g_act && q.isdec);
                if (dm) {
                    double part;
                    if (!sum_k) {
                        // gamma1 >= 0: the step time is monotone in the context length,
                        // so the max step is the step of the longest context
                        const unsigned nmax =
                            __reduce_max_sync(FULL, (g_act && q.isdec) ? m_prompt(mem) + mem.dec + 1u : 0u);
                        part = decode_step_time((long long)nmax, 1, P);
                    } else {
                        const double st = (g_act && q.isdec)
                                              ? decode_step_time((long long)m_prompt(mem) + mem.dec + 1, 1, P)
                                              : 0.0;
                        PySum ps;
                        ps.init();
                        for (int k = 0; uni(k < m); k++) {
                            const double x = __shfl_sync(FULL, st, k);
                            if ((dm >> k) & 1u) ps.push(x);
                        }
                        part = ps.value();
                    }
                    total = ss::add(total, part);
                }
                const double end = ss::add(T.clock, total);

                // ---- per-member progress (engine.py:351-363, 382-421)
                SS_SECT(10);
                bool done = false;
                bool dups = false;
                if (anom_ok && uni(anom)) {
                    const unsigned dupm = __match_any_sync(FULL, g_act ? mem.slot : (0x80000000u | lane));
                    dups = __ballot_sync(FULL, g_act && __popc(dupm) > 1) != 0;
                }
                if (!dups) {
                    int delta = 0;
                    bool newres = false;
                    if (g_act) {
                        const long long g = T.off + mem.slot;
                        if (!(mem.flg & F_FIRST)) {
                            A.out.req.first_scheduled[g] = T.clock;
                            mem.flg |= F_FIRST;
                        }
                        if (q.isdec) {
                            delta = 1;
                            mem.dec += 1;
                        } else {
                            delta = (int)(q.kvh + (m_prompt(mem) - q.pfn));
                            mem.flg = (mem.flg & ~F_STAGE) | ST_DEC | F_PF;
                            newres = true;
                        }
                        mem.flg &= ~F_GRANT;
                        if (mem.dec >= m_tout(mem)) {
                            done = true;
                            delta -= (int)(m_prompt(mem) + mem.dec);
                            A.out.req.finish_time[g] = end;
                            mem.ft = 0.0;
                            mem.flg = (mem.flg & ~F_STAGE) | ST_DONE;
                        } else {
                            mem.ft = remaining_time(m_prompt(mem), m_mid(mem), m_prompt(mem), mem.dec, 0, P);
                        }
                        store_dyn(A, g, mem.ft, mem.dec, mem.flg);
                    }
                    // allocations all fit (admission reserved them); completions release
                    T.used += (long long)__reduce_add_sync(FULL, delta);
                    if (T.used > cap) set_status(T, SS_TRACE_REF_ERROR);  // mem.allocate raises
                    if (T.used < 0) set_status(T, SS_TRACE_INTERNAL);
                    const unsigned nmr = __ballot_sync(FULL, newres);
                    if (nmr) {
                        if (track_res && newres) {
                            const uint32_t idx = (uint32_t)(T.nR + __popc(nmr & lt));
                            A.w.R[T.off + idx] = mem.slot;
                            A.w.rpos[T.off + mem.slot] = idx;
                        }
                        T.nR += __popc(nmr);
                    }
                    unsigned cmk = __ballot_sync(FULL, done);
                    if (cmk) {
                        __syncwarp();
                        while (cmk) {
                            const int k = __ffs(cmk) - 1;
                            cmk &= cmk - 1;
                            const uint32_t s = __shfl_sync(FULL, mem.slot, k);
                            if (track_res && lane == 0) {
                                const uint32_t ri = A.w.rpos[T.off + s];
                                const uint32_t last = A.w.R[T.off + T.nR - 1];
                                A.w.R[T.off + ri] = last;
                                A.w.rpos[T.off + last] = ri;
                            }
                            T.nR -= 1;
                            __syncwarp();
                        }
                    }
                } else {
                    // duplicate copies of a request (stale heap entries): out of
                    // line, the hot general round carries none of this code
                    {
                        const DupOut o = progress_dups(&A, T.off, R.G, T.clock, end, cap, T.used, T.nR, mem);
                        T.used = o.used;
                        T.nR = o.nR;
                        if (o.err) set_status(T, SS_TRACE_REF_ERROR);
                        done = o.done;
                    }
                    if (uni(T.status != SS_TRACE_OK)) {
                        T.rounds += 1;
                        break;
                    }
                    if (g_act) {  // every copy sees the final state
                        const Dyn d = DYN(A)[T.off + mem.slot];
                        mem.dec = d.dec;
                        mem.flg = d.flg;
                        mem.ft = d.ft;
                    }
                }
                // ---- ITERATION_END record (engine.py:365-380) + digest
                SS_SECT(11);
                const unsigned cdone = __ballot_sync(FULL, done);
                const int nc_done = __popc(cdone);
                const int gi = __popc(R.G & lt), ci = __popc(cdone & lt);
                if (want_digest) {
                    // one hash stream: granted lanes hash their slot (pass 0), completing lanes
                    // their completion term (pass 1); header / memory / time as one weighted
                    // sum (ss_round_fields) in lane 31
                    const unsigned long long dsalt = ((r64 << 24) ^ ((unsigned long long)SS_TAG_DONE << 20) ^
                                                      (unsigned long long)ci) * 0x9E3779B97F4A7C15ull;
#pragma unroll 1
                    for (int ps = 0; ps < 2; ps++) {
                        const bool use = ps == 0 ? g_act : (done && cdone != 0);
                        if (!__any_sync(FULL, use)) continue;
                        const unsigned long long x =
                            ps == 0 ? ((unsigned long long)mem.slot ^ ((unsigned long long)(gi + 1) * SS_DG_POS))
                                    : ((unsigned long long)mem.slot ^ dsalt);
                        const unsigned long long h = ss_mix64(x);
                        dig += use ? (ps == 0 ? h * ss_round_mul(r64) : h) : 0ull;
                    }
                    if (lane == 31)
                        dig += ss_round_fields(r64, ss_hdr_word(kind, ng, nc_done, R.ndec), (unsigned long long)T.used,
                                               dbits(end));
                }
                if (logging) {
                    const long long lp = c.logpos;
                    const long long base = lp + SS_LOG_HEADER_WORDS + (long long)SS_LOG_DECISION_WORDS * R.ndec;
                    if (g_act) log_put(c, base + gi, mem.slot);
                    if (done) log_put(c, base + ng + ci, mem.slot);
                    __syncwarp();
                    if (lane == 0) {
                        const unsigned long long mu = (unsigned long long)T.used, tb = dbits(end);
                        log_put(c, lp + 0, (uint32_t)kind);
                        log_put(c, lp + 1, (uint32_t)ng);
                        log_put(c, lp + 2, (uint32_t)nc_done);
                        log_put(c, lp + 3, (uint32_t)R.ndec);
                        log_put(c, lp + 4, (uint32_t)mu);
                        log_put(c, lp + 5, (uint32_t)(mu >> 32));
                        log_put(c, lp + 6, (uint32_t)tb);
                        log_put(c, lp + 7, (uint32_t)(tb >> 32));
                        c.logpos = base + ng + nc_done;
                    }
                }
                if (T.used > peak) peak = T.used;
                T.clock = end;
                T.rounds += 1;
                // ---- ongoing = granted copies not completed, in granted order
                SS_SECT(12);
                const bool stay = g_act && (mem.flg & F_STAGE) != ST_DONE;
                const unsigned smk = __ballot_sync(FULL, stay);
                __syncwarp();
                if (stay) sm->OM[__popc(smk & lt)] = mem;
                T.nO = __popc(smk);
                __syncwarp();
                const bool prefix = smk == FULL || smk == (1u << __popc(smk)) - 1u;
                if (stay && prefix) {
                    okey = mem_key<POL>(mem);  // no compaction: lane keeps its record
                } else if (lane < T.nO) {
                    okey = mem_key<POL>(sm->OM[lane]);
                }
                // keys mirrored to X[32..] (p* and ranking read them from smem);
                // keep the ongoing records sorted by their new keys (usually they are)
                if (lane < T.nO) sm->X[32 + lane] = okey;
                __syncwarp();
                if (POL != SS_POLICY_FCFS &&
                    __ballot_sync(FULL, lane + 1 < T.nO && klt(sm->X[32 + ((lane + 1) & 31)], okey))) {
                    int r = 0;
                    for (int k = 0; uni(k < T.nO); k++) {
                        const Key x = sm->X[32 + k];
                        if (klt(x, okey) || (keq(x, okey) && k < lane)) r++;
                    }
                    MemS mine;
                    if (lane < T.nO) mine = sm->OM[lane];
                    __syncwarp();
                    if (lane < T.nO) {
                        sm->OM[r] = mine;
                        sm->X[32 + r] = okey;
                    }
                    __syncwarp();
                    if (lane < T.nO) okey = sm->X[32 + lane];
                }
            }
            if (logging) {
                __syncwarp();
                if (c.logpos > c.logcap) set_status(T, SS_TRACE_LOG_OVERFLOW);
            }
            if (T.rounds >= round_cap) set_status(T, SS_TRACE_ROUND_CAP);

            // ---- queue rebuild: drop popped FRONT entries, then insert this
            SS_SECT(13);
            //      round's pushed-back / failed / evicted requests with the key
            //      they were queued with (the heap stores keys at insert time)
            f_compact(E, T, R.rmF);
            for (int base = 0; uni(base < T.nins); base += 32) {
                const int i = base + lane;
                bool v = false;
                Key k;
                if (i < T.nins) {
                    k = INS(A)[T.off + i];
                    const uint32_t s = k.aux & SLOT_MASK;
                    if (s != SLOT_MASK) {
                        v = true;
                        atomicAnd(FLG(A, T.off + s), ~F_INS);  // result unused: no round trip
                    }
                }
                const int2 qs = q_insert32(&A, sm, T.off, T.nF, T.nB, T.nRun, k, v);
                T.nF = qs.x;
                T.nB = qs.y;
            }
            T.nins = 0;
        }

        // ---- per-trace results; the per-request outputs and the fused waiting-time
        // statistics (metrics.py:35-56) are finished after this kernel by ss_epilogue.cu
        SS_SECT(4);
        {
            dig = warp_sum_u64(dig);
            ss_trace_stats* st = A.out.stats + t;
            if (lane == 0) {
                st->digest = want_digest ? dig : 0ull;
                st->rounds = T.rounds;
                st->evictions = c.evictions;
                st->mem_used_peak = peak;
                st->log_words = c.log ? (c.logpos < c.logcap ? c.logpos : c.logcap) : 0;
                st->unservable = c.nuns;
                st->status = T.status;
                st->lost_evictions = c.lost;
                st->anomalies = c.anomalies;
#ifdef SS_DEBUG_ANOM
                st->_pad = c.dbg;
#elif defined(SS_DEBUG_TRACE_TIME)  // dev builds: start and duration of the trace (ns, globaltimer)
                unsigned long long dbg_t1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t1));
                st->_pad = (int)(dbg_t1 - dbg_t0);
                st->sum_pool = (long long)dbg_t0;
                {
                    unsigned smid;
                    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                    st->sum_victims = (long long)smid;
                }
#else
                st->_pad = 0;
#endif
#ifndef SS_DEBUG_TRACE_TIME
                st->sum_pool = c.s_pool;
#endif
                st->sum_granted = c.s_granted;
#ifndef SS_DEBUG_TRACE_TIME
                st->sum_victims = c.s_victims;
#endif
                st->sum_resident_evict = c.s_res;
                st->final_clock = T.clock;
            }
        }
#ifdef SS_DEBUG_TIMING
        SS_SECT(0);
        if (lane == 0 && t < SS_DBG_TRACES)
            for (int i = 0; i < SS_DBG_SLOTS; i++) g_dbg_trace[t][i] = dbg_acc[i] - dbg_snap[i];
#endif
        __syncwarp();
    }
#ifdef SS_DEBUG_TIMING
    SS_SECT(0);
    if (lane == 0)
        for (int i = 0; i < SS_DBG_SLOTS; i++) atomicAdd(&g_dbg_cycles[i], dbg_acc[i]);
#endif
}

// --------------------------------------------------------------------------
// host-side launch helpers
// --------------------------------------------------------------------------
static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

static long long tiles_for(int64_t n) { return ((n > 0 ? n : 1) + RS_TILE - 1) / RS_TILE; }
// every trace has ceil(n_t / EPI_TILE) <= n_t / EPI_TILE + 1 epilogue tiles
static size_t epi_tiles_max(int64_t n, int32_t T) {
    return (size_t)(n > 0 ? n : 1) / EPI_TILE + (size_t)(T > 0 ? T : 1) + 1;
}

// Layout: zero-initialised block first (one memset per run), then scratch.
size_t work_bytes(int64_t n, int32_t T) {
    size_t nn = (size_t)(n > 0 ? n : 1), tt = (size_t)(T > 0 ? T : 1);
    size_t zero = 2 * align16(tt * 8) + align16(tt * 4) + align16((size_t)RS_PASSES * 256 * 4) + 16;
    // st, dy, B, ins, S, k0: 16 B; rpos, R, pend, tt0, tt1: 4 B
    return zero + 6 * align16(nn * 16) + 5 * align16(nn * 4) + align16(tt * 4) + align16((tt + 1) * 8) +
           align16((size_t)(RS_PASSES + 1) * 4) + align16((size_t)256 * tiles_for(n) * 4) +
           align16(tt * 4) + align16((tt + 1) * 8) + align16(epi_tiles_max(n, T) * sizeof(EpiPart));
}

size_t work_zero_bytes(int32_t T) {
    size_t tt = (size_t)(T > 0 ? T : 1);
    return 2 * align16(tt * 8) + align16(tt * 4) + align16((size_t)RS_PASSES * 256 * 4) + 16;
}

void carve_work(void* base, int64_t n, int32_t T, Work* w) {
    size_t nn = (size_t)(n > 0 ? n : 1), tt = (size_t)(T > 0 ? T : 1);
    char* p = (char*)base;
    w->tok = (unsigned long long*)p; p += align16(tt * 8);
    w->foot = (unsigned long long*)p; p += align16(tt * 8);
    w->nuns = (uint32_t*)p;  p += align16(tt * 4);
    w->hist = (uint32_t*)p;  p += align16((size_t)RS_PASSES * 256 * 4);
    w->next_trace = (int*)p; w->sel = (int*)p + 1; p += 16;
    w->st = (void*)p;        p += align16(nn * 16);
    w->dy = (void*)p;        p += align16(nn * 16);
    w->B = (void*)p;         p += align16(nn * 16);
    w->ins = (void*)p;       p += align16(nn * 16);
    w->S = (void*)p;         p += align16(nn * 16);
    w->k0 = (void*)p;        p += align16(nn * 16);
    w->rpos = (uint32_t*)p;  p += align16(nn * 4);
    w->R = (uint32_t*)p;     p += align16(nn * 4);
    w->pend = (uint32_t*)p;  p += align16(nn * 4);
    w->tt0 = (uint32_t*)p;   p += align16(nn * 4);
    w->tt1 = (uint32_t*)p;   p += align16(nn * 4);
    w->bulkP = (int*)p;      p += align16(tt * 4);
    w->eoff = (long long*)p; p += align16((tt + 1) * 8);
    w->plan = (int*)p;       p += align16((size_t)(RS_PASSES + 1) * 4);
    w->tcnt = (uint32_t*)p;  p += align16((size_t)256 * tiles_for(n) * 4);
    w->tiles_max = tiles_for(n);
    w->epT = (int*)p;        p += align16(tt * 4);
    w->epoff = (long long*)p; p += align16((tt + 1) * 8);
    w->epart = (void*)p;
}

int sched_smem_bytes() { return (int)(sizeof(WarpSmem) * WPB); }

static int mode_of(uint32_t flags) {
    return ((flags & SS_FLAG_DIGEST) ? 1 : 0) | ((flags & SS_FLAG_ROUND_LOG) ? 2 : 0);
}

// MODE bits: 0 digest, 1 round log, 2 chunked stretches (semantic), 3 no eviction
// possible (with 2), 4 "sum" batch durations
#define SS_K(M) \
    case M: return (const void*)sched_kernel<POL, M>;
template <int POL>
static const void* kernel_ptr(int mode) {
    if constexpr (POL == SS_POLICY_SEMANTIC) {
        switch (mode) {
            SS_K(0) SS_K(1) SS_K(2) SS_K(3) SS_K(4) SS_K(5) SS_K(6) SS_K(7)
            SS_K(12) SS_K(13) SS_K(14) SS_K(15)
            SS_K(16) SS_K(17) SS_K(18) SS_K(19) SS_K(20) SS_K(21) SS_K(22) SS_K(23)
            SS_K(28) SS_K(29) SS_K(30) SS_K(31)
        default: return nullptr;
        }
    } else {  // the stretch / chunk fast paths exist for the semantic policy only
        switch (mode) {
            SS_K(0) SS_K(1) SS_K(2) SS_K(3) SS_K(16) SS_K(17) SS_K(18) SS_K(19)
        default: return nullptr;
        }
    }
}
#undef SS_K

static const void* kernel_for(int policy, int mode) {
    switch (policy) {
    case SS_POLICY_SEMANTIC: return kernel_ptr<SS_POLICY_SEMANTIC>(mode);
    case SS_POLICY_FCFS: return kernel_ptr<SS_POLICY_FCFS>(mode);
    case SS_POLICY_SJF: return kernel_ptr<SS_POLICY_SJF>(mode);
    case SS_POLICY_HPJF: return kernel_ptr<SS_POLICY_HPJF>(mode);
    default: return nullptr;
    }
}

int sched_max_blocks(int policy, int* sm_count) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const void* k = kernel_for(policy, 1);
    if (!k) return 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sched_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * WPB, sched_smem_bytes());
    if (sm_count) *sm_count = sms;
    return per * sms;
}

int launch_sched(const KArgs& a, int blocks, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    size_t smem = (size_t)sched_smem_bytes();
    const int mode = mode_of(a.P.flags) | (a.P.decode_cost_sum ? 16 : 0);
    const void* k = kernel_for(a.P.policy, mode);
    if (!k) return SS_ERR_UNSUPPORTED;
    void* argv[] = {(void*)&a};
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem > (size_t)optin) return SS_ERR_UNSUPPORTED;  // SS_WPB x per-warp state exceeds the SM
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SS_ERR_CUDA;
    if (a.P.policy == SS_POLICY_SEMANTIC) {  // the chunked variants first; the unselected ones exit at once
        for (int v : {12, 4}) {
            const void* kc = kernel_for(a.P.policy, mode | v);
            cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (cudaLaunchKernel(kc, dim3(blocks), dim3(32 * WPB), argv, smem, st) != cudaSuccess) return SS_ERR_CUDA;
        }
    }
    if (cudaLaunchKernel(k, dim3(blocks), dim3(32 * WPB), argv, smem, st) != cudaSuccess) return SS_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

int sched_launches(int policy) { return policy == SS_POLICY_SEMANTIC ? 3 : 1; }

}  // namespace ss

#ifdef SS_DEBUG_TIMING
// debug builds only (not part of include/semsched_b200.h): read and clear the section counters
extern "C" int ss_debug_trace_cycles(unsigned long long* out, int n) {
    cudaDeviceSynchronize();
    if (n > ss::SS_DBG_TRACES) n = ss::SS_DBG_TRACES;
    return cudaMemcpyFromSymbol(out, ss::g_dbg_trace, sizeof(unsigned long long) * ss::SS_DBG_SLOTS * (size_t)n) == cudaSuccess ? 0 : -1;
}
extern "C" int ss_debug_cycles(unsigned long long* out) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, ss::g_dbg_cycles, sizeof(unsigned long long) * ss::SS_DBG_SLOTS) != cudaSuccess) return -1;
    unsigned long long z[ss::SS_DBG_SLOTS] = {0};
    return cudaMemcpyToSymbol(ss::g_dbg_cycles, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif
