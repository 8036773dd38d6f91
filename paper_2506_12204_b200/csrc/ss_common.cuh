// ss_common.cuh — request records, flags and the packed dispatch key shared
// by the scheduler kernel (ss_kernel.cu) and the grid-wide prepass
// (ss_prepass.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ss_kernel.cuh"

namespace ss {

constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t ST_WAIT = 0, ST_DEC = 2, ST_DONE = 5, ST_UNS = 6;
constexpr uint32_t F_STAGE = 7u, F_PF = 8u, F_Q = 16u, F_INS = 32u, F_FIRST = 64u, F_GRANT = 128u;
// set with ST_UNS when the request was DECODING at _mark_unservable (engine.py:402-412 keeps its stage)
constexpr uint32_t F_UDEC = 256u;
// the per-request output state code: stage | prefilled << 8 | (unservable while decoding) << 9
__host__ __device__ __forceinline__ uint32_t state_code(uint32_t flg) {
    return (flg & F_STAGE) | ((flg & F_PF) ? 256u : 0u) | ((flg & F_UDEC) ? 512u : 0u);
}
constexpr uint32_t SLOT_MASK = 0x00FFFFFFu, DEC_BIT = 0x80000000u;

struct __align__(16) Key {
    unsigned long long hi;
    uint32_t lo;
    uint32_t aux;  // slot | decoding << 31
};

// dynamic record of a request in HBM
struct __align__(16) Dyn {
    double ft;
    uint32_t dec;
    uint32_t flg;
};

__device__ __forceinline__ bool klt(const Key& a, const Key& b) {
#ifdef SS_KLT_SHORT
    return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
#else
    return (a.hi < b.hi) | ((a.hi == b.hi) & (a.lo < b.lo));  // branch-free (no short-circuit)
#endif
}
__device__ __forceinline__ bool keq(const Key& a, const Key& b) { return (a.hi == b.hi) & (a.lo == b.lo); }
// branch-free forms for hot warp-synchronous code (no short-circuit branches)
__device__ __forceinline__ bool klt_nb(const Key& a, const Key& b) {
    return (a.hi < b.hi) | ((a.hi == b.hi) & (a.lo < b.lo));
}
__device__ __forceinline__ Key kinf() {
    Key k;
    k.hi = ~0ull;
    k.lo = ~0u;
    k.aux = ~0u;
    return k;
}
// index t with off[t] <= g < off[t+1] (first such t past empty ranges)
template <typename I>
__device__ __forceinline__ int upper_index(const I* off, int n, long long g) {
    int lo = 0, hi = n;  // search in off[0..n]
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if ((long long)off[mid + 1] <= g) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
template <int POL>
__device__ __forceinline__ Key make_key(uint32_t urank, double ft, uint32_t tie, uint32_t slot,
                                        bool decoding) {
    unsigned long long fb = (unsigned long long)__double_as_longlong(ft);
    Key k;
    if (POL == SS_POLICY_SEMANTIC) {
        k.hi = ((unsigned long long)urank << 56) | (fb >> 7);
        k.lo = ((uint32_t)(fb & 127ull) << 25) | tie;
    } else if (POL == SS_POLICY_FCFS) {
        k.hi = 0ull;
        k.lo = tie;
    } else if (POL == SS_POLICY_SJF) {
        k.hi = fb >> 7;
        k.lo = ((uint32_t)(fb & 127ull) << 25) | tie;
    } else {
        k.hi = (unsigned long long)urank << 56;
        k.lo = tie;
    }
    k.aux = slot | (decoding ? DEC_BIT : 0u);
    return k;
}
}  // namespace ss
