// ss_costs.cuh — the reference's analytical cost model on the device.
//
// Every expression keeps the reference's association order
// (/root/reference/pkg/src/semsched/costs.py:99-191); the translation unit is
// compiled with -fmad=false so no multiply-add pair is contracted into an
// FMA (an FMA changes gamma1*n+gamma2 for 2-246 of 4,096 inputs).
// The explicit __dmul_rn/__dadd_rn intrinsics make that independent of the
// compiler flag as well.
#pragma once
#include <stdint.h>

#include "../../include/semsched_b200.h"

#ifndef SS_HDI
#define SS_HDI __host__ __device__ __forceinline__
#endif

namespace ss {

#if defined(__CUDA_ARCH__)
SS_HDI double mul(double a, double b) { return __dmul_rn(a, b); }
SS_HDI double add(double a, double b) { return __dadd_rn(a, b); }
SS_HDI double sub(double a, double b) { return __dsub_rn(a, b); }
SS_HDI double dv(double a, double b) { return __ddiv_rn(a, b); }
#else
SS_HDI double mul(double a, double b) { return a * b; }
SS_HDI double add(double a, double b) { return a + b; }
SS_HDI double sub(double a, double b) { return a - b; }
SS_HDI double dv(double a, double b) { return a / b; }
#endif

// costs.py:99-102   prefill(n) = (a1*n)*n + a2*n
SS_HDI double prefill_time(int64_t n, const ss_profile& p) {
    double d = (double)n;
    return add(mul(mul(p.alpha1, d), d), mul(p.alpha2, d));
}
// costs.py:105-109  gamma1*(n+j-1) + gamma2
SS_HDI double decode_step_time(int64_t n, int64_t j, const ss_profile& p) {
    return add(mul(p.gamma1, (double)(n + j - 1)), p.gamma2);
}
// costs.py:112-116  gamma1*(((0.5*m)*m + n*m) + 0.5*m) + gamma2*m, n*m exact int
SS_HDI double decode_total_time(int64_t n, int64_t m, const ss_profile& p) {
    double dm = (double)m;
    double inner = add(mul(mul(0.5, dm), dm), (double)(n * m));
    inner = add(inner, mul(0.5, dm));
    return add(mul(p.gamma1, inner), mul(p.gamma2, dm));
}
// the same value for 32-bit token counts (n*m < 2^64 exactly; conversions exact-rounded alike)
SS_HDI double decode_total_time_u32(uint32_t n, uint32_t m, const ss_profile& p) {
    double dm = (double)m;
    double inner = add(mul(mul(0.5, dm), dm), (double)((unsigned long long)n * m));
    inner = add(inner, mul(0.5, dm));
    return add(mul(p.gamma1, inner), mul(p.gamma2, dm));
}
// costs.py:119-122
SS_HDI double reload_time(int64_t tokens, const ss_profile& p) {
    return mul(p.beta_load, (double)tokens);
}
// costs.py:125-130  offload iff beta_load < a1*n + a2 (strict)
SS_HDI bool should_cache_prefill(int64_t n, const ss_profile& p) {
    return p.beta_load < add(mul(p.alpha1, (double)n), p.alpha2);
}
// costs.py:133-139
SS_HDI double resume_cost(int64_t n, int64_t m_done, int64_t m_saved, const ss_profile& p) {
    return add(mul(p.beta_load, (double)m_saved), decode_total_time(n, m_done - m_saved, p));
}
// min(m_done, max(0, floor/ceil(s))) with Python-int semantics
SS_HDI int64_t clamp_round(double v, int64_t m_done) {
    if (!(v > 0.0)) return 0;
    if (v >= (double)m_done) return m_done;
    return (int64_t)v;
}
// costs.py:142-171  Eq. 6 integer argmin, ties -> larger save count
SS_HDI int64_t optimal_save_tokens(int64_t n, int64_t m_done, const ss_profile& p) {
    if (m_done == 0) return 0;
    if (p.gamma1 == 0.0) {
        double none = resume_cost(n, m_done, 0, p), all = resume_cost(n, m_done, m_done, p);
        return all <= none ? m_done : 0;
    }
    double k = sub(p.beta_load, mul(p.gamma1, (double)n));
    k = sub(k, dv(p.gamma1, 2.0));
    k = sub(k, p.gamma2);
    k = dv(k, p.gamma1);
    double s_real = sub((double)m_done, k);
    int64_t lo = clamp_round(floor(s_real), m_done);
    int64_t hi = clamp_round(ceil(s_real), m_done);
    if (hi == lo) return lo;
    return resume_cost(n, m_done, hi, p) <= resume_cost(n, m_done, lo, p) ? hi : lo;
}
// costs.py:174-191  f_t = reload(kv_host) + prefill(prompt-prefilled)
//                         + decode_total(prompt+decoded, max(1, mid-decoded))
SS_HDI double remaining_time(int64_t prompt, int64_t mid, int64_t prefilled, int64_t decoded,
                             int64_t kv_host, const ss_profile& p) {
    double total = reload_time(kv_host, p);
    total = add(total, prefill_time(prompt - prefilled, p));
    int64_t left = mid - decoded;
    if (left < 1) left = 1;
    return add(total, decode_total_time(prompt + decoded, left, p));
}

// CPython >= 3.12 float sum() (Neumaier), bltinmodule.c builtin_sum_impl.
struct PySum {
    double s, c;
    int n;
    SS_HDI void init() { s = 0.0; c = 0.0; n = 0; }
    SS_HDI void push(double x) {
        if (n == 0) { s = x; c = 0.0; n = 1; return; }
        double t = add(s, x);
        if (fabs(s) >= fabs(x)) c = add(c, add(sub(s, t), x));
        else c = add(c, add(sub(x, t), s));
        s = t;
        n++;
    }
    SS_HDI double value() const {
        if (n == 0) return 0.0;
        return (c != 0.0 && isfinite(c)) ? add(s, c) : s;
    }
};

}  // namespace ss
