// ss_audit.cu — the completion-order constraint audit (Eq. 2) on the device,
// for one trace or thousands at once.
//
// Reference: metrics.constraint_audit (metrics.py:59-91). Completed records
// are sorted by finish time (stable) and every pair a < b is examined:
//   skip if f_a >= f_b;  comparable += 1;  skip if f_a < arrival_b;
//   skip if rank_a <= rank_b;  else (id_a, id_b) is a violation.
// Because ties in f are skipped, the counted pairs are exactly the ordered
// pairs with f_i < f_j — no sort is needed for the counts. One thread owns a
// row i and sweeps the trace's records staged tile by tile in shared memory
// (O(n^2) compare work, the reference's own complexity, at full SM width).
// The ordered pair list (optional) needs each row's rank in the stable
// finish-time order (counted in the same sweep) and, per row, the later rows
// in that order: rows are scattered to their rank, per-row counts scanned,
// and a second sweep writes (id_i, id_j) in the reference's order.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "../../include/semsched_b200.h"

namespace ss {
namespace {

constexpr int AT = 256;    // rows per CTA
constexpr int TILE = 1024; // records staged per shared-memory tile

struct AuditIn {
    const int64_t* off;
    const double* fin;
    const double* arr;
    const int32_t* rank;
    int32_t n_traces;
};

// per row: comparable / violations with the row first; rank in stable order
__global__ void __launch_bounds__(AT) audit_rows(AuditIn in, long long* viol_t, long long* comp_t,
                                                  uint32_t* row_viol, uint32_t* row_rank, int want_rank) {
    __shared__ double sf[TILE], sa[TILE];
    __shared__ int32_t sr[TILE];
    const int t = blockIdx.x;
    const long long o = in.off[t], n = in.off[t + 1] - o;
    const long long i = (long long)blockIdx.y * AT + threadIdx.x;
    if ((long long)blockIdx.y * AT >= n) return;
    const bool mine = i < n;
    double fi = 0.0;
    int32_t ri = 0;
    bool done_i = false;
    if (mine) {
        fi = in.fin[o + i];
        ri = in.rank[o + i];
        done_i = !isnan(fi);
    }
    unsigned long long c = 0, v = 0, rk = 0;
    for (long long base = 0; base < n; base += TILE) {
        const int m = (int)(n - base < TILE ? n - base : TILE);
        __syncthreads();
        for (int k = threadIdx.x; k < m; k += AT) {
            sf[k] = in.fin[o + base + k];
            sa[k] = in.arr[o + base + k];
            sr[k] = in.rank[o + base + k];
        }
        __syncthreads();
        if (done_i) {
            for (int k = 0; k < m; k++) {
                const double fj = sf[k];  // NaN (not completed) fails every compare
                const bool later = fi < fj;
                c += later;
                v += later && !(fi < sa[k]) && ri > sr[k];
                rk += fj < fi || (fj == fi && base + k < i);
            }
        }
    }
    if (mine) {
        if (row_viol) row_viol[o + i] = (uint32_t)v;
        if (want_rank) row_rank[o + i] = (uint32_t)rk;
    }
    // block totals
    __shared__ unsigned long long bc[AT / 32], bv[AT / 32];
    for (int s = 16; s > 0; s >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, s);
        v += __shfl_xor_sync(0xffffffffu, v, s);
    }
    if ((threadIdx.x & 31) == 0) {
        bc[threadIdx.x >> 5] = c;
        bv[threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long C = 0, V = 0;
        for (int w = 0; w < AT / 32; w++) {
            C += bc[w];
            V += bv[w];
        }
        if (C) atomicAdd((unsigned long long*)&comp_t[t], C);
        if (V) atomicAdd((unsigned long long*)&viol_t[t], V);
    }
}

// completed rows scattered to their stable finish-time rank; per-rank counts
__global__ void audit_scatter(AuditIn in, const uint32_t* row_viol, const uint32_t* row_rank, int32_t* by_rank,
                              uint32_t* cnt_by_rank) {
    const int t = blockIdx.x;
    const long long o = in.off[t], n = in.off[t + 1] - o;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        if (isnan(in.fin[o + i])) continue;
        const uint32_t r = row_rank[o + i];
        by_rank[o + r] = (int32_t)i;
        cnt_by_rank[o + r] = row_viol[o + i];
    }
}

// per trace: exclusive scan of the counts in rank order (+ the trace's base)
__global__ void __launch_bounds__(1024) audit_scan(AuditIn in, const long long* ncomp, const uint32_t* cnt_by_rank,
                                                   const long long* base_t, long long* pos_by_rank) {
    __shared__ long long ws[32];
    __shared__ long long carry;
    const int t = blockIdx.x;
    const long long o = in.off[t], nc = ncomp[t];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = base_t[t];
    __syncthreads();
    for (long long b0 = 0; b0 < nc; b0 += 1024) {
        const long long r = b0 + threadIdx.x;
        const long long x0 = r < nc ? (long long)cnt_by_rank[o + r] : 0;
        long long x = x0;
        for (int s = 1; s < 32; s <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, s);
            if (lane >= s) x += y;
        }
        if (lane == 31) ws[wid] = x;
        __syncthreads();
        if (wid == 0) {
            long long s2 = ws[lane];
            for (int s = 1; s < 32; s <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, s2, s);
                if (lane >= s) s2 += y;
            }
            ws[lane] = s2;
        }
        __syncthreads();
        const long long pre = carry + (wid ? ws[wid - 1] : 0) + x - x0;
        if (r < nc) pos_by_rank[o + r] = pre;
        __syncthreads();
        if (threadIdx.x == 1023) carry = pre + x0;
        __syncthreads();
    }
}

// pairs (id_i, id_j) in the reference's order: rows by rank, j by rank
__global__ void __launch_bounds__(AT) audit_pairs(AuditIn in, const int64_t* ids, const long long* ncomp,
                                                   const int32_t* by_rank, const long long* pos_by_rank,
                                                   int64_t* pairs) {
    const int t = blockIdx.x;
    const long long o = in.off[t], nc = ncomp[t];
    const long long r = (long long)blockIdx.y * AT + threadIdx.x;
    if (r >= nc) return;
    const long long i = by_rank[o + r];
    const double fi = in.fin[o + i];
    const int32_t ri = in.rank[o + i];
    const int64_t idi = ids[o + i];
    long long w = pos_by_rank[o + r];
    for (long long p = r + 1; p < nc; p++) {
        const long long j = by_rank[o + p];
        const double fj = in.fin[o + j];
        if (!(fi < fj)) continue;
        if (fi < in.arr[o + j]) continue;
        if (ri <= in.rank[o + j]) continue;
        pairs[2 * w] = idi;
        pairs[2 * w + 1] = ids[o + j];
        w++;
    }
}

thread_local char g_err[256];
int fail(int code, const char* msg) {
    strncpy(g_err, msg, sizeof g_err - 1);
    return code;
}
size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }
std::mutex g_mu;
void* g_buf = nullptr;
size_t g_cap = 0;
int g_dev = -1;  // device g_buf lives on
thread_local double g_rows_ms = 0.0;

}  // namespace
}  // namespace ss

extern "C" {

const char* ss_audit_last_error(void) { return ss::g_err; }

double ss_audit_last_kernel_ms(void) { return ss::g_rows_ms; }

int ss_audit_host(int32_t n_traces, const int64_t* offsets, const double* finish, const double* arrival,
                  const int32_t* rank, const int64_t* ids, int64_t* violations, int64_t* comparable,
                  int64_t* pairs, int64_t pairs_cap, void* stream) {
    using namespace ss;
    if (n_traces < 0 || (n_traces > 0 && (!offsets || !violations || !comparable)))
        return fail(SS_ERR_INVALID_ARG, "bad arguments");
    if (n_traces == 0) return SS_OK;
    const int64_t n = offsets[n_traces];
    if (n > 0 && (!finish || !arrival || !rank || (pairs && !ids))) return fail(SS_ERR_INVALID_ARG, "null input");
    int64_t maxn = 0;
    for (int32_t t = 0; t < n_traces; t++) {
        const int64_t k = offsets[t + 1] - offsets[t];
        if (k < 0) return fail(SS_ERR_INVALID_ARG, "offsets must be nondecreasing");
        if (k > maxn) maxn = k;
    }
    if (maxn > (int64_t)65535 * AT) return fail(SS_ERR_UNSUPPORTED, "trace longer than 16.7M records");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t T = (size_t)n_traces, nn = (size_t)(n > 0 ? n : 1);
    const bool want = pairs != nullptr;
    size_t need = a16((T + 1) * 8) + 2 * a16(nn * 8) + a16(nn * 4) + a16(nn * 8) + 4 * a16(T * 8) +
                  3 * a16(nn * 4) + a16(nn * 8);
    std::lock_guard<std::mutex> lk(g_mu);
    int cur = 0;
    if (cudaGetDevice(&cur) != cudaSuccess) return fail(SS_ERR_CUDA, "cudaGetDevice");
    if (g_buf && g_dev != cur) {  // the caller moved to another device: release on the old one
        cudaSetDevice(g_dev);
        cudaFree(g_buf);
        cudaSetDevice(cur);
        g_buf = nullptr;
        g_cap = 0;
    }
    g_dev = cur;
    if (g_cap < need) {
        if (g_buf) cudaFree(g_buf);
        g_buf = nullptr;
        g_cap = 0;
        if (cudaMalloc(&g_buf, need) != cudaSuccess) return fail(SS_ERR_CUDA, "cudaMalloc (audit workspace)");
        g_cap = need;
    }
    char* p = (char*)g_buf;
    auto take = [&](size_t b) {
        char* r = p;
        p += a16(b);
        return (void*)r;
    };
    AuditIn in;
    int64_t* d_off = (int64_t*)take((T + 1) * 8);
    double* d_f = (double*)take(nn * 8);
    double* d_a = (double*)take(nn * 8);
    int32_t* d_r = (int32_t*)take(nn * 4);
    int64_t* d_id = (int64_t*)take(nn * 8);
    long long* d_v = (long long*)take(T * 8);
    long long* d_c = (long long*)take(T * 8);
    long long* d_nc = (long long*)take(T * 8);
    long long* d_base = (long long*)take(T * 8);
    uint32_t* d_rv = (uint32_t*)take(nn * 4);
    uint32_t* d_rk = (uint32_t*)take(nn * 4);
    uint32_t* d_cr = (uint32_t*)take(nn * 4);
    long long* d_pos = (long long*)take(nn * 8);
    cudaMemcpyAsync(d_off, offsets, (T + 1) * 8, cudaMemcpyHostToDevice, st);
    if (n > 0) {
        cudaMemcpyAsync(d_f, finish, (size_t)n * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_a, arrival, (size_t)n * 8, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_r, rank, (size_t)n * 4, cudaMemcpyHostToDevice, st);
        if (want) cudaMemcpyAsync(d_id, ids, (size_t)n * 8, cudaMemcpyHostToDevice, st);
    }
    cudaMemsetAsync(d_v, 0, T * 8, st);
    cudaMemsetAsync(d_c, 0, T * 8, st);
    in.off = d_off;
    in.fin = d_f;
    in.arr = d_a;
    in.rank = d_r;
    in.n_traces = n_traces;
    const unsigned yb = (unsigned)((maxn + AT - 1) / AT);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    if (yb > 0) audit_rows<<<dim3((unsigned)T, yb), AT, 0, st>>>(in, d_v, d_c, d_rv, d_rk, want ? 1 : 0);
    cudaError_t le = cudaGetLastError();
    cudaEventRecord(e1, st);
    cudaMemcpyAsync(violations, d_v, T * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(comparable, d_c, T * 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    g_rows_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (le != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(le));
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    if (!want) return SS_OK;
    int64_t total = 0;
    std::vector<long long> base(T), ncomp(T);
    for (size_t t = 0; t < T; t++) {
        base[t] = total;
        total += violations[t];
        long long k = 0;
        for (int64_t i = offsets[t]; i < offsets[t + 1]; i++) k += !isnan(finish[i]);
        ncomp[t] = k;
    }
    if (2 * total > pairs_cap) return fail(SS_ERR_INVALID_ARG, "pairs buffer too small (need 2 x total violations)");
    if (total == 0) return SS_OK;
    int32_t* d_byr = nullptr;
    int64_t* d_pairs = nullptr;
    if (cudaMalloc(&d_byr, nn * 4) != cudaSuccess || cudaMalloc(&d_pairs, (size_t)total * 16) != cudaSuccess) {
        cudaFree(d_byr);
        return fail(SS_ERR_CUDA, "cudaMalloc (audit pairs)");
    }
    cudaMemcpyAsync(d_base, base.data(), T * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_nc, ncomp.data(), T * 8, cudaMemcpyHostToDevice, st);
    audit_scatter<<<(unsigned)T, 256, 0, st>>>(in, d_rv, d_rk, d_byr, d_cr);
    audit_scan<<<(unsigned)T, 1024, 0, st>>>(in, d_nc, d_cr, d_base, d_pos);
    audit_pairs<<<dim3((unsigned)T, yb), AT, 0, st>>>(in, d_id, d_nc, d_byr, d_pos, d_pairs);
    le = cudaGetLastError();
    cudaMemcpyAsync(pairs, d_pairs, (size_t)total * 16, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = le;
    cudaFree(d_byr);
    cudaFree(d_pairs);
    if (e != cudaSuccess) return fail(SS_ERR_CUDA, cudaGetErrorString(e));
    return SS_OK;
}

}  // extern "C"
