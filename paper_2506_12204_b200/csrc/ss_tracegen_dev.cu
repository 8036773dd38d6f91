// ss_tracegen_dev.cu — the bulk trace generator on the device: one thread per
// trace, writing the scheduler's SoA inputs straight into HBM.
//
// Same draws as the host generator (ss_tracegen.cpp) and therefore as the
// reference's generate() + predictor_pipeline() (workload.py:63-93,
// predictors.py:85-149): CPython's MT19937 with init_by_array seeding,
// random() (53-bit), getrandbits / _randbelow, choices() via bisect on the
// cumulative weights. The Mersenne Twister state (624 words) lives in the
// thread's local memory (L1-resident at these occupancies).
//
// Pending order needs no sort: generate() emits arrivals in (arrival, id)
// order, and the prediction server is FIFO (predictors.py:107-148: every
// batch starts at max(fill time, server free) and finishes `latency` later),
// so ready times are non-decreasing in generation order and the reference's
// sort by (ready, arrival, id) is the identity. The kernel checks this and
// reports a violation instead of silently emitting another order.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/semsched_tracegen.h"

namespace {

struct DevMT {
    uint32_t mt[624];
    int mti;
    __device__ void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < 624; mti++) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    __device__ void seed(int64_t s) {
        uint64_t a = s < 0 ? (uint64_t)(-(s + 1)) + 1u : (uint64_t)s;
        uint32_t key[2];
        int n = 0;
        if (a == 0) key[n++] = 0;
        while (a) {
            key[n++] = (uint32_t)(a & 0xffffffffu);
            a >>= 32;
        }
        init_genrand(19650218u);
        int i = 1, j = 0;
        for (int k = 624; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
            if (j >= n) j = 0;
        }
        for (int k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            i++;
            if (i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
        }
        mt[0] = 0x80000000u;
        mti = 624;
    }
    __device__ void twist() {
        int kk;
        uint32_t y;
        for (kk = 0; kk < 624 - 397; kk++) {
            y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
            mt[kk] = mt[kk + 397] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        for (; kk < 623; kk++) {
            y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
            mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
        mt[623] = mt[396] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        mti = 0;
    }
    __device__ uint32_t u32() {
        if (mti >= 624) twist();
        uint32_t y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= (y >> 18);
        return y;
    }
    __device__ double random() {
        const uint32_t a = u32() >> 5, b = u32() >> 6;
        return __dmul_rn(__dadd_rn(__dmul_rn((double)a, 67108864.0), (double)b), 1.0 / 9007199254740992.0);
    }
    __device__ uint32_t getrandbits(int k) { return u32() >> (32 - k); }
    __device__ uint64_t randbelow(uint64_t n) {
        const int k = 64 - __clzll((long long)n);
        if (k <= 32) {
            uint32_t r = getrandbits(k);
            while (r >= n) r = getrandbits(k);
            return r;
        }
        for (;;) {
            const uint64_t lo = u32();
            const uint64_t hi = u32() >> (64 - k);
            const uint64_t r = lo | (hi << 32);
            if (r < n) return r;
        }
    }
    __device__ int64_t randint(int64_t a, int64_t b) { return a + (int64_t)randbelow((uint64_t)(b - a + 1)); }
};

struct DevSpec {
    ss_gen_spec s;
    const double* cum;        // [levels] cumulative urgency weights (host-computed, same adds)
    const uint32_t* reps;     // [buckets]
    const int64_t* seeds;
    const int64_t* pseeds;
    int64_t n_traces;
    int* bad;                 // set when the ready order is not monotone
};

__global__ void __launch_bounds__(64) gen_kernel(const DevSpec D, const ss_gen_out O) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= D.n_traces) return;
    const ss_gen_spec& S = D.s;
    const int64_t N = S.total_requests, off = t * N;
    DevMT g;
    // ---- workload.generate (workload.py:63-93)
    g.seed(D.seeds[t]);
    const double total = __dadd_rn(D.cum[S.levels - 1], 0.0);
    int64_t placed = 0, tick = 0;
    while (placed < N) {
        int64_t k = S.concurrent_fixed ? S.concurrent : g.randint(1, S.concurrent);
        if (k > N - placed) k = N - placed;
        const double at = __dmul_rn((double)tick, S.gap_s);
        for (int64_t q = 0; q < k; q++) {
            const double x = __dmul_rn(g.random(), total);
            int lo = 0, hi = S.levels - 1;  // bisect_right(cum, x, 0, levels - 1)
            while (lo < hi) {
                const int mid = (lo + hi) / 2;
                if (x < D.cum[mid]) hi = mid;
                else lo = mid + 1;
            }
            const int64_t pl = g.randint(S.prompt_lo, S.prompt_hi);
            const int64_t ol = g.randint(S.out_lo, S.out_hi);
            const int64_t g2 = off + placed;
            O.arrival[g2] = at;
            O.prompt[g2] = (uint32_t)pl;
            O.true_out[g2] = (uint32_t)ol;
            O.true_urg[g2] = (uint8_t)lo;
            O.tie[g2] = (uint32_t)placed;
            if (O.ids) O.ids[g2] = placed;
            if (O.record_pos) O.record_pos[g2] = placed;
            placed++;
        }
        tick++;
    }
    // ---- predictors.predictor_pipeline (predictors.py:85-149)
    g.seed(D.pseeds[t]);
    for (int64_t i = 0; i < N; i++) {
        const int64_t g2 = off + i;
        int64_t u = O.true_urg[g2];
        if (!(g.random() >= S.urgency_error)) {
            const int64_t d = S.urgency_disp, hi = S.levels - 1;
            const int64_t step = g.random() < 0.5 ? d : -d;
            int64_t o = u + step < 0 ? 0 : (u + step > hi ? hi : u + step);
            if (o == u) o = u - step < 0 ? 0 : (u - step > hi ? hi : u - step);
            u = o;
        }
        int64_t len = O.true_out[g2];
        if (g.random() < S.length_error) {
            const int64_t d = S.length_disp, hi = S.max_output_len;
            const int64_t step = g.random() < 0.5 ? d : -d;
            int64_t o = len + step < 0 ? 0 : (len + step > hi ? hi : len + step);
            if (o == len) o = len - step < 0 ? 0 : (len - step > hi ? hi : len - step);
            len = o;
        }
        if (len > S.max_output_len) len = S.max_output_len;
        int64_t idx = (len * S.buckets) / S.max_output_len;
        if (idx > S.buckets - 1) idx = S.buckets - 1;
        O.pred_urg[g2] = (uint8_t)u;
        O.pred_len[g2] = D.reps[idx];
    }
    // FIFO prediction server: ready times (non-decreasing in generation order)
    double free_at = 0.0;
    auto serve = [&](int64_t a, int64_t b, double filled) {
        const double start = filled >= free_at ? filled : free_at;
        const double done = __dadd_rn(start, S.latency_s);
        free_at = done;
        for (int64_t i = a; i < b; i++) O.ready[off + i] = done;
    };
    if (!S.full_batching) {
        int64_t i = 0;
        while (i < N) {
            const double at = O.arrival[off + i];
            int64_t j = i;
            while (j < N && O.arrival[off + j] == at) j++;
            for (int64_t k = i; k < j; k += S.pred_batch) serve(k, k + S.pred_batch < j ? k + S.pred_batch : j, at);
            i = j;
        }
    } else {
        int64_t start = 0;
        for (int64_t i = 0; i < N; i++) {
            if (i + 1 - start >= S.pred_batch) {
                serve(start, i + 1, O.arrival[off + i]);
                start = i + 1;
            }
        }
        if (start < N) serve(start, N, O.arrival[off + N - 1]);
    }
    for (int64_t i = 1; i < N; i++)
        if (O.ready[off + i] < O.ready[off + i - 1]) atomicExch(D.bad, 1);
}

}  // namespace

extern "C" int ss_generate_traces_device(const ss_gen_spec* spec, int64_t n_traces, const int64_t* seeds,
                                         const int64_t* pred_seeds, const ss_gen_out* out, void* stream) {
    if (!spec || !out || (n_traces > 0 && (!seeds || !pred_seeds))) return 1;
    const ss_gen_spec S = *spec;
    if (S.total_requests < 0 || S.levels < 1 || S.levels > 255 || S.concurrent < 1 || S.buckets < 1 ||
        S.max_output_len < 1 || S.pred_batch < 1 || S.out_hi > S.max_output_len || S.prompt_lo < 1 ||
        S.out_lo < 1 || !S.bucket_reps)
        return 1;
    if (n_traces == 0 || S.total_requests == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    // cumulative weights with the host's (and Python's) left-to-right adds
    double cum[256];
    double acc = 0.0;
    for (int l = 0; l < S.levels; l++) {
        acc += S.urgency_weights ? S.urgency_weights[l] : 1.0;
        cum[l] = acc;
    }
    const size_t nb = (size_t)S.levels * 8 + (size_t)S.buckets * 4 + (size_t)n_traces * 16 + 16;
    char* buf = nullptr;
    if (cudaMalloc(&buf, nb) != cudaSuccess) return 2;
    double* d_cum = (double*)buf;
    uint32_t* d_reps = (uint32_t*)(buf + (size_t)S.levels * 8);
    int64_t* d_seeds = (int64_t*)(buf + (((size_t)S.levels * 8 + (size_t)S.buckets * 4 + 7) & ~(size_t)7));
    int64_t* d_pseeds = d_seeds + n_traces;
    int* d_bad = (int*)(d_pseeds + n_traces);
    cudaMemcpyAsync(d_cum, cum, (size_t)S.levels * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_reps, S.bucket_reps, (size_t)S.buckets * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_seeds, seeds, (size_t)n_traces * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_pseeds, pred_seeds, (size_t)n_traces * 8, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(d_bad, 0, sizeof(int), st);
    DevSpec D;
    D.s = S;
    D.cum = d_cum;
    D.reps = d_reps;
    D.seeds = d_seeds;
    D.pseeds = d_pseeds;
    D.n_traces = n_traces;
    D.bad = d_bad;
    gen_kernel<<<(unsigned)((n_traces + 63) / 64), 64, 0, st>>>(D, *out);
    int bad = 0;
    cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(buf);
    if (e != cudaSuccess) return 2;
    return bad ? 3 : 0;
}
