// ss_tracegen.cpp — native bulk trace preparation (host, multi-threaded).
//
// Produces, for many seeds at once, exactly the SoA the Python path builds
// from the reference's
//   generate(WorkloadSpec(seed=s))                 workload.py:63-93
//   predictor_pipeline(arrivals, cfg, Random(seed)) predictors.py:85-149
// by re-implementing the CPython `random.Random` calls those functions make:
// MT19937 with init_by_array seeding (Modules/_randommodule.c), random()
// (53-bit), getrandbits(k<=32), randint/randrange via _randbelow_with_
// getrandbits (Lib/random.py), choices() with cumulative weights + bisect.
// Checked against the Python implementation seed by seed in
// tests/test_tracegen.py. This is input preparation, outside the timed
// scheduler path.
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/semsched_tracegen.h"

namespace {

struct MT {
    uint32_t mt[624];
    int mti;
    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < 624; mti++) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t* key, size_t n) {
        init_genrand(19650218u);
        size_t i = 1, j = 0;
        size_t k = 624 > n ? 624 : n;
        for (; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= 624) {
                mt[0] = mt[623];
                i = 1;
            }
            if (j >= n) j = 0;
        }
        for (k = 623; k; k--) {
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
    // random.Random(seed) for a Python int seed: key = 32-bit words of |seed|
    void seed(int64_t s) {
        uint64_t a = s < 0 ? (uint64_t)(-(s + 1)) + 1u : (uint64_t)s;
        uint32_t key[2];
        size_t n = 0;
        if (a == 0) key[n++] = 0;
        while (a) {
            key[n++] = (uint32_t)(a & 0xffffffffu);
            a >>= 32;
        }
        init_by_array(key, n);
    }
    uint32_t u32() {
        static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
        uint32_t y;
        if (mti >= 624) {
            int kk;
            for (kk = 0; kk < 624 - 397; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < 623; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[623] = mt[396] ^ (y >> 1) ^ mag01[y & 1u];
            mti = 0;
        }
        y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= (y >> 18);
        return y;
    }
    double random() {
        uint32_t a = u32() >> 5, b = u32() >> 6;
        return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
    }
    uint32_t getrandbits(int k) { return u32() >> (32 - k); }  // 1 <= k <= 32
    // Random._randbelow_with_getrandbits
    uint64_t randbelow(uint64_t n) {
        int k = 64 - __builtin_clzll(n);
        if (k <= 32) {
            uint32_t r = getrandbits(k);
            while (r >= n) r = getrandbits(k);
            return r;
        }
        // k in 33..64: getrandbits fills 32-bit words little-endian
        for (;;) {
            uint64_t lo = u32();
            uint64_t hi = u32() >> (64 - k);
            uint64_t r = lo | (hi << 32);
            if (r < n) return r;
        }
    }
    int64_t randint(int64_t a, int64_t b) { return a + (int64_t)randbelow((uint64_t)(b - a + 1)); }
};

struct Req {
    int64_t id;
    double arrival;
    uint32_t prompt, out;
    uint8_t urg;
};

// bisect_right(cum, x, 0, hi)
int bisect_right(const double* cum, double x, int hi) {
    int lo = 0;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (x < cum[mid]) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// workload.generate: N requests in generation (= record) order
void gen_arrivals(const ss_gen_spec& S, MT& g, Req* rq) {
    const int64_t N = S.total_requests;
    std::vector<double> cum((size_t)S.levels);
    double acc = 0.0;
    for (int l = 0; l < S.levels; l++) {
        acc += S.urgency_weights ? S.urgency_weights[l] : 1.0;
        cum[(size_t)l] = acc;
    }
    const double total = cum[(size_t)S.levels - 1] + 0.0;
    int64_t placed = 0, tick = 0;
    while (placed < N) {
        int64_t k = S.concurrent_fixed ? S.concurrent : g.randint(1, S.concurrent);
        if (k > N - placed) k = N - placed;
        double t = (double)tick * S.gap_s;
        for (int64_t q = 0; q < k; q++) {
            int u = bisect_right(cum.data(), g.random() * total, S.levels - 1);
            int64_t pl = g.randint(S.prompt_lo, S.prompt_hi);
            int64_t ol = g.randint(S.out_lo, S.out_hi);
            Req& r = rq[placed];
            r.id = placed;
            r.arrival = t;
            r.prompt = (uint32_t)pl;
            r.out = (uint32_t)ol;
            r.urg = (uint8_t)u;
            placed++;
        }
        tick++;
    }
}

// Error-model displacement: +-d with a drawn sign, clamped; the other sign
// when clamping would leave the value unchanged.
int64_t displace(MT& p, int64_t value, int64_t lo, int64_t hi, int64_t d) {
    int64_t step = p.random() < 0.5 ? d : -d;
    int64_t o = std::min(hi, std::max(lo, value + step));
    if (o == value) o = std::min(hi, std::max(lo, value - step));
    return o;
}

// predictors.predictor_pipeline over N time-ordered requests: per request the
// urgency draw(s) then the length draw(s) (`what` bit 0 / bit 1), then the
// single FIFO prediction server's ready times (bit 2). fe: predicted rank,
// bucket: predicted length bucket index.
void predict(const ss_gen_spec& S, MT& p, int64_t N, const Req* rq, int what, uint8_t* fe, uint32_t* bucket,
             double* ready) {
    for (int64_t i = 0; i < N; i++) {
        const Req& r = rq[i];
        if (what & 1) {
            int64_t u = r.urg;
            if (!(p.random() >= S.urgency_error)) u = displace(p, u, 0, S.levels - 1, S.urgency_disp);
            fe[i] = (uint8_t)u;
        }
        if (what & 2) {
            int64_t len = r.out;
            if (p.random() < S.length_error) len = displace(p, len, 0, S.max_output_len, S.length_disp);
            if (len > S.max_output_len) len = S.max_output_len;
            bucket[i] = (uint32_t)std::min<int64_t>(S.buckets - 1, (len * S.buckets) / S.max_output_len);
        }
    }
    if (!(what & 4)) return;
    double free_at = 0.0;
    auto serve = [&](int64_t a, int64_t b, double filled) {
        double start = filled >= free_at ? filled : free_at;  // max(fill_time, server_free)
        double done = start + S.latency_s;
        free_at = done;
        for (int64_t i = a; i < b; i++) ready[i] = done;
    };
    if (!S.full_batching) {
        int64_t i = 0;
        while (i < N) {
            double t = rq[i].arrival;
            int64_t j = i;
            while (j < N && rq[j].arrival == t) j++;
            for (int64_t k = i; k < j; k += S.pred_batch) serve(k, std::min(j, k + S.pred_batch), t);
            i = j;
        }
    } else {
        int64_t start = 0;
        for (int64_t i = 0; i < N; i++) {
            if (i + 1 - start >= S.pred_batch) {
                serve(start, i + 1, rq[i].arrival);
                start = i + 1;
            }
        }
        if (start < N) serve(start, N, rq[N - 1].arrival);
    }
}

void gen_one(const ss_gen_spec& S, int64_t seed, int64_t pred_seed, int64_t off, const ss_gen_out& O) {
    const int64_t N = S.total_requests;
    std::vector<Req> rq((size_t)N);
    MT g;
    g.seed(seed);
    gen_arrivals(S, g, rq.data());
    MT p;
    p.seed(pred_seed);
    std::vector<uint8_t> fe((size_t)N);
    std::vector<uint32_t> bucket((size_t)N);
    std::vector<double> ready((size_t)N);
    predict(S, p, N, rq.data(), 7, fe.data(), bucket.data(), ready.data());
    // pending order: (ready, arrival, id); generate() ids ascend with arrival
    std::vector<int64_t> ord((size_t)N);
    for (int64_t i = 0; i < N; i++) ord[(size_t)i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        if (ready[(size_t)a] != ready[(size_t)b]) return ready[(size_t)a] < ready[(size_t)b];
        if (rq[(size_t)a].arrival != rq[(size_t)b].arrival) return rq[(size_t)a].arrival < rq[(size_t)b].arrival;
        return rq[(size_t)a].id < rq[(size_t)b].id;
    });
    for (int64_t s = 0; s < N; s++) {
        int64_t i = ord[(size_t)s];
        const Req& r = rq[(size_t)i];
        int64_t g2 = off + s;
        O.ready[g2] = ready[(size_t)i];
        O.arrival[g2] = r.arrival;
        O.prompt[g2] = r.prompt;
        O.true_out[g2] = r.out;
        O.pred_len[g2] = S.bucket_reps[bucket[(size_t)i]];
        O.pred_urg[g2] = fe[(size_t)i];
        O.true_urg[g2] = r.urg;
        O.tie[g2] = (uint32_t)i;  // rank of (arrival, id): the generation order
        if (O.ids) O.ids[g2] = r.id;
        if (O.record_pos) O.record_pos[g2] = i;
    }
}

bool spec_ok(const ss_gen_spec& S) {
    return !(S.total_requests < 0 || S.levels < 1 || S.levels > 255 || S.concurrent < 1 || S.buckets < 1 ||
             S.max_output_len < 1 || S.pred_batch < 1 || S.out_hi > S.max_output_len || S.prompt_lo < 1 ||
             S.out_lo < 1 || !S.bucket_reps);
}

}  // namespace

extern "C" int ss_generate_traces(const ss_gen_spec* spec, int64_t n_traces, const int64_t* seeds,
                                  const int64_t* pred_seeds, const ss_gen_out* out, int n_threads) {
    if (!spec || !out || (n_traces > 0 && (!seeds || !pred_seeds))) return 1;
    const ss_gen_spec S = *spec;
    if (!spec_ok(S)) return 1;
    std::atomic<int64_t> next(0);
    auto work = [&]() {
        for (;;) {
            int64_t t = next.fetch_add(1);
            if (t >= n_traces) break;
            gen_one(S, seeds[t], pred_seeds[t], t * S.total_requests, *out);
        }
    };
    int nt = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    if (nt > n_traces) nt = (int)(n_traces > 0 ? n_traces : 1);
    std::vector<std::thread> th;
    for (int i = 1; i < nt; i++) th.emplace_back(work);
    work();
    for (auto& x : th) x.join();
    return 0;
}

extern "C" int ss_generate_arrivals(const ss_gen_spec* spec, int64_t seed, double* arrival, uint32_t* prompt,
                                    uint32_t* true_out, uint8_t* true_urg) {
    if (!spec || !spec_ok(*spec)) return 1;
    const int64_t N = spec->total_requests;
    if (N > 0 && (!arrival || !prompt || !true_out || !true_urg)) return 1;
    std::vector<Req> rq((size_t)N);
    MT g;
    g.seed(seed);
    gen_arrivals(*spec, g, rq.data());
    for (int64_t i = 0; i < N; i++) {
        arrival[i] = rq[(size_t)i].arrival;
        prompt[i] = rq[(size_t)i].prompt;
        true_out[i] = rq[(size_t)i].out;
        true_urg[i] = rq[(size_t)i].urg;
    }
    return 0;
}

extern "C" int ss_predict(const ss_gen_spec* spec, int64_t n, const double* arrival, const uint32_t* true_out,
                          const uint8_t* true_urg, int32_t what, uint32_t* mt_state, uint8_t* pred_urg,
                          uint32_t* pred_bucket, double* ready) {
    if (!spec || !mt_state || n < 0 || (what & ~7) || spec->levels < 1 || spec->levels > 255 || spec->buckets < 1 ||
        spec->max_output_len < 1 || spec->pred_batch < 1)
        return 1;
    if (n > 0 && (((what & 1) && (!true_urg || !pred_urg)) || ((what & 2) && (!true_out || !pred_bucket)) ||
                  ((what & 4) && (!arrival || !ready))))
        return 1;
    if (mt_state[624] > 624) return 1;
    std::vector<Req> rq((size_t)n);
    for (int64_t i = 0; i < n; i++) {
        rq[(size_t)i].id = i;
        rq[(size_t)i].arrival = arrival ? arrival[i] : 0.0;
        rq[(size_t)i].out = true_out ? true_out[i] : 0u;
        rq[(size_t)i].urg = true_urg ? true_urg[i] : 0u;
    }
    MT p;
    memcpy(p.mt, mt_state, sizeof p.mt);
    p.mti = (int)mt_state[624];
    predict(*spec, p, n, rq.data(), what, pred_urg, pred_bucket, ready);
    memcpy(mt_state, p.mt, sizeof p.mt);
    mt_state[624] = (uint32_t)p.mti;
    return 0;
}
