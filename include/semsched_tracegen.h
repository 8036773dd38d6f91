/*
 * semsched_tracegen.h — native bulk trace preparation (host side).
 *
 * Replaces, for many seeds per call, the reference's input producers
 *   workload.generate(WorkloadSpec)           workload.py:63-93
 *   predictors.predictor_pipeline(...)        predictors.py:85-149
 * reproducing CPython's random.Random draw for draw, and lays the result out
 * as the ss_trace_batch SoA of semsched_b200.h (pending order).
 */
#ifndef SEMSCHED_TRACEGEN_H
#define SEMSCHED_TRACEGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ss_gen_spec {
    /* WorkloadSpec (workload.py:19-45) */
    int64_t total_requests;
    double gap_s;
    int32_t concurrent;
    int32_t concurrent_fixed;      /* concurrent_mode == "fixed"                  */
    int32_t levels;
    int32_t buckets;
    const double* urgency_weights; /* [levels] or NULL (all 1.0)                  */
    int64_t prompt_lo, prompt_hi;
    int64_t out_lo, out_hi;
    int64_t max_output_len;
    const uint32_t* bucket_reps;   /* [buckets] representative length per bucket  */
    /* PredictorConfig (predictors.py:41-53) */
    double latency_s;
    int32_t pred_batch;
    int32_t full_batching;         /* Strategy.FULL_BATCHING                      */
    double urgency_error, length_error;
    int64_t urgency_disp, length_disp;  /* ErrorModel.displacement               */
} ss_gen_spec;

typedef struct ss_gen_out {         /* [n_traces * total_requests], pending order */
    double* ready;
    double* arrival;
    uint32_t* prompt;
    uint32_t* true_out;
    uint32_t* pred_len;
    uint8_t* pred_urg;
    uint8_t* true_urg;
    uint32_t* tie;
    int64_t* ids;                   /* nullable */
    int64_t* record_pos;            /* nullable */
} ss_gen_out;

/* Trace t uses Random(seeds[t]) for the workload and Random(pred_seeds[t])
 * for the predictors (ScenarioConfig.seed). Returns 0 on success. */
int ss_generate_traces(const ss_gen_spec* spec, int64_t n_traces, const int64_t* seeds,
                       const int64_t* pred_seeds, const ss_gen_out* out, int n_threads);

/* The same generator on the device: one thread per trace, `out` holds DEVICE
 * pointers (the scheduler's inputs stay in HBM). seeds / pred_seeds and the
 * spec's arrays are host memory. Synchronises `stream` (a cudaStream_t, NULL
 * = default). Returns 0 on success, 1 on an invalid spec, 2 on a CUDA error,
 * 3 if a trace's ready times are not non-decreasing in generation order (the
 * generator relies on the FIFO prediction server for the pending order). */
int ss_generate_traces_device(const ss_gen_spec* spec, int64_t n_traces, const int64_t* seeds,
                              const int64_t* pred_seeds, const ss_gen_out* out, void* stream);

/* One trace's arrivals as workload.generate(spec) with Random(seed)
 * (workload.py:63-93): N = spec->total_requests requests in generation order
 * (id = index). Only the workload fields of `spec` are read (bucket_reps must
 * be non-NULL). Returns 0 on success, 1 on an invalid spec. */
int ss_generate_arrivals(const ss_gen_spec* spec, int64_t seed, double* arrival, uint32_t* prompt,
                         uint32_t* true_out, uint8_t* true_urg);

/* predictors.predictor_pipeline (predictors.py:85-149) over n time-ordered
 * requests, continuing the caller's CPython Random: `mt_state` holds the 624
 * MT19937 words and the position (Random.getstate()[1]) and is advanced in
 * place. `what`: bit 0 urgency predictions (pred_urg, spec levels /
 * urgency_error / urgency_disp), bit 1 length buckets (pred_bucket: bucket
 * index; max_output_len / buckets / length_error / length_disp), bit 2 the
 * FIFO prediction server's ready times (latency_s, pred_batch,
 * full_batching). Returns 0 on success, 1 on invalid arguments. */
int ss_predict(const ss_gen_spec* spec, int64_t n, const double* arrival, const uint32_t* true_out,
               const uint8_t* true_urg, int32_t what, uint32_t* mt_state, uint8_t* pred_urg,
               uint32_t* pred_bucket, double* ready);

#ifdef __cplusplus
}
#endif
#endif
