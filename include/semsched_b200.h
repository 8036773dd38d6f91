/*
 * semsched_b200.h — C-ABI of the B200-native semantic-scheduling hot path.
 *
 * Drop-in boundary for the reference's simulation entry points
 * (reference = arXiv 2506.12204 package `semsched`, paths relative to
 * /root/reference/pkg/src/semsched):
 *
 *   ss_run_traces / ss_run_traces_host
 *       replace `run(cfg, arrivals) -> Trace`           engine.py:444-450
 *       and `Simulator(cfg).run(arrivals)`               engine.py:152-243
 *       batched over many independent traces (the reference runs one
 *       trace per call; `sweeps.sweep` loops them, sweeps.py:25-47).
 *       One call runs every scheduler round of every trace:
 *         per round  `Simulator._schedule`              engine.py:246-254
 *                    -> `stage_aware_schedule`          batching.py:57-88
 *                    `Simulator._execute`               engine.py:288-380
 *                    -> `priority_based_eviction`       kvcache.py:137-179
 *                    -> `should_recompute`              kvcache.py:81-134
 *   ss_trace_stats (output) replaces the waiting-time statistics of
 *       `metrics.average_waiting_time` / `normalized_waiting_time` /
 *       `overall_normalized_waiting_time`               metrics.py:35-56
 *
 * Every entry point takes plain pointers and sizes; no torch types.
 * Inputs are structure-of-arrays, all traces concatenated, each trace's
 * requests in the reference's *pending* order, i.e. sorted by
 * (prediction-ready time, arrival time, id)        predictors.py:148.
 *
 * Error behaviour mirrors the reference: invalid arguments -> SS_ERR_INVALID_ARG
 * (reference: ValueError, engine.py:102-108); unservable requests are
 * RETURNED (never raised), exactly like Trace.unservable (engine.py:82).
 * A trace whose state stops changing (the reference would spin forever in
 * engine.py:202-224) reports SS_TRACE_LIVELOCK instead.
 */
#ifndef SEMSCHED_B200_H
#define SEMSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SS_OK                 0
#define SS_ERR_INVALID_ARG    1  /* reference: ValueError / ConfigError       */
#define SS_ERR_CUDA           2  /* CUDA runtime failure (message via ss_last_error) */
#define SS_ERR_TRACE_FAILED   3  /* >=1 trace ended with a non-OK trace status */
#define SS_ERR_NO_DEVICE      4  /* no CUDA device: there is no CPU fallback   */
#define SS_ERR_UNSUPPORTED    5  /* configuration outside the kernel's limits  */

/* ---- per-trace status (ss_trace_stats.status) --------------------------- */
#define SS_TRACE_OK           0
#define SS_TRACE_LIVELOCK     1  /* round made no progress and state repeats    */
#define SS_TRACE_ROUND_CAP    2  /* params.max_rounds reached                    */
#define SS_TRACE_LOG_OVERFLOW 3  /* round log region too small                   */
#define SS_TRACE_INTERNAL     4  /* invariant violated (allocation > free, ...)  */
#define SS_TRACE_REF_ERROR    6  /* the reference raises an exception on this
                                    trace (IllegalTransitionError,
                                    DuplicateRequestError, ValueError from
                                    estimate_kv_size on a completed request or an
                                    uncaught AdmissionFailure)  */

/* ---- policies (engine.py:40-44, keys engine.py:114-123) ---------------- */
#define SS_POLICY_SEMANTIC 0
#define SS_POLICY_FCFS     1
#define SS_POLICY_SJF      2
#define SS_POLICY_HPJF     3

/* ---- flags ----------------------------------------------------------- */
#define SS_FLAG_ROUND_LOG  1u   /* write per-round ITERATION_END records     */
#define SS_FLAG_DIGEST     2u   /* accumulate the per-trace schedule digest   */
/* Scheduler variant (results are identical; speed differs). By default the run
 * uses chunked stretches of same-batch decode rounds (32 rounds per warp step)
 * when no trace's KV footprint bound can reach the budget, else one round per
 * step. These flags force one variant (tests cover both on every case). */
#define SS_FLAG_FORCE_CHUNKED  4u
#define SS_FLAG_FORCE_PERROUND 8u

/* limits of the device path */
#define SS_MAX_BATCH       32   /* one scheduler candidate per lane of a warp */
#define SS_MAX_LEVELS      16   /* true-urgency levels in ss_trace_stats      */
#define SS_MAX_TRACE_REQS  (1u << 24)  /* tie rank packs into 24 bits        */

/* Analytical cost profile, costs.py:21-41 (GpuProfile). */
typedef struct ss_profile {
    double alpha1, alpha2;   /* prefill(n)  = alpha1*n*n + alpha2*n          */
    double gamma1, gamma2;   /* decode step = gamma1*(n+j-1) + gamma2        */
    double beta_load;        /* reload(k)   = beta_load*k                     */
    double beta_save;        /* carried for API completeness (unused by ref) */
} ss_profile;

/* ScenarioConfig knobs the hot path reads (engine.py:89-111). */
typedef struct ss_params {
    ss_profile profile;
    int64_t memory_capacity;   /* token slots, DeviceMemory.capacity          */
    int32_t batch_size;        /* b, 1..SS_MAX_BATCH                          */
    int32_t policy;            /* SS_POLICY_*                                 */
    int32_t dependency_rule;   /* kvcache.py:111                              */
    int32_t decode_cost_sum;   /* 0: "max", 1: "sum"   (engine.py:148)        */
    int32_t levels;            /* true-urgency levels for the stats (<=16)    */
    uint32_t flags;            /* SS_FLAG_*                                    */
    int64_t max_rounds;        /* per-trace round cap; 0 = automatic:
                                  64 * (requests + sum of true output lengths)
                                  + 100000, far above any progressing schedule */
    int64_t bulk_min;          /* bulk admission: a trace whose first round admits
                                  >= bulk_min requests (config C: 1M at t = 0) gets
                                  them as one sorted run built by the grid-wide
                                  radix sort instead of per-warp queue inserts.
                                  0 = SS_BULK_MIN_DEFAULT, < 0 = never. Results
                                  are identical either way (tests force 1).      */
    int64_t epilogue_min;      /* grid-wide end of trace: a trace of >= epilogue_min
                                  requests (config C: one pool of 1M) leaves its
                                  per-request outputs and waiting-time sums
                                  (metrics.py:35-56) to two grid-wide kernels
                                  (exact double-double tile sums, 1e-15 relative to
                                  CPython's sum); every shorter trace is finished
                                  by one warp of the short-trace epilogue kernel
                                  (sequential CPython sum, bit-exact).
                                  0 = SS_EPILOGUE_MIN_DEFAULT, < 0 = never.      */
} ss_params;

#define SS_BULK_MIN_DEFAULT 1024
#define SS_EPILOGUE_MIN_DEFAULT 16384

/* Requests of all traces, concatenated; trace t owns
 * [trace_offsets[t], trace_offsets[t+1]), in pending order. */
typedef struct ss_trace_batch {
    int32_t  n_traces;
    int32_t  _pad;
    int64_t  n_requests;
    const int64_t*  trace_offsets;    /* [n_traces+1]                            */
    const double*   ready_time;       /* prediction_ready_time                   */
    const double*   arrival_time;     /* Request.arrival_time                    */
    const uint32_t* prompt_len;       /* Request.prompt_len (>=1)                */
    const uint32_t* true_output_len;  /* Request.true_output_len (>=1)           */
    const uint32_t* pred_len;         /* predicted_bucket.representative_len     */
    const uint8_t*  pred_urgency;     /* f_e.rank (dispatch key)                 */
    const uint8_t*  true_urgency;     /* true_urgency.rank (stats only)          */
    const uint32_t* tie_rank;         /* rank of (arrival_time, id) in the trace */
} ss_trace_batch;

/* Per-trace result record (fixed size, gathered across ranks). */
typedef struct ss_trace_stats {
    uint64_t digest;           /* schedule digest (SS_FLAG_DIGEST)                 */
    int64_t  rounds;           /* _schedule+_execute rounds = scheduler decisions  */
    int64_t  evictions;        /* Trace.eviction_count                             */
    int64_t  mem_used_peak;    /* max ITERATION_END mem_used                       */
    int64_t  log_words;        /* words written to the round log                   */
    int32_t  completed;
    int32_t  unservable;       /* len(Trace.unservable)                            */
    int32_t  status;           /* SS_TRACE_*                                       */
    int32_t  lost_evictions;   /* evictions made by an admission that then failed:
                                  applied but, as in the reference, not recorded   */
    int32_t  anomalies;        /* grants of a request that still had a heap entry
                                  (the reference then carries a stale key and
                                  duplicate batch members; emulated) */
    int32_t  _pad;
    /* per-round tallies for the algorithmic byte model         */
    int64_t  sum_pool;         /* sum over rounds of live requests (heap+buffer+ongoing) */
    int64_t  sum_granted;      /* sum of granted batch members                     */
    int64_t  sum_victims;      /* victims processed (recorded + lost decisions)    */
    int64_t  sum_resident_evict; /* residents, summed over rounds that evict       */
    double   final_clock;      /* RUN_END time                                     */
    /* CPython-3.12 float sum() (Neumaier) over completed records in trace order  */
    double   sum_wait;         /* sum(finish - arrival)                            */
    double   sum_norm_wait;    /* sum((finish - arrival)/generated)                */
    double   level_norm_sum[SS_MAX_LEVELS];
    int32_t  level_count[SS_MAX_LEVELS];
} ss_trace_stats;

/* Per-request outputs, same indexing as the inputs. NaN encodes None. */
typedef struct ss_request_out {
    double*   first_scheduled;  /* RequestRecord.first_scheduled  */
    double*   finish_time;      /* RequestRecord.finish_time      */
    uint32_t* generated;        /* RequestRecord.generated_tokens */
    uint32_t* evictions;        /* RequestRecord.evictions        */
    double*   f_t;              /* final Request.f_t  (optional, may be NULL)      */
    uint32_t* state;            /* final stage | prefilled<<8 | unservable-while-decoding<<9 (optional, NULL ok) */
} ss_request_out;

/* Whole-call outputs. */
typedef struct ss_outputs {
    ss_request_out req;
    ss_trace_stats* stats;          /* [n_traces]                                  */
    uint32_t* unservable_slots;     /* [n_requests]: trace t's list starts at
                                       trace_offsets[t]; slots are trace-local     */
    uint32_t* round_log;            /* SS_FLAG_ROUND_LOG: words                    */
    const int64_t* log_offsets;     /* [n_traces+1] word ranges into round_log     */
} ss_outputs;

/* Stage encoding of ss_request_out.state (requests.py:17-23). */
#define SS_STAGE_WAITING    0
#define SS_STAGE_DECODING   2
#define SS_STAGE_COMPLETED  5
#define SS_STAGE_UNSERVABLE 6   /* removed by _mark_unservable (engine.py:402-412) */

/* ---- round log record (one per ITERATION_END event, engine.py:329-380) ----
 * word 0 kind (0 decode, 1 prefill, 2 nothing granted), 1 m granted,
 * 2 c completed, 3 v decisions, 4-5 mem_used (u64), 6-7 time (f64 bits),
 * then v decisions of SS_LOG_DECISION_WORDS words each (in eviction order):
 *   victim slot, action (0 offload, 1 discard), decode_saved, decode_discarded,
 *   freed_slots, f_t_before (2 words), f_t_after (2 words),
 * then m granted slots (batch order), then c completed slots (granted order).
 * Slots are trace-local pending-order row indices.
 */
#define SS_LOG_HEADER_WORDS    8
#define SS_LOG_DECISION_WORDS  9
#define SS_KIND_DECODE   0
#define SS_KIND_PREFILL  1
#define SS_KIND_NONE     2

/* ---- schedule digest -------------------------------------------------
 * Order-sensitive and lane-parallel: a sum (mod 2^64) of one hashed term per
 * (round, field, position). Shared verbatim by the oracle (tests) and the
 * device so full-size parity reduces to comparing one u64 per trace.
 * The granted list of round r contributes
 *     ss_round_mul(r) * sum_pos ss_grant_term(pos, slot_pos)      (mod 2^64)
 * (an odd round multiplier times a position-tagged hash of the list), so a
 * batch that stays the same over a stretch of rounds hashes once; the header,
 * memory and time fields are ss_round_fields(round, ...) below; a completion is
 * one ss_term(round, SS_TAG_DONE, index, slot), an eviction decision one
 * ss_decision_term(round, index, fields...). */
#if defined(__CUDACC__)
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD static inline
#endif
SS_HD uint64_t ss_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
SS_HD uint64_t ss_term(uint64_t round, uint32_t tag, uint32_t idx, uint64_t v) {
    return ss_mix64(v ^ (((round << 24) ^ ((uint64_t)tag << 20) ^ (uint64_t)idx) * 0x9E3779B97F4A7C15ull));
}
#define SS_DG_POS   0xD6E8FEB86659FD93ull
#define SS_DG_ROUND 0xA0761D6478BD642Full
SS_HD uint64_t ss_grant_term(uint32_t pos, uint64_t slot) {
    return ss_mix64(slot ^ ((uint64_t)(pos + 1u) * SS_DG_POS));
}
SS_HD uint64_t ss_round_mul(uint64_t round) { return (2u * round + 1u) * SS_DG_ROUND; }
/* The three fields every round has (header word, KV slots in use, round end
 * time bits) enter as one weighted sum, linear in each field:
 *     ss_round_fields(r, hdr, mem, t) =
 *         (2r+1) * (K_H (hdr ^ S_H) + K_M (mem ^ S_M) + K_T (t ^ S_T))   (mod 2^64)
 * With odd weights a change of any one field changes the digest, and a round's
 * fields cost three multiply-adds instead of three 64-bit mixes (in the kernel's
 * stretches of same-batch rounds this was a third of the scheduler's time). */
#define SS_DG_HDR  0xD1B54A32D192ED03ull
#define SS_DG_MEM  0xAEF17502108EF2D9ull
#define SS_DG_TIME 0xF1357AEA2E62A9C5ull
#define SS_DS_HDR  0x5851F42D4C957F2Dull
#define SS_DS_MEM  0x14057B7EF767814Full
#define SS_DS_TIME 0x2545F4914F6CDD1Dull
SS_HD uint64_t ss_round_fields(uint64_t round, uint64_t hdr, uint64_t mem, uint64_t tbits) {
    return (2u * round + 1u) *
           (SS_DG_HDR * (hdr ^ SS_DS_HDR) + SS_DG_MEM * (mem ^ SS_DS_MEM) + SS_DG_TIME * (tbits ^ SS_DS_TIME));
}
#define SS_TAG_HDR   1u   /* unused since ss_round_fields */
#define SS_TAG_MEM   2u   /* unused since ss_round_fields */
#define SS_TAG_TIME  3u   /* unused since ss_round_fields */
#define SS_TAG_GRANT 4u   /* unused since the grant terms above */
#define SS_TAG_DONE  5u
#define SS_TAG_EV0   6u   /* unused since ss_decision_term */
#define SS_TAG_EV1   7u
#define SS_TAG_EV2   8u
#define SS_TAG_EV3   9u
#define SS_TAG_EV4  10u
/* Eviction decision d of round r: one mixed (round, index) weight times a linear
 * sum of its five fields w0 = victim | action<<32, w1 = saved | discarded<<32,
 * w2 = freed, w3 / w4 = f_t before / after bits (odd field weights). */
#define SS_DG_DEC 0x8CB92BA72F3D8DD7ull
SS_HD uint64_t ss_decision_term(uint64_t round, uint32_t d, uint64_t w0, uint64_t w1, uint64_t w2, uint64_t w3,
                                uint64_t w4) {
    const uint64_t W = ss_mix64(((round << 24) ^ (uint64_t)d) * SS_DG_DEC) | 1u;
    return W * (0xC2B2AE3D27D4EB4Full * (w0 ^ 0x165667B19E3779F9ull) + 0x27D4EB2F165667C5ull * (w1 ^ 0x85EBCA77C2B2AE63ull) +
                0x9E3779B185EBCA87ull * (w2 ^ 0xFF51AFD7ED558CCDull) + 0xC4CEB9FE1A85EC53ull * (w3 ^ 0x62A9D9ED799705F5ull) +
                0x4CF5AD432745937Full * (w4 ^ 0x1B873593CC9E2D51ull));
}
SS_HD uint64_t ss_hdr_word(uint32_t kind, uint32_t m, uint32_t c, uint32_t v) {
    return (uint64_t)kind | ((uint64_t)m << 8) | ((uint64_t)c << 24) | ((uint64_t)v << 40);
}

/* ---- entry points ----------------------------------------------------- */

/* Last error message of the calling thread ("" if none). */
const char* ss_last_error(void);

/* Library / device info. Returns SS_OK, or SS_ERR_NO_DEVICE. */
int ss_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor);

/* Device workspace the run needs (bytes), for callers that pre-allocate. */
int ss_workspace_bytes(const ss_params* params, int32_t n_traces, int64_t n_requests,
                       size_t* bytes);

/* Run every trace to completion. All pointers in `batch` and `out` are DEVICE
 * pointers; `workspace` is a device buffer of >= ss_workspace_bytes bytes
 * (NULL: the library allocates and frees one). `stream` is a cudaStream_t
 * (NULL = legacy default stream). Asynchronous w.r.t. the host unless the
 * library allocated the workspace. `kernel_ms` (nullable) receives the
 * scheduler kernel's device time measured with events on `stream`
 * (forces a sync). Returns SS_OK, SS_ERR_TRACE_FAILED (see stats[].status),
 * or an error. */
int ss_run_traces(const ss_params* params, const ss_trace_batch* batch,
                  const ss_outputs* out, void* workspace, size_t workspace_bytes,
                  void* stream, float* kernel_ms);

/* Same, with every pointer in `batch` and `out` on the HOST (pinned or
 * pageable). Copies in, runs, copies out, synchronises. This is the
 * reference-facing plugin call (host buffers in, host buffers out).
 * Batches of >= 1,024 traces run as up to 8 equal slices of consecutive traces on
 * library-owned streams (which first wait for `stream`): uploads, kernels and
 * downloads of different slices overlap. Pinned buffers give full overlap.
 * `kernel_ms` then reports the span from the first slice's prepass to the
 * last kernel's end. Serialised by a library mutex. */
int ss_run_traces_host(const ss_params* params, const ss_trace_batch* batch,
                       const ss_outputs* out, void* stream, float* kernel_ms);

/* Device times of the calling thread's last ss_run_traces made with a
 * non-NULL kernel_ms: the grid-wide prepass (request init + bulk-admission
 * radix sort) and the scheduler kernel. */
int ss_last_timings(float* prepass_ms, float* kernel_ms);

/* Number of warps the scheduler kernel keeps resident (for reporting). */
int ss_kernel_config(const ss_params* params, int32_t n_traces, int* blocks,
                     int* warps_per_block, int* smem_bytes_per_block);

/* ---- per-step entry points (ss_step.cu) -----------------------------------
 * The reference's public per-step functions, for callers that drive their own
 * loop over heaps of Request objects (the Python shim's batching / kvcache
 * modules). HOST buffers in and out; the call stages them through a device
 * workspace, runs, and synchronises. */

/* A key tuple of the reference (requests.py:81-97): (urgency rank, remaining
 * seconds, arrival, id), a baseline policy's shorter tuple (engine.py:114-123)
 * padded with -inf, or an eviction key (every component negated). Compared
 * lexicographically with IEEE `<`; equal tuples keep pool order. */
typedef struct ss_key4 { double k[4]; } ss_key4;

#define SS_SELECT_TOP_B        0  /* extract_top_b only            batching.py:46-54  */
#define SS_SELECT_STAGE_AWARE  1  /* stage_aware_schedule          batching.py:57-88  */
#define SS_SELECT_PREEMPTIVE   2  /* SJF / HPJF top-b of the merge engine.py:270-285  */
#define SS_SELECT_FCFS         3  /* ongoing + b - |ongoing| pops  engine.py:256-267  */

/* Replaces extract_top_b / stage_aware_schedule (batching.py:46-88) and the
 * baselines' selection (engine.py:256-285).
 *   stored[n_pool]   the dispatch heap's keys as stored at insertion: pop order
 *   current[n_pool]  key_fn(r) now (p* and merge order); NULL = same as stored
 *   pool_decoding    1 where r.stage is DECODING (batching.py:39-43)
 *   ongoing[n_ongoing], ongoing_decoding: the ongoing requests, current keys
 * Out: cand[<= b]  pool indices of the popped candidates, in pop order;
 *      merged[<= b + n_ongoing] the merge in batch order, entries j < n_cand
 *        name candidate j, entries >= n_cand name ongoing (j - n_cand);
 *      n_selected = members taken (min(b, n_merged)); kind SS_KIND_PREFILL /
 *        SS_KIND_DECODE. Candidates absent from merged were pushed back as
 *        prefill work; merged[n_selected:] are pushed back (batching.py:80-87).
 * b and n_ongoing <= SS_MAX_BATCH. */
int ss_select_batch(const ss_key4* stored, const ss_key4* current, const uint8_t* pool_decoding,
                    int64_t n_pool, const ss_key4* ongoing, const uint8_t* ongoing_decoding,
                    int32_t n_ongoing, int32_t b, int32_t mode, int32_t* cand, int32_t* n_cand,
                    int32_t* merged, int32_t* n_merged, int32_t* n_selected, int32_t* kind,
                    void* stream);

/* One eviction decision (kvcache.py:59-67) plus the victim's new counters. */
typedef struct ss_victim {
    int32_t index;            /* resident index in the call's arrays            */
    int32_t action;           /* 0 offload, 1 discard (prefill_action)          */
    int64_t decode_saved, decode_discarded, freed_slots;
    int64_t prefilled;        /* prefilled_tokens after the decision             */
    int64_t kv_host;          /* kv_host_tokens after the decision               */
    double  f_t_before, f_t_after;
    int64_t _pad;
} ss_victim;

/* Replaces priority_based_eviction (kvcache.py:137-179) with should_recompute
 * (kvcache.py:81-134) applied to every victim.
 *   ev_keys[n]: the eviction heap's stored keys (smallest pops first);
 *   per resident: prompt_len, prefilled_tokens, decoded_tokens,
 *   kv_device_tokens, predicted representative length, f_t; protected[n].
 *   select = 1: the eviction loop — pop in key order, skip protected, evict
 *     until demand + used <= capacity; *failed = 1 when every unprotected
 *     resident went and it still does not fit (AdmissionFailure; the victims
 *     stand). skipped[] = protected entries popped (re-inserted by the caller).
 *   select = 0: should_recompute on every entry, in the given order.
 * victims[] are in eviction order. */
int ss_evict(const ss_key4* ev_keys, const uint32_t* prompt, const uint32_t* prefilled,
             const uint32_t* decoded, const uint32_t* kv_device, const uint32_t* pred_len,
             const double* f_t, const uint8_t* protected_, int64_t n, int64_t demand, int64_t used,
             int64_t capacity, const ss_profile* profile, int32_t dependency_rule, int32_t select,
             ss_victim* victims, int64_t* n_victims, int32_t* skipped, int64_t* n_skipped,
             int32_t* failed, void* stream);

/* Completion-order constraint audit, Eq. 2 (metrics.constraint_audit,
 * metrics.py:59-91), for many traces at once. Trace t owns records
 * [offsets[t], offsets[t+1]) in any order; finish = NaN marks a request that
 * did not complete (excluded, as in the reference). rank = true or predicted
 * urgency rank. Out: violations[t], comparable[t] (violation_rate =
 * violations / comparable, 0 if none comparable). pairs (nullable): when
 * given, receives 2 x sum(violations) int64 (id_a, id_b) in the reference's
 * order (traces in order; within a trace by the stable finish-time order of
 * a, then of b); pairs_cap is its length in int64s. HOST pointers. */
int ss_audit_host(int32_t n_traces, const int64_t* offsets, const double* finish, const double* arrival,
                  const int32_t* rank, const int64_t* ids, int64_t* violations, int64_t* comparable,
                  int64_t* pairs, int64_t pairs_cap, void* stream);
const char* ss_audit_last_error(void);
/* Device time (ms) of the calling thread's last ss_audit_host pair sweep. */
double ss_audit_last_kernel_ms(void);

/* Message of the calling thread's last failed per-step call. */
const char* ss_step_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SEMSCHED_B200_H */
