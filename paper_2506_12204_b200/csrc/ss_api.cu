// ss_api.cu — the C-ABI (include/semsched_b200.h): validation, workspace,
// launch, optional host staging. No torch types cross this boundary.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>

#include "ss_kernel.cuh"

namespace {

thread_local std::string g_err;
thread_local float g_prepass_ms = 0.f, g_kernel_ms = 0.f;

int fail(int code, const char* msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    char buf[256];
    snprintf(buf, sizeof buf, "%s: %s", where, cudaGetErrorString(e));
    g_err = buf;
    return SS_ERR_CUDA;
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t e_ = (call);                            \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

int validate(const ss_params* p, const ss_trace_batch* b, const ss_outputs* o) {
    if (!p || !b || !o) return fail(SS_ERR_INVALID_ARG, "null argument");
    if (p->batch_size < 1) return fail(SS_ERR_INVALID_ARG, "batch size must be >= 1");
    if (p->memory_capacity < 1) return fail(SS_ERR_INVALID_ARG, "memory capacity must be >= 1");
    if (p->decode_cost_sum != 0 && p->decode_cost_sum != 1)
        return fail(SS_ERR_INVALID_ARG, "decode_batch_cost must be 'max' or 'sum'");
    if (p->batch_size > SS_MAX_BATCH) return fail(SS_ERR_UNSUPPORTED, "batch size above SS_MAX_BATCH (32)");
    if (p->policy < SS_POLICY_SEMANTIC || p->policy > SS_POLICY_HPJF) return fail(SS_ERR_INVALID_ARG, "unknown policy");
    if (b->n_traces < 0 || b->n_requests < 0) return fail(SS_ERR_INVALID_ARG, "negative sizes");
    if (b->n_traces > 0 && (!b->trace_offsets)) return fail(SS_ERR_INVALID_ARG, "trace_offsets is null");
    if (b->n_requests > 0 &&
        (!b->ready_time || !b->arrival_time || !b->prompt_len || !b->true_output_len || !b->pred_len ||
         !b->pred_urgency || !b->true_urgency || !b->tie_rank))
        return fail(SS_ERR_INVALID_ARG, "null input array");
    if (b->n_traces > 0 && (!o->stats)) return fail(SS_ERR_INVALID_ARG, "stats output is null");
    if (b->n_requests > 0 && (!o->req.first_scheduled || !o->req.finish_time || !o->req.generated ||
                              !o->req.evictions || !o->unservable_slots))
        return fail(SS_ERR_INVALID_ARG, "null output array");
    if ((p->flags & SS_FLAG_ROUND_LOG) && (!o->round_log || !o->log_offsets))
        return fail(SS_ERR_INVALID_ARG, "round log requested without buffers");
    return SS_OK;
}

struct HostStage {
    std::mutex mu;
    void* buf = nullptr;
    size_t cap = 0;
};
HostStage g_stage;

size_t a16(size_t x) { return (x + 15) & ~(size_t)15; }

}  // namespace

extern "C" {

const char* ss_last_error(void) { return g_err.c_str(); }

int ss_last_timings(float* prepass_ms, float* kernel_ms) {
    if (prepass_ms) *prepass_ms = g_prepass_ms;
    if (kernel_ms) *kernel_ms = g_kernel_ms;
    return SS_OK;
}

int ss_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    int d = 0;
    CK(cudaGetDevice(&d));
    if (device) *device = d;
    if (sm_count) CK(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, d));
    if (cc_major) CK(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, d));
    if (cc_minor) CK(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, d));
    return SS_OK;
}

int ss_workspace_bytes(const ss_params* params, int32_t n_traces, int64_t n_requests, size_t* bytes) {
    (void)params;
    if (!bytes) return fail(SS_ERR_INVALID_ARG, "null bytes");
    if (n_traces < 0 || n_requests < 0) return fail(SS_ERR_INVALID_ARG, "negative sizes");
    *bytes = ss::work_bytes(n_requests, n_traces);
    return SS_OK;
}

int ss_kernel_config(const ss_params* params, int32_t n_traces, int* blocks, int* warps_per_block,
                     int* smem_bytes_per_block) {
    int sms = 0;
    int maxb = ss::sched_max_blocks(params ? params->policy : 0, &sms);
    if (maxb <= 0) return fail(SS_ERR_UNSUPPORTED, "kernel not available");
    int need = (n_traces + ss::WPB - 1) / ss::WPB;
    if (blocks) *blocks = need < maxb ? (need > 0 ? need : 1) : maxb;
    if (warps_per_block) *warps_per_block = ss::WPB;
    if (smem_bytes_per_block) *smem_bytes_per_block = ss::sched_smem_bytes();
    return SS_OK;
}

int ss_run_traces(const ss_params* params, const ss_trace_batch* batch, const ss_outputs* out,
                  void* workspace, size_t workspace_bytes, void* stream, float* kernel_ms) {
    int rc = validate(params, batch, out);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    if (batch->n_traces == 0) {
        if (kernel_ms) *kernel_ms = 0.f;
        return SS_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    size_t need = ss::work_bytes(batch->n_requests, batch->n_traces);
    void* ws = workspace;
    bool own = false;
    if (!ws) {
        CK(cudaMallocAsync(&ws, need, st));
        own = true;
    } else if (workspace_bytes < need) {
        return fail(SS_ERR_INVALID_ARG, "workspace too small");
    }
    ss::KArgs a;
    a.P = *params;
    a.in = *batch;
    a.out = *out;
    ss::carve_work(ws, batch->n_requests, batch->n_traces, &a.w);
    CK(cudaMemsetAsync(ws, 0, ss::work_zero_bytes(batch->n_traces), st));
    int blocks = 0;
    rc = ss_kernel_config(params, batch->n_traces, &blocks, nullptr, nullptr);
    if (rc) return rc;
    cudaEvent_t e0 = nullptr, em = nullptr, e1 = nullptr;
    if (kernel_ms) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&em));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, st));
    }
    rc = ss::launch_prepass(a, stream);
    if (rc) {
        cudaError_t e = cudaGetLastError();
        return e != cudaSuccess ? cuda_fail(e, "prepass launch") : fail(rc, "prepass launch failed");
    }
    if (kernel_ms) CK(cudaEventRecord(em, st));
    rc = ss::launch_sched(a, blocks, stream);
    if (rc) {
        cudaError_t e = cudaGetLastError();
        return e != cudaSuccess ? cuda_fail(e, "sched_kernel launch") : fail(rc, "launch failed");
    }
    if (kernel_ms) {
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&g_prepass_ms, e0, em));
        CK(cudaEventElapsedTime(&g_kernel_ms, em, e1));
        *kernel_ms = g_kernel_ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(em);
        cudaEventDestroy(e1);
    }
    if (own) {
        CK(cudaFreeAsync(ws, st));
        CK(cudaStreamSynchronize(st));
    }
    return SS_OK;
}

int ss_run_traces_host(const ss_params* params, const ss_trace_batch* hb, const ss_outputs* ho,
                       void* stream, float* kernel_ms) {
    int rc = validate(params, hb, ho);
    if (rc) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SS_ERR_NO_DEVICE, "no CUDA device");
    const int64_t n = hb->n_requests;
    const int32_t T = hb->n_traces;
    if (T == 0) {
        if (kernel_ms) *kernel_ms = 0.f;
        return SS_OK;
    }
    const size_t nn = (size_t)(n > 0 ? n : 1);
    const bool logr = (params->flags & SS_FLAG_ROUND_LOG) != 0;
    int64_t log_words = 0;
    if (logr) log_words = ho->log_offsets[T];
    // one device allocation: inputs | outputs | log | workspace
    size_t in_b = a16((T + 1) * 8) + 2 * a16(nn * 8) + 3 * a16(nn * 4) + 2 * a16(nn) + a16(nn * 4);
    size_t out_b = 2 * a16(nn * 8) + 2 * a16(nn * 4) + a16(nn * 8) + a16(nn * 4) +
                   a16((size_t)T * sizeof(ss_trace_stats)) + a16(nn * 4);
    size_t log_b = logr ? a16((size_t)log_words * 4) + a16((T + 1) * 8) : 0;
    size_t ws_b = ss::work_bytes(n, T);
    // no trace long enough for a bulk first round: skip the bulk-sort stage
    ss_params pp = *params;
    if (pp.bulk_min == 0) {
        int64_t maxlen = 0;
        for (int32_t t = 0; t < T; t++) {
            const int64_t k = hb->trace_offsets[t + 1] - hb->trace_offsets[t];
            if (k > maxlen) maxlen = k;
        }
        if (maxlen < SS_BULK_MIN_DEFAULT) pp.bulk_min = -1;
    }
    params = &pp;
    size_t total = in_b + out_b + log_b + ws_b;
    std::lock_guard<std::mutex> lk(g_stage.mu);
    cudaStream_t st = (cudaStream_t)stream;
    if (g_stage.cap < total) {
        if (g_stage.buf) CK(cudaFree(g_stage.buf));
        g_stage.buf = nullptr;
        g_stage.cap = 0;
        CK(cudaMalloc(&g_stage.buf, total));
        g_stage.cap = total;
    }
    char* p = (char*)g_stage.buf;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += a16(bytes);
        return (void*)r;
    };
    ss_trace_batch db = *hb;
    ss_outputs dout;
    memset(&dout, 0, sizeof dout);
    int64_t* d_off = (int64_t*)take((T + 1) * 8);
    CK(cudaMemcpyAsync(d_off, hb->trace_offsets, (T + 1) * 8, cudaMemcpyHostToDevice, st));
    db.trace_offsets = d_off;
#define H2D(field, bytes)                                                               \
    do {                                                                                \
        void* d_ = take(bytes);                                                         \
        if (n > 0) CK(cudaMemcpyAsync(d_, hb->field, bytes, cudaMemcpyHostToDevice, st)); \
        db.field = (decltype(db.field))d_;                                              \
    } while (0)
    H2D(ready_time, nn * 8);
    H2D(arrival_time, nn * 8);
    H2D(prompt_len, nn * 4);
    H2D(true_output_len, nn * 4);
    H2D(pred_len, nn * 4);
    H2D(pred_urgency, nn);
    H2D(true_urgency, nn);
    H2D(tie_rank, nn * 4);
#undef H2D
    dout.req.first_scheduled = (double*)take(nn * 8);
    dout.req.finish_time = (double*)take(nn * 8);
    dout.req.generated = (uint32_t*)take(nn * 4);
    dout.req.evictions = (uint32_t*)take(nn * 4);
    void* d_ft = take(nn * 8);
    void* d_state = take(nn * 4);
    dout.req.f_t = ho->req.f_t ? (double*)d_ft : nullptr;
    dout.req.state = ho->req.state ? (uint32_t*)d_state : nullptr;
    dout.stats = (ss_trace_stats*)take((size_t)T * sizeof(ss_trace_stats));
    dout.unservable_slots = (uint32_t*)take(nn * 4);
    if (logr) {
        dout.round_log = (uint32_t*)take((size_t)log_words * 4);
        int64_t* d_loff = (int64_t*)take((T + 1) * 8);
        CK(cudaMemcpyAsync(d_loff, ho->log_offsets, (T + 1) * 8, cudaMemcpyHostToDevice, st));
        dout.log_offsets = d_loff;
    }
    void* ws = take(ws_b);
    rc = ss_run_traces(params, &db, &dout, ws, ws_b, stream, kernel_ms);
    if (rc) return rc;
#define D2H(dst, src, bytes) \
    if ((dst) && (bytes) > 0) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st))
    size_t nb = (size_t)n;
    D2H(ho->req.first_scheduled, dout.req.first_scheduled, nb * 8);
    D2H(ho->req.finish_time, dout.req.finish_time, nb * 8);
    D2H(ho->req.generated, dout.req.generated, nb * 4);
    D2H(ho->req.evictions, dout.req.evictions, nb * 4);
    D2H(ho->req.f_t, dout.req.f_t, nb * 8);
    D2H(ho->req.state, dout.req.state, nb * 4);
    D2H(ho->stats, dout.stats, (size_t)T * sizeof(ss_trace_stats));
    D2H(ho->unservable_slots, dout.unservable_slots, nb * 4);
    if (logr) D2H(ho->round_log, dout.round_log, (size_t)log_words * 4);
#undef D2H
    CK(cudaStreamSynchronize(st));
    for (int32_t t = 0; t < T; t++)
        if (ho->stats[t].status != SS_TRACE_OK) return fail(SS_ERR_TRACE_FAILED, "a trace ended with a non-OK status");
    return SS_OK;
}

}  // extern "C"
