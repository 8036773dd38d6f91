// ss_api.cu — the C-ABI (include/semsched_b200.h): validation, workspace,
// launch, optional host staging. No torch types cross this boundary.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>

#include "ss_costs.cuh"
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

#ifndef SS_SLICE_TRACES
#define SS_SLICE_TRACES 512  // ss_run_traces_host pipelines batches of >= 2 slices of this size
#endif
#ifndef SS_MAX_SLICES
#define SS_MAX_SLICES 8
#endif
struct HostStage {
    std::mutex mu;
    void* buf = nullptr;   // device: inputs | outputs | log | offsets | workspaces
    size_t cap = 0;
    void* hbuf = nullptr;  // pinned host: the slices' rebased offsets
    size_t hcap = 0;
    cudaStream_t streams[SS_MAX_SLICES] = {};
    int dev = -1;  // device the buffer and streams live on
};
constexpr int32_t SLICE_TRACES = SS_SLICE_TRACES;
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
    if (const char* e = getenv("SS_BLOCKS_PER_SM")) {  // dev: occupancy experiments
        int per = atoi(e);
        if (per > 0 && per * sms < maxb) maxb = per * sms;
    }
    if (const char* e = getenv("SS_MAX_BLOCKS")) {  // dev: wave-balance experiments
        int mb = atoi(e);
        if (mb > 0 && mb < maxb) maxb = mb;
    }
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
    a.z0 = ss::add(ss::reload_time(0, params->profile), ss::prefill_time(0, params->profile));
    {
        const double g1 = params->profile.gamma1, g2 = params->profile.gamma2;
        a.screen = (g1 >= 0.0 && g2 >= 0.0 && g1 < 1e300 && g2 < 1e300 && a.z0 == 0.0) ? 1 : 0;
    }
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
    rc = ss::launch_epilogue(a, stream);
    if (rc) return cuda_fail(cudaGetLastError(), "epilogue launch");
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
    const bool logr = (params->flags & SS_FLAG_ROUND_LOG) != 0;
    // host offsets: the copies below read [offsets[t], offsets[t+1]) of every array
    if (hb->trace_offsets[0] != 0 || hb->trace_offsets[T] != n)
        return fail(SS_ERR_INVALID_ARG, "trace_offsets must start at 0 and end at n_requests");
    for (int32_t t = 0; t < T; t++)
        if (hb->trace_offsets[t + 1] < hb->trace_offsets[t])
            return fail(SS_ERR_INVALID_ARG, "trace_offsets must be nondecreasing");
    if (logr) {
        if (ho->log_offsets[0] != 0) return fail(SS_ERR_INVALID_ARG, "log_offsets must start at 0");
        for (int32_t t = 0; t < T; t++)
            if (ho->log_offsets[t + 1] < ho->log_offsets[t])
                return fail(SS_ERR_INVALID_ARG, "log_offsets must be nondecreasing");
    }
    // Slices of consecutive traces, each on its own stream: slice s+1's inputs
    // upload while slice s computes, slice s's outputs download while later
    // slices compute, and a later slice's CTAs fill the SM slots an earlier
    // slice's finished warps free. Every slice is an independent ss_run_traces.
    int S = (int)(T / SLICE_TRACES);
    S = S < 1 ? 1 : (S > SS_MAX_SLICES ? SS_MAX_SLICES : S);
    if (const char* e = getenv("SS_HOST_SLICES")) {  // dev: slice-count experiments
        const int v = atoi(e);
        if (v >= 1 && v <= SS_MAX_SLICES) S = v;
    }
    int32_t t0s[SS_MAX_SLICES + 1];
    for (int s = 0; s <= S; s++) t0s[s] = (int32_t)((int64_t)T * s / S);
    size_t in_b = 2 * a16((size_t)(n > 0 ? n : 1) * 8) + 4 * a16((size_t)(n > 0 ? n : 1) * 4) +
                  2 * a16((size_t)(n > 0 ? n : 1));
    const size_t nn = (size_t)(n > 0 ? n : 1);
    size_t out_b = 3 * a16(nn * 8) + 3 * a16(nn * 4) + a16((size_t)T * sizeof(ss_trace_stats)) + a16(nn * 4);
    const int64_t log_words = logr ? ho->log_offsets[T] : 0;
    size_t log_b = logr ? a16((size_t)log_words * 4) : 0;
    size_t off_b = 0, ws_b = 0;
    for (int s = 0; s < S; s++) {
        const int32_t Ts = t0s[s + 1] - t0s[s];
        const int64_t ns = hb->trace_offsets[t0s[s + 1]] - hb->trace_offsets[t0s[s]];
        off_b += a16((size_t)(Ts + 1) * 8) * (logr ? 2 : 1);
        ws_b += a16(ss::work_bytes(ns, Ts));
    }
    const size_t total = a16(in_b) + a16(out_b) + a16(log_b) + a16(off_b) + a16(ws_b);
    std::lock_guard<std::mutex> lk(g_stage.mu);
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if (g_stage.dev != dev && (g_stage.buf || g_stage.streams[0])) {
        // the staging buffer and streams belong to the device of an earlier call: release them there
        CK(cudaSetDevice(g_stage.dev));
        if (g_stage.buf) cudaFree(g_stage.buf);
        for (auto& st : g_stage.streams)
            if (st) cudaStreamDestroy(st), st = nullptr;
        g_stage.buf = nullptr;
        g_stage.cap = 0;
        CK(cudaSetDevice(dev));
    }
    g_stage.dev = dev;
    if (g_stage.cap < total) {
        if (g_stage.buf) CK(cudaFree(g_stage.buf));
        g_stage.buf = nullptr;
        g_stage.cap = 0;
        CK(cudaMalloc(&g_stage.buf, total));
        g_stage.cap = total;
    }
    if (g_stage.hcap < off_b) {  // pinned staging of the slices' rebased offsets
        if (g_stage.hbuf) CK(cudaFreeHost(g_stage.hbuf));
        g_stage.hbuf = nullptr;
        g_stage.hcap = 0;
        CK(cudaMallocHost(&g_stage.hbuf, off_b));
        g_stage.hcap = off_b;
    }
    for (int s = 0; s < S; s++)
        if (!g_stage.streams[s]) CK(cudaStreamCreateWithFlags(&g_stage.streams[s], cudaStreamNonBlocking));
    char* p = (char*)g_stage.buf;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += a16(bytes);
        return (void*)r;
    };
    // whole-batch device arrays; slice s works on its request / trace range
    ss_trace_batch db = *hb;
    db.ready_time = (double*)take(nn * 8);
    db.arrival_time = (double*)take(nn * 8);
    db.prompt_len = (uint32_t*)take(nn * 4);
    db.true_output_len = (uint32_t*)take(nn * 4);
    db.pred_len = (uint32_t*)take(nn * 4);
    db.pred_urgency = (uint8_t*)take(nn);
    db.true_urgency = (uint8_t*)take(nn);
    db.tie_rank = (uint32_t*)take(nn * 4);
    ss_outputs dout;
    memset(&dout, 0, sizeof dout);
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
    if (logr) dout.round_log = (uint32_t*)take((size_t)log_words * 4);
    char* d_offs = (char*)take(off_b);
    char* d_ws = (char*)take(ws_b);
    char* h_offs = (char*)g_stage.hbuf;
    // the slices start after the caller's stream work
    cudaStream_t cs = (cudaStream_t)stream;
    cudaEvent_t ev_in = nullptr, ev_k0 = nullptr, ev_k1[SS_MAX_SLICES] = {};
    auto drop_events = [&]() {
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_k0) cudaEventDestroy(ev_k0);
        for (auto& e : ev_k1)
            if (e) cudaEventDestroy(e), e = nullptr;
        ev_in = ev_k0 = nullptr;
    };
    // every slice's uploads, kernels and downloads; an error return leaves
    // work queued on the slice streams, which must drain before the staging
    // buffers (and the g_stage lock) are given up
    auto run_slices = [&]() -> int {
        // the round log is copied back whole: its words past each trace's log_words
        // are defined (zero) rather than left over from earlier calls (initcheck)
        if (logr) CK(cudaMemsetAsync(dout.round_log, 0, (size_t)log_words * 4, cs));
        CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        CK(cudaEventRecord(ev_in, cs));
        if (kernel_ms && S > 1) {
            CK(cudaEventCreate(&ev_k0));
            for (int s = 0; s < S; s++) CK(cudaEventCreate(&ev_k1[s]));
        }
        size_t ooff = 0, wsoff = 0;
        ss_outputs so_s[SS_MAX_SLICES];
        int64_t ra_s[SS_MAX_SLICES], ns_s[SS_MAX_SLICES], la_s[SS_MAX_SLICES], lw_s[SS_MAX_SLICES];
        int32_t ta_s[SS_MAX_SLICES], Ts_s[SS_MAX_SLICES];
        for (int s = 0; s < S; s++) {
            cudaStream_t st = g_stage.streams[s];
            CK(cudaStreamWaitEvent(st, ev_in, 0));
            const int32_t ta = t0s[s], Ts = t0s[s + 1] - t0s[s];
            const int64_t ra = hb->trace_offsets[ta], ns = hb->trace_offsets[t0s[s + 1]] - ra;
            // rebased trace (and log) offsets of this slice
            int64_t* ho_off = (int64_t*)(h_offs + ooff);
            int64_t* do_off = (int64_t*)(d_offs + ooff);
            for (int32_t t = 0; t <= Ts; t++) ho_off[t] = hb->trace_offsets[ta + t] - ra;
            CK(cudaMemcpyAsync(do_off, ho_off, (size_t)(Ts + 1) * 8, cudaMemcpyHostToDevice, st));
            ooff += a16((size_t)(Ts + 1) * 8);
            ss_trace_batch sb = db;
            sb.n_traces = Ts;
            sb.n_requests = ns;
            sb.trace_offsets = do_off;
#define H2D(field, esz)                                                                                  \
        do {                                                                                                 \
            sb.field = db.field + ra;                                                                        \
            if (ns > 0) CK(cudaMemcpyAsync((void*)sb.field, hb->field + ra, (size_t)ns * (esz), cudaMemcpyHostToDevice, st)); \
        } while (0)
            H2D(ready_time, 8);
            H2D(arrival_time, 8);
            H2D(prompt_len, 4);
            H2D(true_output_len, 4);
            H2D(pred_len, 4);
            H2D(pred_urgency, 1);
            H2D(true_urgency, 1);
            H2D(tie_rank, 4);
#undef H2D
            ss_outputs so = dout;
            so.req.first_scheduled += ra;
            so.req.finish_time += ra;
            so.req.generated += ra;
            so.req.evictions += ra;
            if (so.req.f_t) so.req.f_t += ra;
            if (so.req.state) so.req.state += ra;
            so.stats += ta;
            so.unservable_slots += ra;
            int64_t la = 0, lw = 0;
            if (logr) {
                la = ho->log_offsets[ta];
                lw = ho->log_offsets[t0s[s + 1]] - la;
                int64_t* hl = (int64_t*)(h_offs + ooff);
                int64_t* dl = (int64_t*)(d_offs + ooff);
                for (int32_t t = 0; t <= Ts; t++) hl[t] = ho->log_offsets[ta + t] - la;
                CK(cudaMemcpyAsync(dl, hl, (size_t)(Ts + 1) * 8, cudaMemcpyHostToDevice, st));
                ooff += a16((size_t)(Ts + 1) * 8);
                so.round_log += la;
                so.log_offsets = dl;
            }
            // no trace of the slice long enough for a bulk first round: skip the bulk-sort stage
            ss_params pp = *params;
            if (pp.bulk_min == 0) {
                int64_t maxlen = 0;
                for (int32_t t = ta; t < ta + Ts; t++) {
                    const int64_t k = hb->trace_offsets[t + 1] - hb->trace_offsets[t];
                    if (k > maxlen) maxlen = k;
                }
                if (maxlen < SS_BULK_MIN_DEFAULT) pp.bulk_min = -1;
            }
            if (pp.epilogue_min >= 0) {  // no trace long enough for the grid-wide end: skip its launches
                int64_t maxlen = 0;
                for (int32_t t = ta; t < ta + Ts; t++) {
                    const int64_t k = hb->trace_offsets[t + 1] - hb->trace_offsets[t];
                    if (k > maxlen) maxlen = k;
                }
                if (maxlen < ss::epilogue_threshold(pp)) pp.epilogue_min = -1;
            }
            const size_t wsz = ss::work_bytes(ns, Ts);
            if (ev_k0 && s == 0) CK(cudaEventRecord(ev_k0, st));
            // one slice: the call times its prepass and kernel itself (ss_last_timings)
            rc = ss_run_traces(&pp, &sb, &so, d_ws + wsoff, wsz, (void*)st, S == 1 ? kernel_ms : nullptr);
            if (rc) return rc;
            wsoff += a16(wsz);
            if (ev_k0) CK(cudaEventRecord(ev_k1[s], st));
            so_s[s] = so;
            ra_s[s] = ra;
            ns_s[s] = ns;
            ta_s[s] = ta;
            Ts_s[s] = Ts;
            la_s[s] = la;
            lw_s[s] = lw;
        }
        // downloads only after every slice's work is queued: a pageable destination makes
        // cudaMemcpyAsync block the host, which must not delay the later slices' uploads
        for (int s = 0; s < S; s++) {
            cudaStream_t st = g_stage.streams[s];
            const ss_outputs& so = so_s[s];
            const int64_t ra = ra_s[s], la = la_s[s], lw = lw_s[s];
            const int32_t ta = ta_s[s], Ts = Ts_s[s];
#define D2H(dst, src, bytes) \
        if ((dst) && (bytes) > 0) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st))
            const size_t nb = (size_t)ns_s[s];
            D2H(ho->req.first_scheduled + ra, so.req.first_scheduled, nb * 8);
            D2H(ho->req.finish_time + ra, so.req.finish_time, nb * 8);
            D2H(ho->req.generated + ra, so.req.generated, nb * 4);
            D2H(ho->req.evictions + ra, so.req.evictions, nb * 4);
            if (ho->req.f_t) D2H(ho->req.f_t + ra, so.req.f_t, nb * 8);
            if (ho->req.state) D2H(ho->req.state + ra, so.req.state, nb * 4);
            D2H(ho->stats + ta, so.stats, (size_t)Ts * sizeof(ss_trace_stats));
            D2H(ho->unservable_slots + ra, so.unservable_slots, nb * 4);
            if (logr) D2H(ho->round_log + la, so.round_log, (size_t)lw * 4);
#undef D2H
        }
        for (int s = 0; s < S; s++) CK(cudaStreamSynchronize(g_stage.streams[s]));
        return SS_OK;
    };
    rc = run_slices();
    if (rc) {
        for (int s = 0; s < S; s++)
            if (g_stage.streams[s]) cudaStreamSynchronize(g_stage.streams[s]);
        drop_events();
        return rc;
    }
    if (kernel_ms && S > 1) {
        // span from the first slice's prepass to the last kernel to finish
        float mx = 0.f;
        for (int s = 0; s < S; s++) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, ev_k0, ev_k1[s]) == cudaSuccess) mx = ms > mx ? ms : mx;
        }
        *kernel_ms = g_kernel_ms = mx;
        g_prepass_ms = 0.f;
    }
    drop_events();
    for (int32_t t = 0; t < T; t++)
        if (ho->stats[t].status != SS_TRACE_OK) return fail(SS_ERR_TRACE_FAILED, "a trace ended with a non-OK status");
    return SS_OK;
}

}  // extern "C"
