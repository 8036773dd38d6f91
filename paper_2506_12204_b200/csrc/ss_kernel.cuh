// ss_kernel.cuh — device-side argument block of the scheduler kernel.
#pragma once
#include <stdint.h>

#include "../../include/semsched_b200.h"

namespace ss {

// select_kernel's choice: one round per step / chunked stretches with no eviction
// possible (resident list not kept) / chunked stretches forced by the caller
constexpr int SS_SEL_PERROUND = 0, SS_SEL_NO_EVICT = 1, SS_SEL_CHUNKED = 2;
constexpr int FCAP = 64;  // sorted queue-front capacity per trace (shared memory)
#ifndef SS_WPB
#define SS_WPB 4
#endif
constexpr int WPB = SS_WPB;  // traces (warps) per CTA

// Per-request scratch in HBM, indexed like the inputs (trace offset + slot).
struct Work {
    void* st;            // static record: prompt, true_out, pred_len, rank << 24 | tie
    void* dy;            // dynamic record: f_t, decoded, flags (stage | prefilled | queued | ...)
    uint32_t* rpos;      // position in the resident list
    void* B;             // queue BACK: 16-byte packed keys
    uint32_t* R;         // resident list (eviction candidates)
    uint32_t* pend;      // servable requests in pending order
    void* ins;           // this round's re-queue list: 16-byte keys (prepass: sort ping-pong)
    void* k0;            // dispatch key of each request at admission (prepass; read by the admission loop)
    // ---- prepass (ss_prepass.cu) -------------------------------------------
    void* S;                  // sorted bulk runs: 16-byte keys, trace t at [eoff[t], eoff[t] + bulkP[t])
    uint32_t* tt0;            // radix sort payload: trace index of each key (ping-pong pair)
    uint32_t* tt1;
    unsigned long long* tok;  // per trace: sum of true output lengths (round cap)
    unsigned long long* foot; // per trace: sum of prompt + max(true, predicted) output + 1 (KV footprint bound)
    int* sel;                 // scheduler variant for this run (SS_SEL_*)
    uint32_t* nuns;           // per trace: unservable requests (0 -> identity pending list)
    int* bulkP;               // per trace: bulk prefix length (0: no bulk admission)
    long long* eoff;          // per trace + 1: exclusive scan of bulkP
    uint32_t* hist;           // [RS_PASSES][256] global digit histograms
    int* plan;                // [RS_PASSES] source buffer of each pass (-1: skipped), [RS_PASSES]: final
    uint32_t* tcnt;           // [256][tiles] per-tile digit counts -> scanned offsets
    long long tiles_max;      // capacity of tcnt in tiles
    // ---- grid-wide end of trace (ss_epilogue.cu) ----------------------------
    int* epT;                 // per trace: epilogue tiles (0: the scheduler warp finishes the trace)
    long long* epoff;         // per trace + 1: exclusive scan of epT
    void* epart;              // per epilogue tile: partial sums (EpiPart)
    int* next_trace;     // work counter for persistent warps
};

struct KArgs {
    ss_params P;
    ss_trace_batch in;
    ss_outputs out;
    Work w;
    double z0;  // reload(0) + prefill(0) of a decoding request's remaining time (costs.py:174-191), host-computed
    int screen; // the chunk's order screen is valid: gamma1, gamma2 >= 0 and finite, z0 == 0 (ss_kernel.cu)
};

constexpr int PP_THREADS = 256;               // prepass CTA size
constexpr int RS_ITEMS = 16;                  // radix sort: keys per thread per tile
constexpr int RS_TILE = PP_THREADS * RS_ITEMS;
constexpr int RS_PASSES = 16;                 // 8-bit digits: lo 4, hi 8, trace index 4
constexpr int EPI_TILE = 4096;                // requests per epilogue tile (one CTA)
constexpr int EPI_CH = SS_MAX_LEVELS + 2;     // sums: level 0..15, normalized wait, wait

// per-tile partial sums of the grid-wide epilogue: double-double per channel
struct __align__(16) EpiPart {
    double hi[EPI_CH], lo[EPI_CH];
    int cnt[SS_MAX_LEVELS + 1];  // per level, completed
    int _pad[3];
};

// traces of >= this many requests finish in the grid-wide epilogue (0 = never)
__host__ __device__ __forceinline__ long long epilogue_threshold(const ss_params& P) {
    return P.epilogue_min == 0 ? (long long)SS_EPILOGUE_MIN_DEFAULT : (P.epilogue_min < 0 ? 0 : P.epilogue_min);
}

size_t work_bytes(int64_t n_requests, int32_t n_traces);
void carve_work(void* base, int64_t n_requests, int32_t n_traces, Work* w);
size_t work_zero_bytes(int32_t n_traces);  // leading bytes of the workspace zeroed per run
// grid-wide prepass: request init, per-trace tallies, bulk-admission sort
int launch_prepass(const KArgs& a, void* stream);
int launch_sched(const KArgs& a, int blocks, void* stream);
// grid-wide end of trace for long traces (per-request outputs + statistics)
int launch_epilogue(const KArgs& a, void* stream);
int sched_launches(int policy);  // scheduler kernel launches per run
int sched_smem_bytes();
int sched_max_blocks(int policy, int* sm_count);

}  // namespace ss
