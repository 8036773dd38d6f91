// ss_kernel.cuh — device-side argument block of the scheduler kernel.
#pragma once
#include <stdint.h>

#include "../../include/semsched_b200.h"

namespace ss {

constexpr int FCAP = 64;  // sorted queue-front capacity per trace (shared memory)
constexpr int WPB = 4;    // traces (warps) per CTA

// Per-request scratch in HBM, indexed like the inputs (trace offset + slot).
struct Work {
    void* st;            // static record: prompt, true_out, pred_len, rank << 24 | tie
    void* dy;            // dynamic record: f_t, decoded, flags (stage | prefilled | queued | ...)
    uint32_t* rpos;      // position in the resident list
    void* B;             // queue BACK: 16-byte packed keys
    uint32_t* R;         // resident list (eviction candidates)
    uint32_t* pend;      // servable requests in pending order
    void* ins;           // this round's re-queue list: 16-byte keys
    int* next_trace;     // work counter for persistent warps
};

struct KArgs {
    ss_params P;
    ss_trace_batch in;
    ss_outputs out;
    Work w;
};

size_t work_bytes(int64_t n_requests);
void carve_work(void* base, int64_t n_requests, Work* w);
int launch_sched(const KArgs& a, int blocks, void* stream);
int sched_smem_bytes();
int sched_max_blocks(int policy, int* sm_count);

}  // namespace ss
