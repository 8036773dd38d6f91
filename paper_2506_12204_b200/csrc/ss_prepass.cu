// ss_prepass.cu — grid-wide work that precedes the per-trace scheduler warps.
//
// 1. Request init (engine.py:183-199), one thread per request over every
//    trace at once: static / dynamic records (f_t of a fresh request), output
//    initialisation, per-trace tallies (unservable count -> identity pending
//    list when zero; token sum -> automatic round cap). Coalesced, HBM-bound.
//
// 2. Bulk admission. The first round of a trace admits every request whose
//    prediction-ready time is within 1e-12 of the first one (engine.py:204-206).
//    When that group is large (config C: 1,000,000 requests at t = 0) the
//    reference pushes each into its dispatch heap (heaps.py:32-113, and the
//    O(n^2) ArrivalBuffer drain, heaps.py:233). Here the group's packed
//    dispatch keys (requests.py:81-91; the f_t of a fresh request is static)
//    are sorted ONCE by a grid-wide LSD radix sort over 8-bit digits of
//    (trace, key-hi, key-lo), stable, with digits that are constant over the
//    whole input skipped (decided on the device from one histogram pass). The
//    scheduler warp then consumes the sorted run from its front (ss_kernel.cu
//    refill), so a million-request pool costs O(1) per round instead of a scan.
//
// Every kernel reads its sizes from device memory (bulk element count,
// per-pass plan): the host launches a fixed sequence with no synchronisation,
// and kernels with nothing to do exit at once.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ss_common.cuh"
#include "ss_costs.cuh"
#include "ss_kernel.cuh"

namespace ss {

namespace {

__device__ __forceinline__ unsigned lanemask_lt_pp() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ long long bulk_threshold(const ss_params& P) {
    return P.bulk_min == 0 ? (long long)SS_BULK_MIN_DEFAULT : P.bulk_min;
}

// ---- 1. bulk detection: one thread per trace -------------------------------
// The first admission threshold follows Simulator.run (engine.py:202-211):
// clock 0; if the first servable request is not ready by 0 + 1e-12 the loop
// jumps the clock to its ready time, then admits ready <= clock + 1e-12.
__global__ void detect_kernel(const __grid_constant__ KArgs A) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= A.in.n_traces) return;
    const long long off = A.in.trace_offsets[t];
    const long long n = A.in.trace_offsets[t + 1] - off;
    int P = 0;
    const long long bm = bulk_threshold(A.P);
    if (bm > 0 && n >= bm) {
        long long i0 = 0;
        while (i0 < n && (long long)A.in.prompt_len[off + i0] + 1 > A.P.memory_capacity) i0++;
        if (i0 < n) {
            const double r0 = A.in.ready_time[off + i0];
            const double c0 = r0 <= add(0.0, 1e-12) ? 0.0 : r0;
            const double thr = add(c0, 1e-12);
            long long lo = i0, hi = n;  // ready is sorted (pending order)
            while (lo < hi) {
                long long mid = (lo + hi) >> 1;
                if (A.in.ready_time[off + mid] <= thr) lo = mid + 1;
                else hi = mid;
            }
            if (lo >= bm) P = (int)lo;
        }
    }
    A.w.bulkP[t] = P;
    // grid-wide end of trace (ss_epilogue.cu) for long traces
    const long long em = epilogue_threshold(A.P);
    A.w.epT[t] = (em > 0 && n >= em) ? (int)((n + EPI_TILE - 1) / EPI_TILE) : 0;
}

// exclusive scan of in[0..T) -> out[0..T] (single CTA, chunked)
__device__ void block_scan(const int* in, long long* out, int T) {
    __shared__ long long wsum[32];
    __shared__ long long carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < T; base += 1024) {
        const int t = base + threadIdx.x;
        long long v = t < T ? (long long)in[t] : 0;
        long long x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            long long s = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                long long y = __shfl_up_sync(FULL, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const long long pre = carry + (wid ? wsum[wid - 1] : 0) + x - v;
        if (t < T) out[t] = pre;
        __syncthreads();
        if (threadIdx.x == 1023) carry = pre + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[T] = carry;
    __syncthreads();
}

// bulkP -> eoff (bulk runs), epT -> epoff (epilogue tiles)
__global__ void __launch_bounds__(1024) eoff_scan_kernel(const __grid_constant__ KArgs A) {
    block_scan(A.w.bulkP, A.w.eoff, A.in.n_traces);
    block_scan(A.w.epT, A.w.epoff, A.in.n_traces);
}

// ---- 2. request init: one thread per request --------------------------------
__global__ void __launch_bounds__(PP_THREADS) init_kernel(const __grid_constant__ KArgs A) {
    const long long n = A.in.n_requests;
    const int T = A.in.n_traces;
    const ss_profile& P = A.P.profile;
    const long long cap = A.P.memory_capacity;
    const long long stride = (long long)gridDim.x * blockDim.x;
    uint4* STA = reinterpret_cast<uint4*>(A.w.st);
    Dyn* DYN = reinterpret_cast<Dyn*>(A.w.dy);
    const int lane = threadIdx.x & 31;
    // uniform trip count so the warp-aggregated tallies see every lane
    for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += stride) {
        const long long g = base + threadIdx.x;
        const bool v = g < n;
        int t = -1;
        unsigned long long tok = 0, foot = 0;
        uint32_t uns = 0;
        if (v) {
            t = upper_index(A.in.trace_offsets, T, g);
            const long long i = g - A.in.trace_offsets[t];
            const uint32_t prompt = A.in.prompt_len[g], mid = A.in.pred_len[g], tout = A.in.true_output_len[g];
            uint4 st;
            st.x = prompt;
            st.y = tout;
            st.z = mid;
            st.w = ((uint32_t)A.in.pred_urgency[g] << 24) | A.in.tie_rank[g];
            STA[g] = st;
            const bool serv = (long long)prompt + 1 <= cap;
            uint32_t flg = serv ? ST_WAIT : ST_UNS;
            if (serv && i < A.w.bulkP[t]) flg |= F_Q;  // admitted in bulk: queued from the start
            Dyn d;
            d.ft = remaining_time(prompt, mid, 0, 0, 0, P);  // engine.py:183-184
            d.dec = 0u;
            d.flg = flg;
            DYN[g] = d;
            // dispatch key at admission (engine.py:204-206 -> heaps.py insert)
            const uint32_t rk = A.in.pred_urgency[g], tie = A.in.tie_rank[g], sl = (uint32_t)i;
            Key k;
            switch (A.P.policy) {
            case SS_POLICY_FCFS: k = make_key<SS_POLICY_FCFS>(rk, d.ft, tie, sl, false); break;
            case SS_POLICY_SJF: k = make_key<SS_POLICY_SJF>(rk, d.ft, tie, sl, false); break;
            case SS_POLICY_HPJF: k = make_key<SS_POLICY_HPJF>(rk, d.ft, tie, sl, false); break;
            default: k = make_key<SS_POLICY_SEMANTIC>(rk, d.ft, tie, sl, false); break;
            }
            reinterpret_cast<Key*>(A.w.k0)[g] = k;
            A.out.req.first_scheduled[g] = __longlong_as_double(0x7ff8000000000000ll);
            A.out.req.finish_time[g] = __longlong_as_double(0x7ff8000000000000ll);
            A.out.req.evictions[g] = 0u;
            A.out.unservable_slots[g] = 0xFFFFFFFFu;  // defined contents past the trace's list
            tok = tout;
            foot = (unsigned long long)prompt + (tout > mid ? tout : mid) + 1u;
            uns = serv ? 0u : 1u;
        }
        // warp-aggregated per-trace tallies (traces are contiguous in g, so a
        // warp touches few traces); 16-bit halves keep the lane sums exact
        const unsigned peers = __match_any_sync(FULL, v ? t : -1 - lane);
        const uint32_t s_lo = __reduce_add_sync(peers, (uint32_t)(tok & 0xffffu));
        const uint32_t s_hi = __reduce_add_sync(peers, (uint32_t)(tok >> 16));
        const uint32_t s_un = __reduce_add_sync(peers, uns);
        const uint32_t f_lo = __reduce_add_sync(peers, (uint32_t)(foot & 0xffffu));
        const uint32_t f_hi = __reduce_add_sync(peers, (uint32_t)(foot >> 16));
        if (v && lane == __ffs(peers) - 1) {
            atomicAdd(&A.w.tok[t], (unsigned long long)s_lo + ((unsigned long long)s_hi << 16));
            atomicAdd(&A.w.foot[t], (unsigned long long)f_lo + ((unsigned long long)f_hi << 16));
            if (s_un) atomicAdd(&A.w.nuns[t], s_un);
        }
    }
}

#ifndef SS_CHUNK_TIGHTNESS
#define SS_CHUNK_TIGHTNESS 0.55  // KV budget / (b x mean footprint bound) above which chunks run
#endif

// ---- 2b. scheduler variant: the no-eviction chunked kernel where the KV budget
// can never bind (twice the largest per-trace footprint bound fits), i.e. no
// trace can ever evict; otherwise the evicting chunked kernel when the budget
// holds SS_CHUNK_TIGHTNESS of a full batch's mean footprint, else the
// per-round kernel (heavy eviction: short stretches).
__global__ void __launch_bounds__(1024) select_kernel(const __grid_constant__ KArgs A) {
    __shared__ unsigned long long wmax[32];
    __shared__ double wfoot[32], wn[32];
    const int T = A.in.n_traces;
    unsigned long long mx = 0;
    double fs = 0.0, ns = 0.0;  // footprint bounds and requests over all traces
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        mx = A.w.foot[t] > mx ? A.w.foot[t] : mx;
        fs += (double)A.w.foot[t];
        ns += (double)(A.in.trace_offsets[t + 1] - A.in.trace_offsets[t]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(FULL, mx, o);
        mx = y > mx ? y : mx;
        fs += __shfl_xor_sync(FULL, fs, o);
        ns += __shfl_xor_sync(FULL, ns, o);
    }
    if ((threadIdx.x & 31) == 0) {
        wmax[threadIdx.x >> 5] = mx;
        wfoot[threadIdx.x >> 5] = fs;
        wn[threadIdx.x >> 5] = ns;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); i++) {
            mx = wmax[i] > mx ? wmax[i] : mx;
            fs += wfoot[i];
            ns += wn[i];
        }
        const long long cap = A.P.memory_capacity;
        int sel = (cap > 0 && mx <= (unsigned long long)cap / 2) ? SS_SEL_NO_EVICT : SS_SEL_PERROUND;
        // evicting regime: chunks pay when the budget holds most of a full batch's
        // footprint (config A, ratio ~0.71: chunked 22% faster); under heavy eviction
        // (config D, ~0.40) stretches are short and the per-round kernel is ahead
        const double per_req = ns > 0.0 ? fs / ns : 0.0;
        if (sel == SS_SEL_PERROUND && per_req > 0.0 &&
            (double)cap >= SS_CHUNK_TIGHTNESS * (double)A.P.batch_size * per_req)
            sel = SS_SEL_CHUNKED;
        if ((A.P.flags & SS_FLAG_FORCE_CHUNKED) && sel != SS_SEL_NO_EVICT) sel = SS_SEL_CHUNKED;
        if (A.P.flags & SS_FLAG_FORCE_PERROUND) sel = SS_SEL_PERROUND;
        *A.w.sel = sel;
    }
}

// ---- 3. bulk keys: one thread per bulk element ------------------------------
template <int POL>
__device__ __forceinline__ Key bulk_key(const KArgs& A, long long g, uint32_t i) {
    const uint32_t prompt = A.in.prompt_len[g];
    if ((long long)prompt + 1 > A.P.memory_capacity) {
        Key k = kinf();
        k.aux = SLOT_MASK;  // unservable: sorts behind the trace's run
        return k;
    }
    const double ft = remaining_time(prompt, A.in.pred_len[g], 0, 0, 0, A.P.profile);
    return make_key<POL>(A.in.pred_urgency[g], ft, A.in.tie_rank[g], i, false);
}

__global__ void __launch_bounds__(PP_THREADS) keys_kernel(const __grid_constant__ KArgs A) {
    const int T = A.in.n_traces;
    const long long E = A.w.eoff[T];
    Key* S = reinterpret_cast<Key*>(A.w.S);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const int t = upper_index(A.w.eoff, T, e);
        const long long i = e - A.w.eoff[t];
        const long long g = A.in.trace_offsets[t] + i;
        Key k;
        switch (A.P.policy) {
        case SS_POLICY_FCFS: k = bulk_key<SS_POLICY_FCFS>(A, g, (uint32_t)i); break;
        case SS_POLICY_SJF: k = bulk_key<SS_POLICY_SJF>(A, g, (uint32_t)i); break;
        case SS_POLICY_HPJF: k = bulk_key<SS_POLICY_HPJF>(A, g, (uint32_t)i); break;
        default: k = bulk_key<SS_POLICY_SEMANTIC>(A, g, (uint32_t)i); break;
        }
        S[e] = k;
        A.w.tt0[e] = (uint32_t)t;
    }
}

// ---- 4. LSD radix sort over (trace, hi, lo) ----------------------------------
__device__ __forceinline__ uint32_t digit_of(const Key& k, uint32_t tr, int p) {
    if (p < 4) return (k.lo >> (8 * p)) & 255u;
    if (p < 12) return (uint32_t)(k.hi >> (8 * (p - 4))) & 255u;
    return (tr >> (8 * (p - 12))) & 255u;
}

// all RS_PASSES digit histograms in one read of the keys
__global__ void __launch_bounds__(PP_THREADS) hist_kernel(const __grid_constant__ KArgs A) {
    __shared__ uint32_t h[RS_PASSES * 256];
    const long long E = A.w.eoff[A.in.n_traces];
    if (E == 0) return;
    for (int i = threadIdx.x; i < RS_PASSES * 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const Key* S = reinterpret_cast<const Key*>(A.w.S);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) {
        const Key k = S[e];
        const uint32_t tr = A.w.tt0[e];
#pragma unroll
        for (int p = 0; p < RS_PASSES; p++) atomicAdd(&h[p * 256 + digit_of(k, tr, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < RS_PASSES * 256; i += blockDim.x)
        if (h[i]) atomicAdd(&A.w.hist[i], h[i]);
}

// pass plan: a digit held by every key is skipped; sources alternate S / ins
__global__ void plan_kernel(const __grid_constant__ KArgs A) {
    __shared__ int trivial[RS_PASSES];
    const long long E = A.w.eoff[A.in.n_traces];
    if (threadIdx.x < RS_PASSES) trivial[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < RS_PASSES * 256; i += blockDim.x)
        if ((long long)A.w.hist[i] == E) trivial[i >> 8] = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        int src = 0;
        for (int p = 0; p < RS_PASSES; p++) {
            if (E == 0 || trivial[p]) {
                A.w.plan[p] = -1;
            } else {
                A.w.plan[p] = src;
                src ^= 1;
            }
        }
        A.w.plan[RS_PASSES] = src;  // buffer holding the sorted keys
    }
}

__device__ __forceinline__ const Key* src_keys(const KArgs& A, int s) {
    return reinterpret_cast<const Key*>(s ? A.w.ins : A.w.S);
}
__device__ __forceinline__ Key* dst_keys(const KArgs& A, int s) {
    return reinterpret_cast<Key*>(s ? A.w.S : A.w.ins);
}

// per-tile digit counts, stored digit-major: tcnt[d * tiles + tile]
__global__ void __launch_bounds__(PP_THREADS) count_kernel(const __grid_constant__ KArgs A, int p) {
    const int s = A.w.plan[p];
    if (s < 0) return;
    __shared__ uint32_t c[256];
    const long long E = A.w.eoff[A.in.n_traces];
    const long long tiles = (E + RS_TILE - 1) / RS_TILE;
    const Key* K = src_keys(A, s);
    const uint32_t* TT = s ? A.w.tt1 : A.w.tt0;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        c[threadIdx.x] = 0;
        __syncthreads();
        const long long b0 = tile * RS_TILE;
#pragma unroll 4
        for (int j = 0; j < RS_ITEMS; j++) {
            const long long e = b0 + j * PP_THREADS + threadIdx.x;
            if (e < E) atomicAdd(&c[digit_of(K[e], TT[e], p)], 1u);
        }
        __syncthreads();
        A.w.tcnt[(long long)threadIdx.x * tiles + tile] = c[threadIdx.x];
        __syncthreads();
    }
}

// exclusive scan of tcnt in digit-major order (single CTA, chunked)
__global__ void __launch_bounds__(1024) tscan_kernel(const __grid_constant__ KArgs A, int p) {
    if (A.w.plan[p] < 0) return;
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    const long long E = A.w.eoff[A.in.n_traces];
    const long long tiles = (E + RS_TILE - 1) / RS_TILE;
    const long long N = 256 * tiles;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (long long base = 0; base < N; base += 1024) {
        const long long i = base + threadIdx.x;
        const uint32_t v = i < N ? A.w.tcnt[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULL, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t sm = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(FULL, sm, o);
                if (lane >= o) sm += y;
            }
            wsum[lane] = sm;
        }
        __syncthreads();
        const uint32_t pre = carry + (wid ? wsum[wid - 1] : 0u) + x - v;
        if (i < N) A.w.tcnt[i] = pre;
        __syncthreads();
        if (threadIdx.x == 1023) carry = pre + v;
        __syncthreads();
    }
}

// stable scatter: keys of a tile ranked in input order within each digit
__global__ void __launch_bounds__(PP_THREADS) scatter_kernel(const __grid_constant__ KArgs A, int p) {
    const int s = A.w.plan[p];
    if (s < 0) return;
    constexpr int NW = PP_THREADS / 32;
    __shared__ uint32_t wc[NW][256];
    __shared__ uint32_t run[256];
    __shared__ uint32_t base[256];
    const long long E = A.w.eoff[A.in.n_traces];
    const long long tiles = (E + RS_TILE - 1) / RS_TILE;
    const Key* K = src_keys(A, s);
    Key* D = dst_keys(A, s);
    const uint32_t* TT = s ? A.w.tt1 : A.w.tt0;
    uint32_t* TD = s ? A.w.tt0 : A.w.tt1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt_pp();
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        base[threadIdx.x] = A.w.tcnt[(long long)threadIdx.x * tiles + tile];
        run[threadIdx.x] = 0;
        const long long b0 = tile * RS_TILE;
        for (int j = 0; j < RS_ITEMS; j++) {
#pragma unroll
            for (int w = 0; w < NW; w++) wc[w][threadIdx.x] = 0;
            __syncthreads();
            const long long e = b0 + j * PP_THREADS + threadIdx.x;
            const bool v = e < E;
            Key k;
            uint32_t tr = 0, d = 0;
            if (v) {
                k = K[e];
                tr = TT[e];
                d = digit_of(k, tr, p);
            }
            const unsigned peers = __match_any_sync(FULL, v ? (int)d : -1 - lane);
            const uint32_t rk = __popc(peers & lt);
            if (v && rk == 0) wc[wid][d] = __popc(peers);
            __syncthreads();
            {
                uint32_t acc = run[threadIdx.x];
#pragma unroll
                for (int w = 0; w < NW; w++) {
                    const uint32_t c = wc[w][threadIdx.x];
                    wc[w][threadIdx.x] = acc;
                    acc += c;
                }
                run[threadIdx.x] = acc;
            }
            __syncthreads();
            if (v) {
                const uint32_t pos = base[d] + wc[wid][d] + rk;
                D[pos] = k;
                TD[pos] = tr;
            }
            __syncthreads();
        }
    }
}

// the sorted keys end in S whatever the number of executed passes
__global__ void __launch_bounds__(PP_THREADS) final_kernel(const __grid_constant__ KArgs A) {
    if (A.w.plan[RS_PASSES] == 0) return;  // already in S
    const long long E = A.w.eoff[A.in.n_traces];
    const Key* src = reinterpret_cast<const Key*>(A.w.ins);
    Key* dst = reinterpret_cast<Key*>(A.w.S);
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += stride) dst[e] = src[e];
}

}  // namespace

int launch_prepass(const KArgs& a, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int T = a.in.n_traces;
    const long long n = a.in.n_requests;
    const int grid = sms * 8;  // 8 x 256 threads per SM, grid-stride
    detect_kernel<<<(T + 255) / 256, 256, 0, st>>>(a);
    eoff_scan_kernel<<<1, 1024, 0, st>>>(a);
    if (n > 0) {
        long long need = (n + PP_THREADS - 1) / PP_THREADS;
        init_kernel<<<(int)(need < grid ? need : grid), PP_THREADS, 0, st>>>(a);
    }
    select_kernel<<<1, 1024, 0, st>>>(a);
    if (a.P.bulk_min < 0 || n == 0) return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
    keys_kernel<<<grid, PP_THREADS, 0, st>>>(a);
    hist_kernel<<<sms * 2, PP_THREADS, 0, st>>>(a);
    plan_kernel<<<1, 256, 0, st>>>(a);
    const long long tiles_max = a.w.tiles_max;
    const int tgrid = (int)(tiles_max < grid ? tiles_max : grid);
    for (int p = 0; p < RS_PASSES; p++) {
        count_kernel<<<tgrid, PP_THREADS, 0, st>>>(a, p);
        tscan_kernel<<<1, 1024, 0, st>>>(a, p);
        scatter_kernel<<<tgrid, PP_THREADS, 0, st>>>(a, p);
    }
    final_kernel<<<grid, PP_THREADS, 0, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

}  // namespace ss
