// Speculative start-state runs with warp-level convergence detection.
//
// Device form of the speculative part of match_chunk_kernel
// (kmerscan/_kernels.py:89-112): for one chunk, run R0 = pss[0] and every
// other candidate start state pss[i] in lock step for at most
// weff = min(window, chunk length) symbols; run i converges at the first
// step j where its state equals R0's (then it would coincide forever, the
// transition function being a function).  One warp = one chunk x up to 31
// candidates: lane 0 carries R0, lanes 1..31 the speculative runs; the
// convergence test of the whole warp is a single __match_any_sync on the
// states (lane 0's equivalence class = the converged lanes), and the warp
// retires as soon as __all_sync says every live lane has converged.
//
// Outputs per run: conv (step, or -1) and optionally the count correction
// delta_i = sum_{t < conv_i} out(s_i(t)) - out(s_0(t)), so that a converged
// run's counts are counts(R0) + delta_i, exactly the reference's
// `counts[i] += counts[0] - fr_counts[j]` reconciliation.
#include <algorithm>

#include "scan_kernels.cuh"

namespace ks {
namespace {

struct SpecTask {
    int32_t chunk;
    int32_t first;  // pss index (>= 1) carried by lane 1
};


__device__ __forceinline__ void add_outputs(long long* row, uint32_t s, int32_t n_accept,
                                            const int32_t* off, const int32_t* ids, long long v) {
    if (s >= uint32_t(n_accept)) return;
    for (int k = off[s]; k < off[s + 1]; ++k)
        atomicAdd(reinterpret_cast<unsigned long long*>(&row[ids[k]]), (unsigned long long)v);
}

__global__ void speculate_kernel(SeqView seq, const int64_t* cbeg, const int64_t* cend,
                                 const int64_t* pss_off, const uint16_t* pss, int32_t window,
                                 const SpecTask* tasks, int32_t ntasks, const uint16_t* t1,
                                 int32_t n_accept, const int32_t* off, const int32_t* ids,
                                 int32_t ne, int32_t* conv_out, long long* delta) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (wid >= ntasks) return;  // warp-uniform
    const SpecTask task = tasks[wid];
    const int64_t o = pss_off[task.chunk];
    const int64_t nr = pss_off[task.chunk + 1] - o;
    const int64_t cb = cbeg[task.chunk];
    const int64_t weff = min64(window, cend[task.chunk] - cb);
    const int64_t run = lane == 0 ? 0 : task.first + lane - 1;
    const bool live = lane > 0 && run < nr;
    uint32_t s = pss[o + (live ? run : 0)];
    int32_t conv = -1;
    for (int64_t j = 0; j < weff; ++j) {
        const uint32_t sym = seq_sym(seq, cb + j);
        s = t1[s * 5u + sym];
        const uint32_t s0 = __shfl_sync(0xffffffffu, s, 0);
        const unsigned same = __match_any_sync(0xffffffffu, s) & 1u;
        if (live && conv < 0) {
            if (same) {
                conv = int32_t(j);
            } else if (delta) {
                long long* row = delta + (o + run) * int64_t(ne);
                add_outputs(row, s, n_accept, off, ids, 1);
                add_outputs(row, s0, n_accept, off, ids, -1);
            }
        }
        if (__all_sync(0xffffffffu, !live || conv >= 0)) break;
    }
    if (live) conv_out[o + run] = conv;
    if (lane == 0 && task.first == 1) conv_out[o] = -1;
}

}  // namespace

int launch_speculate(ks_ctx* ctx, const SeqView& seq, int32_t n_chunks, const int64_t* d_cbeg,
                     const int64_t* d_cend, const int64_t* d_pss_off, const uint16_t* d_pss,
                     const int64_t* h_pss_off, int32_t window, const uint16_t* t1,
                     int32_t n_accept, const int32_t* off, const int32_t* ids, int32_t ne,
                     int32_t* d_conv, long long* d_delta, void* d_tasks_buf, int* launches) {
    std::vector<SpecTask> tasks;
    for (int32_t k = 0; k < n_chunks; ++k) {
        const int64_t nr = h_pss_off[k + 1] - h_pss_off[k];
        if (nr <= 0) continue;
        int64_t first = 1;
        do {
            tasks.push_back(SpecTask{k, int32_t(first)});
            first += 31;
        } while (first < nr);
    }
    if (tasks.empty()) return KS_OK;
    KS_CUDA(cudaMemcpyAsync(d_tasks_buf, tasks.data(), tasks.size() * sizeof(SpecTask),
                            cudaMemcpyHostToDevice, ctx->stream));
    const int threads = 256;
    const int64_t total = int64_t(tasks.size()) * 32;
    const int blocks = int((total + threads - 1) / threads);
    speculate_kernel<<<blocks, threads, 0, ctx->stream>>>(
        seq, d_cbeg, d_cend, d_pss_off, d_pss, window, static_cast<const SpecTask*>(d_tasks_buf),
        int32_t(tasks.size()), t1, n_accept, off, ids, ne, d_conv, d_delta);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    // the task list lives in pageable host memory: finish before it goes away
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    return KS_OK;
}

size_t speculate_task_bytes(int32_t n_chunks, const int64_t* h_pss_off) {
    size_t n = 0;
    for (int32_t k = 0; k < n_chunks; ++k) {
        const int64_t nr = h_pss_off[k + 1] - h_pss_off[k];
        if (nr > 0) n += size_t(max64(1, (nr - 1 + 30) / 31));
    }
    return n * sizeof(SpecTask) + 16;
}

}  // namespace ks
