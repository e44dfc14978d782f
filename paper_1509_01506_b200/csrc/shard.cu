// The multi-GPU and speculation entry points of the C ABI
// (include/kmerscan_b200.h): shard boundary maps (ks_segment_map[_async]),
// a shard's count from maps gathered over NCCL or from a loaded halo
// (ks_count_shard_async), and the reference's speculative runs with their
// reconciliation (ks_speculate, for engine.match_chunk metadata).
//
// A shard's boundary map is its start -> end state map over all states: one
// state per thread walking the shard (SPECULATE), the uniform image of its
// last D bases (LOOKBACK), or the action of the product of its chunk
// elements (MAPSCAN).  Rank r's entry state is START pushed through the maps
// of ranks < r (the reference's chain walk, engine.py:155-163, lifted to
// GPU shards).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "runtime.h"

namespace ks {
namespace {

// map_out[q_orig] = original id of walking [begin, end) from q (all q), or of
// walking [end - D, end) from any state (uniform) for definite automata.
template <class T>
__global__ void segment_map_kernel(SeqView seq, int64_t begin, int64_t end, const T* t1, int32_t nq,
                                   int32_t uniform_start, const int32_t* new_of_old, const int32_t* old_of_new,
                                   int32_t* map_out) {
    __shared__ uint32_t shared_state;
    if (uniform_start >= 0) {
        if (threadIdx.x == 0 && blockIdx.x == 0) {
            uint32_t s = uint32_t(uniform_start);
            for (int64_t p = begin; p < end; ++p) s = t1[size_t(s) * 5 + seq_sym(seq, p)];
            shared_state = s;
        }
        __syncthreads();
        const int32_t v = old_of_new[shared_state];
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) map_out[q] = v;
        return;
    }
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        uint32_t s = uint32_t(new_of_old[q]);
        for (int64_t p = begin; p < end; ++p) s = t1[size_t(s) * 5 + seq_sym(seq, p)];
        map_out[q] = old_of_new[s];
    }
}

// map_out[q_orig] = original id of action(element *d_elem)(q)
__global__ void action_map_kernel(const uint16_t* d_elem, const uint16_t* action, int32_t nq,
                                  const int32_t* new_of_old, const int32_t* old_of_new, int32_t* map_out) {
    const uint32_t m = *d_elem;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x)
        map_out[q] = old_of_new[action[size_t(m) * nq + new_of_old[q]]];
}

// entry of shard `rank`: START pushed through the gathered maps of ranks < rank
__global__ void compose_entry_kernel(const int32_t* maps, int32_t nq, int32_t rank, int32_t start_orig,
                                     const int32_t* new_of_old, uint16_t* entry_internal) {
    int32_t s = start_orig;
    for (int r = 0; r < rank; ++r) s = maps[size_t(r) * nq + s];
    *entry_internal = uint16_t(new_of_old[s]);
}


// cuStreamWaitValue32 / cuStreamWriteValue32 through the runtime's driver
// entry points (no -lcuda link).
using StreamValueFn = int (*)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
StreamValueFn stream_value_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return reinterpret_cast<StreamValueFn>(fn);
}
int stream_write_value(cudaStream_t st, unsigned int* addr, unsigned int value) {
    static const StreamValueFn fn = stream_value_fn("cuStreamWriteValue32");
    if (!fn) return fail(KS_E_UNSUPPORTED, "cuStreamWriteValue32 unavailable");
    if (fn(st, reinterpret_cast<unsigned long long>(addr), value, 0u) != 0)
        return fail(KS_E_CUDA, "cuStreamWriteValue32 failed");
    return KS_OK;
}

}  // namespace

int count_shard_impl(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                     const int32_t* d_maps, int32_t rank, unsigned long long* d_counts, unsigned int* d_signal,
                     unsigned int signal_value);
}  // namespace ks

using namespace ks;

extern "C" {

int ks_segment_map(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                   int32_t* map_out) {
    CtxLock lock_(ctx);
    if (!ctx || !dfa || !seq || !map_out) return fail(KS_E_INVALID, "null argument");
    if (begin < 0 || end < begin || end > seq->n) return fail(KS_E_INVALID, "segment out of bounds");
    DeviceGuard guard(ctx->device);
    const HostDfa& h = dfa->host;
    std::vector<uint32_t> img(h.nq);
    int launches = 0;
    if (h.strategy != KS_STRATEGY_MAPSCAN) {   // SPECULATE: every state walks the segment
        Arena ar;
        int rc = ensure_scratch(ctx, size_t(h.nq) * 4 + 1024, &ar);
        if (rc) return rc;
        uint32_t* d = static_cast<uint32_t*>(ar.take(size_t(h.nq) * 4));
        if (h.strategy == KS_STRATEGY_LOOKBACK && end - begin >= h.sync_depth) {
            rc = launch_walk(ctx, dfa, seq, end - h.sync_depth, end, 1, h.start_internal, d);
            if (rc) return rc;
            uint32_t v = 0;
            KS_CUDA(cudaMemcpyAsync(&v, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
            std::fill(img.begin(), img.end(), v);
        } else {
            rc = launch_walk(ctx, dfa, seq, begin, end, h.nq, -1, d);
            if (rc) return rc;
            KS_CUDA(cudaMemcpyAsync(img.data(), d, size_t(h.nq) * 4, cudaMemcpyDeviceToHost, ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
        }
    } else {
        int64_t origin, L, nch;
        geometry(seq, begin, end, &origin, &L, &nch);
        uint16_t m = 0;
        if (end > begin) {
            Arena ar;
            int rc = ensure_scratch(ctx, size_t(nch) * 4 + 4096, &ar);
            if (rc) return rc;
            uint16_t* elems = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
            uint16_t* tot = static_cast<uint16_t*>(ar.take(16));
            rc = monoid_prefix(ctx, dfa, seq, begin, end, origin, L, nch, elems, nullptr, 0, nullptr, tot, &launches);
            if (rc) return rc;
            KS_CUDA(cudaMemcpyAsync(&m, tot, 2, cudaMemcpyDeviceToHost, ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        for (int q = 0; q < h.nq; ++q) img[q] = h.action[size_t(m) * h.nq + q];
    }
    for (int q = 0; q < h.nq; ++q) map_out[q] = h.old_of_new[img[h.new_of_old[q]]];
    return KS_OK;
}

int ks_segment_map_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                         int32_t* d_map_out) {
    CtxLock lock_(ctx);
    if (!ctx || !dfa || !seq || !d_map_out) return fail(KS_E_INVALID, "null argument");
    if (begin < 0 || end < begin || end > seq->n) return fail(KS_E_INVALID, "segment out of bounds");
    DeviceGuard guard(ctx->device);
    const HostDfa& h = dfa->host;
    const int threads = 256;
    const int blocks = std::max(1, std::min((h.nq + threads - 1) / threads, 1024));
    if (h.strategy != KS_STRATEGY_MAPSCAN) {   // SPECULATE: every state walks the segment
        const bool uniform = h.strategy == KS_STRATEGY_LOOKBACK && end - begin >= h.sync_depth;
        if (h.wide)
            segment_map_kernel<uint32_t><<<uniform ? 1 : blocks, threads, 0, ctx->stream>>>(
                view_of(seq), uniform ? end - h.sync_depth : begin, end, dfa->scan.t1w, h.nq,
                uniform ? h.start_internal : -1, dfa->d_new_of_old, dfa->d_old_of_new, d_map_out);
        else
            segment_map_kernel<uint16_t><<<uniform ? 1 : blocks, threads, 0, ctx->stream>>>(
                view_of(seq), uniform ? end - h.sync_depth : begin, end, dfa->scan.t1, h.nq,
                uniform ? h.start_internal : -1, dfa->d_new_of_old, dfa->d_old_of_new, d_map_out);
        KS_CUDA(cudaGetLastError());
        ctx->async_launches += 1;
        ++ctx->async_calls;
        return KS_OK;
    }
    int64_t origin, L, nch;
    geometry(seq, begin, end, &origin, &L, &nch);
    Arena ar;
    int rc = ensure_scratch(ctx, size_t(nch) * 4 + 4096, &ar);
    if (rc) return rc;
    uint16_t* elems = static_cast<uint16_t*>(ar.take(size_t(nch) * 2 + 2));
    uint16_t* tot = static_cast<uint16_t*>(ar.take(16));
    int launches = 0;
    if (nch > 0) {
        rc = monoid_prefix(ctx, dfa, seq, begin, end, origin, L, nch, elems, nullptr, 0, nullptr, tot, &launches);
        if (rc) return rc;
    } else {
        KS_CUDA(cudaMemsetAsync(tot, 0, 2, ctx->stream));  // identity element
    }
    action_map_kernel<<<blocks, threads, 0, ctx->stream>>>(tot, dfa->d_action, h.nq, dfa->d_new_of_old,
                                                           dfa->d_old_of_new, d_map_out);
    KS_CUDA(cudaGetLastError());
    ctx->async_launches += launches + 1;
    ++ctx->async_calls;
    return KS_OK;
}


int ks_count_shard_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                         const int32_t* d_maps, int32_t rank, unsigned long long* d_counts) {
    return count_shard_impl(ctx, dfa, seq, begin, end, d_maps, rank, d_counts, nullptr, 0u);
}

int ks_count_shard_async_signal(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                                const int32_t* d_maps, int32_t rank, unsigned long long* d_counts,
                                uint32_t* d_signal, uint32_t signal_value) {
    if (!d_signal) return fail(KS_E_INVALID, "null signal");
    return count_shard_impl(ctx, dfa, seq, begin, end, d_maps, rank, d_counts, d_signal, signal_value);
}

int ks_stream_wait_value32(void* stream, const uint32_t* d_addr, uint32_t value) {
    static const StreamValueFn fn = stream_value_fn("cuStreamWaitValue32");
    if (!d_addr) return fail(KS_E_INVALID, "null address");
    if (!fn) return fail(KS_E_UNSUPPORTED, "cuStreamWaitValue32 unavailable");
    if (fn(static_cast<cudaStream_t>(stream), reinterpret_cast<unsigned long long>(d_addr), value, 0u /* GEQ */) != 0)
        return fail(KS_E_CUDA, "cuStreamWaitValue32 failed");
    return KS_OK;
}

}  // extern "C"

int ks::count_shard_impl(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                         const int32_t* d_maps, int32_t rank, unsigned long long* d_counts, unsigned int* d_signal,
                         unsigned int signal_value) {
    CtxLock lock_(ctx);
    if (!ctx || !dfa || !seq || !d_counts) return fail(KS_E_INVALID, "null argument");
    if (begin < 0 || end < begin || end > seq->n) return fail(KS_E_INVALID, "range out of bounds");
    DeviceGuard guard(ctx->device);
    const HostDfa& h = dfa->host;
    // halo mode (rank > 0, no maps): the bases before `begin` are the previous
    // shard's tail, at least the synchronisation depth long (LOOKBACK only)
    const bool halo = rank > 0 && !d_maps;
    if (h.wide && rank > 0 && !halo)
        return fail(KS_E_UNSUPPORTED, "wide automata shard in halo mode only (no map exchange)");
    if (halo && end > begin && (h.strategy != KS_STRATEGY_LOOKBACK || begin < h.sync_depth))
        return fail(KS_E_INVALID, "shard without maps needs a definite automaton and a halo of sync_depth bases");
    int64_t origin, L, nch;
    geometry(seq, begin, end, &origin, &L, &nch);
    const bool mapscan = h.strategy == KS_STRATEGY_MAPSCAN;
    const bool spec = h.strategy == KS_STRATEGY_SPECULATE;
    Arena ar;
    size_t need = size_t(h.n_accept) * 8 + size_t(nch) * 2 + 64 * kAlign;
    if (mapscan) need += size_t(nch) * 6;
    if (spec) need += size_t(nch) * 2;
    int rc = ensure_scratch(ctx, need, &ar);
    if (rc) return rc;
    const ScanPlan plan = plan_for(ctx, dfa, dfa->scan);
    // the fast kernel's last CTA finalizes the counts straight into d_counts
    // (it zeroes them first) from the dfa's persistent visit block, which it
    // leaves zeroed: a halo-mode shard count is then one launch
    const bool fused = plan.fast && nch > 0;
    unsigned long long* visits = fused ? static_cast<unsigned long long*>(dfa->d_cnt)
                                       : static_cast<unsigned long long*>(ar.take(size_t(h.n_accept) * 8));
    uint16_t* entry = static_cast<uint16_t*>(ar.take(16));
    uint16_t* chunk_exit = static_cast<uint16_t*>(ar.take(size_t(nch) * 2 + 2));
    int launches = 0;
    if (!fused) {
        if (h.n_accept > 0) KS_CUDA(cudaMemsetAsync(visits, 0, size_t(h.n_accept) * 8, ctx->stream));
        KS_CUDA(cudaMemsetAsync(d_counts, 0, size_t(std::max(h.ne, 1)) * 8, ctx->stream));
    }
    // rank 0 enters in START: a constant, so no compose launch and (LOOKBACK)
    // a scan whose wait for the preceding kernel is deferred
    const bool const_entry = !halo && rank == 0;
    if (!halo && !const_entry) {
        compose_entry_kernel<<<1, 1, 0, ctx->stream>>>(d_maps, h.nq, rank, 0, dfa->d_new_of_old, entry);
        KS_CUDA(cudaGetLastError());
    }
    if (nch > 0) {
        ScanArgs a = base_args(dfa, dfa->scan, seq);
        a.begin = begin;
        a.end = end;
        a.origin = origin;
        a.chunk_len = L;
        a.nchunks = nch;
        a.visits = visits;
        a.chunk_exit = chunk_exit;
        if (mapscan) {
            uint16_t* elems = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
            uint16_t* centry = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
            uint16_t* mtot = static_cast<uint16_t*>(ar.take(16));
            rc = monoid_prefix(ctx, dfa, seq, begin, end, origin, L, nch, elems, centry,
                               const_entry ? h.start_internal : 0, const_entry ? nullptr : entry, mtot, &launches);
            if (rc) return rc;
            a.chunk_entry = centry;
        } else if (spec) {
            uint16_t* centry = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
            rc = spec_entries(ctx, dfa, seq, begin, end, origin, L, nch, const_entry ? h.start_internal : -1,
                              const_entry ? nullptr : entry, centry, nullptr, &launches);
            if (rc) return rc;
            a.chunk_entry = centry;
        } else {
            a.lookback = h.sync_depth;
            a.base_pos = halo ? 0 : begin;   // halo: every chunk, the first included, looks back
            a.base_state = h.start_internal;
            a.base_state_ptr = (halo || const_entry) ? nullptr : entry;
            a.any_state = h.start_internal;
        }
        if (fused) {
            char* blk = static_cast<char*>(dfa->d_cnt);
            int32_t* err = reinterpret_cast<int32_t*>(blk + size_t(h.n_accept) * 8 + size_t(std::max(h.ne, 1)) * 8);
            a.fin_counts = d_counts;
            a.fin_exit_src = chunk_exit + (nch - 1);
            a.fin_exit_dst = reinterpret_cast<uint16_t*>(err + 2);
            a.fin_done = reinterpret_cast<unsigned int*>(err + 1);   // zero between calls
            a.dyn_items = 1;   // fused: the finalizing CTA resets the dynamic-item counters
            a.fin_host = nullptr;
            a.n_expr = h.ne;
            a.fin_signal = d_signal;   // the finalizing CTA raises the flag after the counts
            a.fin_signal_value = signal_value;
        }
        rc = dispatch(ctx, dfa, dfa->scan, plan, a, kModeCount, &launches);
        if (rc) return rc;
    }
    if (!fused) {
        rc = launch_finalize_counts(ctx, visits, h.n_accept, dfa->d_acc_out_off, dfa->d_acc_out_ids, d_counts,
                                    nullptr, nullptr, &launches);
        if (rc) return rc;
        launches += 2;   // the memsets
        if (d_signal) {   // no fused kernel raised it: a stream write after the finalize
            rc = stream_write_value(ctx->stream, d_signal, signal_value);
            if (rc) return rc;
        }
    }
    ctx->async_launches += launches;
    ++ctx->async_calls;
    return KS_OK;
}

extern "C" {

int ks_speculate(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int32_t n_chunks, const int64_t* chunk_begin,
                 const int64_t* chunk_end, const int64_t* pss_off, const int32_t* pss_data, int32_t window,
                 int32_t* conv_out, int64_t* delta_out) {
    CtxLock lock_(ctx);
    if (!ctx || !dfa || !seq || n_chunks < 0 || window < 0) return fail(KS_E_INVALID, "bad argument");
    if (n_chunks == 0) return KS_OK;
    if (!chunk_begin || !chunk_end || !pss_off || !conv_out) return fail(KS_E_INVALID, "null argument");
    DeviceGuard guard(ctx->device);
    const HostDfa& h = dfa->host;
    if (pss_off[0] != 0) return fail(KS_E_INVALID, "pss_off[0] must be 0");
    for (int32_t k = 0; k < n_chunks; ++k) {
        if (pss_off[k + 1] < pss_off[k]) return fail(KS_E_INVALID, "pss_off not monotone");
        if (chunk_begin[k] < 0 || chunk_end[k] < chunk_begin[k] || chunk_end[k] > seq->n)
            return fail(KS_E_INVALID, "chunk out of bounds");
    }
    const int64_t total = pss_off[n_chunks];
    std::vector<uint32_t> pss(size_t(std::max<int64_t>(total, 1)));   // internal ids
    for (int64_t i = 0; i < total; ++i) {
        if (pss_data[i] < 0 || pss_data[i] >= h.nq) return fail(KS_E_INVALID, "pss state out of range");
        pss[i] = uint32_t(h.new_of_old[pss_data[i]]);
    }
    std::vector<uint16_t> pss16;
    if (!h.wide) pss16.assign(pss.begin(), pss.end());
    const size_t id_bytes = h.wide ? 4 : 2;
    const size_t task_bytes = speculate_task_bytes(n_chunks, pss_off);
    const size_t delta_bytes = delta_out ? size_t(total) * size_t(std::max(h.ne, 1)) * 8 : 0;
    Arena ar;
    int rc = ensure_scratch(ctx, size_t(n_chunks) * 16 + size_t(n_chunks + 1) * 8 + size_t(total) * 8 +
                                     task_bytes + delta_bytes + 16 * 1024,
                            &ar);
    if (rc) return rc;
    int64_t* d_cb = static_cast<int64_t*>(ar.take(size_t(n_chunks) * 8));
    int64_t* d_ce = static_cast<int64_t*>(ar.take(size_t(n_chunks) * 8));
    int64_t* d_off = static_cast<int64_t*>(ar.take(size_t(n_chunks + 1) * 8));
    void* d_pss = ar.take(size_t(total) * id_bytes + 4);
    int32_t* d_conv = static_cast<int32_t*>(ar.take(size_t(total) * 4 + 4));
    void* d_tasks = ar.take(task_bytes);
    long long* d_delta = delta_out ? static_cast<long long*>(ar.take(delta_bytes)) : nullptr;
    KS_CUDA(cudaMemcpyAsync(d_cb, chunk_begin, size_t(n_chunks) * 8, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(d_ce, chunk_end, size_t(n_chunks) * 8, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(d_off, pss_off, size_t(n_chunks + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(d_pss, h.wide ? static_cast<const void*>(pss.data()) : static_cast<const void*>(pss16.data()),
                            size_t(total) * id_bytes, cudaMemcpyHostToDevice, ctx->stream));
    if (d_delta) KS_CUDA(cudaMemsetAsync(d_delta, 0, delta_bytes, ctx->stream));
    int launches = 0;
    rc = launch_speculate(ctx, view_of(seq), n_chunks, d_cb, d_ce, d_off, d_pss, h.wide, pss_off, window,
                          h.wide ? static_cast<const void*>(dfa->scan.t1w) : static_cast<const void*>(dfa->scan.t1),
                          h.n_accept, dfa->d_acc_out_off, dfa->d_acc_out_ids, h.ne, d_conv, d_delta, d_tasks,
                          &launches);
    if (rc) return rc;
    KS_CUDA(cudaMemcpyAsync(conv_out, d_conv, size_t(total) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (d_delta) KS_CUDA(cudaMemcpyAsync(delta_out, d_delta, delta_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    return KS_OK;
}

}  // extern "C"
