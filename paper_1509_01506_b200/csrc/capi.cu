// C ABI (include/kmerscan_b200.h): contexts, count / locate / async count,
// and the host orchestration of one scan (scan_impl).  Uploads live in
// upload.cu, shard maps / shard counts / speculation in shard.cu, the
// streamed host-bytes count in stream.cu.
//
// Strategy LOOKBACK (definite automata -- every Aho-Corasick table built by
// build_dfa): one launch.  Each lane chunk derives its true entry state by
// scanning the D bases before it; chunks are independent, so the reference's
// PSS speculation + chain reduction (engine.py:80-91, 137-204) collapses to
// nothing and the single HBM pass is the whole job.
//
// Strategy MAPSCAN (non-converging automata with a small transition monoid,
// e.g. the BASELINE's 1024-state permutation DFA): pass 1 scans every chunk
// with the monoid automaton (chunk -> its start->end map as an element id),
// an exclusive device-wide scan composes the maps into each chunk's true
// entry state, pass 2 counts.  Speculation can never converge there, and the
// reference pays |Q| runs per chunk; this pays two passes.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "runtime.h"

namespace ks {

thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_error = std::string("CUDA error: ") + cudaGetErrorString(e) + " (" + what + ")";
    return KS_E_CUDA;
}


int ensure_scratch(ks_ctx* ctx, size_t bytes, Arena* a) {
    bytes = up(bytes) + 64 * kAlign;
    if (ctx->scratch_bytes < bytes) {
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->scratch) KS_CUDA(cudaFree(ctx->scratch));
        ctx->scratch = nullptr;
        ctx->scratch_bytes = 0;
        KS_CUDA(cudaMalloc(&ctx->scratch, bytes));
        ctx->scratch_bytes = bytes;
    }
    a->base = static_cast<char*>(ctx->scratch);
    a->off = 0;
    a->cap = ctx->scratch_bytes;
    return KS_OK;
}

int ensure_pinned(ks_ctx* ctx, size_t bytes) {
    if (ctx->pinned_bytes >= bytes) return KS_OK;
    if (ctx->pinned) KS_CUDA(cudaFreeHost(ctx->pinned));
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    bytes = std::max<size_t>(bytes, 1 << 16);
    KS_CUDA(cudaMallocHost(&ctx->pinned, bytes));
    ctx->pinned_bytes = bytes;
    return KS_OK;
}

bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}

// Pinned host memory the device can write through the same address (UVA).
bool host_is_device_visible(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost && at.devicePointer == p;
}

namespace {

// ------------------------------------------------------------ tiny kernels
// Rows [0, *n_dev) into pinned host staging; with res_src, block 0 also
// copies the results block (counts | err | exit, res_words words) and the
// row / log totals to pinned memory, so one synchronisation returns all.
__global__ void copy_rows_kernel(const longlong2* __restrict__ src, const int64_t* __restrict__ n_dev,
                                 longlong2* __restrict__ dst, const unsigned int* res_src, uint32_t res_words,
                                 unsigned int* res_dst, const unsigned long long* log_n, int64_t* tot_dst) {
    const int64_t n = *n_dev;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
    if (res_src && blockIdx.x == 0) {
        for (uint32_t i = threadIdx.x; i < res_words; i += blockDim.x) res_dst[i] = __ldcg(&res_src[i]);
        if (threadIdx.x == 0) {
            tot_dst[0] = n;
            tot_dst[1] = int64_t(__ldcg(log_n));
        }
    }
}

template <class T>   // T: uint16_t tables, uint32_t for wide automata
__global__ void walk_kernel(SeqView seq, int64_t begin, int64_t end, const T* t1, int32_t nq,
                            int32_t uniform_start, uint32_t* out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    uint32_t s = uniform_start >= 0 ? uint32_t(uniform_start) : uint32_t(q);
    for (int64_t p = begin; p < end; ++p) s = t1[size_t(s) * 5 + seq_sym(seq, p)];
    out[q] = s;
}

}  // namespace

// Walk [begin, end) from every state (uniform_start < 0, nlanes = |Q|) or
// from one state; internal ids into out (uint32).
int launch_walk(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end, int32_t nlanes,
                int32_t uniform_start, uint32_t* out) {
    const int threads = nlanes == 1 ? 32 : 128;
    const int blocks = (nlanes + threads - 1) / threads;
    if (dfa->host.wide)
        walk_kernel<uint32_t><<<blocks, threads, 0, ctx->stream>>>(view_of(seq), begin, end, dfa->scan.t1w, nlanes,
                                                                     uniform_start, out);
    else
        walk_kernel<uint16_t><<<blocks, threads, 0, ctx->stream>>>(view_of(seq), begin, end, dfa->scan.t1, nlanes,
                                                                     uniform_start, out);
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

SeqView view_of(const ks_seq* s) {
    SeqView v;
    v.bases = s->d_bases;
    v.nmask = s->d_nmask;
    v.rowmask = s->sealed ? s->d_rowmask : nullptr;
    v.n = s->n;
    v.lb = s->lb;
    return v;
}

ScanArgs base_args(const ks_dfa* dfa, const DevTable& T, const ks_seq* seq) {
    ScanArgs a;
    a.seq = view_of(seq);
    a.t1 = T.t1;
    a.t1w = T.t1w;
    a.ht = T.ht;
    a.hot_lo = T.hot_lo;
    a.hot_n = T.hot_n;
    a.tk = T.tk;
    a.nq = T.nq;
    a.n_accept = T.n_accept;
    a.reset_state = T.reset_state;
    a.tk_pad = int32_t(T.tk_bytes / 2);
    a.t1_pad = int32_t(T.t1_bytes / 2);
    a.acc_out_off = dfa->d_acc_out_off;
    a.acc_out_ids = dfa->d_acc_out_ids;
    a.acc_outcnt = dfa->d_acc_outcnt;
    return a;
}

ScanPlan plan_for(const ks_ctx* ctx, const ks_dfa* dfa, const DevTable& T) {
    ScanPlan p;
    const int32_t A = T.n_accept;
    if (T.fast_k > 0 && dfa->tables_in_smem &&
        fast_smem_bytes(kModeCount, int32_t(T.t1z_bytes / 2), A, fast_threads()) + 256 <= ctx->smem_optin) {
        p.fast = true;  // the fast kernel keeps its visit histogram in shared memory
        p.hist_smem = true;
        return p;
    }
    const size_t tables = dfa->tables_in_smem ? T.tk_bytes + T.t1_bytes : 0;
    p.hist_smem = tables + size_t(A) * 4 + 1024 <= ctx->smem_optin;
    return p;
}

// Lane chunks are the sequence's units (64 << lb bases, see SeqView): chunk c
// of a scan over [begin, end) is unit begin / S + c, clipped to the range.
void geometry(const ks_seq* seq, int64_t begin, int64_t end, int64_t* origin, int64_t* L, int64_t* nch) {
    const int64_t S = int64_t(64) << seq->lb;
    const int64_t u0 = begin / S;
    *origin = u0 * S;
    *L = S;
    *nch = end > begin ? (end - 1) / S - u0 + 1 : 0;
}

int dispatch(ks_ctx* ctx, const ks_dfa* dfa, const DevTable& T, const ScanPlan& p, ScanArgs a, int mode,
             int* launches) {
    if (dfa->host.wide) return launch_scan_wide(ctx, a, mode, launches);
    a.hist_smem = p.hist_smem ? 1 : 0;
    if (p.fast) {
        a.tk = T.tkc;
        a.t1 = T.t1z;
        a.t1_pad = int32_t(T.t1z_bytes / 2);
        a.t1_cols = T.t1z_cols;
        // rare hits (expected < 5% of warp-blocks): scan blocks without hit
        // bookkeeping, re-run the few that hit (KS_LEAN=0/1 overrides)
        a.lean = T.hit_rate * 64.0 * 32.0 < 0.05 ? 1 : 0;
        if (const char* e = std::getenv("KS_LEAN"); e && *e) a.lean = std::atoi(e) != 0;
        // a fused K = 2 count takes the visit-class table when it has one
        // and its histogram fits beside the tables (KS_NO_CLS=1: the ring)
        if (mode == kModeCount && T.fast_k == 2 && !a.lean && a.fin_counts && &T == &dfa->scan && T.cls_rows > 0 &&
            dfa->d_cls_visits && !env_flag("KS_NO_CLS") &&
            fast_fixed_bytes(int32_t(T.cls_t1_bytes / 2), T.cls_nhist) + 256 + 1024 <= ctx->smem_optin) {   // + the class kernel's window shift
            a.cls = 1;
            a.tk = T.cls_tk;
            a.t1 = T.cls_t1;
            a.t1_pad = int32_t(T.cls_t1_bytes / 2);
            a.visits = dfa->d_cls_visits;
            a.acc_out_off = T.cls_out_off;
            a.acc_out_ids = T.cls_out_ids;
            a.n_hist = T.cls_nhist;
            a.cls_prim = T.cls_prim;
            a.cls_used = T.cls_used;
            a.n_used = T.cls_nused;
        }
        return launch_scan_fast(ctx, a, mode, T.fast_k, launches);
    }
    return launch_scan(ctx, a, mode, T.stride, dfa->tables_in_smem, launches);
}

// Map pass + single-pass monoid scan over [begin, end): the entry state of
// every chunk into centry (if not null; the range starts in entry_val >= 0
// or *entry_ptr) and the product of all chunk elements into *d_total.
int monoid_prefix(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                  int64_t origin, int64_t L, int64_t nch, uint16_t* elems, uint16_t* centry, int32_t entry_val,
                  const uint16_t* entry_ptr, uint16_t* d_total, int* launches, PhaseTrace* trace) {
    const HostDfa& h = dfa->host;
    ScanArgs m = base_args(dfa, dfa->mono, seq);
    m.begin = begin;
    m.end = end;
    m.origin = origin;
    m.chunk_len = L;
    m.nchunks = nch;
    m.uniform_entry = 0;  // identity element
    m.n_accept = 0;
    m.chunk_exit = elems;
    if (h.mono_sub) m.map_dirty = dfa->d_prod + size_t(h.mono_other) * h.nm;
    int rc = dispatch(ctx, dfa, dfa->mono, plan_for(ctx, dfa, dfa->mono), m, kModeMap, launches);
    if (rc != KS_OK) return rc;
    if (trace) trace->mark("map pass");
    const size_t window = size_t(reinterpret_cast<const char*>(dfa->d_action + size_t(h.nm) * h.nq) -
                                 reinterpret_cast<const char*>(dfa->d_prod));
    rc = monoid_scan_entries(ctx, elems, nch, dfa->d_prod, h.nm, dfa->d_action, h.nq, entry_val, entry_ptr, centry,
                             d_total, window, launches);
    if (trace) trace->mark("monoid scan");
    return rc;
}

// True internal state of the sequence at position pos (state after pos bases).
// SPECULATE entries of every chunk of [begin, end) (spec.cu), map memory in
// ctx->spec_buf (grow-only, <= 256 MiB per segment of chunks).
int spec_entries(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end, int64_t origin,
                 int64_t L, int64_t nch, int32_t entry_val, const uint16_t* entry_ptr, uint16_t* centry,
                 uint16_t* d_exit, int* launches) {
    const HostDfa& h = dfa->host;
    const int64_t per_chunk = int64_t(h.pss_max) * 2 + 4;
    const int64_t seg = std::max<int64_t>(1, std::min<int64_t>(nch, (int64_t(256) << 20) / per_chunk));
    const size_t bytes = speculate_entries_bytes(seg, h.pss_max) + 64 * kAlign;
    if (ctx->spec_bytes < bytes) {
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->spec_buf) KS_CUDA(cudaFree(ctx->spec_buf));
        ctx->spec_buf = nullptr;
        ctx->spec_bytes = 0;
        KS_CUDA(cudaMalloc(&ctx->spec_buf, bytes));
        ctx->spec_bytes = bytes;
    }
    return speculate_entries(ctx, view_of(seq), begin, end, origin, L, nch, dfa->scan.t1, h.nq, dfa->d_pss,
                             dfa->d_pss_off, dfa->d_pss_inv, h.pss_max, entry_val, entry_ptr, centry, d_exit,
                             ctx->spec_buf, seg, launches);
}

int true_state_at(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t pos, int* out,
                  int* launches) {
    const HostDfa& h = dfa->host;
    if (pos == 0) {
        *out = h.start_internal;
        return KS_OK;
    }
    Arena ar;
    if (h.strategy == KS_STRATEGY_LOOKBACK) {
        int rc = ensure_scratch(ctx, 4096, &ar);
        if (rc) return rc;
        uint32_t* d = static_cast<uint32_t*>(ar.take(16));
        const int64_t lb = std::max<int64_t>(0, pos - h.sync_depth);
        rc = launch_walk(ctx, dfa, seq, lb, pos, 1, h.start_internal, d);
        if (rc) return rc;
        if (launches) ++*launches;
        uint32_t v = 0;
        KS_CUDA(cudaMemcpyAsync(&v, d, 4, cudaMemcpyDeviceToHost, ctx->stream));
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = int(v);
        return KS_OK;
    }
    int64_t origin, L, nch;
    geometry(seq, 0, pos, &origin, &L, &nch);
    if (h.strategy == KS_STRATEGY_SPECULATE) {
        int rc = ensure_scratch(ctx, size_t(nch) * 2 + 4096, &ar);
        if (rc) return rc;
        uint16_t* centry = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
        uint16_t* d = static_cast<uint16_t*>(ar.take(16));
        rc = spec_entries(ctx, dfa, seq, 0, pos, origin, L, nch, h.start_internal, nullptr, centry, d, launches);
        if (rc) return rc;
        uint16_t v = 0;
        KS_CUDA(cudaMemcpyAsync(&v, d, 2, cudaMemcpyDeviceToHost, ctx->stream));
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = v;
        return KS_OK;
    }
    int rc = ensure_scratch(ctx, size_t(nch) * 4 + 4096, &ar);
    if (rc) return rc;
    uint16_t* elems = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
    uint16_t* tot = static_cast<uint16_t*>(ar.take(16));
    rc = monoid_prefix(ctx, dfa, seq, 0, pos, origin, L, nch, elems, nullptr, 0, nullptr, tot, launches);
    if (rc) return rc;
    uint16_t m = 0;
    KS_CUDA(cudaMemcpyAsync(&m, tot, 2, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = h.act0[m];
    return KS_OK;
}

int scan_impl(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
              int32_t entry_orig, int64_t row_base, int64_t* counts_out, int32_t* exit_out,
              int64_t** rows_out, int64_t* n_rows, int64_t* async_dst = nullptr) {
    if (!ctx || !dfa || !seq) return fail(KS_E_INVALID, "null handle");
    if (dfa->ctx != ctx || seq->ctx != ctx) return fail(KS_E_INVALID, "handle belongs to another context");
    const HostDfa& h = dfa->host;
    if (begin < 0 || end < begin || end > seq->n) return fail(KS_E_INVALID, "scan range out of bounds");
    if (entry_orig < -1 || entry_orig >= h.nq) return fail(KS_E_INVALID, "entry state out of range");
    const bool locate = rows_out != nullptr;
    if (locate && !n_rows) return fail(KS_E_INVALID, "n_rows is required with rows_out");
    DeviceGuard guard(ctx->device);
    ctx->stats = ks_stats{};
    int launches = 0;
    // async counts record no timing events unless KS_ASYNC_EVENTS=1: event
    // records between back-to-back scans cost ~2% of a C3 step and keep the
    // next scan from launching early (programmatic dependent launch)
    const bool timed = !async_dst || env_flag("KS_ASYNC_EVENTS");
    if (timed) KS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));

    int entry = entry_orig >= 0 ? h.new_of_old[entry_orig] : -1;
    if (entry < 0 && h.strategy != KS_STRATEGY_LOOKBACK) {
        int rc = true_state_at(ctx, dfa, seq, begin, &entry, &launches);
        if (rc) return rc;
    }

    int64_t origin, L, nch;
    const ScanPlan plan = plan_for(ctx, dfa, dfa->scan);
    geometry(seq, begin, end, &origin, &L, &nch);
    if (end == begin) nch = 0;

    const bool mapscan = h.strategy == KS_STRATEGY_MAPSCAN;
    const bool spec = h.strategy == KS_STRATEGY_SPECULATE;
    size_t need = size_t(h.n_accept) * 8 + size_t(std::max(h.ne, 1)) * 8 + size_t(nch) * 2 + 4096;
    if (locate) need += size_t(nch) * 4 + size_t(nch + 1) * 8 + exclusive_scan_rows_tmp_bytes(nch) + 8 * kAlign;
    if (mapscan) need += size_t(nch) * 6 + 4 * kAlign;
    if (spec) need += size_t(nch) * 2 + 2 * kAlign;
    Arena ar;
    int rc = ensure_scratch(ctx, need, &ar);
    if (rc) return rc;
    // visits | counts | err | exit: one memset before, one D2H after -- or,
    // for a plain count on the fast kernel (the last CTA finalizes), the
    // dfa's persistent block (kept zero by the kernel) and results written
    // by the kernel straight into pinned host memory
    const size_t res_bytes = size_t(std::max(h.ne, 1)) * 8 + 16;
    const bool fused = !locate && plan.fast && nch > 0;
    char* scratch_blk = static_cast<char*>(ar.take(size_t(h.n_accept) * 8 + res_bytes));
    char* blk = fused ? static_cast<char*>(dfa->d_cnt) : scratch_blk;
    char* direct = nullptr;   // pinned host destination the kernel writes (counts | err | exit)
    if (fused && !env_flag("KS_NO_DIRECT_RESULTS")) {
        if (!async_dst) {
            rc = ensure_pinned(ctx, res_bytes + 64);
            if (rc) return rc;
        }
        char* host = async_dst ? reinterpret_cast<char*>(async_dst) : static_cast<char*>(ctx->pinned);
        if (host_is_device_visible(host)) direct = host;
    }
    unsigned long long* visits = reinterpret_cast<unsigned long long*>(blk);
    unsigned long long* counts = reinterpret_cast<unsigned long long*>(blk + size_t(h.n_accept) * 8);
    int32_t* err = reinterpret_cast<int32_t*>(counts + std::max(h.ne, 1));
    uint16_t* exit_slot = reinterpret_cast<uint16_t*>(err + 2);   // uint32 for wide automata
    void* exit_region = ar.take(size_t(nch) * 4 + 4);
    uint16_t* chunk_exit = static_cast<uint16_t*>(exit_region);
    uint32_t* chunk_rows = nullptr;
    int64_t* row_off = nullptr;
    void* rows_tmp = nullptr;
    if (locate) {
        chunk_rows = static_cast<uint32_t*>(ar.take(size_t(nch) * 4));
        row_off = static_cast<int64_t*>(ar.take(size_t(nch + 1) * 8));
        rows_tmp = ar.take(exclusive_scan_rows_tmp_bytes(nch));
    }
    uint16_t *elems = nullptr, *centry = nullptr, *mtot = nullptr;
    if (mapscan) {
        elems = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
        centry = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
        mtot = static_cast<uint16_t*>(ar.take(16));
    }
    if (spec) centry = static_cast<uint16_t*>(ar.take(size_t(nch) * 2));
    if (!fused) KS_CUDA(cudaMemsetAsync(blk, 0, size_t(h.n_accept) * 8 + res_bytes, ctx->stream));
    if (direct && !async_dst) *reinterpret_cast<int32_t*>(direct + size_t(std::max(h.ne, 1)) * 8) = 0;   // err word

    ScanArgs a = base_args(dfa, dfa->scan, seq);
    a.begin = begin;
    a.end = end;
    a.origin = origin;
    a.chunk_len = L;
    a.nchunks = nch;
    a.visits = visits;
    a.chunk_exit = h.wide ? nullptr : chunk_exit;
    a.chunk_exit32 = h.wide ? static_cast<uint32_t*>(exit_region) : nullptr;
    a.error = err;
    a.row_base = row_base;
    if (h.strategy == KS_STRATEGY_LOOKBACK) {
        a.lookback = h.sync_depth;
        a.base_pos = entry >= 0 ? begin : 0;
        a.base_state = entry >= 0 ? entry : h.start_internal;
        a.any_state = h.start_internal;
    }

    cudaEvent_t ev_a = ctx->ev[1], ev_b = ctx->ev[2];
    if (async_dst && timed) {  // count-only, no host synchronisation: events per call
        const size_t need_ev = size_t(2 * (ctx->n_async + 1));
        while (ctx->aev.size() < need_ev) {
            cudaEvent_t e;
            KS_CUDA(cudaEventCreate(&e));
            ctx->aev.push_back(e);
        }
        ev_a = ctx->aev[2 * ctx->n_async];
        ev_b = ctx->aev[2 * ctx->n_async + 1];
        ++ctx->n_async;
    }
    if (async_dst) ++ctx->async_calls;
    if (timed) KS_CUDA(cudaEventRecord(ev_a, ctx->stream));
    PhaseTrace trace(ctx->stream);
    trace.mark("start");
    if (mapscan && nch > 0) {
        rc = monoid_prefix(ctx, dfa, seq, begin, end, origin, L, nch, elems, centry, entry, nullptr, mtot, &launches,
                           &trace);
        if (rc) return rc;
        trace.mark("chunk_entry");
        a.chunk_entry = centry;
    }
    if (spec && nch > 0) {
        rc = spec_entries(ctx, dfa, seq, begin, end, origin, L, nch, entry, nullptr, centry, nullptr, &launches);
        if (rc) return rc;
        a.chunk_entry = centry;
    }
    if (locate) a.chunk_rows = chunk_rows;
    // locate on the fast kernel: one pass that logs every accepting visit
    // (position, chunk, rank inside the chunk); rows are scattered from the
    // log once the chunk offsets are known.  A log overflow falls back to the
    // two-pass form (row counts, then an emitting re-scan).
    const int64_t cap = std::max<int64_t>(int64_t(1) << 16, std::min<int64_t>((end - begin) / 64, int64_t(4) << 20));
    // hit-dense automata (expected visits beyond the log) go straight to two passes
    const bool use_log = locate && plan.fast && nch > 0 && dfa->scan.hit_rate * double(end - begin) < 0.5 * double(cap);
    unsigned long long* log_n = nullptr;
    if (use_log) {
        const size_t bytes = size_t(cap) * sizeof(LogEntry) + 64 + 4096 * 4;   // entries | total | per-CTA counts
        if (ctx->log_bytes < bytes) {
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
            if (ctx->log_buf) KS_CUDA(cudaFree(ctx->log_buf));
            ctx->log_buf = nullptr;
            ctx->log_bytes = 0;
            KS_CUDA(cudaMalloc(&ctx->log_buf, bytes));
            ctx->log_bytes = bytes;
        }
        log_n = reinterpret_cast<unsigned long long*>(static_cast<char*>(ctx->log_buf) + size_t(cap) * sizeof(LogEntry));
        KS_CUDA(cudaMemsetAsync(log_n, 0, 8, ctx->stream));
        a.log = static_cast<LogEntry*>(ctx->log_buf);
        a.log_n = log_n;
        a.log_cta_n = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(log_n) + 64);
        a.log_cap = cap;
    }
    // plain counts on the fast kernel: its last CTA finalizes (one launch per call)
    if (fused) {
        a.fin_counts = counts;
        a.fin_exit_src = chunk_exit + (nch - 1);
        a.fin_exit_dst = direct && !async_dst
                             ? reinterpret_cast<uint16_t*>(direct + size_t(std::max(h.ne, 1)) * 8 + 8)
                             : exit_slot;
        a.fin_done = reinterpret_cast<unsigned int*>(err + 1);   // zero between calls
        a.dyn_items = 1;   // fused: the finalizing CTA resets the dynamic-item counters
        a.fin_host = reinterpret_cast<unsigned long long*>(direct);
        a.n_expr = h.ne;
    }
    rc = dispatch(ctx, dfa, dfa->scan, plan, a, use_log ? kModeLog : locate ? kModeRows : kModeCount, &launches);
    if (rc) return rc;
    trace.mark("scan");
    if (timed) KS_CUDA(cudaEventRecord(ev_b, ctx->stream));
    if (!fused) {
        rc = launch_finalize_counts(ctx, visits, h.n_accept, dfa->d_acc_out_off, dfa->d_acc_out_ids, counts,
                                    nch > 0 && !h.wide ? chunk_exit + (nch - 1) : nullptr, exit_slot, &launches);
        if (rc) return rc;
        if (h.wide && nch > 0)
            KS_CUDA(cudaMemcpyAsync(exit_slot, a.chunk_exit32 + (nch - 1), 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (async_dst) {
        if (h.ne > 0 && !direct)
            KS_CUDA(cudaMemcpyAsync(async_dst, counts, size_t(h.ne) * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->async_launches += launches;
        return KS_OK;
    }

    int64_t total_rows = 0;
    int64_t* d_rows = nullptr;
    // single round trip: rows scattered straight into pinned host staging
    // (bounded by log capacity x max outputs per state), totals and counts
    // copied back, one synchronisation; an overflowed log falls through to the
    // two-pass form below
    if (locate && nch > 0 && use_log) {
        const size_t cap_bytes = size_t(a.log_cap) * size_t(std::max(h.max_outcnt, 1)) * 16;
        bool staged = cap_bytes <= (size_t(256) << 20) && !env_flag("KS_LOCATE_TWO_SYNC");
        if (staged && ctx->rstage_bytes < cap_bytes) {
            if (ctx->rstage) KS_CUDA(cudaFreeHost(ctx->rstage));
            ctx->rstage = nullptr;
            ctx->rstage_bytes = 0;
            staged = cudaMallocHost(&ctx->rstage, cap_bytes) == cudaSuccess;
            if (staged) ctx->rstage_bytes = cap_bytes;
            else cudaGetLastError();
        }
        if (staged && ctx->rdev_bytes < cap_bytes) {
            if (ctx->rdev) KS_CUDA(cudaFree(ctx->rdev));
            ctx->rdev = nullptr;
            ctx->rdev_bytes = 0;
            staged = cudaMalloc(&ctx->rdev, cap_bytes) == cudaSuccess;
            if (staged) ctx->rdev_bytes = cap_bytes;
            else cudaGetLastError();
        }
        staged = staged && host_is_device_visible(ctx->rstage);
        if (staged) {
            rc = exclusive_scan_rows(ctx, chunk_rows, nch, row_off, row_off + nch, rows_tmp, &launches);
            if (rc) return rc;
            rc = launch_log_scatter(ctx, a.log, a.log_cta_n, ctx->log_segs, ctx->log_part, log_n, a.log_cap, row_off,
                                    dfa->d_acc_out_off, dfa->d_acc_out_ids, static_cast<int64_t*>(ctx->rdev),
                                    &launches);
            if (rc) return rc;
            rc = ensure_pinned(ctx, size_t(std::max(h.ne, 1)) * 8 + 64 + 16);
            if (rc) return rc;
            char* pin = static_cast<char*>(ctx->pinned);
            int64_t* tot = reinterpret_cast<int64_t*>(pin + size_t(std::max(h.ne, 1)) * 8 + 32);
            // rows [0, total) -> pinned host memory, coalesced (the total is read
            // on the device); the same kernel writes counts | err | exit, the
            // row total and the log total there (no copy operations to wait on)
            const bool dev_visible = host_is_device_visible(pin);
            copy_rows_kernel<<<std::max(1, std::min(ctx->num_sms * 4, int((a.log_cap + 255) / 256))), 256, 0,
                               ctx->stream>>>(static_cast<const longlong2*>(ctx->rdev), row_off + nch,
                                              static_cast<longlong2*>(ctx->rstage),
                                              dev_visible ? reinterpret_cast<const unsigned int*>(counts) : nullptr,
                                              uint32_t(res_bytes / 4), reinterpret_cast<unsigned int*>(pin), log_n,
                                              tot);
            KS_CUDA(cudaGetLastError());
            ++launches;
            trace.mark("rows (staged)");
            if (!dev_visible) {
                KS_CUDA(cudaMemcpyAsync(pin, counts, res_bytes, cudaMemcpyDeviceToHost, ctx->stream));
                KS_CUDA(cudaMemcpyAsync(tot, row_off + nch, 8, cudaMemcpyDeviceToHost, ctx->stream));
                KS_CUDA(cudaMemcpyAsync(tot + 1, log_n, 8, cudaMemcpyDeviceToHost, ctx->stream));
            }
            KS_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
            trace.mark("sync");
            if (uint64_t(tot[1]) <= uint64_t(a.log_cap)) {
                total_rows = tot[0];
                if (*reinterpret_cast<int32_t*>(pin + size_t(std::max(h.ne, 1)) * 8))
                    return fail(KS_E_CHAIN, "internal invariant failed: chunk row count mismatch");
                int64_t* host_rows = static_cast<int64_t*>(std::malloc(size_t(std::max<int64_t>(total_rows, 1)) * 16));
                if (!host_rows) return fail(KS_E_NOMEM, "host allocation of match rows failed");
                std::memcpy(host_rows, ctx->rstage, size_t(total_rows) * 16);
                std::memcpy(counts_out, pin, size_t(h.ne) * 8);
                if (exit_out) {
                    const uint16_t* pin_exit = reinterpret_cast<const uint16_t*>(pin + size_t(std::max(h.ne, 1)) * 8 + 8);
                    *exit_out = h.old_of_new[int(*pin_exit)];
                }
                *rows_out = host_rows;
                *n_rows = total_rows;
                float ms = 0;
                cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
                ctx->stats.scan_ms = ms;
                cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
                ctx->stats.total_ms = ms;
                ctx->stats.kernel_launches = launches;
                ctx->stats.chunks = int32_t(nch);
                ctx->stats.chunk_len = L;
                ctx->stats.rows = total_rows;
                return KS_OK;
            }
        }
    }
    if (locate && nch > 0) {
        rc = exclusive_scan_rows(ctx, chunk_rows, nch, row_off, row_off + nch, rows_tmp, &launches);
        if (rc) return rc;
        trace.mark("row scan");
        KS_CUDA(cudaMemcpyAsync(&total_rows, row_off + nch, 8, cudaMemcpyDeviceToHost, ctx->stream));
        unsigned long long logged = 0;
        if (use_log) KS_CUDA(cudaMemcpyAsync(&logged, log_n, 8, cudaMemcpyDeviceToHost, ctx->stream));
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        trace.mark("sync totals");
        if (total_rows > 0 && use_log && logged <= (unsigned long long)a.log_cap) {
            KS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_rows), size_t(total_rows) * 16, ctx->stream));
            rc = launch_log_scatter(ctx, a.log, a.log_cta_n, ctx->log_segs, ctx->log_part, log_n, a.log_cap, row_off,
                                    dfa->d_acc_out_off, dfa->d_acc_out_ids, d_rows, &launches);
            if (rc) {
                cudaFreeAsync(d_rows, ctx->stream);
                return rc;
            }
        } else if (total_rows > 0) {
            KS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_rows), size_t(total_rows) * 16, ctx->stream));
            ScanArgs e = a;
            e.log = nullptr;
            e.chunk_rows = nullptr;
            e.chunk_row_off = row_off;
            e.rows = d_rows;
            e.visits = nullptr;
            ScanPlan pe = plan;
            pe.hist_smem = false;
            rc = dispatch(ctx, dfa, dfa->scan, pe, e, kModeEmit, &launches);
            if (rc) {
                cudaFreeAsync(d_rows, ctx->stream);
                return rc;
            }
        }
    }

    trace.mark("rows");
    // results; rows below 32 MiB go through the pinned staging buffer (DMA
    // speed, then one host memcpy), larger ones into the page-locked result
    const size_t rbytes = locate ? size_t(std::max<int64_t>(total_rows, 0)) * 16 : 0;
    const bool stage_rows = rbytes > 0 && rbytes < (size_t(32) << 20);
    const size_t stage_off = (size_t(std::max(h.ne, 1)) * 8 + 64 + 255) & ~size_t(255);
    rc = ensure_pinned(ctx, stage_rows ? stage_off + rbytes : size_t(std::max(h.ne, 1)) * 8 + 64);
    if (rc) {
        if (d_rows) cudaFreeAsync(d_rows, ctx->stream);
        return rc;
    }
    char* pin = static_cast<char*>(ctx->pinned);
    if (!direct) KS_CUDA(cudaMemcpyAsync(pin, counts, res_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    uint16_t* pin_exit = reinterpret_cast<uint16_t*>(pin + size_t(std::max(h.ne, 1)) * 8 + 8);
    int64_t* host_rows = nullptr;
    if (locate) {
        host_rows = static_cast<int64_t*>(std::malloc(size_t(std::max<int64_t>(total_rows, 1)) * 16));
        if (!host_rows) {
            if (d_rows) cudaFreeAsync(d_rows, ctx->stream);
            return fail(KS_E_NOMEM, "host allocation of match rows failed");
        }
        if (total_rows > 0) {
            // large results: page-lock the destination so the copy runs at DMA speed
            bool registered = false;
            if (!stage_rows)
                registered = cudaHostRegister(host_rows, rbytes, cudaHostRegisterDefault) == cudaSuccess;
            cudaError_t ce = cudaMemcpyAsync(stage_rows ? static_cast<void*>(pin + stage_off) : host_rows, d_rows,
                                             rbytes, cudaMemcpyDeviceToHost, ctx->stream);
            if (registered) {
                if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
                cudaHostUnregister(host_rows);
            }
            if (ce != cudaSuccess) {
                std::free(host_rows);
                cudaFreeAsync(d_rows, ctx->stream);
                return cuda_fail(ce, "rows D2H");
            }
        }
        if (d_rows) cudaFreeAsync(d_rows, ctx->stream);
    }
    trace.mark("results D2H");
    KS_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
    cudaError_t se = cudaStreamSynchronize(ctx->stream);
    if (se != cudaSuccess) {
        std::free(host_rows);
        return cuda_fail(se, "scan");
    }
    const int32_t err_flag = *reinterpret_cast<int32_t*>(pin + size_t(std::max(h.ne, 1)) * 8);
    if (err_flag) {
        std::free(host_rows);
        return fail(KS_E_CHAIN, "internal invariant failed: chunk row count mismatch");
    }
    std::memcpy(counts_out, pin, size_t(h.ne) * 8);
    if (stage_rows) std::memcpy(host_rows, pin + stage_off, rbytes);
    if (exit_out) {
        int ex;
        if (nch > 0) ex = h.wide ? int(*reinterpret_cast<uint32_t*>(pin_exit)) : int(*pin_exit);
        else if (entry >= 0) ex = entry;
        else {
            rc = true_state_at(ctx, dfa, seq, begin, &ex, &launches);
            if (rc) {
                std::free(host_rows);
                return rc;
            }
        }
        *exit_out = h.old_of_new[ex];
    }
    if (locate) {
        *rows_out = host_rows;
        *n_rows = total_rows;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]);
    ctx->stats.scan_ms = ms;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
    ctx->stats.total_ms = ms;
    ctx->stats.kernel_launches = launches;
    ctx->stats.chunks = int32_t(nch);
    ctx->stats.chunk_len = L;
    ctx->stats.rows = total_rows;
    return KS_OK;
}

}  // namespace ks

using namespace ks;

extern "C" {

const char* ks_last_error(void) { return g_error.c_str(); }
const char* ks_version(void) { return "kmerscan_b200 0.1 (sm_100a)"; }
void ks_free(void* p) { std::free(p); }

int ks_open(int device, ks_ctx** out) {
    if (!out) return fail(KS_E_INVALID, "out is null");
    int n = 0;
    KS_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(KS_E_INVALID, "no such CUDA device");
    KS_CUDA(cudaSetDevice(device));
    ks_ctx* c = new ks_ctx();
    c->device = device;
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaGetDeviceProperties");
    }
    if (prop.major < 10) {
        delete c;
        return fail(KS_E_UNSUPPORTED, "kmerscan_b200 requires an sm_100 (Blackwell) device");
    }
    c->sms_total = prop.multiProcessorCount;
    c->num_sms = c->sms_total;
    if (const char* r = std::getenv("KS_RESERVE_SMS"); r && *r)
        c->num_sms = std::max(1, c->sms_total - std::max(0, std::atoi(r)));
    c->l2_persist_max = size_t(prop.persistingL2CacheMaxSize);
    c->smem_optin = prop.sharedMemPerBlockOptin;
    e = cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaStreamCreate");
    }
    c->stream = c->own_stream;
    for (auto& ev : c->ev) cudaEventCreate(&ev);
    l2_persist_acquire(device);
    // keep freed stream-ordered allocations (match rows, upload staging) in
    // the pool instead of returning them to the driver at every sync
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = 1ull << 32;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    *out = c;
    return KS_OK;
}

int ks_close(ks_ctx* ctx) {
    if (!ctx) return KS_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);   // before freeing what it reads
    l2_persist_release(ctx);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    if (ctx->sbuf) cudaFree(ctx->sbuf);
    if (ctx->spec_buf) cudaFree(ctx->spec_buf);
    if (ctx->mstat) cudaFree(ctx->mstat);
    if (ctx->rowstat) cudaFree(ctx->rowstat);
    if (ctx->rstage) cudaFreeHost(ctx->rstage);
    if (ctx->rdev) cudaFree(ctx->rdev);
    if (ctx->log_buf) cudaFree(ctx->log_buf);
    if (ctx->wctr) cudaFree(ctx->wctr);
    if (ctx->tctr) cudaFree(ctx->tctr);
    delete ctx->pool;
    if (ctx->hstage) cudaFreeHost(ctx->hstage);
    for (auto& ev : ctx->hev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
    }
    for (auto& ev : ctx->sev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->aev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    return KS_OK;
}

int ks_set_stream(ks_ctx* ctx, void* stream) {
    CtxLock lock_(ctx);
    if (!ctx) return fail(KS_E_INVALID, "null context");
    cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    if (next != ctx->stream) {
        // the context's scratch, result blocks and look-back status words
        // assume one stream: order everything queued on the old stream before
        // any work the new one receives
        DeviceGuard guard(ctx->device);
        KS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
        KS_CUDA(cudaStreamWaitEvent(next, ctx->ev[0], 0));
        ctx->stream = next;
    }
    return KS_OK;
}

int ks_set_reserved_sms(ks_ctx* ctx, int32_t n_sms) {
    CtxLock lock_(ctx);
    if (!ctx) return fail(KS_E_INVALID, "null context");
    if (n_sms < 0 || n_sms >= ctx->sms_total) return fail(KS_E_INVALID, "reserved SMs out of range");
    ctx->num_sms = ctx->sms_total - n_sms;
    return KS_OK;
}

int ks_synchronize(ks_ctx* ctx) {
    CtxLock lock_(ctx);
    if (!ctx) return fail(KS_E_INVALID, "null context");
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    return KS_OK;
}

int ks_get_stats(const ks_ctx* ctx, ks_stats* out) {
    CtxLock lock_(ctx);
    if (!ctx || !out) return fail(KS_E_INVALID, "null argument");
    *out = ctx->stats;
    return KS_OK;
}

int ks_count(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_out) {
    CtxLock lock_(ctx);
    if (!counts_out) return fail(KS_E_INVALID, "counts_out is null");
    return scan_impl(ctx, dfa, seq, 0, seq ? seq->n : 0, -1, 0, counts_out, nullptr, nullptr, nullptr);
}

int ks_locate(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_out, int64_t** rows_out,
              int64_t* n_rows) {
    CtxLock lock_(ctx);
    if (!counts_out || !rows_out || !n_rows) return fail(KS_E_INVALID, "null output");
    return scan_impl(ctx, dfa, seq, 0, seq ? seq->n : 0, -1, 0, counts_out, nullptr, rows_out, n_rows);
}

int ks_count_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_pinned) {
    CtxLock lock_(ctx);
    if (!counts_pinned) return fail(KS_E_INVALID, "counts_pinned is null");
    int64_t dummy = 0;
    return scan_impl(ctx, dfa, seq, 0, seq ? seq->n : 0, -1, 0, &dummy, nullptr, nullptr, nullptr, counts_pinned);
}

int ks_async_wait(ks_ctx* ctx, float* scan_ms_total, int32_t* calls, int32_t* launches) {
    CtxLock lock_(ctx);
    if (!ctx) return fail(KS_E_INVALID, "null context");
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    float total = 0;
    for (int i = 0; i < ctx->n_async; ++i) {
        float ms = 0;
        KS_CUDA(cudaEventElapsedTime(&ms, ctx->aev[2 * i], ctx->aev[2 * i + 1]));
        total += ms;
    }
    if (scan_ms_total) *scan_ms_total = total;
    PhaseTrace::flush();
    if (calls) *calls = ctx->async_calls;
    if (launches) *launches = ctx->async_launches;
    ctx->n_async = 0;
    ctx->async_calls = 0;
    ctx->async_launches = 0;
    return KS_OK;
}

int ks_scan_range(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                  int32_t entry_state, int64_t row_offset_base, int64_t* counts_out, int32_t* exit_state,
                  int64_t** rows_out, int64_t* n_rows) {
    CtxLock lock_(ctx);
    if (!counts_out) return fail(KS_E_INVALID, "counts_out is null");
    return scan_impl(ctx, dfa, seq, begin, end, entry_state, row_offset_base, counts_out, exit_state, rows_out,
                     n_rows);
}

}  // extern "C"
