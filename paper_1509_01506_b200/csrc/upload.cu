// Upload side of the C ABI (include/kmerscan_b200.h): automata (compiled on
// the host by dfa_compile.cpp into one device blob: stride tables, 1-base
// tables, output CSR, monoid / speculation tables) and sequences (2-bit
// lane-tiled bases + OTHER / soft-mask bitmaps, from codes, host ASCII or
// device bytes through the encode kernels), plus their download helpers.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "runtime.h"

namespace ks {

int upload_table(const CompiledTable& t, DevTable* d, char* blob, size_t* off, bool dry) {
    auto place = [&](const void* src, size_t bytes) -> char* {
        *off = up(*off);
        char* p = blob + *off;
        if (!dry && bytes) std::memcpy(p, src, bytes);
        *off += align16(bytes) + 16;
        return p;
    };
    d->nq = t.nq;
    d->n_accept = t.n_accept;
    d->stride = t.stride;
    d->reset_state = t.reset_state;
    d->tk_bytes = align16(t.tk.size() * 2);
    d->t1_bytes = align16(t.t1.size() * 2);
    d->tk = reinterpret_cast<const uint16_t*>(place(t.tk.data(), t.tk.size() * 2));
    d->t1 = reinterpret_cast<const uint16_t*>(place(t.t1.data(), t.t1.size() * 2));
    if (!t.t1w.empty()) d->t1w = reinterpret_cast<const uint32_t*>(place(t.t1w.data(), t.t1w.size() * 4));
    if (!t.ht.empty()) d->ht = reinterpret_cast<const uint16_t*>(place(t.ht.data(), t.ht.size() * 2));
    d->hot_lo = t.hot_lo;
    d->hot_n = t.ht.empty() ? 0 : t.hot_n;
    d->fast_k = t.fast_k;
    d->hit_rate = t.hit_rate;
    d->t1z_bytes = align16(t.t1z.size() * 2);
    d->t1z_cols = t.t1z_cols;
    if (t.fast_k) {
        d->tkc = reinterpret_cast<const uint16_t*>(place(t.tkc.data(), t.tkc.size() * 2));
        d->t1z = reinterpret_cast<const uint16_t*>(place(t.t1z.data(), t.t1z.size() * 2));
    }
    d->cls_rows = t.cls_rows;
    d->cls_nhist = t.cls_nhist;
    d->cls_t1_bytes = align16(t.cls_t1.size() * 2);
    if (t.cls_rows) {
        d->cls_tk = reinterpret_cast<const uint16_t*>(place(t.cls_tk.data(), t.cls_tk.size() * 2));
        d->cls_t1 = reinterpret_cast<const uint16_t*>(place(t.cls_t1.data(), t.cls_t1.size() * 2));
        d->cls_prim = reinterpret_cast<const uint16_t*>(place(t.cls_prim.data(), t.cls_prim.size() * 2));
        d->cls_out_off = reinterpret_cast<const int32_t*>(place(t.cls_out_off.data(), t.cls_out_off.size() * 4));
        d->cls_out_ids = reinterpret_cast<const int32_t*>(place(t.cls_out_ids.data(), t.cls_out_ids.size() * 4));
        d->cls_used = reinterpret_cast<const int32_t*>(place(t.cls_used.data(), t.cls_used.size() * 4));
        d->cls_nused = int(t.cls_used.size());
    }
    return KS_OK;
}

// Blocks per unit (2^lb): the fast scan gives each warp one tile (32 units)
// at a time, so pick the unit size that minimises (rounds of tiles over the
// SMs' warps, with the CTA size fast_warps_per_cta picks) x (unit length +
// per-unit overhead), i.e. wave quantisation vs entry overhead.
int choose_lb(const ks_ctx* ctx, int64_t n) {
    if (const char* e = std::getenv("KS_TILE_LB"); e && *e) return std::min(6, std::max(0, std::atoi(e)));
    int best = 2;
    double best_cost = 1e300;
    for (int lb = 0; lb <= 6; ++lb) {
        const int64_t tile = int64_t(2048) << lb;
        const int64_t tiles = std::max<int64_t>(1, (n + tile - 1) / tile);
        const int64_t slots = int64_t(ctx->num_sms) * fast_warps_per_cta(tiles, ctx->num_sms);
        const int64_t rounds = (tiles + slots - 1) / slots;
        const double cost = double(rounds) * double((64 << lb) + 128);   // ~128 bases of per-unit overhead
        if (cost <= best_cost) {
            best_cost = cost;
            best = lb;
        }
    }
    return best;
}

int seq_alloc(ks_ctx* ctx, int64_t n_capacity, ks_seq** out) {
    ks_seq* s = new ks_seq();
    s->ctx = ctx;
    s->lb = choose_lb(ctx, n_capacity);
    const int64_t tile_blocks = int64_t(32) << s->lb;
    const int64_t blocks = (n_capacity + 63) / 64;
    s->n_blocks = ((blocks + tile_blocks - 1) / tile_blocks + 1) * tile_blocks;
    const size_t rm_bytes = size_t(s->n_blocks / tile_blocks) * 8;
    const size_t bytes = size_t(s->n_blocks) * 32 + rm_bytes;
    cudaError_t e = cudaMalloc(&s->d_blob, bytes);
    if (e != cudaSuccess) {
        delete s;
        return cuda_fail(e, "cudaMalloc(sequence)");
    }
    char* p = static_cast<char*>(s->d_blob);
    s->d_bases = reinterpret_cast<uint64_t*>(p);
    s->d_nmask = reinterpret_cast<uint64_t*>(p + size_t(s->n_blocks) * 16);
    s->d_soft = reinterpret_cast<uint64_t*>(p + size_t(s->n_blocks) * 24);
    s->d_rowmask = reinterpret_cast<uint64_t*>(p + size_t(s->n_blocks) * 32);
    e = cudaMemsetAsync(s->d_blob, 0, bytes, ctx->stream);
    if (e != cudaSuccess) {
        cudaFree(s->d_blob);
        delete s;
        return cuda_fail(e, "cudaMemset(sequence)");
    }
    *out = s;
    return KS_OK;
}

// Row flags of a finished upload (SeqView::rowmask): one warp per tile ORs
// the 32 lanes' OTHER bitmaps of every block row.
__global__ void seq_rowmask_kernel(const uint64_t* __restrict__ nmask, int64_t n_tiles, int lb,
                                   uint64_t* __restrict__ rowmask) {
    const int64_t t = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (t >= n_tiles) return;
    const int lane = threadIdx.x & 31;
    const uint64_t* p = nmask + (t << (5 + lb)) + lane;
    uint64_t m = 0;
    for (int k = 0; k < (1 << lb); ++k)
        if (__any_sync(0xffffffffu, __ldg(p + 32 * k) != 0ull)) m |= 1ull << k;
    if (lane == 0) rowmask[t] = m;
}

int seq_seal(ks_ctx* ctx, ks_seq* s) {
    if (!s->d_rowmask) return KS_OK;
    const int64_t n_tiles = s->n_blocks >> (5 + s->lb);
    const int threads = 256;
    const int64_t blocks = (n_tiles * 32 + threads - 1) / threads;
    seq_rowmask_kernel<<<unsigned(blocks), threads, 0, ctx->stream>>>(s->d_nmask, n_tiles, s->lb, s->d_rowmask);
    KS_CUDA(cudaGetLastError());
    s->sealed = true;
    return KS_OK;
}

void seq_destroy(ks_seq* s) {
    if (!s) return;
    if (s->d_blob) cudaFree(s->d_blob);
    delete s;
}

}  // namespace ks

using namespace ks;

namespace ks {
// Codes (1 B/symbol, often pageable numpy memory) packed on the host by the
// worker pool into the tile-slot layout (0.375 B/symbol) in the pinned
// staging ring, pieces of whole tiles copied on the copy stream while the
// next piece is packed: a pageable 1 B/symbol copy runs at a fraction of the
// link, the packed wire at the link rate.
int upload_codes_host(ks_ctx* ctx, const uint8_t* codes, int64_t n, ks_seq* s) {
    const int64_t tb = int64_t(32) << s->lb;   // blocks per tile
    const int64_t nb = (n + 63) / 64;
    const int64_t ntiles = (nb + tb - 1) / tb;
    const int64_t tiles_per_piece = std::max<int64_t>(1, (int64_t(64) << 20) / 64 / tb);
    const int64_t piece_slots = tiles_per_piece * tb;
    const size_t stage = up(size_t(piece_slots) * 24);
    if (!ctx->copy_stream) {
        KS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (auto& e : ctx->sev) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->hev) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (ctx->hstage_bytes < 3 * stage) {
        KS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
        if (ctx->hstage) KS_CUDA(cudaFreeHost(ctx->hstage));
        ctx->hstage = nullptr;
        ctx->hstage_bytes = 0;
        KS_CUDA(cudaMallocHost(&ctx->hstage, 3 * stage));
        ctx->hstage_bytes = 3 * stage;
    }
    if (!ctx->pool) ctx->pool = new HostPool(host_pack_threads());
    // the sequence's zeroing memset (seq_alloc, compute stream) precedes the copies
    KS_CUDA(cudaEventRecord(ctx->sev[2], ctx->stream));
    KS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->sev[2], 0));
    std::atomic<int> bad{0};
    const int64_t npieces = (ntiles + tiles_per_piece - 1) / tiles_per_piece;
    for (int64_t p = 0; p < npieces; ++p) {
        const int st = int(p % 3);
        uint64_t* hb = reinterpret_cast<uint64_t*>(static_cast<char*>(ctx->hstage) + st * stage);
        uint64_t* hn = hb + 2 * piece_slots;
        if (p >= 3) KS_CUDA(cudaEventSynchronize(ctx->hev[st]));   // staging slot free again
        const int64_t t0 = p * tiles_per_piece, t1 = std::min(ntiles, t0 + tiles_per_piece);
        const int64_t sbase = t0 * tb;
        constexpr int64_t kTilesPerTask = 4;
        ctx->pool->run((t1 - t0 + kTilesPerTask - 1) / kTilesPerTask, [&](int64_t k) {
            const int64_t a0 = t0 + k * kTilesPerTask, a1 = std::min(t1, a0 + kTilesPerTask);
            if (!pack_codes_blocks(codes, n, a0 * tb, a1 * tb, s->lb, hb, hn, sbase)) bad.store(1);
        });
        const size_t ns = size_t(t1 - t0) * size_t(tb);
        KS_CUDA(cudaMemcpyAsync(s->d_bases + 2 * sbase, hb, ns * 16, cudaMemcpyHostToDevice, ctx->copy_stream));
        KS_CUDA(cudaMemcpyAsync(s->d_nmask + sbase, hn, ns * 8, cudaMemcpyHostToDevice, ctx->copy_stream));
        KS_CUDA(cudaEventRecord(ctx->hev[st], ctx->copy_stream));
    }
    // later work on the compute stream sees the sequence
    KS_CUDA(cudaEventRecord(ctx->sev[2], ctx->copy_stream));
    KS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->sev[2], 0));
    KS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    if (bad.load()) return fail(KS_E_INVALID, "symbol code out of range (expected 0..4)");
    s->n = n;
    return KS_OK;
}

}  // namespace ks

extern "C" {

int ks_dfa_upload_ex(ks_ctx* ctx, const int32_t* transitions, int32_t n_states, const int32_t* out_offsets,
                     const int32_t* out_ids, int32_t n_expressions, int32_t force_strategy, ks_dfa** out) {
    CtxLock lock_(ctx);
    if (!ctx || !out) return fail(KS_E_INVALID, "null argument");
    DeviceGuard guard(ctx->device);
    ks_dfa* d = new ks_dfa();
    d->ctx = ctx;
    const size_t budget = ctx->smem_optin > 2048 ? ctx->smem_optin - 2048 : 0;
    int rc = compile_dfa(transitions, n_states, out_offsets, out_ids, n_expressions, force_strategy, budget,
                         &d->host);
    if (rc != KS_OK) {
        delete d;
        return rc;
    }
    const HostDfa& h = d->host;
    // one blob: tables, CSR, monoid tables
    auto layout = [&](char* blob, bool dry) -> size_t {
        size_t off = 0;
        upload_table(h.scan, &d->scan, blob, &off, dry);
        auto place = [&](const void* src, size_t bytes) -> char* {
            off = up(off);
            char* p = blob + off;
            if (!dry && bytes) std::memcpy(p, src, bytes);
            off += align16(bytes) + 16;
            return p;
        };
        d->d_acc_out_off = reinterpret_cast<int32_t*>(place(h.acc_out_off.data(), h.acc_out_off.size() * 4));
        d->d_acc_out_ids = reinterpret_cast<int32_t*>(place(h.acc_out_ids.data(), h.acc_out_ids.size() * 4));
        d->d_acc_outcnt = reinterpret_cast<uint16_t*>(place(h.acc_outcnt.data(), h.acc_outcnt.size() * 2));
        d->d_new_of_old = reinterpret_cast<int32_t*>(place(h.new_of_old.data(), h.new_of_old.size() * 4));
        d->d_old_of_new = reinterpret_cast<int32_t*>(place(h.old_of_new.data(), h.old_of_new.size() * 4));
        if (h.strategy == KS_STRATEGY_MAPSCAN) {
            upload_table(h.mono, &d->mono, blob, &off, dry);
            d->d_prod = reinterpret_cast<uint16_t*>(place(h.prod.data(), h.prod.size() * 2));
            d->d_act0 = reinterpret_cast<uint16_t*>(place(h.act0.data(), h.act0.size() * 2));
            d->d_action = reinterpret_cast<uint16_t*>(place(h.action.data(), h.action.size() * 2));
        }
        if (h.strategy == KS_STRATEGY_SPECULATE) {
            d->d_pss = reinterpret_cast<uint16_t*>(place(h.pss.data(), h.pss.size() * 2));
            d->d_pss_off = reinterpret_cast<int32_t*>(place(h.pss_off.data(), h.pss_off.size() * 4));
            d->d_pss_inv = reinterpret_cast<int16_t*>(place(h.pss_inv.data(), h.pss_inv.size() * 2));
        }
        return up(off);
    };
    const size_t bytes = layout(nullptr, true);
    std::vector<char> host(bytes, 0);
    layout(host.data(), false);
    cudaError_t e = cudaMalloc(&d->d_blob, bytes);
    if (e != cudaSuccess) {
        delete d;
        return cuda_fail(e, "cudaMalloc(dfa)");
    }
    // on the context's (non-blocking) stream and waited for: a pageable
    // cudaMemcpy may return before its DMA lands, and nothing would order the
    // legacy stream against the kernels that read these tables
    e = cudaMemcpyAsync(d->d_blob, host.data(), bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        cudaFree(d->d_blob);
        delete d;
        return cuda_fail(e, "cudaMemcpy(dfa)");
    }
    // rebase host-blob pointers onto the device blob
    const ptrdiff_t delta = static_cast<char*>(d->d_blob) - host.data();
    auto rebase = [&](auto*& p) {
        using Ptr = std::remove_reference_t<decltype(p)>;
        if (p) p = (Ptr)((const char*)p + delta);
    };
    rebase(d->scan.tk);
    rebase(d->scan.t1);
    rebase(d->scan.t1w);
    rebase(d->scan.ht);
    rebase(d->scan.tkc);
    rebase(d->scan.t1z);
    rebase(d->scan.cls_tk);
    rebase(d->scan.cls_t1);
    rebase(d->scan.cls_prim);
    rebase(d->scan.cls_out_off);
    rebase(d->scan.cls_out_ids);
    rebase(d->scan.cls_used);
    rebase(d->d_acc_out_off);
    rebase(d->d_acc_out_ids);
    rebase(d->d_acc_outcnt);
    rebase(d->d_new_of_old);
    rebase(d->d_old_of_new);
    if (h.strategy == KS_STRATEGY_MAPSCAN) {
        rebase(d->mono.tk);
        rebase(d->mono.t1);
        rebase(d->mono.tkc);
        rebase(d->mono.t1z);
        rebase(d->d_prod);
        rebase(d->d_act0);
        rebase(d->d_action);
    }
    if (h.strategy == KS_STRATEGY_SPECULATE) {
        rebase(d->d_pss);
        rebase(d->d_pss_off);
        rebase(d->d_pss_inv);
    }
    const size_t cnt_bytes = size_t(h.n_accept) * 8 + size_t(std::max(h.ne, 1)) * 8 + 16;
    if (cudaMalloc(&d->d_cnt, cnt_bytes) != cudaSuccess ||
        cudaMemsetAsync(d->d_cnt, 0, cnt_bytes, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        if (d->d_cnt) cudaFree(d->d_cnt);
    if (d->d_cls_visits) cudaFree(d->d_cls_visits);
        cudaFree(d->d_blob);
        delete d;
        return fail(KS_E_CUDA, "cudaMalloc(dfa result block)");
    }
    if (d->scan.cls_rows) {
        const size_t vb = size_t(d->scan.cls_nhist) * 8;
        if (cudaMalloc(&d->d_cls_visits, vb) != cudaSuccess ||
            cudaMemsetAsync(d->d_cls_visits, 0, vb, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
            cudaGetLastError();
            if (d->d_cls_visits) cudaFree(d->d_cls_visits);
            cudaFree(d->d_cnt);
            cudaFree(d->d_blob);
            delete d;
            return fail(KS_E_CUDA, "cudaMalloc(dfa class counters)");
        }
    }
    const size_t smem_scan = d->scan.tk_bytes + d->scan.t1_bytes;
    const size_t smem_mono = h.strategy == KS_STRATEGY_MAPSCAN ? d->mono.tk_bytes + d->mono.t1_bytes : 0;
    d->tables_in_smem = !h.wide && std::max(smem_scan, smem_mono) + 1024 <= ctx->smem_optin;
    if (const char* g = std::getenv("KS_FORCE_GLOBAL_TABLES"); g && *g == '1') d->tables_in_smem = false;
    *out = d;
    return KS_OK;
}

int ks_dfa_upload(ks_ctx* ctx, const int32_t* transitions, int32_t n_states, const int32_t* out_offsets,
                  const int32_t* out_ids, int32_t n_expressions, ks_dfa** out) {
    CtxLock lock_(ctx);
    return ks_dfa_upload_ex(ctx, transitions, n_states, out_offsets, out_ids, n_expressions, 0, out);
}

int ks_dfa_info_get(const ks_dfa* d, ks_dfa_info* out) {
    if (!d || !out) return fail(KS_E_INVALID, "null argument");
    const HostDfa& h = d->host;
    out->n_states = h.nq;
    out->n_expressions = h.ne;
    out->n_accepting = h.n_accept;
    out->strategy = h.strategy;
    out->sync_depth = h.strategy == KS_STRATEGY_LOOKBACK ? h.sync_depth : -1;
    const bool fast = d->scan.fast_k > 0 && d->tables_in_smem;
    out->stride = fast ? d->scan.fast_k : h.scan.stride;
    out->monoid_size = h.strategy == KS_STRATEGY_MAPSCAN ? h.nm : 0;
    out->other_resets = h.scan.reset_state >= 0 ? 1 : 0;
    out->table_bytes = int64_t(d->scan.tk_bytes + d->scan.t1_bytes);
    out->tables_in_smem = d->tables_in_smem ? 1 : 0;
    out->reserved = 0;
    return KS_OK;
}

int ks_dfa_free(ks_dfa* d) {
    CtxLock lock_(d ? d->ctx : nullptr);
    if (!d) return KS_OK;
    DeviceGuard guard(d->ctx->device);
    if (d->d_blob) cudaFree(d->d_blob);
    if (d->d_cnt) cudaFree(d->d_cnt);
    if (d->d_cls_visits) cudaFree(d->d_cls_visits);
    delete d;
    return KS_OK;
}

int ks_seq_upload_codes(ks_ctx* ctx, const uint8_t* codes, int64_t n, ks_seq** out) {
    CtxLock lock_(ctx);
    if (!ctx || !out || n < 0 || (n > 0 && !codes)) return fail(KS_E_INVALID, "bad argument");
    DeviceGuard guard(ctx->device);
    ks_seq* s = nullptr;
    int rc = seq_alloc(ctx, n, &s);
    if (rc) return rc;
    if (n >= (int64_t(8) << 20) && !env_flag("KS_DEVICE_PACK_CODES")) {   // host-packed wire, pipelined
        rc = upload_codes_host(ctx, codes, n, s);
        if (rc) {
            seq_destroy(s);
            return rc;
        }
        if ((rc = seq_seal(ctx, s)) != KS_OK) {
            seq_destroy(s);
            return rc;
        }
        *out = s;
        return KS_OK;
    }
    Arena ar;
    rc = ensure_scratch(ctx, size_t(n) + 1024, &ar);
    if (rc) {
        seq_destroy(s);
        return rc;
    }
    uint8_t* d_codes = static_cast<uint8_t*>(ar.take(size_t((n + 63) / 64 * 64) + 64));
    int* flag = static_cast<int*>(ar.take(16));
    int launches = 0;
    cudaError_t e = cudaMemsetAsync(flag, 0, 16, ctx->stream);
    if (e == cudaSuccess && n > 0) e = cudaMemcpyAsync(d_codes, codes, size_t(n), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) {
        seq_destroy(s);
        return cuda_fail(e, "sequence upload");
    }
    rc = pack_codes_device(ctx, d_codes, n, s, flag, &launches);
    int bad = 0;
    if (rc == KS_OK) {
        e = cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "pack codes");
    }
    if (rc == KS_OK && bad) rc = fail(KS_E_INVALID, "symbol code out of range (expected 0..4)");
    if (rc == KS_OK) rc = seq_seal(ctx, s);
    if (rc) {
        seq_destroy(s);
        return rc;
    }
    *out = s;
    return KS_OK;
}

static int encode_common(ks_ctx* ctx, const uint8_t* d_bytes, int64_t n_bytes, int32_t fasta, ks_seq** out) {
    ks_seq* s = nullptr;
    int rc = seq_alloc(ctx, n_bytes, &s);
    if (rc) return rc;
    Arena ar;
    const size_t staged = d_bytes ? 0 : 0;
    (void)staged;
    rc = ensure_scratch(ctx, encode_scratch_bytes(n_bytes) + 4096, &ar);
    if (rc) {
        seq_destroy(s);
        return rc;
    }
    int launches = 0;
    rc = encode_ascii_device(ctx, d_bytes, n_bytes, fasta != 0, s, ar.take(encode_scratch_bytes(n_bytes)),
                             &launches);
    if (rc == KS_OK) rc = seq_seal(ctx, s);
    if (rc) {
        seq_destroy(s);
        return rc;
    }
    *out = s;
    return KS_OK;
}

int ks_seq_encode_device(ks_ctx* ctx, const uint8_t* d_bytes, int64_t n_bytes, int32_t fasta, ks_seq** out) {
    CtxLock lock_(ctx);
    if (!ctx || !out || n_bytes < 0 || (n_bytes > 0 && !d_bytes)) return fail(KS_E_INVALID, "bad argument");
    DeviceGuard guard(ctx->device);
    return encode_common(ctx, d_bytes, n_bytes, fasta, out);
}

int ks_seq_upload_ascii(ks_ctx* ctx, const uint8_t* bytes, int64_t n_bytes, int32_t fasta, ks_seq** out) {
    CtxLock lock_(ctx);
    if (!ctx || !out || n_bytes < 0 || (n_bytes > 0 && !bytes)) return fail(KS_E_INVALID, "bad argument");
    DeviceGuard guard(ctx->device);
    uint8_t* d_in = nullptr;
    KS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_in), size_t(n_bytes) + 64, ctx->stream));
    cudaError_t e = n_bytes ? cudaMemcpyAsync(d_in, bytes, size_t(n_bytes), cudaMemcpyHostToDevice, ctx->stream)
                            : cudaSuccess;
    int rc = e == cudaSuccess ? encode_common(ctx, d_in, n_bytes, fasta, out) : cuda_fail(e, "ascii upload");
    cudaFreeAsync(d_in, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    return rc;
}

int ks_seq_length(const ks_seq* s, int64_t* n) {
    if (!s || !n) return fail(KS_E_INVALID, "null argument");
    *n = s->n;
    return KS_OK;
}

int ks_seq_download_codes(ks_ctx* ctx, const ks_seq* s, uint8_t* out) {
    CtxLock lock_(ctx);
    if (!ctx || !s || (s->n > 0 && !out)) return fail(KS_E_INVALID, "null argument");
    DeviceGuard guard(ctx->device);
    Arena ar;
    int rc = ensure_scratch(ctx, size_t(s->n) + 256, &ar);
    if (rc) return rc;
    uint8_t* d = static_cast<uint8_t*>(ar.take(size_t(s->n) + 16));
    rc = unpack_codes_device(ctx, s, d);
    if (rc) return rc;
    if (s->n) KS_CUDA(cudaMemcpyAsync(out, d, size_t(s->n), cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    return KS_OK;
}

int ks_seq_download_softmask(ks_ctx* ctx, const ks_seq* s, uint64_t* out, int64_t n_words) {
    CtxLock lock_(ctx);
    if (!ctx || !s || !out) return fail(KS_E_INVALID, "null argument");
    DeviceGuard guard(ctx->device);
    const int64_t have = (s->n + 63) / 64;
    if (n_words < have) return fail(KS_E_INVALID, "softmask buffer too small");
    if (have) {
        Arena ar;
        int rc = ensure_scratch(ctx, size_t(have) * 8 + 256, &ar);
        if (rc) return rc;
        uint64_t* d = static_cast<uint64_t*>(ar.take(size_t(have) * 8));
        rc = linear_softmask_device(ctx, s, d);
        if (rc) return rc;
        KS_CUDA(cudaMemcpyAsync(out, d, size_t(have) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    return KS_OK;
}

int ks_seq_free(ks_seq* s) {
    CtxLock lock_(s ? s->ctx : nullptr);
    if (!s) return KS_OK;
    DeviceGuard guard(s->ctx->device);
    cudaStreamSynchronize(s->ctx->stream);
    seq_destroy(s);
    return KS_OK;
}

}  // extern "C"
