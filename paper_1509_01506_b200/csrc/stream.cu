// Streamed count straight from host bytes (ks_count_host_bytes and the
// host packers' C-ABI entry points).  The wire formats and the pipeline are
// described on stream_count_impl; DESIGN.md "End-to-end path".
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "runtime.h"

namespace ks {

// Streaming count from a host buffer (ks_count_host_bytes).  Two wire
// formats, both double-buffered on the device, every piece entering in the
// state the previous piece left (a device-resident uint16), visits
// accumulating across pieces:
//  * host pack (raw input without whitespace, the default): host worker
//    threads pack piece i (AVX-512, host_pack.cpp) straight into the
//    tile-slot layout in pinned staging slot i%3; the copy stream moves
//    0.25-0.375 B/base while piece i+1 is packed and piece i-1 scanned.  A
//    piece holding whitespace sets *fallback (positions would shift).
//  * device encode (FASTA, whitespace, or KS_DEVICE_ENCODE=1): raw bytes go
//    over PCIe (1 B/base) into buffer i%2 while the previous piece is
//    encoded -- line state (FASTA headers) carried across pieces on the
//    device -- compacted and scanned.  One host sync per piece reads the
//    piece's retained length for the scan geometry; the next piece's copy is
//    already queued, so the link never idles.
int stream_count_impl(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes, bool fasta,
                      int stream_mode, int64_t* counts_out, bool* fallback) {
    const bool host_pack = stream_mode == kStreamPacked;
    const bool wire = stream_mode == kStreamWire;
    const HostDfa& h = dfa->host;
    *fallback = false;
    // piece size: 64 MiB (inputs below 128 MiB: a quarter of the input, at
    // least 16 MiB, so packing, copy and scan still overlap -- C2 +4%);
    // KS_PIECE_KB overrides (tests use small pieces to cross many boundaries)
    const char* pk = std::getenv("KS_PIECE_KB");
    const int64_t piece_bytes = pk && std::atoll(pk) > 0 ? std::atoll(pk) << 10
                                : n_bytes < (int64_t(128) << 20) ? std::max<int64_t>(int64_t(16) << 20, n_bytes / 4)
                                                                 : int64_t(64) << 20;
    const int64_t piece = std::min<int64_t>(std::max<int64_t>(n_bytes, 64), piece_bytes);
    const int64_t npieces = (n_bytes + piece - 1) / piece;
    ks_seq tmpl;
    tmpl.lb = choose_lb(ctx, piece);
    const int64_t tile_blocks = int64_t(32) << tmpl.lb;
    const int64_t blocks = (piece + 63) / 64;
    const int64_t slots = ((blocks + tile_blocks - 1) / tile_blocks + 1) * tile_blocks;
    const int64_t ntiles = slots / tile_blocks;
    // device input region per buffer: the compacted OTHER bitmaps + their tile
    // ids (host pack) or the raw bytes (device encode)
    // host pack with pinned input also ships every raw_every-th piece raw
    // (1 B/base over PCIe, encoded on the device): the link then carries what
    // the host's memory bandwidth cannot pack (KS_RAW_EVERY, 0 = off)
    int raw_every = 0;
    if (host_pack) {
        cudaPointerAttributes pa{};
        const bool pinned_in = cudaPointerGetAttributes(&pa, bytes) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        const char* re = std::getenv("KS_RAW_EVERY");
        raw_every = pinned_in ? (re && *re ? std::atoi(re) : 6) : 0;   // measured: 6 best (C3 e2e +6%)
    }
    auto raw_piece = [&](int64_t i) { return raw_every > 0 && (i % raw_every) == raw_every - 2; };
    const size_t in_bytes = host_pack ? up(std::max(size_t(slots) * 8 + size_t(ntiles) * 4 + 64,
                                                    raw_every > 0 ? size_t(piece) + 64 : size_t(0)))
                            : wire ? up(size_t(blocks) * 24 + 64)   // linear codes + special masks
                                   : up(size_t(piece) + 64);
    const size_t seq_bytes = up(size_t(slots) * 32);
    const size_t need = 2 * (in_bytes + seq_bytes);
    if (ctx->sbuf_bytes < need) {
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->sbuf) KS_CUDA(cudaFree(ctx->sbuf));
        ctx->sbuf = nullptr;
        ctx->sbuf_bytes = 0;
        KS_CUDA(cudaMalloc(&ctx->sbuf, need));
        ctx->sbuf_bytes = need;
    }
    if (!ctx->copy_stream) {
        KS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (auto& e : ctx->sev) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        for (auto& e : ctx->hev) KS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // staging slot: bases (16 B per block slot), compacted OTHER bitmaps (<= 8 B per slot), tile ids
    const size_t stage = wire ? up(size_t(blocks) * 24) : up(size_t(slots) * 24 + size_t(ntiles) * 4);
    if (host_pack || wire) {
        if (ctx->hstage_bytes < 3 * stage) {
            KS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
            if (ctx->hstage) KS_CUDA(cudaFreeHost(ctx->hstage));
            ctx->hstage = nullptr;
            ctx->hstage_bytes = 0;
            KS_CUDA(cudaMallocHost(&ctx->hstage, 3 * stage));
            ctx->hstage_bytes = 3 * stage;
        }
        if (!ctx->pool) ctx->pool = new HostPool(host_pack_threads());
    }
    uint8_t* din[2];
    ks_seq pseq[2];
    for (int b = 0; b < 2; ++b) {
        char* base = static_cast<char*>(ctx->sbuf) + b * (in_bytes + seq_bytes);
        din[b] = reinterpret_cast<uint8_t*>(base);
        pseq[b].ctx = ctx;
        pseq[b].lb = tmpl.lb;
        pseq[b].n_blocks = slots;
        pseq[b].d_bases = reinterpret_cast<uint64_t*>(base + in_bytes);
        pseq[b].d_nmask = reinterpret_cast<uint64_t*>(base + in_bytes + size_t(slots) * 16);
        pseq[b].d_soft = reinterpret_cast<uint64_t*>(base + in_bytes + size_t(slots) * 24);
    }
    int64_t origin, L, nch_max;
    geometry(&pseq[0], 0, piece, &origin, &L, &nch_max);
    const bool mapscan = h.strategy == KS_STRATEGY_MAPSCAN;
    const bool spec = h.strategy == KS_STRATEGY_SPECULATE;
    Arena ar;
    size_t scratch = size_t(h.n_accept) * 8 + size_t(std::max(h.ne, 1)) * 8 + size_t(nch_max) * 2 + 16 * kAlign;
    if (mapscan) scratch += size_t(nch_max) * 6 + 4 * kAlign;
    if (spec) scratch += size_t(nch_max) * 2 + 2 * kAlign;
    if (stream_mode == kStreamDevice) scratch += encode_scratch_bytes(piece) + 2 * kAlign;
    if (wire) scratch += size_t(blocks + 1) * 12 + exclusive_scan_rows_tmp_bytes(blocks + 1) + 4 * kAlign;
    if (raw_every > 0) scratch += size_t(blocks + 1) * 4 + 2 * kAlign;
    int rc = ensure_scratch(ctx, scratch, &ar);
    if (rc) return rc;
    unsigned long long* visits = static_cast<unsigned long long*>(ar.take(size_t(h.n_accept) * 8));
    unsigned long long* counts = static_cast<unsigned long long*>(ar.take(size_t(std::max(h.ne, 1)) * 8));
    uint16_t* chunk_exit = static_cast<uint16_t*>(ar.take(size_t(nch_max) * 2 + 2));
    uint16_t* state = static_cast<uint16_t*>(ar.take(16));
    int* d_carry = static_cast<int*>(ar.take(16));           // FASTA line state between pieces
    int64_t* d_total = static_cast<int64_t*>(ar.take(16));   // retained symbols of the piece
    void* enc_scratch = stream_mode == kStreamDevice ? ar.take(encode_scratch_bytes(piece)) : nullptr;
    uint32_t* w_kept = wire ? static_cast<uint32_t*>(ar.take(size_t(blocks + 1) * 4)) : nullptr;
    int64_t* w_pos = wire ? static_cast<int64_t*>(ar.take(size_t(blocks + 1) * 8)) : nullptr;
    void* w_tmp = wire ? ar.take(exclusive_scan_rows_tmp_bytes(blocks + 1)) : nullptr;
    uint32_t* kept = raw_every > 0 ? static_cast<uint32_t*>(ar.take(size_t(blocks + 1) * 4)) : nullptr;
    int* ws_flag = static_cast<int*>(ar.take(16));           // raw pieces of the host-pack stream
    uint16_t *elems = nullptr, *centry = nullptr, *mtot = nullptr;
    if (mapscan) {
        elems = static_cast<uint16_t*>(ar.take(size_t(nch_max) * 2));
        centry = static_cast<uint16_t*>(ar.take(size_t(nch_max) * 2));
        mtot = static_cast<uint16_t*>(ar.take(16));
    }
    if (spec) centry = static_cast<uint16_t*>(ar.take(size_t(nch_max) * 2));
    rc = ensure_pinned(ctx, size_t(std::max(h.ne, 1)) * 8 + 64);
    if (rc) return rc;
    char* pin = static_cast<char*>(ctx->pinned);
    int64_t* pin_total = reinterpret_cast<int64_t*>(pin + size_t(std::max(h.ne, 1)) * 8 + 16);
    *reinterpret_cast<uint16_t*>(pin) = uint16_t(h.start_internal);
    if (h.n_accept > 0) KS_CUDA(cudaMemsetAsync(visits, 0, size_t(h.n_accept) * 8, ctx->stream));
    KS_CUDA(cudaMemsetAsync(counts, 0, size_t(std::max(h.ne, 1)) * 8, ctx->stream));
    KS_CUDA(cudaMemsetAsync(d_carry, 0, 16, ctx->stream));
    KS_CUDA(cudaMemsetAsync(ws_flag, 0, 16, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(state, pin, 2, cudaMemcpyHostToDevice, ctx->stream));
    // the copy stream must not overwrite a buffer before the compute stream is done with it
    KS_CUDA(cudaEventRecord(ctx->sev[2], ctx->stream));
    KS_CUDA(cudaEventRecord(ctx->sev[3], ctx->stream));
    const ScanPlan plan = plan_for(ctx, dfa, dfa->scan);
    int launches = 0;
    int64_t h2d = 2;   // the entry state
    int line_state = 0;   // wire mode, FASTA: line state before the next piece (input start = line start)
    int64_t d2h = 0;
    auto issue_raw_copy = [&](int64_t i) -> int {   // device-encode mode: raw piece i -> din[i % 2]
        const int b = int(i & 1);
        const int64_t off = i * piece;
        const int64_t len = std::min(piece, n_bytes - off);
        KS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->sev[2 + b], 0));
        KS_CUDA(cudaMemcpyAsync(din[b], bytes + off, size_t(len), cudaMemcpyHostToDevice, ctx->copy_stream));
        KS_CUDA(cudaEventRecord(ctx->sev[b], ctx->copy_stream));
        h2d += len;
        return KS_OK;
    };
    if (stream_mode == kStreamDevice && npieces > 0) {
        rc = issue_raw_copy(0);
        if (rc) return rc;
    }
    for (int64_t i = 0; i < npieces; ++i) {
        const int b = int(i & 1);
        const int64_t off = i * piece;
        const int64_t len = std::min(piece, n_bytes - off);
        int64_t nsym = len;   // symbols this piece contributes
        if (host_pack && raw_piece(i)) {
            KS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->sev[2 + b], 0));
            KS_CUDA(cudaMemcpyAsync(din[b], bytes + off, size_t(len), cudaMemcpyHostToDevice, ctx->copy_stream));
            KS_CUDA(cudaEventRecord(ctx->sev[b], ctx->copy_stream));
            h2d += len;
            KS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->sev[b], 0));
            rc = encode_raw_piece(ctx, din[b], len, &pseq[b], kept, ws_flag, &launches);
            if (rc) return rc;
        } else if (host_pack) {
            const int st = int(i % 3);
            uint64_t* hb = reinterpret_cast<uint64_t*>(static_cast<char*>(ctx->hstage) + st * stage);
            uint64_t* hn = hb + 2 * slots;
            int32_t* hid = reinterpret_cast<int32_t*>(hn + slots);
            if (i >= 3) KS_CUDA(cudaEventSynchronize(ctx->hev[st]));   // staging slot free again
            const int64_t nt = ((len + 63) / 64 + tile_blocks - 1) / tile_blocks;   // tiles in this piece
            const int64_t used = nt * tile_blocks;
            const int64_t per_task = 4;   // tiles
            std::atomic<int> fl{0};
            std::atomic<int32_t> ncomp{0};
            const uint8_t* src = bytes + off;
            ctx->pool->run((nt + per_task - 1) / per_task, [&](int64_t t) {
                const PackFlags f = pack_ascii_tiles(src, len, t * per_task, std::min(nt, (t + 1) * per_task),
                                                     tmpl.lb, hb, hn, hid, &ncomp);
                if (f.whitespace) fl.fetch_or(1);
            });
            if (fl.load() & 1) {   // whitespace: positions shift, use the compacting path
                KS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
                KS_CUDA(cudaStreamSynchronize(ctx->stream));
                *fallback = true;
                return KS_OK;
            }
            const int nc = ncomp.load();
            uint64_t* d_comp = reinterpret_cast<uint64_t*>(din[b]);
            int32_t* d_ids = reinterpret_cast<int32_t*>(din[b] + size_t(slots) * 8);
            KS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->sev[2 + b], 0));
            KS_CUDA(cudaMemcpyAsync(pseq[b].d_bases, hb, size_t(used) * 16, cudaMemcpyHostToDevice,
                                    ctx->copy_stream));
            KS_CUDA(cudaMemsetAsync(pseq[b].d_nmask, 0, size_t(used) * 8, ctx->copy_stream));
            h2d += used * 16;
            if (nc > 0) {
                KS_CUDA(cudaMemcpyAsync(d_comp, hn, size_t(nc) * tile_blocks * 8, cudaMemcpyHostToDevice,
                                        ctx->copy_stream));
                KS_CUDA(cudaMemcpyAsync(d_ids, hid, size_t(nc) * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d += int64_t(nc) * (tile_blocks * 8 + 4);
            }
            KS_CUDA(cudaEventRecord(ctx->hev[st], ctx->copy_stream));
            KS_CUDA(cudaEventRecord(ctx->sev[b], ctx->copy_stream));
            KS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->sev[b], 0));
            rc = scatter_tile_masks_device(ctx, d_comp, d_ids, nc, int(tile_blocks), pseq[b].d_nmask, &launches);
            if (rc) return rc;
        } else if (wire) {
            const int st = int(i % 3);
            const int64_t nbk = (len + 63) / 64;
            char* sp = static_cast<char*>(ctx->hstage) + st * stage;
            uint64_t* hb = reinterpret_cast<uint64_t*>(sp);
            uint64_t* hs = reinterpret_cast<uint64_t*>(sp + size_t(nbk) * 16);
            if (i >= 3) KS_CUDA(cudaEventSynchronize(ctx->hev[st]));   // staging slot free again
            // 256 KiB of input per task (KS_WIRE_TASK_BLOCKS: tests cut tasks small)
            const char* tb = std::getenv("KS_WIRE_TASK_BLOCKS");
            const int64_t kTaskBlocks = tb && std::atoll(tb) > 0 ? std::atoll(tb) : 4096;
            const int64_t ntask = (nbk + kTaskBlocks - 1) / kTaskBlocks;
            std::vector<WireTask> res(static_cast<size_t>(ntask));
            const uint8_t* src = bytes + off;
            const int first_state = line_state;
            ctx->pool->run(ntask, [&](int64_t t) {
                const int64_t b0 = t * kTaskBlocks, b1 = std::min(nbk, b0 + kTaskBlocks);
                int ss = 1;
                if (fasta) {
                    if (t == 0) ss = first_state;
                    else ss = (src[(b0 << 6) - 1] == '\n' || src[(b0 << 6) - 1] == '\r') ? 0 : -1;
                }
                res[size_t(t)] = pack_wire_task(src, len, b0, b1, fasta, ss, hb, hs);
            });
            // resolve the tasks that assumed "sequence line" at their start
            int64_t kept = 0;
            for (int64_t t = 0; t < ntask; ++t) {
                WireTask& r = res[size_t(t)];
                if (!r.exact && line_state == 2) {
                    const int64_t b0 = t * kTaskBlocks, b1 = std::min(nbk, b0 + kTaskBlocks);
                    wire_drop_prefix(b0, b1, r.first_term, hb, hs);
                    r.kept -= r.prefix_kept;
                }
                kept += r.kept;
                if (r.exact || r.first_term >= 0) line_state = r.end_state;
            }
            const size_t wire_bytes = size_t(nbk) * 24;
            KS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->sev[2 + b], 0));
            KS_CUDA(cudaMemcpyAsync(din[b], sp, wire_bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
            h2d += int64_t(wire_bytes);
            KS_CUDA(cudaEventRecord(ctx->hev[st], ctx->copy_stream));
            KS_CUDA(cudaEventRecord(ctx->sev[b], ctx->copy_stream));
            KS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->sev[b], 0));
            const uint64_t* d_lin = reinterpret_cast<const uint64_t*>(din[b]);
            rc = wire_compact_device(ctx, d_lin, d_lin + 2 * nbk, nbk, &pseq[b], w_kept, w_pos, w_tmp, d_total,
                                     &launches);
            if (rc) return rc;
            nsym = kept;
        } else {
            if (i + 1 < npieces) {   // keep the link busy: the next piece's copy goes first
                rc = issue_raw_copy(i + 1);
                if (rc) return rc;
            }
            KS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->sev[b], 0));
            rc = encode_compact_device(ctx, din[b], len, fasta, d_carry, &pseq[b], enc_scratch, d_total,
                                       &launches);
            if (rc) return rc;
            KS_CUDA(cudaEventRecord(ctx->sev[2 + b], ctx->stream));  // din[b] consumed
            KS_CUDA(cudaMemcpyAsync(pin_total, d_total, 8, cudaMemcpyDeviceToHost, ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));
            d2h += 8;
            nsym = *pin_total;
        }
        pseq[b].n = nsym;
        if (nsym > 0) {
            int64_t o2, L2, nch;
            geometry(&pseq[b], 0, nsym, &o2, &L2, &nch);
            ScanArgs a = base_args(dfa, dfa->scan, &pseq[b]);
            a.begin = 0;
            a.end = nsym;
            a.origin = o2;
            a.chunk_len = L2;
            a.nchunks = nch;
            a.visits = visits;
            a.chunk_exit = chunk_exit;
            if (mapscan) {
                rc = monoid_prefix(ctx, dfa, &pseq[b], 0, nsym, o2, L2, nch, elems, centry, 0, state, mtot, &launches);
                if (rc) return rc;
                a.chunk_entry = centry;
            } else if (spec) {
                rc = spec_entries(ctx, dfa, &pseq[b], 0, nsym, o2, L2, nch, -1, state, centry, nullptr, &launches);
                if (rc) return rc;
                a.chunk_entry = centry;
            } else {
                a.lookback = h.sync_depth;
                a.base_pos = 0;
                a.base_state_ptr = state;
                a.any_state = h.start_internal;
            }
            rc = dispatch(ctx, dfa, dfa->scan, plan, a, kModeCount, &launches);
            if (rc) return rc;
            KS_CUDA(cudaMemcpyAsync(state, chunk_exit + (nch - 1), 2, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if (host_pack || wire) KS_CUDA(cudaEventRecord(ctx->sev[2 + b], ctx->stream));  // device buffer b consumed
    }
    rc = launch_finalize_counts(ctx, visits, h.n_accept, dfa->d_acc_out_off, dfa->d_acc_out_ids, counts,
                                nullptr, nullptr, &launches);
    if (rc) return rc;
    KS_CUDA(cudaMemcpyAsync(pin, counts, size_t(h.ne) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    int* pin_ws = reinterpret_cast<int*>(pin + size_t(std::max(h.ne, 1)) * 8 + 8);
    KS_CUDA(cudaMemcpyAsync(pin_ws, ws_flag, 4, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (*pin_ws) {   // a raw piece held whitespace: redo on the compacting path
        *fallback = true;
        return KS_OK;
    }
    std::memcpy(counts_out, pin, size_t(h.ne) * 8);
    ctx->stats.kernel_launches = launches;
    ctx->stats.h2d_bytes = h2d;
    ctx->stats.d2h_bytes = d2h + int64_t(h.ne) * 8;
    return KS_OK;
}

}  // namespace ks

using namespace ks;

extern "C" {

int ks_pack_host_ascii(const uint8_t* bytes, int64_t n_bytes, int32_t lb, uint64_t* bases, uint64_t* nmask,
                       int32_t* flags) {
    if (n_bytes < 0 || (n_bytes > 0 && (!bytes || !bases || !nmask)) || lb < 0 || lb > 12)
        return fail(KS_E_INVALID, "bad argument");
    const int64_t tb = int64_t(32) << lb;
    const int64_t used = (n_bytes + 63) / 64 + tb - 1 - ((n_bytes + 63) / 64 + tb - 1) % tb;
    const PackFlags f = pack_ascii_blocks(bytes, n_bytes, 0, used, lb, bases, nmask);
    if (flags) *flags = (f.whitespace ? 1 : 0) | (f.other ? 2 : 0);
    return KS_OK;
}

int ks_pack_host_codes(const uint8_t* codes, int64_t n, int32_t lb, uint64_t* bases, uint64_t* nmask) {
    if (n < 0 || (n > 0 && (!codes || !bases || !nmask)) || lb < 0 || lb > 12) return fail(KS_E_INVALID, "bad argument");
    const int64_t tb = int64_t(32) << lb;
    const int64_t used = (n + 63) / 64 + tb - 1 - ((n + 63) / 64 + tb - 1) % tb;
    if (!pack_codes_blocks(codes, n, 0, used, lb, bases, nmask))
        return fail(KS_E_INVALID, "symbol code out of range (expected 0..4)");
    return KS_OK;
}

int ks_pack_host_wire(const uint8_t* bytes, int64_t n_bytes, int32_t fasta, uint64_t* bases, uint64_t* special,
                      int64_t* kept) {
    if (n_bytes < 0 || (n_bytes > 0 && (!bytes || !bases || !special)) || !kept)
        return fail(KS_E_INVALID, "bad argument");
    const WireTask t = pack_wire_task(bytes, n_bytes, 0, (n_bytes + 63) / 64, fasta != 0, 0, bases, special);
    *kept = t.kept;
    return KS_OK;
}

int ks_count_host_bytes(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes, int32_t fasta,
                        int64_t* counts_out) {
    CtxLock lock_(ctx);
    if (!ctx || !dfa || !counts_out || n_bytes < 0 || (n_bytes > 0 && !bytes))
        return fail(KS_E_INVALID, "bad argument");
    if (dfa->ctx != ctx) return fail(KS_E_INVALID, "handle belongs to another context");
    DeviceGuard guard(ctx->device);
    if (n_bytes == 0) {
        std::memset(counts_out, 0, size_t(dfa->host.ne) * 8);
        return KS_OK;
    }
    if (dfa->host.wide) {   // wide automata: one device upload + the plain scan (no streaming form)
        ks_seq* seq = nullptr;
        int rc = ks_seq_upload_ascii(ctx, bytes, n_bytes, fasta, &seq);
        if (rc) return rc;
        rc = ks_count(ctx, dfa, seq, counts_out);
        ks_seq_free(seq);
        return rc;
    }
    ctx->stats = ks_stats{};
    KS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
    bool fallback = false;
    const bool device_encode = std::getenv("KS_DEVICE_ENCODE") != nullptr;
    const int second = device_encode ? kStreamDevice : kStreamWire;   // input with whitespace / FASTA
    const int first = fasta ? second : device_encode ? kStreamDevice : kStreamPacked;
    int rc = stream_count_impl(ctx, dfa, bytes, n_bytes, fasta != 0, first, counts_out, &fallback);
    if (rc) return rc;
    if (fallback) {  // whitespace in raw input: the device-encode stream compacts it
        ctx->stats = ks_stats{};
        KS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
        rc = stream_count_impl(ctx, dfa, bytes, n_bytes, false, second, counts_out, &fallback);
        if (rc) return rc;
    }
    KS_CUDA(cudaEventRecord(ctx->ev[3], ctx->stream));
    KS_CUDA(cudaEventSynchronize(ctx->ev[3]));
    float ms = 0;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
    ctx->stats.total_ms = ms;
    return KS_OK;
}

int ks_count_host_ascii(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes,
                        int64_t* counts_out) {
    CtxLock lock_(ctx);
    return ks_count_host_bytes(ctx, dfa, bytes, n_bytes, 0, counts_out);
}

}  // extern "C"
