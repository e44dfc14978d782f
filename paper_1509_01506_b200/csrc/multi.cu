// Multi-device contexts: one sequence sharded over several GPUs of one
// process (the reference's run() spreading one call over all its workers,
// engine.py:207-237, lifted to devices).
//
// A ks_mctx owns one ks_ctx (device + stream) per rank and, when the ranks
// are distinct devices, one NCCL communicator per rank (ncclCommInitAll,
// single process; libnccl is loaded at run time, so the library itself has no
// link dependency on it).  A ks_mseq holds rank r's contiguous slice of the
// sequence on its device; slices of a code upload carry the previous
// slice's last kHalo symbols in front (halo), slices of an ASCII upload are
// cut at byte (FASTA: line) boundaries and encoded on their device.
//
// Count step (all enqueued, one host synchronisation at the end):
//   * definite automaton + halo: every rank scans its slice from the halo's
//     lookback (ks_count_shard_async, one fused launch) -> NCCL all-reduce of
//     the uint64 counts;
//   * otherwise: every rank writes its slice's boundary map
//     (ks_segment_map_async) -> NCCL all-gather of the maps -> each rank
//     composes START through the maps of ranks < r on the device and scans
//     from there -> NCCL all-reduce.
// When two ranks share a device (tests on a one-GPU box) or NCCL is absent,
// the same exchanges run as stream-ordered peer copies (cudaMemcpyPeerAsync,
// events between the ranks' streams) and a summing kernel on rank 0.
// Locate: per-rank ks_scan_range with global row offsets; rows concatenated
// in rank order are the globally sorted list.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime.h"

namespace {

// ncclCommInitAll & co, resolved from libnccl.so.2 at run time.
struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
};

Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            n.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (n.lib) break;
        }
        if (!n.lib) return;
        auto sym = [](const char* s) { return dlsym(n.lib, s); };
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
        n.ok = n.CommInitAll && n.CommDestroy && n.AllReduce && n.AllGather && n.GroupStart && n.GroupEnd &&
               n.GetErrorString;
    });
    return &n;
}

int nccl_fail(ncclResult_t r, const char* what) {
    Nccl* n = nccl();
    return ks::fail(KS_E_CUDA, std::string(what) + ": " + (n->GetErrorString ? n->GetErrorString(r) : "nccl error"));
}

#define KS_NCCL(call)                                          \
    do {                                                       \
        ncclResult_t _r = (call);                              \
        if (_r != ncclSuccess) return nccl_fail(_r, #call);    \
    } while (0)

constexpr int64_t kHalo = 2048;   // >= kMaxSyncDepth: covers every definite automaton

// counts[0..ne) = sum over ranks of parts[r][0..ne)
__global__ void sum_parts_kernel(const unsigned long long* __restrict__ parts, int n_parts, int ne,
                                 unsigned long long* __restrict__ out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
        unsigned long long v = 0;
        for (int r = 0; r < n_parts; ++r) v += parts[size_t(r) * ne + e];
        out[e] = v;
    }
}

}  // namespace

struct ks_mctx {
    std::mutex mu;
    std::vector<int> dev;
    std::vector<ks_ctx*> ctx;
    std::vector<ncclComm_t> comm;          // empty: peer-copy transport
    std::vector<cudaEvent_t> ev;           // one per rank (peer-copy ordering)
    // per rank: maps (world x nq int32) and counts (ne uint64); rank 0 also
    // gathers the ranks' counts (world x ne) for the peer-copy transport
    std::vector<void*> buf;
    std::vector<size_t> buf_bytes;
    unsigned long long* gather = nullptr;
    size_t gather_bytes = 0;
    int64_t* host = nullptr;               // pinned result staging
    size_t host_bytes = 0;
};

struct ks_mdfa {
    ks_mctx* m = nullptr;
    std::vector<ks_dfa*> d;
    int nq = 0, ne = 0, strategy = 0, sync_depth = -1;
};

struct ks_mseq {
    ks_mctx* m = nullptr;
    std::vector<ks_seq*> s;
    std::vector<int64_t> base;   // global position of each slice's first symbol
    std::vector<int64_t> halo;   // symbols of the previous slice in front of it
    std::vector<int64_t> len;    // the slice's own symbols
    int64_t n = 0;
};

namespace {

int world(const ks_mctx* m) { return int(m->ctx.size()); }

int ensure_buf(ks_mctx* m, int r, size_t bytes) {
    if (m->buf_bytes[r] >= bytes) return KS_OK;
    ks::DeviceGuard g(m->dev[r]);
    KS_CUDA(cudaStreamSynchronize(m->ctx[r]->stream));
    if (m->buf[r]) KS_CUDA(cudaFree(m->buf[r]));
    m->buf[r] = nullptr;
    m->buf_bytes[r] = 0;
    KS_CUDA(cudaMalloc(&m->buf[r], bytes));
    m->buf_bytes[r] = bytes;
    return KS_OK;
}

int sync_all(ks_mctx* m) {
    for (int r = 0; r < world(m); ++r) {
        ks::DeviceGuard g(m->dev[r]);
        KS_CUDA(cudaStreamSynchronize(m->ctx[r]->stream));
    }
    return KS_OK;
}

// Rank r's stream waits for rank k's stream (peer-copy ordering).
int order_after(ks_mctx* m, int r, int k) {
    {
        ks::DeviceGuard g(m->dev[k]);
        KS_CUDA(cudaEventRecord(m->ev[k], m->ctx[k]->stream));
    }
    ks::DeviceGuard g(m->dev[r]);
    KS_CUDA(cudaStreamWaitEvent(m->ctx[r]->stream, m->ev[k], 0));
    return KS_OK;
}

// Definite automaton and every non-empty slice after the first carries at
// least sync_depth symbols of its predecessor: entry states by lookback.
bool use_halo(const ks_mdfa* d, const ks_mseq* s) {
    if (d->strategy != KS_STRATEGY_LOOKBACK) return false;
    for (size_t r = 1; r < s->halo.size(); ++r)
        if (s->len[r] > 0 && s->halo[r] < std::max(d->sync_depth, 1)) return false;
    return true;
}

// Entry state (original id) of every rank from the slices' boundary maps,
// composed on the host (locate: the rows come back to the host anyway).
int host_entries(ks_mctx* m, const ks_mdfa* d, const ks_mseq* s, std::vector<int32_t>* entry) {
    const int W = world(m);
    entry->assign(size_t(W), 0);
    std::vector<int32_t> map(size_t(d->nq));
    int32_t state = 0;   // START
    for (int r = 0; r < W; ++r) {
        (*entry)[r] = state;
        if (r + 1 == W) break;
        int rc = ks_segment_map(m->ctx[r], d->d[r], s->s[r], s->halo[r], s->halo[r] + s->len[r], map.data());
        if (rc) return rc;
        if (s->len[r] > 0) state = map[size_t(state)];
    }
    return KS_OK;
}

}  // namespace

extern "C" {

int ks_open_multi(int32_t n_dev, const int32_t* dev_ids, ks_mctx** out) {
    using namespace ks;
    if (n_dev < 1 || !dev_ids || !out) return fail(KS_E_INVALID, "ks_open_multi: bad argument");
    ks_mctx* m = new ks_mctx();
    for (int r = 0; r < n_dev; ++r) {
        ks_ctx* c = nullptr;
        int rc = ks_open(dev_ids[r], &c);
        if (rc) {
            ks_close_multi(m);
            return rc;
        }
        m->dev.push_back(dev_ids[r]);
        m->ctx.push_back(c);
        m->buf.push_back(nullptr);
        m->buf_bytes.push_back(0);
        cudaEvent_t e;
        {
            DeviceGuard g(dev_ids[r]);
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        }
        m->ev.push_back(e);
    }
    std::vector<int> sorted(m->dev);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const char* env = std::getenv("KS_MULTI_NCCL");
    const bool want = !(env && *env == '0');
    if (n_dev > 1 && distinct && want && nccl()->ok) {
        m->comm.resize(size_t(n_dev));
        ncclResult_t r = nccl()->CommInitAll(m->comm.data(), n_dev, m->dev.data());
        if (r != ncclSuccess) {
            m->comm.clear();
            int rc = nccl_fail(r, "ncclCommInitAll");
            ks_close_multi(m);
            return rc;
        }
    }
    *out = m;
    return KS_OK;
}

int ks_close_multi(ks_mctx* m) {
    if (!m) return KS_OK;
    for (size_t r = 0; r < m->ctx.size(); ++r) {
        ks::DeviceGuard g(m->dev[r]);
        cudaStreamSynchronize(m->ctx[r]->stream);
        if (r < m->comm.size() && m->comm[r]) nccl()->CommDestroy(m->comm[r]);
        if (m->buf[r]) cudaFree(m->buf[r]);
        if (r < m->ev.size()) cudaEventDestroy(m->ev[r]);
    }
    if (m->gather) {
        ks::DeviceGuard g(m->dev[0]);
        cudaFree(m->gather);
    }
    if (m->host) cudaFreeHost(m->host);
    for (ks_ctx* c : m->ctx) ks_close(c);
    delete m;
    return KS_OK;
}

int ks_multi_info(const ks_mctx* m, int32_t* n_dev, int32_t* uses_nccl) {
    if (!m) return ks::fail(KS_E_INVALID, "null context");
    if (n_dev) *n_dev = int32_t(m->ctx.size());
    if (uses_nccl) *uses_nccl = m->comm.empty() ? 0 : 1;
    return KS_OK;
}

int ks_mdfa_upload(ks_mctx* m, const int32_t* transitions, int32_t n_states, const int32_t* out_offsets,
                   const int32_t* out_ids, int32_t n_expressions, ks_mdfa** out) {
    using namespace ks;
    if (!m || !out) return fail(KS_E_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(m->mu);
    ks_mdfa* d = new ks_mdfa();
    d->m = m;
    for (int r = 0; r < world(m); ++r) {
        ks_dfa* h = nullptr;
        int rc = ks_dfa_upload(m->ctx[r], transitions, n_states, out_offsets, out_ids, n_expressions, &h);
        if (rc) {
            for (ks_dfa* x : d->d) ks_dfa_free(x);
            delete d;
            return rc;
        }
        d->d.push_back(h);
    }
    ks_dfa_info info{};
    ks_dfa_info_get(d->d[0], &info);
    d->nq = info.n_states;
    d->ne = info.n_expressions;
    d->strategy = info.strategy;
    d->sync_depth = info.sync_depth;
    *out = d;
    return KS_OK;
}

int ks_mdfa_free(ks_mdfa* d) {
    if (!d) return KS_OK;
    for (ks_dfa* x : d->d) ks_dfa_free(x);
    delete d;
    return KS_OK;
}

int ks_mseq_upload_codes(ks_mctx* m, const uint8_t* codes, int64_t n, ks_mseq** out) {
    using namespace ks;
    if (!m || !out || n < 0 || (n > 0 && !codes)) return fail(KS_E_INVALID, "bad argument");
    std::lock_guard<std::mutex> lk(m->mu);
    const int W = world(m);
    ks_mseq* s = new ks_mseq();
    s->m = m;
    s->n = n;
    // contiguous slices on 64-symbol boundaries (distributed.shard_bounds)
    const int64_t blocks = (n + 63) / 64, per = blocks / W, extra = blocks % W;
    int64_t b = 0;
    for (int r = 0; r < W; ++r) {
        const int64_t nb = per + (r < extra ? 1 : 0);
        const int64_t lo = std::min(b * 64, n), hi = r + 1 < W ? std::min((b + nb) * 64, n) : n;
        b += nb;
        const int64_t h = std::min(lo, kHalo);
        ks_seq* q = nullptr;
        int rc = ks_seq_upload_codes(m->ctx[r], codes + (lo - h), hi - lo + h, &q);
        if (rc) {
            ks_mseq_free(s);
            return rc;
        }
        s->s.push_back(q);
        s->base.push_back(lo);
        s->halo.push_back(h);
        s->len.push_back(hi - lo);
    }
    *out = s;
    return KS_OK;
}

int ks_mseq_upload_ascii(ks_mctx* m, const uint8_t* bytes, int64_t n_bytes, int32_t fasta, ks_mseq** out) {
    using namespace ks;
    if (!m || !out || n_bytes < 0 || (n_bytes > 0 && !bytes)) return fail(KS_E_INVALID, "bad argument");
    std::lock_guard<std::mutex> lk(m->mu);
    const int W = world(m);
    ks_mseq* s = new ks_mseq();
    s->m = m;
    // byte cut points; FASTA pieces start at line starts so that every piece
    // is parsed from a known line state (ingest.py:65-66 line model)
    std::vector<int64_t> cut(size_t(W) + 1, n_bytes);
    cut[0] = 0;
    for (int r = 1; r < W; ++r) {
        int64_t c = std::max(cut[r - 1], n_bytes * r / W);
        if (fasta) {
            while (c < n_bytes && c > 0 && bytes[c - 1] != '\n' && bytes[c - 1] != '\r') ++c;
            if (c < n_bytes && c > 0 && bytes[c - 1] == '\r' && bytes[c] == '\n') ++c;   // CRLF stays whole
        }
        cut[r] = c;
    }
    int64_t pos = 0;
    for (int r = 0; r < W; ++r) {
        ks_seq* q = nullptr;
        int rc = ks_seq_upload_ascii(m->ctx[r], bytes + cut[r], cut[r + 1] - cut[r], fasta, &q);
        if (rc) {
            ks_mseq_free(s);
            return rc;
        }
        int64_t len = 0;
        ks_seq_length(q, &len);
        s->s.push_back(q);
        s->base.push_back(pos);
        s->halo.push_back(0);
        s->len.push_back(len);
        pos += len;
    }
    s->n = pos;
    *out = s;
    return KS_OK;
}

int ks_mseq_length(const ks_mseq* s, int64_t* n) {
    if (!s || !n) return ks::fail(KS_E_INVALID, "null argument");
    *n = s->n;
    return KS_OK;
}

int ks_mseq_free(ks_mseq* s) {
    if (!s) return KS_OK;
    for (ks_seq* q : s->s) ks_seq_free(q);
    delete s;
    return KS_OK;
}

int ks_mcount(ks_mctx* m, const ks_mdfa* d, const ks_mseq* s, int64_t* counts_out) {
    using namespace ks;
    if (!m || !d || !s || !counts_out) return fail(KS_E_INVALID, "null argument");
    if (d->m != m || s->m != m) return fail(KS_E_INVALID, "handles belong to another multi-device context");
    std::lock_guard<std::mutex> lk(m->mu);
    const int W = world(m);
    const int ne = std::max(d->ne, 1);
    const size_t maps_bytes = size_t(W) * size_t(d->nq) * 4;
    const size_t cnt_off = (maps_bytes + 255) & ~size_t(255);
    for (int r = 0; r < W; ++r) {
        int rc = ensure_buf(m, r, cnt_off + size_t(ne) * 8);
        if (rc) return rc;
    }
    auto maps = [&](int r) { return static_cast<int32_t*>(m->buf[r]); };
    auto cnts = [&](int r) {
        return reinterpret_cast<unsigned long long*>(static_cast<char*>(m->buf[r]) + cnt_off);
    };
    const bool halo = use_halo(d, s);
    const bool nc = !m->comm.empty();
    if (!halo && W > 1) {
        // boundary maps -> all-gather (every rank sees the maps of all ranks)
        for (int r = 0; r < W; ++r) {
            int rc = ks_segment_map_async(m->ctx[r], d->d[r], s->s[r], s->halo[r], s->halo[r] + s->len[r],
                                          maps(r) + size_t(r) * d->nq);
            if (rc) return rc;
        }
        if (nc) {
            KS_NCCL(nccl()->GroupStart());
            for (int r = 0; r < W; ++r)
                KS_NCCL(nccl()->AllGather(maps(r) + size_t(r) * d->nq, maps(r), size_t(d->nq), ncclInt32,
                                          m->comm[r], m->ctx[r]->stream));
            KS_NCCL(nccl()->GroupEnd());
        } else {
            for (int r = 0; r < W; ++r)
                for (int k = 0; k < r; ++k) {   // rank r composes the maps of ranks < r
                    int rc = order_after(m, r, k);
                    if (rc) return rc;
                    DeviceGuard g(m->dev[r]);
                    KS_CUDA(cudaMemcpyPeerAsync(maps(r) + size_t(k) * d->nq, m->dev[r], maps(k) + size_t(k) * d->nq,
                                                m->dev[k], size_t(d->nq) * 4, m->ctx[r]->stream));
                }
        }
    }
    // per-rank shard counts (rank 0 from START; halo ranks by lookback)
    for (int r = 0; r < W; ++r) {
        const int32_t* dm = (halo || W == 1) ? nullptr : maps(r);
        int rc = ks_count_shard_async(m->ctx[r], d->d[r], s->s[r], s->halo[r], s->halo[r] + s->len[r], dm,
                                      halo ? (s->halo[r] > 0 ? r : 0) : r, cnts(r));
        if (rc) return rc;
    }
    // sum over ranks into rank 0's counts
    if (W > 1 && nc) {
        KS_NCCL(nccl()->GroupStart());
        for (int r = 0; r < W; ++r)
            KS_NCCL(nccl()->AllReduce(cnts(r), cnts(r), size_t(ne), ncclUint64, ncclSum, m->comm[r],
                                      m->ctx[r]->stream));
        KS_NCCL(nccl()->GroupEnd());
    } else if (W > 1) {
        DeviceGuard g(m->dev[0]);
        const size_t gb = size_t(W) * size_t(ne) * 8;
        if (m->gather_bytes < gb) {
            KS_CUDA(cudaStreamSynchronize(m->ctx[0]->stream));
            if (m->gather) KS_CUDA(cudaFree(m->gather));
            m->gather = nullptr;
            m->gather_bytes = 0;
            KS_CUDA(cudaMalloc(&m->gather, gb));
            m->gather_bytes = gb;
        }
        for (int k = 0; k < W; ++k) {
            if (k > 0) {
                int rc = order_after(m, 0, k);
                if (rc) return rc;
            }
            DeviceGuard g2(m->dev[0]);
            KS_CUDA(cudaMemcpyPeerAsync(m->gather + size_t(k) * ne, m->dev[0], cnts(k), m->dev[k], size_t(ne) * 8,
                                        m->ctx[0]->stream));
        }
        DeviceGuard g3(m->dev[0]);
        sum_parts_kernel<<<std::max(1, std::min((ne + 255) / 256, 64)), 256, 0, m->ctx[0]->stream>>>(
            m->gather, W, ne, cnts(0));
        KS_CUDA(cudaGetLastError());
    }
    {
        DeviceGuard g(m->dev[0]);
        if (m->host_bytes < size_t(ne) * 8) {
            if (m->host) KS_CUDA(cudaFreeHost(m->host));
            m->host = nullptr;
            m->host_bytes = 0;
            KS_CUDA(cudaMallocHost(&m->host, size_t(ne) * 8));
            m->host_bytes = size_t(ne) * 8;
        }
        KS_CUDA(cudaMemcpyAsync(m->host, cnts(0), size_t(ne) * 8, cudaMemcpyDeviceToHost, m->ctx[0]->stream));
    }
    int rc = sync_all(m);
    if (rc) return rc;
    for (int r = 0; r < W; ++r) {   // the async calls' bookkeeping
        rc = ks_async_wait(m->ctx[r], nullptr, nullptr, nullptr);
        if (rc) return rc;
    }
    std::memcpy(counts_out, m->host, size_t(d->ne) * 8);
    return KS_OK;
}

int ks_mlocate(ks_mctx* m, const ks_mdfa* d, const ks_mseq* s, int64_t* counts_out, int64_t** rows_out,
               int64_t* n_rows) {
    using namespace ks;
    if (!m || !d || !s || !counts_out || !rows_out || !n_rows) return fail(KS_E_INVALID, "null argument");
    if (d->m != m || s->m != m) return fail(KS_E_INVALID, "handles belong to another multi-device context");
    std::lock_guard<std::mutex> lk(m->mu);
    const int W = world(m);
    std::vector<int32_t> entry;
    const bool halo = use_halo(d, s);
    if (!halo) {
        int rc = host_entries(m, d, s, &entry);
        if (rc) return rc;
    }
    std::vector<std::vector<int64_t>> cnt(size_t(W), std::vector<int64_t>(size_t(std::max(d->ne, 1)), 0));
    std::vector<int64_t*> rows(size_t(W), nullptr);
    std::vector<int64_t> nr(size_t(W), 0);
    std::vector<int> rcs(size_t(W), 0);
    std::vector<std::thread> th;
    for (int r = 0; r < W; ++r)   // the ranks' scans run concurrently (one host thread each)
        th.emplace_back([&, r] {
            const int32_t e = halo ? (s->halo[r] > 0 ? -1 : 0) : entry[r];
            rcs[r] = ks_scan_range(m->ctx[r], d->d[r], s->s[r], s->halo[r], s->halo[r] + s->len[r], e,
                                   s->base[r] - s->halo[r], cnt[r].data(), nullptr, &rows[r], &nr[r]);
        });
    for (auto& t : th) t.join();
    int64_t total = 0;
    int rc = KS_OK;
    for (int r = 0; r < W; ++r) {
        if (rcs[r] && !rc) rc = rcs[r];
        total += nr[r];
    }
    if (!rc) {
        int64_t* all = static_cast<int64_t*>(std::malloc(size_t(std::max<int64_t>(total, 1)) * 16));
        if (!all) {
            rc = fail(KS_E_NOMEM, "ks_mlocate: rows");
        } else {
            int64_t at = 0;
            for (int r = 0; r < W; ++r) {
                if (nr[r]) std::memcpy(all + 2 * at, rows[r], size_t(nr[r]) * 16);
                at += nr[r];
            }
            for (int e = 0; e < d->ne; ++e) {
                int64_t v = 0;
                for (int r = 0; r < W; ++r) v += cnt[r][e];
                counts_out[e] = v;
            }
            *rows_out = all;
            *n_rows = total;
        }
    }
    for (int r = 0; r < W; ++r)
        if (rows[r]) ks_free(rows[r]);
    return rc;
}

}  // extern "C"
