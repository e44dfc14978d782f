// Internal declarations shared by the host C++ and the CUDA translation units.
#pragma once

#include <cstdint>
#include <string>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/kmerscan_b200.h"

namespace ks {

class HostPool;

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define KS_CUDA(call)                                              \
    do {                                                           \
        cudaError_t _e = (call);                                   \
        if (_e != cudaSuccess) return ::ks::cuda_fail(_e, #call);  \
    } while (0)

// ---------------------------------------------------------------- limits
constexpr int kMaxStates = 32767;        // uint16 entries, bit 15 = hit flag
constexpr uint16_t kFlag = 0x8000u;
constexpr uint16_t kStateMask = 0x7FFFu;
constexpr int kMaxSyncDepth = 2048;      // longest lookback (AC automata: the longest literal)
constexpr int kMaxMonoid = 4096;         // product table <= 32 MiB
constexpr int kBlockBases = 64;          // bases per packed block (one nmask word)
constexpr int kScanThreads = 512;

// ---------------------------------------------------------------- DFA forms
// Host-compiled device form of one automaton.  States are renumbered so that
// accepting states are [0, n_accept): a hit test is `s < n_accept`.
struct CompiledTable {
    int nq = 0;                      // states of this table
    int n_accept = 0;                // internal ids < n_accept have outputs
    int stride = 1;                  // K: bases per stride-table lookup
    int reset_state = -1;            // internal id all states enter on OTHER, or -1
    std::vector<uint16_t> t1;        // nq x 5 single-symbol table (internal ids)
    std::vector<uint32_t> t1w;       // the same with 32-bit ids (automata above kMaxStates)
    std::vector<uint16_t> tk;        // nq x 4^K, entry = next | (hit on path ? kFlag : 0)
    // fast form (nq <= 4096): 128 KiB column-major K-stride table with a
    // row nq (unused padding); entry at [(w << (16 - 2K)) + s] = (next << 1) | hit
    int fast_k = 0;                  // 0 = not eligible
    double hit_rate = 0;             // accepting-state visits per base on uniform random input
    std::vector<uint16_t> tkc;       // 65536 entries
    std::vector<uint16_t> t1z;       // (nq + 1) x t1z_cols (4: OTHER resets, not stored)
    int t1z_cols = 5;
    // wide automata (> kMaxStates): the hot states [hot_lo, hot_lo + hot_n)
    // (the shallowest, where a scan spends nearly all its steps) get a
    // 4-column shared-memory table of hot indices, 0xFFFF = the next state is
    // cold (read the 32-bit 1-base table from L2)
    std::vector<uint16_t> ht;
    int hot_lo = 0, hot_n = 0;
    // visit-class form of the K = 2 fast table (count mode; scan_fast.cu CLS):
    // a row is a state plus, for the K-steps whose intermediate state
    // accepts, the output multiset of that intermediate state.  Entry =
    // (row << 1) | (sub << 13) | (hit << 15); the step's visits are counted
    // once, in histogram slot (sub << 12) | row, whose output multiset is
    // out(intermediate) + out(final).  Rows [0, nq) are the states, row nq
    // the padding row, rows > nq copies of a state for its 4th, 5th, ...
    // accepting intermediate multiset.
    std::vector<uint16_t> cls_tk;        // 65536 entries, column-major like tkc
    std::vector<uint16_t> cls_t1;        // (cls_rows + 1) x t1z_cols: 1-base table over rows
    std::vector<uint16_t> cls_prim;      // cls_rows: the state of each row
    std::vector<int32_t> cls_out_off;    // cls_nhist + 1: CSR of each slot's output multiset
    std::vector<int32_t> cls_out_ids;
    std::vector<int32_t> cls_used;       // the slots with a non-empty multiset (the only ones ever counted)
    int cls_rows = 0, cls_nhist = 0;     // 0 = no class form
};

struct HostDfa {
    int nq = 0, ne = 0, n_accept = 0;
    bool wide = false;                  // > kMaxStates states: 32-bit ids, LOOKBACK, generic K = 1 scan
    int strategy = 0;
    int sync_depth = -1;
    int start_internal = 0;
    std::vector<int32_t> new_of_old, old_of_new;
    std::vector<int32_t> acc_out_off;   // n_accept + 1 (CSR over internal accepting ids)
    std::vector<int32_t> acc_out_ids;
    std::vector<uint16_t> acc_outcnt;   // n_accept
    int max_outcnt = 0;
    CompiledTable scan;                 // the automaton itself
    // MAPSCAN
    int nm = 0;
    CompiledTable mono;                 // transition-monoid automaton (no hits)
    // mono_sub: when OTHER resets the automaton, `mono` covers only the
    // OTHER-free submonoid (ids [0, mono.nq), numbered first; its OTHER column
    // is the identity) and a chunk holding OTHER maps to const(reset) times
    // the element of what follows its last OTHER: prod[mono_other][e]
    bool mono_sub = false;
    int mono_other = -1;                // id of const(reset) = identity . OTHER
    std::vector<uint16_t> prod;         // nm x nm: element(a then b)
    std::vector<uint16_t> act0;         // nm: internal state reached from START
    std::vector<uint16_t> action;       // nm x nq: internal state reached from q
    // SPECULATE
    std::vector<uint16_t> pss;          // candidate entry states after symbol x: pss[pss_off[x]..pss_off[x+1])
    std::vector<int32_t> pss_off;       // 6
    std::vector<int16_t> pss_inv;       // 5 x nq: index of q in pss of x, or -1
    int pss_max = 0;
};

int compile_dfa(const int32_t* trans, int nq, const int32_t* out_off, const int32_t* out_ids,
                int ne, int force_strategy, size_t smem_budget, HostDfa* out);

// ---------------------------------------------------------------- device views
struct DevTable {
    const uint16_t* t1 = nullptr;   // nq x 5
    const uint32_t* t1w = nullptr;  // nq x 5, 32-bit ids (wide automata)
    const uint16_t* tk = nullptr;   // nq x 4^K
    int nq = 0, n_accept = 0, stride = 1, reset_state = -1;
    size_t tk_bytes = 0, t1_bytes = 0;
    const uint16_t* tkc = nullptr;  // fast form (see CompiledTable)
    const uint16_t* t1z = nullptr;
    int t1z_cols = 5;
    int fast_k = 0;
    size_t t1z_bytes = 0;
    double hit_rate = 0;
    const uint16_t* ht = nullptr;   // wide automata: hot table (CompiledTable::ht)
    int hot_lo = 0, hot_n = 0;
    const uint16_t* cls_tk = nullptr;   // visit-class form (CompiledTable::cls_*)
    const uint16_t* cls_t1 = nullptr;
    const uint16_t* cls_prim = nullptr;
    const int32_t* cls_out_off = nullptr;
    const int32_t* cls_out_ids = nullptr;
    const int32_t* cls_used = nullptr;
    int cls_nused = 0;
    size_t cls_t1_bytes = 0;
    int cls_rows = 0, cls_nhist = 0;
};

// Packed sequence layout ("lane-tiled").  The sequence is cut into units of
// B = 2^lb blocks (64 bases each); 32 consecutive units form a tile.  Within a
// tile, block k of unit l is stored at block slot (k << 5) | l, so the 32
// lanes of a warp that scan the 32 units of a tile read block k with one
// fully coalesced 512-byte load.  bases: 16 B per block slot (2-bit codes,
// base i of the block at bit 2i); nmask/soft: 8 B per block slot.
struct SeqView {
    const uint64_t* bases = nullptr;
    const uint64_t* nmask = nullptr;
    int64_t n = 0;
    int32_t lb = 4;   // log2(blocks per unit)
    // per tile: bit k = some block of row k (the 32 lanes' k-th blocks) holds
    // OTHER; null when not computed (streamed pieces).  The fast scan skips
    // the OTHER-bitmap loads of clear rows.
    const uint64_t* rowmask = nullptr;
};

// Block slot of global block g (= position >> 6).
__host__ __device__ inline int64_t blk_slot(int64_t g, int lb) {
    const int64_t u = g >> lb;
    return ((u >> 5) << (5 + lb)) | ((g & ((int64_t(1) << lb) - 1)) << 5) | (u & 31);
}

#ifdef __CUDACC__
// Symbol code (0..4) at position p.
__device__ __forceinline__ uint32_t seq_sym(const SeqView& q, int64_t p) {
    const int64_t slot = blk_slot(p >> 6, q.lb);
    const int i = int(p & 63);
    if ((__ldg(&q.nmask[slot]) >> i) & 1ull) return 4u;
    return uint32_t(__ldg(&q.bases[2 * slot + (i >> 5)]) >> (2 * (i & 31))) & 3u;
}
#endif

}  // namespace ks

struct ks_ctx {
    std::recursive_mutex mu;   // public calls on one context are serialised (CtxLock)
    int device = 0;
    int num_sms = 148;          // SMs the grids are sized for (sms_total - reserved)
    int sms_total = 148;
    size_t smem_optin = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    ks_stats stats{};
    // grow-only device scratch
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    void* pinned = nullptr;   // small pinned host staging
    size_t pinned_bytes = 0;
    // streaming host-input path (ks_count_host_ascii): copy stream, events,
    // double-buffered device input + packed piece buffers
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t sev[4] = {nullptr, nullptr, nullptr, nullptr};
    void* sbuf = nullptr;
    size_t sbuf_bytes = 0;
    // host-packed wire format: worker pool + pinned staging ring
    ks::HostPool* pool = nullptr;
    void* hstage = nullptr;
    size_t hstage_bytes = 0;
    cudaEvent_t hev[3] = {nullptr, nullptr, nullptr};
    // SPECULATE chunk maps (grow-only, separate from `scratch`)
    void* spec_buf = nullptr;
    size_t spec_bytes = 0;
    // single-pass monoid scan: per-tile status words (epoch | flag | element),
    // zeroed once at allocation; every launch uses a fresh epoch
    unsigned long long* mstat = nullptr;
    int64_t mstat_cap = 0;
    uint32_t mepoch = 0;
    // single-pass row-offset scan: per-tile flags (epoch | flag) and the
    // tiles' sums / inclusive prefixes, zeroed once at allocation
    void* rowstat = nullptr;
    int64_t rowstat_cap = 0;
    uint32_t rowepoch = 0;
    size_t l2_persist = 0;      // persisting-L2 set-aside requested so far (monoid tables)
    size_t l2_persist_max = 0;  // the device's limit
    // pinned host staging the locate scatter writes rows into (grow-only)
    void* rstage = nullptr;
    size_t rstage_bytes = 0;
    void* rdev = nullptr;      // device rows of the same capacity (scatter target)
    size_t rdev_bytes = 0;
    // single-pass locate log (grow-only)
    void* log_buf = nullptr;
    unsigned int* wctr = nullptr;   // task counter of the wide count kernel
    unsigned int* tctr = nullptr;   // dynamic-item counters of the fast count kernel (32 x 128 B)
    size_t log_bytes = 0;
    int32_t log_segs = 0;           // segments (scan CTAs) of the last logged scan
    int64_t log_part = 0;           // entries per segment
    // ks_count_async: one event pair per call until ks_async_wait
    std::vector<cudaEvent_t> aev;
    int n_async = 0;            // per-call event pairs in use (KS_ASYNC_EVENTS=1)
    int async_calls = 0;        // async enqueues since the last ks_async_wait
    int async_launches = 0;
};

struct ks_dfa {
    ks_ctx* ctx = nullptr;
    ks::HostDfa host;
    ks::DevTable scan;
    ks::DevTable mono;
    int32_t* d_acc_out_off = nullptr;
    int32_t* d_acc_out_ids = nullptr;
    uint16_t* d_acc_outcnt = nullptr;
    uint16_t* d_prod = nullptr;
    uint16_t* d_act0 = nullptr;
    uint16_t* d_action = nullptr;   // nm x nq
    uint16_t* d_pss = nullptr;      // SPECULATE candidate sets (HostDfa::pss)
    int32_t* d_pss_off = nullptr;
    int16_t* d_pss_inv = nullptr;
    int32_t* d_new_of_old = nullptr;
    int32_t* d_old_of_new = nullptr;
    void* d_blob = nullptr;   // single allocation backing the above
    // persistent result block of the fused count (visits | counts | err |
    // done | exit, the layout of scan_impl's result block); zero between
    // calls: the kernel's last CTA cleans it, so a count needs no memset
    void* d_cnt = nullptr;
    // visit-class counters of the fused K = 2 count (cls_nhist), kept zero
    // between calls like d_cnt
    unsigned long long* d_cls_visits = nullptr;
    bool tables_in_smem = true;
};

struct ks_seq {
    ks_ctx* ctx = nullptr;
    int64_t n = 0;
    uint64_t* d_bases = nullptr;
    uint64_t* d_nmask = nullptr;
    uint64_t* d_soft = nullptr;
    void* d_blob = nullptr;
    int64_t n_blocks = 0;   // block slots allocated (whole tiles + one padding tile)
    int32_t lb = 4;         // log2(blocks per unit), see SeqView
    // SeqView::rowmask, one word per tile; filled by seq_seal() once an
    // upload has finished (resident sequences are immutable from then on)
    uint64_t* d_rowmask = nullptr;
    bool sealed = false;
};

// Held for the duration of every public call that uses a context.
struct CtxLock {
    std::unique_lock<std::recursive_mutex> lk;
    explicit CtxLock(const ks_ctx* c) {
        if (c) lk = std::unique_lock<std::recursive_mutex>(const_cast<ks_ctx*>(c)->mu);
    }
};
