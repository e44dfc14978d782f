// Chunked DFA scan kernels (sm_100a) -- shared declarations.
//
// Replaces the reference's hot loops (kmerscan/_kernels.py:25-28 scan_from,
// :77-87 the full run of match_chunk_kernel):
//     s = trans[s, sym[j]]; for k in out_off[s]..out_off[s+1]: counts[out_ids[k]] += 1
//
// B200 layout: every thread owns one contiguous lane chunk of L bases
// (L multiple of 64) and walks it with a K-base stride table staged in
// shared memory: one LDS.U16 advances K bases.  Bit 15 of an entry flags
// "a state with outputs was entered during these K bases"; only then the K
// bases are re-walked with the 1-base table and the visited accepting
// states are histogrammed (shared-memory atomics; per-expression counts are
// formed once at the end from the per-state visit histogram).  The sequence
// is read as 2-bit packed bases (16 B per 64 bases) plus one OTHER-bitmap
// word per 64 bases, prefetched one block ahead.
//
// OTHER handling: a 64-base block whose bitmap is all ones (inside an N run)
// rides the warp's fast path and is fixed up afterwards when OTHER sends
// every state to one state (always true for built automata); a partially
// OTHER block, a block cut by the chunk/segment edge, or a non-resetting
// automaton sends the warp through the per-base path for that block.
#pragma once

#include <cstdint>

#include "ks_internal.h"

namespace ks {

enum ScanMode : int { kModeCount = 0, kModeRows = 1, kModeEmit = 2, kModeMap = 3, kModeLog = 4 };

// One accepting-state visit of a locate pass (kModeLog, fast kernel): where
// its rows start inside its chunk; log_scatter turns it into rows once the
// chunk offsets are known.  Single-pass locate while hits fit the log.
struct LogEntry {
    int64_t pos1;     // row offset (row_base + position + 1)
    uint32_t chunk;   // chunk index of the launch
    uint32_t local;   // rows of this chunk before this visit
    uint32_t state;   // internal accepting state
    uint32_t pad;
};

struct ScanArgs {
    SeqView seq;
    int64_t begin = 0, end = 0;      // positions scanned: [begin, end)
    int64_t origin = 0;              // 64-aligned: chunk c starts at origin + c*chunk_len
    int64_t chunk_len = 64;          // multiple of 64
    int64_t nchunks = 0;
    // entry state of each chunk (first match wins):
    const uint16_t* chunk_entry = nullptr;  // per-chunk entry states (MAPSCAN pass 2)
    int32_t uniform_entry = -1;      // >= 0: every chunk enters in this state (MAP pass)
    int32_t lookback = 0;            // else: scan max(base_pos, cb - lookback) .. cb
    int64_t base_pos = 0;            //   starting in base_state when at base_pos,
    int32_t base_state = 0;          //   in any_state otherwise (synchronising word)
    const uint16_t* base_state_ptr = nullptr;  // if set: base_state read from device memory
    int32_t any_state = 0;
    // automaton
    const uint16_t* t1 = nullptr;    // nq x 5 (global)
    const uint32_t* t1w = nullptr;   // nq x 5, 32-bit ids (wide automata, scan_wide_kernel)
    uint32_t* chunk_exit32 = nullptr;   // wide automata: per chunk exit state (optional)
    const uint16_t* ht = nullptr;    // wide automata: hot table (hot_n x 4, hot indices, 0xFFFF = cold)
    int32_t hot_lo = 0, hot_n = 0;
    const uint16_t* tk = nullptr;    // nq x 4^K (global)
    int32_t nq = 0, n_accept = 0, reset_state = -1;
    int32_t tk_pad = 0, t1_pad = 0;  // uint16 entries, multiples of 8
    int32_t t1_cols = 5;             // fast kernel: columns of t1 (4: OTHER -> reset_state)
    int32_t lean = 0;                // fast kernel: hits so rare that blocks run without recording
                                     // and a warp re-runs a block only when one of its lanes hit
    int32_t hist_smem = 0;           // histogram in shared memory
    int32_t ring_depth = 0;          // fast kernel: deferred hits per lane (set by launch_scan_fast)
    // outputs
    unsigned long long* visits = nullptr;   // n_accept, global accumulation
    uint16_t* chunk_exit = nullptr;         // per chunk exit state (optional)
    uint32_t* chunk_rows = nullptr;         // kModeRows
    const int64_t* chunk_row_off = nullptr; // kModeEmit (nchunks + 1)
    const int32_t* acc_out_off = nullptr;
    const int32_t* acc_out_ids = nullptr;
    const uint16_t* acc_outcnt = nullptr;
    int64_t* rows = nullptr;
    int64_t row_base = 0;                   // row offset = position + 1 + row_base
    int32_t* error = nullptr;               // set to 1 on an internal invariant failure
    // fast kernel, count mode: the last CTA turns visits into counts (fused
    // finalize_counts).  visits and fin_done must be zero at launch; the last
    // CTA leaves them zero again (so a persistent block needs no memset),
    // zeroes fin_counts itself, and copies the counts to fin_host (a device
    // view of pinned host memory, so no D2H copy follows) when it is set.
    unsigned long long* fin_counts = nullptr;
    const uint16_t* fin_exit_src = nullptr;
    uint16_t* fin_exit_dst = nullptr;
    unsigned int* fin_done = nullptr;
    unsigned long long* fin_host = nullptr;
    int32_t n_expr = 0;
    unsigned int* fin_signal = nullptr;     // optional: set to fin_signal_value once the counts are final
    unsigned int fin_signal_value = 0;
    // kModeMap over the OTHER-free submonoid (HostDfa::mono_sub): a chunk
    // that holds OTHER (the table resets to the identity there) exits with
    // map_dirty[element since its last OTHER]
    const uint16_t* map_dirty = nullptr;
    LogEntry* log = nullptr;                // kModeLog: log_cap entries, one segment of log_part per CTA
    unsigned long long* log_n = nullptr;    // kModeLog: total logged (> log_cap when a segment overflowed)
    unsigned int* log_cta_n = nullptr;      // kModeLog: entries of each CTA's segment
    int64_t log_cap = 0;
    int64_t log_part = 0;                   // set by launch_scan_fast
    unsigned int* work_ctr = nullptr;       // wide count kernel: task counter (zeroed per launch)
    int32_t run_blocks = 0;                 // wide count kernel: blocks per run
    // fast kernel, count mode: dynamic work items (dyn_items: the caller's
    // fused finalize allows them; tile_ctr = the context's counters, zero at
    // launch and reset by the finalizing CTA)
    int32_t dyn_items = 0;
    unsigned int* tile_ctr = nullptr;
    int32_t split_tiles = 0, split_parts = 1;
    // the last split2_tiles of the split tiles are cut finer still (split2_parts ranges):
    // the items handed out last are the smallest
    int32_t split2_tiles = 0, split2_parts = 1;
    int64_t static_items = 0;               // items below this go round-robin
    int32_t early_wait = 0;                 // fast kernel: wait for the preceding kernel up front (KS_EARLY_WAIT=1)
    // fast K = 2 count with the visit-class table (CompiledTable::cls_*): tk/t1
    // are the class forms, visits / acc_out_* the n_hist class slots
    int32_t cls = 0;
    int32_t n_hist = 0;
    const uint16_t* cls_prim = nullptr;     // row -> state (chunk exits)
    const int32_t* cls_used = nullptr;      // the slots the finalize reads (n_used of them)
    int32_t n_used = 0;
    uint32_t one = 1;                       // a 1 the compiler cannot fold (multiply-add / add operands)
    int32_t ktime = 0;                      // fast kernel: per-phase timestamps (KS_KTIME=1, diagnostic)
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

#ifdef __CUDACC__
// ---- table staging with bulk copies (the TMA engine: UBLKCP + SYNCS) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
// global -> shared bulk copy; completion counted in bytes on the mbarrier
__device__ __forceinline__ void bulk_copy_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbarrier_wait0(uint32_t mbar) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t"
        "@!done bra WAIT_%=;\n\t}"
        ::"r"(mbar) : "memory");
}
// Stage up to two global regions (16-byte aligned, sizes multiples of 16)
// into shared memory: one thread arms the CTA's mbarrier and issues 32 KiB
// bulk copies while the other threads go on (histogram clears etc.); call
// stage_wait before reading the staged bytes.  Every thread calls both.
struct BulkStage {
    uint32_t mbar;
    __device__ __forceinline__ void begin(unsigned long long* bar, uint32_t d0, const void* s0, uint32_t n0,
                                          uint32_t d1 = 0, const void* s1 = nullptr, uint32_t n1 = 0) {
        mbar = smem_u32(bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(n0 + n1)
                         : "memory");
            constexpr uint32_t kPart = 32768;
            for (uint32_t o = 0; o < n0; o += kPart)
                bulk_copy_g2s(d0 + o, static_cast<const char*>(s0) + o, n0 - o < kPart ? n0 - o : kPart, mbar);
            for (uint32_t o = 0; o < n1; o += kPart)
                bulk_copy_g2s(d1 + o, static_cast<const char*>(s1) + o, n1 - o < kPart ? n1 - o : kPart, mbar);
        }
    }
    __device__ __forceinline__ void wait() const { mbarrier_wait0(mbar); }
};
#endif

// Launch attribute keeping [base, base + bytes) in the persisting part of L2
// (constant automaton tables: they survive the sequence streaming through L2
// and the calls in between).  Grows the device's set-aside as needed; false
// (attribute not filled) when unavailable or KS_NO_L2_PERSIST is set.
bool l2_persist_attr(ks_ctx* ctx, const void* base, size_t bytes, cudaLaunchAttribute* attr);
void l2_persist_acquire(int device);     // ks_open: one more context on the device
void l2_persist_release(ks_ctx* ctx);    // ks_close: the last one restores the set-aside

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

// Launch one scan over [a.begin, a.end); fills chunk geometry, grid and smem.
// Returns KS_OK or a KS_E_* code (error text set).
int launch_scan(ks_ctx* ctx, ScanArgs a, int mode, int stride, bool smem_tables, int* launches);
// Automata above kMaxStates (32-bit ids): one base per lookup from the
// 1-base table through L1/L2, lookback entries only.
int launch_scan_wide(ks_ctx* ctx, ScanArgs a, int mode, int* launches);

// Chunk geometry used by launch_scan for a span (so callers can size arrays).
void scan_geometry(const ks_ctx* ctx, int64_t begin, int64_t end, int stride, bool smem_tables,
                   int32_t tk_pad, int32_t t1_pad, int32_t hist_words, int64_t* origin,
                   int64_t* chunk_len, int64_t* nchunks);

void chunk_geometry(int64_t begin, int64_t end, int64_t threads, int64_t* origin, int64_t* chunk_len,
                    int64_t* nchunks);

// Fast shared-memory kernel for tables with a fast form (csrc/scan_fast.cu).
int launch_scan_fast(ks_ctx* ctx, ScanArgs a, int mode, int k, int* launches);
size_t fast_fixed_bytes(int32_t t1_pad, int32_t hist_words);
size_t fast_smem_bytes(int mode, int32_t t1_pad, int32_t hist_words, int threads);
// Warps per CTA of the fast scan for `tiles` tiles of 32 units: 32, or fewer
// when that makes the tiles fill whole rounds over all SMs.
int fast_warps_per_cta(int64_t tiles, int num_sms);
int fast_threads();
// rows of the logged visits: rows[row_off[chunk] + local + k] = (pos1, id_k)
// Rows of the visit log at their chunk offsets.  With n_dev the count is read
// on the device (n is then the log capacity; an overflowed log writes nothing).
int launch_log_scatter(ks_ctx* ctx, const LogEntry* log, const unsigned int* seg_n, int32_t segs, int64_t part,
                       const unsigned long long* n_dev, int64_t cap, const int64_t* row_off, const int32_t* acc_out_off,
                       const int32_t* acc_out_ids, int64_t* rows, int* launches);

// Prefix scans (csrc/prefix_scan.cu).
int exclusive_scan_rows(ks_ctx* ctx, const uint32_t* in, int64_t n, int64_t* out_excl,
                        int64_t* d_total, void* tmp, int* launches);
size_t exclusive_scan_rows_tmp_bytes(int64_t n);
// exclusive running maximum (identity -1); tmp sized like the rows scan
int exclusive_scan_max(ks_ctx* ctx, const int64_t* in, int64_t n, int64_t* out_excl, int64_t* d_total,
                       void* tmp, int* launches);
// Single-pass (decoupled look-back) monoid scan fused with the chunk entry
// states: centry[i] = action[(in[0] ... in[i-1])][q0] with q0 = entry_val
// (>= 0) or *entry_ptr; centry may be null.  *d_total = the product of all n
// elements.  One launch, no temporaries beyond ctx->mstat.
// The product and action tables (window_bytes from prod on) are kept in the
// persisting part of L2, so the dependent lookups stay L2 hits while the
// sequence streams through (and across calls).
int monoid_scan_entries(ks_ctx* ctx, const uint16_t* in, int64_t n, const uint16_t* prod, int32_t nm,
                        const uint16_t* action, int32_t nq, int32_t entry_val, const uint16_t* entry_ptr,
                        uint16_t* centry, uint16_t* d_total, size_t window_bytes, int* launches);

// Small helper kernels (csrc/scan.cu).
int launch_finalize_counts(ks_ctx* ctx, const unsigned long long* visits, int32_t n_accept,
                           const int32_t* acc_out_off, const int32_t* acc_out_ids,
                           unsigned long long* counts, const uint16_t* exit_src, uint16_t* exit_dst,
                           int* launches);
// SPECULATE strategy (spec.cu): entry state of every chunk of [begin, end)
// from per-chunk candidate maps, processed seg_chunks chunks at a time in
// `buf` (speculate_entries_bytes).  The range's entry is entry_val (>= 0) or
// *entry_ptr; *d_exit (optional) receives the state after `end`.
size_t speculate_entries_bytes(int64_t seg_chunks, int32_t pss_max);
int speculate_entries(ks_ctx* ctx, const SeqView& seq, int64_t begin, int64_t end, int64_t origin, int64_t L,
                      int64_t nch, const uint16_t* t1, int32_t nq, const uint16_t* pss, const int32_t* pss_off,
                      const int16_t* inv, int32_t pss_max, int32_t entry_val, const uint16_t* entry_ptr,
                      uint16_t* centry, uint16_t* d_exit, void* buf, int64_t seg_chunks, int* launches);


}  // namespace ks
