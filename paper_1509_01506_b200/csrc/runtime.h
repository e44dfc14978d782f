// Host-side runtime shared by the C-ABI translation units (capi.cu,
// stream.cu): scratch arenas, the scan plan/dispatch, strategy helpers and
// the device helpers of encode.cu / spec.cu / scan_fast.cu.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "host_pack.h"
#include "scan_kernels.cuh"

namespace ks {

constexpr size_t kAlign = 256;
inline size_t up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Bump allocator over the context's grow-only scratch buffer.
struct Arena {
    char* base = nullptr;
    size_t off = 0;
    size_t cap = 0;
    void* take(size_t n) {
        off = up(off);
        void* p = base + off;
        off += up(n ? n : 1);
        return p;
    }
};

int ensure_scratch(ks_ctx* ctx, size_t bytes, Arena* a);
int ensure_pinned(ks_ctx* ctx, size_t bytes);
bool env_flag(const char* name);
bool host_is_device_visible(const void* p);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Kernel choice for one table: the fast column-major kernel when the table
// has a fast form and fits, else the generic row-major kernel.
struct ScanPlan {
    bool fast = false;
    bool hist_smem = false;
};

SeqView view_of(const ks_seq* s);
ScanArgs base_args(const ks_dfa* dfa, const DevTable& T, const ks_seq* seq);
ScanPlan plan_for(const ks_ctx* ctx, const ks_dfa* dfa, const DevTable& T);
void geometry(const ks_seq* seq, int64_t begin, int64_t end, int64_t* origin, int64_t* L, int64_t* nch);
int dispatch(ks_ctx* ctx, const ks_dfa* dfa, const DevTable& T, const ScanPlan& p, ScanArgs a, int mode,
             int* launches);
// KS_PHASE_TRACE=1: stream-ordered events between the phases of a scan,
// printed to stderr once the call completes (diagnostics only).
// KS_PHASE_TRACE=2: the same, deferred -- no synchronisation per call; the
// phases of every call are printed by ks_async_wait (async pipelines).
struct PhaseTrace {
    using Marks = std::vector<std::pair<const char*, cudaEvent_t>>;
    cudaStream_t st = nullptr;
    bool deferred = false;
    Marks marks;
    explicit PhaseTrace(cudaStream_t s) {
        if (env_flag("KS_PHASE_TRACE")) {
            st = s;
            const char* v = std::getenv("KS_PHASE_TRACE");
            deferred = v[0] == '2';
        }
    }
    void mark(const char* name) {
        if (!st) return;
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        cudaEventRecord(e, st);
        marks.emplace_back(name, e);
    }
    static std::vector<Marks>& pending() {
        static std::vector<Marks> p;
        return p;
    }
    static void print(Marks& m) {
        for (size_t i = 1; i < m.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, m[i - 1].second, m[i].second);
            std::fprintf(stderr, "[ks phase] %-14s %9.1f us\n", m[i].first, ms * 1e3f);
        }
        for (auto& x : m) cudaEventDestroy(x.second);
        m.clear();
    }
    static void flush() {   // after a synchronisation
        for (auto& m : pending()) print(m);
        pending().clear();
    }
    ~PhaseTrace() {
        if (!st || marks.empty()) return;
        if (deferred) {
            pending().push_back(std::move(marks));
            return;
        }
        cudaStreamSynchronize(st);
        print(marks);
    }
};

// Walk [begin, end) from every state (uniform_start < 0, nlanes = |Q|) or
// from one state; internal ids into out (uint32).
int launch_walk(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end, int32_t nlanes,
                int32_t uniform_start, uint32_t* out);
int monoid_prefix(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end,
                  int64_t origin, int64_t L, int64_t nch, uint16_t* elems, uint16_t* centry, int32_t entry_val,
                  const uint16_t* entry_ptr, uint16_t* d_total, int* launches, PhaseTrace* trace = nullptr);
int spec_entries(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin, int64_t end, int64_t origin,
                 int64_t L, int64_t nch, int32_t entry_val, const uint16_t* entry_ptr, uint16_t* centry,
                 uint16_t* d_exit, int* launches);
int choose_lb(const ks_ctx* ctx, int64_t n);

// the streamed count from host bytes (stream.cu)
enum StreamMode { kStreamPacked = 0, kStreamWire = 1, kStreamDevice = 2 };
int stream_count_impl(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes, bool fasta,
                      int stream_mode, int64_t* counts_out, bool* fallback);

// encode.cu / spec.cu
size_t encode_scratch_bytes(int64_t n_bytes);
int encode_compact_device(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, bool fasta, int* d_carry,
                          ks_seq* seq, void* scratch, int64_t* d_total, int* launches);
int encode_ascii_device(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, bool fasta, ks_seq* seq, void* scratch,
                        int* launches);
int pack_codes_device(ks_ctx* ctx, const uint8_t* d_codes, int64_t n, ks_seq* seq, int* d_flag,
                      int* launches);
int wire_compact_device(ks_ctx* ctx, const uint64_t* d_lin, const uint64_t* d_special, int64_t n_blocks, ks_seq* seq,
                        uint32_t* kept, int64_t* pos, void* tmp, int64_t* d_total, int* launches);
int encode_raw_piece(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, ks_seq* seq, uint32_t* kept, int* ws_flag,
                     int* launches);
int scatter_tile_masks_device(ks_ctx* ctx, const uint64_t* d_compact, const int32_t* d_ids, int n_tiles,
                              int tile_words, uint64_t* d_nmask, int* launches);
int unpack_codes_device(ks_ctx* ctx, const ks_seq* seq, uint8_t* d_out);
int linear_softmask_device(ks_ctx* ctx, const ks_seq* seq, uint64_t* d_out);
int launch_speculate(ks_ctx* ctx, const SeqView& seq, int32_t n_chunks, const int64_t* d_cbeg,
                     const int64_t* d_cend, const int64_t* d_pss_off, const void* d_pss, bool wide,
                     const int64_t* h_pss_off, int32_t window, const void* t1, int32_t n_accept,
                     const int32_t* off, const int32_t* ids, int32_t ne, int32_t* d_conv,
                     long long* d_delta, void* d_tasks_buf, int* launches);
size_t speculate_task_bytes(int32_t n_chunks, const int64_t* h_pss_off);

}  // namespace ks
