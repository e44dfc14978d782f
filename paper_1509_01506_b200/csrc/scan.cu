// Chunked DFA scan kernels and their launchers (see scan_kernels.cuh).
#include <cstdlib>
#include <algorithm>

#include "scan_kernels.cuh"

namespace ks {
namespace {

// --------------------------------------------------------------- hit sinks
// What a visit to an accepting state (internal id s < n_accept) at sequence
// position `pos` does, per mode.  Visits are the reference's inner CSR loop
// (_kernels.py:26-28 / :80-84) deferred: counts[e] = sum_s visits[s]*mult(s,e).
template <int MODE>
struct Sink {
    unsigned int* shist;
    unsigned long long* visits;
    const uint16_t* outcnt;
    const int32_t* off;
    const int32_t* ids;
    int64_t* rows;
    int64_t row_base;
    uint32_t nrows;
    int64_t cur;

    __device__ __forceinline__ void add(uint32_t s, uint32_t times) {
        if (shist) atomicAdd(&shist[s], times);
        else atomicAdd(&visits[s], (unsigned long long)times);
    }

    __device__ __forceinline__ void hit(int64_t pos, uint32_t s) {
        if constexpr (MODE == kModeCount || MODE == kModeRows) {
            add(s, 1u);
            if constexpr (MODE == kModeRows) nrows += __ldg(&outcnt[s]);
        } else if constexpr (MODE == kModeEmit) {
            const int k1 = __ldg(&off[s + 1]);
            const long long o = row_base + pos + 1;
            for (int k = __ldg(&off[s]); k < k1; ++k, ++cur) {
                longlong2 r;
                r.x = o;
                r.y = __ldg(&ids[k]);
                reinterpret_cast<longlong2*>(rows)[cur] = r;
            }
        }
    }

    // `n` consecutive positions starting at pos0 all entering state s.
    __device__ __forceinline__ void hit_run(int64_t pos0, int n, uint32_t s) {
        if constexpr (MODE == kModeCount || MODE == kModeRows) {
            add(s, uint32_t(n));
            if constexpr (MODE == kModeRows) nrows += uint32_t(n) * __ldg(&outcnt[s]);
        } else if constexpr (MODE == kModeEmit) {
            for (int i = 0; i < n; ++i) hit(pos0 + i, s);
        }
    }
};

template <bool SM>
struct Tables {
    const uint16_t* tk;
    const uint16_t* t1;
    __device__ __forceinline__ uint32_t k(uint32_t i) const {
        if constexpr (SM) return tk[i];
        else return __ldg(tk + i);
    }
    __device__ __forceinline__ uint32_t one(uint32_t i) const {
        if constexpr (SM) return t1[i];
        else return __ldg(t1 + i);
    }
};

// Bits [off, off+width) of the 128-bit value w1:w0 (off, width compile-time
// after unrolling).
__device__ __forceinline__ uint32_t bits128(uint64_t w0, uint64_t w1, int off, int width) {
    uint64_t v;
    if (off >= 64) v = w1 >> (off - 64);
    else if (off + width > 64) v = (w0 >> off) | (w1 << (64 - off));
    else v = w0 >> off;
    return uint32_t(v) & ((1u << width) - 1u);
}


// Re-walk the K bases of a flagged stride step with the 1-base table,
// recording every accepting state entered.
template <int K, int MODE, bool SM>
__device__ __forceinline__ void rewalk(uint32_t s, uint32_t word, int64_t pos, int32_t n_accept,
                                       const Tables<SM>& T, Sink<MODE>& sink) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
        s = T.one(s * 5u + ((word >> (2 * i)) & 3u));
        if (s < uint32_t(n_accept)) sink.hit(pos + i, s);
    }
}

// Advance one full, OTHER-free 64-base block with the K-stride table.
template <int K, int MODE, bool SM>
__device__ __forceinline__ uint32_t fast_block(uint32_t s, uint64_t w0, uint64_t w1, bool live,
                                               int64_t p0, int32_t n_accept, const Tables<SM>& T,
                                               Sink<MODE>& sink) {
    constexpr int W = 2 * K;
    constexpr int NL = 64 / K;
    if constexpr (K == 1) {   // large automata: the 1-base table itself, hits by the accepting-first ids
#pragma unroll 16
        for (int j = 0; j < 64; ++j) {
            s = T.one(s * 5u + bits128(w0, w1, 2 * j, 2));
            if constexpr (MODE != kModeMap) {
                if (live && s < uint32_t(n_accept)) sink.hit(p0 + j, s);
            }
        }
        return s;
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        const uint32_t word = bits128(w0, w1, W * j, W);
        const uint32_t e = T.k((s << W) | word);
        if constexpr (MODE != kModeMap) {
            if (e & kFlag) {
                if (live) rewalk<K, MODE, SM>(s, word, p0 + K * j, n_accept, T, sink);
            }
        }
        s = e & kStateMask;
    }
#pragma unroll
    for (int r = NL * K; r < 64; ++r) {  // K == 3 leaves one base
        s = T.one(s * 5u + bits128(w0, w1, 2 * r, 2));
        if constexpr (MODE != kModeMap) {
            if (live && s < uint32_t(n_accept)) sink.hit(p0 + r, s);
        }
    }
    return s;
}

extern __shared__ __align__(16) unsigned char g_smem[];

template <int K, int MODE, bool SM>
__global__ void __launch_bounds__(1024, 1) scan_kernel(const ScanArgs a) {
    uint16_t* s_tk = reinterpret_cast<uint16_t*>(g_smem);
    uint16_t* s_t1 = s_tk + (SM ? a.tk_pad : 0);
    unsigned int* s_hist = reinterpret_cast<unsigned int*>(s_t1 + (SM ? a.t1_pad : 0));

    __shared__ __align__(8) unsigned long long staged;
    BulkStage st;
    if constexpr (SM)   // both tables by bulk copies (TMA engine) while the threads clear the histogram
        st.begin(&staged, smem_u32(s_tk), a.tk, uint32_t(a.tk_pad) * 2u, smem_u32(s_t1), a.t1,
                 uint32_t(a.t1_pad) * 2u);
    const bool hist_smem = (MODE == kModeCount || MODE == kModeRows) && a.hist_smem;
    if (hist_smem)
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x) s_hist[i] = 0u;
    if constexpr (SM) st.wait();
    __syncthreads();

    Tables<SM> T;
    T.tk = SM ? s_tk : a.tk;
    T.t1 = SM ? s_t1 : a.t1;
    const uint32_t n_accept = uint32_t(a.n_accept);
    const uint4* bases4 = reinterpret_cast<const uint4*>(a.seq.bases);
    const uint64_t* nmask = a.seq.nmask;

    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < a.nchunks; c += stride) {
        const int64_t cb = max64(a.begin, a.origin + c * a.chunk_len);
        const int64_t ce = min64(a.end, a.origin + (c + 1) * a.chunk_len);

        uint32_t s;
        if (a.chunk_entry) {
            s = a.chunk_entry[c];
        } else if (a.uniform_entry >= 0) {
            s = uint32_t(a.uniform_entry);
        } else {
            const int64_t lb = max64(a.base_pos, cb - a.lookback);
            s = uint32_t(lb == a.base_pos ? (a.base_state_ptr ? int32_t(*a.base_state_ptr) : a.base_state) : a.any_state);
            for (int64_t p = lb; p < cb; ++p) s = T.one(s * 5u + seq_sym(a.seq, p));
        }

        Sink<MODE> sink;
        sink.shist = hist_smem ? s_hist : nullptr;
        sink.visits = a.visits;
        sink.outcnt = a.acc_outcnt;
        sink.off = a.acc_out_off;
        sink.ids = a.acc_out_ids;
        sink.rows = a.rows;
        sink.row_base = a.row_base;
        sink.nrows = 0;
        sink.cur = (MODE == kModeEmit) ? a.chunk_row_off[c] : 0;

        int64_t b = cb >> 6;
        const int64_t bend = (ce + 63) >> 6;
        const int lb = a.seq.lb;
        bool dirty = false;   // kModeMap over the submonoid: OTHER inside the chunk
        uint4 wb = __ldg(bases4 + blk_slot(b, lb));
        uint64_t wm = __ldg(nmask + blk_slot(b, lb));
        for (; b < bend; ++b) {
            // arrays are padded by a whole tile: the prefetch never faults
            const int64_t ns = blk_slot(b + 1, lb);
            const uint4 nb = __ldg(bases4 + ns);
            const uint64_t nm = __ldg(nmask + ns);
            const int64_t p0 = b << 6;
            const int lo = int(max64(cb - p0, 0));
            const int hi = int(min64(ce - p0, 64));
            const uint64_t w0 = (uint64_t(wb.y) << 32) | wb.x;
            const uint64_t w1 = (uint64_t(wb.w) << 32) | wb.z;
            const bool full = (lo == 0) && (hi == 64);
            const bool alln = wm == ~0ull;
            if constexpr (MODE == kModeMap) {
                if (wm && a.map_dirty)
                    dirty |= (wm & ((hi >= 64 ? ~0ull : ((1ull << hi) - 1ull)) & (~0ull << lo))) != 0ull;
            }
            const bool fast = full && (wm == 0ull || (alln && a.reset_state >= 0));
            if (__all_sync(__activemask(), fast)) {
                const uint32_t s2 = fast_block<K, MODE, SM>(s, w0, w1, !alln, p0, a.n_accept, T, sink);
                if (alln) {
                    s = uint32_t(a.reset_state);
                    if constexpr (MODE != kModeMap) {
                        if (s < n_accept) sink.hit_run(p0, 64, s);
                    }
                } else {
                    s = s2;
                }
            } else {
                for (int i = lo; i < hi; ++i) {
                    const uint32_t sym = ((wm >> i) & 1ull)
                                             ? 4u
                                             : uint32_t((i < 32 ? w0 >> (2 * i) : w1 >> (2 * (i - 32)))) & 3u;
                    s = T.one(s * 5u + sym);
                    if constexpr (MODE != kModeMap) {
                        if (s < n_accept) sink.hit(p0 + i, s);
                    }
                }
            }
            wb = nb;
            wm = nm;
        }
        if constexpr (MODE == kModeMap) {
            if (dirty) s = __ldg(&a.map_dirty[s]);
        }
        if (a.chunk_exit) a.chunk_exit[c] = uint16_t(s);
        if constexpr (MODE == kModeRows) a.chunk_rows[c] = sink.nrows;
        if constexpr (MODE == kModeEmit) {
            if (sink.cur != a.chunk_row_off[c + 1]) atomicExch(a.error, 1);
        }
    }

    if (hist_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&a.visits[i], (unsigned long long)s_hist[i]);
    }
}

// Wide automata (> 32767 states, 32-bit ids): one thread per chunk, one
// 1-base lookup per symbol (__ldg, the table lives in L2), entry states by
// lookback only (definite automata), hits as in scan_kernel.
template <int MODE>
__global__ void __launch_bounds__(256) scan_wide_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) unsigned int w_hist[];
    const bool hist_smem = (MODE == kModeCount || MODE == kModeRows) && a.hist_smem;
    if (hist_smem) {
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x) w_hist[i] = 0u;
        __syncthreads();
    }
    const uint32_t n_accept = uint32_t(a.n_accept);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < a.nchunks; c += stride) {
        const int64_t cb = max64(a.begin, a.origin + c * a.chunk_len);
        const int64_t ce = min64(a.end, a.origin + (c + 1) * a.chunk_len);
        const int64_t lb = max64(a.base_pos, cb - a.lookback);
        uint32_t s = uint32_t(lb == a.base_pos ? a.base_state : a.any_state);
        for (int64_t p = lb; p < cb; ++p) s = __ldg(&a.t1w[size_t(s) * 5 + seq_sym(a.seq, p)]);
        Sink<MODE> sink;
        sink.shist = hist_smem ? w_hist : nullptr;
        sink.visits = a.visits;
        sink.outcnt = a.acc_outcnt;
        sink.off = a.acc_out_off;
        sink.ids = a.acc_out_ids;
        sink.rows = a.rows;
        sink.row_base = a.row_base;
        sink.nrows = 0;
        sink.cur = (MODE == kModeEmit) ? a.chunk_row_off[c] : 0;
        for (int64_t p = cb; p < ce; ++p) {
            s = __ldg(&a.t1w[size_t(s) * 5 + seq_sym(a.seq, p)]);
            if constexpr (MODE != kModeMap) {
                if (s < n_accept) sink.hit(p, s);
            }
        }
        if (a.chunk_exit32) a.chunk_exit32[c] = s;
        if constexpr (MODE == kModeRows) a.chunk_rows[c] = sink.nrows;
        if constexpr (MODE == kModeEmit) {
            if (sink.cur != a.chunk_row_off[c + 1]) atomicExch(a.error, 1);
        }
    }
    if (hist_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x)
            if (w_hist[i]) atomicAdd(&a.visits[i], (unsigned long long)w_hist[i]);
    }
}

// Wide automata with a hot table (CompiledTable::ht): states in
// [hot_lo, hot_lo + hot_n) step through the shared-memory table (2-byte hot
// indices), every other transition -- from a cold state, or into one (0xFFFF)
// -- reads the 32-bit 1-base table through L1/L2.  One thread per unit chunk
// (a warp's 32 chunks are one tile: each block load is one coalesced 512 B
// read), whole 64-base blocks stepped from registers, hits into the
// shared-memory visit histogram when it fits (global atomics otherwise).
__device__ __forceinline__ uint32_t wide_hot_step(const uint16_t* ht, const uint32_t* __restrict__ t1w, uint32_t s,
                                                  uint32_t sym, uint32_t lo, uint32_t H) {
    const uint32_t hs = s - lo;
    if (hs < H) {
        const uint32_t e = ht[hs * 4u + sym];
        if (e != 0xFFFFu) return e + lo;
    }
    return __ldg(&t1w[size_t(s) * 5 + sym]);
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) scan_wide_hot_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) unsigned char wh_smem[];
    uint16_t* ht = reinterpret_cast<uint16_t*>(wh_smem);
    const size_t ht_bytes = (size_t(a.hot_n) * 8 + 15) & ~size_t(15);
    unsigned int* shist = reinterpret_cast<unsigned int*>(wh_smem + ht_bytes);
    const bool hist_smem = (MODE == kModeCount || MODE == kModeRows) && a.hist_smem;
    // the hot table (8-byte rows, padded to 16 bytes in the blob) by bulk copies
    __shared__ __align__(8) unsigned long long staged;
    BulkStage st;
    st.begin(&staged, smem_u32(ht), a.ht, uint32_t(ht_bytes));
    if (hist_smem)
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x) shist[i] = 0u;
    st.wait();
    __syncthreads();
    const uint32_t A = uint32_t(a.n_accept), lo = uint32_t(a.hot_lo), H = uint32_t(a.hot_n);
    const uint32_t reset = uint32_t(a.reset_state);
    const uint4* bases4 = reinterpret_cast<const uint4*>(a.seq.bases);
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < a.nchunks; c += stride) {
        const int64_t cb = max64(a.begin, a.origin + c * a.chunk_len);
        const int64_t ce = min64(a.end, a.origin + (c + 1) * a.chunk_len);
        const int64_t lb = max64(a.base_pos, cb - a.lookback);
        uint32_t s = uint32_t(lb == a.base_pos ? a.base_state : a.any_state);
        for (int64_t p = lb; p < cb; ++p) {
            const uint32_t y = seq_sym(a.seq, p);
            s = y == 4u ? reset : wide_hot_step(ht, a.t1w, s, y, lo, H);
        }
        Sink<MODE> sink;
        sink.shist = hist_smem ? shist : nullptr;
        sink.visits = a.visits;
        sink.outcnt = a.acc_outcnt;
        sink.off = a.acc_out_off;
        sink.ids = a.acc_out_ids;
        sink.rows = a.rows;
        sink.row_base = a.row_base;
        sink.nrows = 0;
        sink.cur = (MODE == kModeEmit) ? a.chunk_row_off[c] : 0;
        for (int64_t g = cb >> 6; g <= (ce - 1) >> 6 && cb < ce; ++g) {
            const int64_t slot = blk_slot(g, a.seq.lb);
            const uint4 xb = __ldg(bases4 + slot);
            const uint64_t xm = __ldg(a.seq.nmask + slot);
            const int64_t p0 = g << 6;
            const int q0 = int(max64(cb - p0, 0)), q1 = int(min64(ce - p0, 64));
            if (q0 == 0 && q1 == 64 && xm == 0ull) {   // a whole OTHER-free block
#pragma unroll
                for (int q = 0; q < 64; ++q) {
                    const uint32_t w = q < 16 ? xb.x : q < 32 ? xb.y : q < 48 ? xb.z : xb.w;
                    s = wide_hot_step(ht, a.t1w, s, (w >> (2 * (q & 15))) & 3u, lo, H);
                    if constexpr (MODE != kModeMap) {
                        if (s < A) sink.hit(p0 + q, s);
                    }
                }
            } else {
                for (int q = q0; q < q1; ++q) {
                    const uint32_t w = q < 16 ? xb.x : q < 32 ? xb.y : q < 48 ? xb.z : xb.w;
                    const uint32_t y = ((xm >> q) & 1ull) ? 4u : (w >> (2 * (q & 15))) & 3u;
                    s = y == 4u ? reset : wide_hot_step(ht, a.t1w, s, y, lo, H);
                    if constexpr (MODE != kModeMap) {
                        if (s < A) sink.hit(p0 + q, s);
                    }
                }
            }
        }
        if (a.chunk_exit32) a.chunk_exit32[c] = s;
        if constexpr (MODE == kModeRows) a.chunk_rows[c] = sink.nrows;
        if constexpr (MODE == kModeEmit) {
            if (sink.cur != a.chunk_row_off[c + 1]) atomicExch(a.error, 1);
        }
    }
    if (hist_smem) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x)
            if (shist[i]) atomicAdd(&a.visits[i], (unsigned long long)shist[i]);
    }
}

// Count mode, lean steps and dynamic work: warps take tasks of 32 runs of
// U blocks (one run per lane) from a counter, so warps the scheduler favours
// take more and none idles at the end (a static split left 28% of warp time
// at the final barrier).  A run enters by its own lookback (the automaton is
// definite).  A step from a hot state is one shared lookup in the hot table
// -- whose row hot_n is all 0xFFFF, the target of cold states, so there is
// no predicate -- and the warp takes the L2 path only when some lane's next
// state is cold (a warp-uniform branch).  Hits are predicated reductions
// into the shared (HSM) or global visit histogram.  Blocks with OTHER or cut
// by the span edge take the per-symbol path.
template <bool HSM>
__device__ __forceinline__ void red_hit(bool p, uint32_t saddr, unsigned long long* g) {
    if constexpr (HSM) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.add.u32 [%1], 1;\n\t}"
                     :: "r"(uint32_t(p)), "r"(saddr) : "memory");
    } else {
        if (p) atomicAdd(g, 1ull);
    }
}

__device__ __forceinline__ uint32_t lds16u(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

template <bool HSM>
__global__ void __launch_bounds__(1024, 1) scan_wide_hot_ilp_kernel(const ScanArgs a) {
    extern __shared__ __align__(16) unsigned char wh_smem[];
    uint16_t* ht = reinterpret_cast<uint16_t*>(wh_smem);
    const uint32_t H = uint32_t(a.hot_n);
    const size_t ht_bytes = (size_t(H + 1) * 8 + 15) & ~size_t(15);   // + the all-cold row H
    unsigned int* shist = reinterpret_cast<unsigned int*>(wh_smem + ht_bytes);
    // the H hot rows by bulk copies (8-byte rows; an odd H copies 8 bytes of
    // the blob's padding too), then the all-cold sentinel row over them
    __shared__ __align__(8) unsigned long long staged;
    BulkStage st;
    st.begin(&staged, smem_u32(ht), a.ht, uint32_t((size_t(H) * 8 + 15) & ~size_t(15)));
    if (HSM)
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x) shist[i] = 0u;
    st.wait();
    for (size_t i = size_t(H) * 4 + threadIdx.x; i < ht_bytes / 2; i += blockDim.x) ht[i] = 0xFFFFu;
    __syncthreads();
    const uint32_t A = uint32_t(a.n_accept), lo = uint32_t(a.hot_lo);
    const uint32_t reset = uint32_t(a.reset_state);
    const uint32_t ht_s = uint32_t(__cvta_generic_to_shared(ht));
    const uint32_t hist_s = uint32_t(__cvta_generic_to_shared(shist));
    const uint4* bases4 = reinterpret_cast<const uint4*>(a.seq.bases);
    const uint32_t* t1w = a.t1w;
    const int lane = threadIdx.x & 31;
    const int64_t B0 = a.begin >> 6, nB = ((a.end - 1) >> 6) - B0 + 1;
    const int64_t U = a.run_blocks;
    const int64_t ntasks = (nB + U * 32 - 1) / (U * 32);
    auto step = [&](uint32_t x, uint32_t y) -> uint32_t {   // one symbol 0..3 (per-symbol paths)
        const uint32_t e = lds16u(ht_s + min(x - lo, H) * 8u + y * 2u);
        return e != 0xFFFFu ? e + lo : __ldg(&t1w[size_t(x) * 5 + y]);
    };
    for (;;) {
        unsigned int task = 0;
        if (lane == 0) task = atomicAdd(a.work_ctr, 1u);
        task = __shfl_sync(0xffffffffu, task, 0);
        if (int64_t(task) >= ntasks) break;
        const int64_t r = int64_t(task) * 32 + lane;
        const int64_t b0 = min64(B0 + r * U, B0 + nB), b1 = min64(B0 + (r + 1) * U, B0 + nB);
        const int64_t rb = max64(a.begin, b0 << 6), re = min64(a.end, b1 << 6);
        const int nb = int(b1 - b0);
        const int nmax = __reduce_max_sync(0xffffffffu, nb);
        uint32_t Aj = nb > 0 ? A : 0u;   // idle lanes ride along without hits
        uint32_t s = lo;
        if (nb > 0) {   // lookback
            const int64_t lbp = max64(a.base_pos, rb - a.lookback);
            s = uint32_t(lbp == a.base_pos ? a.base_state : a.any_state);
            if ((rb & 63) == 0 && rb - lbp <= 64 && rb > lbp) {
                // the tail of the previous block, from registers (one load)
                const int64_t slot = blk_slot((rb >> 6) - 1, a.seq.lb);
                const uint4 pb = __ldg(bases4 + slot);
                const uint64_t pm = __ldg(a.seq.nmask + slot);
                for (int q = int(64 - (rb - lbp)); q < 64; ++q) {
                    const uint32_t w = q < 16 ? pb.x : q < 32 ? pb.y : q < 48 ? pb.z : pb.w;
                    const uint32_t y = ((pm >> q) & 1ull) ? 4u : (w >> (2 * (q & 15))) & 3u;
                    s = y == 4u ? reset : step(s, y);
                }
            } else {
                for (int64_t p = lbp; p < rb; ++p) {
                    const uint32_t y = seq_sym(a.seq, p);
                    s = y == 4u ? reset : step(s, y);
                }
            }
        }
        uint32_t ex = s;
        for (int k = 0; k < nmax; ++k) {
            uint4 xb = make_uint4(0, 0, 0, 0);
            uint64_t xm = 0;
            bool fast = true;
            const int64_t gb = b0 + k;
            if (k < nb) {
                const int64_t slot = blk_slot(gb, a.seq.lb);
                xm = __ldg(a.seq.nmask + slot);
                xb = __ldg(bases4 + slot);
                fast = xm == 0ull && (gb << 6) >= rb && (gb << 6) + 64 <= re;
            } else {
                if (k == nb) ex = s;
                Aj = 0u;
            }
            if (__all_sync(0xffffffffu, fast)) {
#pragma unroll 1
                for (int wi = 0; wi < 4; ++wi) {
                    const uint32_t w = wi == 0 ? xb.x : wi == 1 ? xb.y : wi == 2 ? xb.z : xb.w;
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const uint32_t y2 = (q == 0 ? (w << 1) : (w >> (2 * q - 1))) & 6u;   // symbol * 2
                        uint32_t e = lds16u(ht_s + min(s - lo, H) * 8u + y2);
                        const bool cold = e == 0xFFFFu;
                        if (__any_sync(0xffffffffu, cold)) {
                            const uint32_t g2 = cold ? __ldg(&t1w[size_t(s) * 5 + (y2 >> 1)]) : 0u;
                            e = cold ? g2 - lo : e;
                        }
                        s = e + lo;
                        red_hit<HSM>(s < Aj, hist_s + s * 4u, a.visits + s);
                    }
                }
            } else if (k < nb) {
                const int64_t p0 = gb << 6;
                const int q0 = int(max64(rb - p0, 0)), q1 = int(min64(re - p0, 64));
                for (int q = q0; q < q1; ++q) {
                    const uint32_t w = q < 16 ? xb.x : q < 32 ? xb.y : q < 48 ? xb.z : xb.w;
                    const uint32_t y = ((xm >> q) & 1ull) ? 4u : (w >> (2 * (q & 15))) & 3u;
                    s = y == 4u ? reset : step(s, y);
                    red_hit<HSM>(s < Aj, hist_s + s * 4u, a.visits + s);
                }
            }
        }
        if (nb == nmax) ex = s;
        if (a.chunk_exit32 && a.nchunks > 0 && nb > 0 && re == a.end) a.chunk_exit32[a.nchunks - 1] = ex;
    }
    if (HSM) {
        __syncthreads();
        for (int i = threadIdx.x; i < a.n_accept; i += blockDim.x)
            if (shist[i]) atomicAdd(&a.visits[i], (unsigned long long)shist[i]);
    }
}

using ScanFn = void (*)(const ScanArgs);

template <int K, bool SM>
ScanFn pick_mode(int mode) {
    switch (mode) {
        case kModeCount: return scan_kernel<K, kModeCount, SM>;
        case kModeRows: return scan_kernel<K, kModeRows, SM>;
        case kModeEmit: return scan_kernel<K, kModeEmit, SM>;
        case kModeMap: return scan_kernel<K, kModeMap, SM>;
    }
    return nullptr;
}

ScanFn pick_kernel(int mode, int stride, bool sm) {
    switch (stride) {
        case 1: return sm ? pick_mode<1, true>(mode) : pick_mode<1, false>(mode);
        case 2: return sm ? pick_mode<2, true>(mode) : pick_mode<2, false>(mode);
        case 3: return sm ? pick_mode<3, true>(mode) : pick_mode<3, false>(mode);
        case 4: return sm ? pick_mode<4, true>(mode) : pick_mode<4, false>(mode);
    }
    return nullptr;
}

size_t scan_smem_bytes(bool smem_tables, int32_t tk_pad, int32_t t1_pad, int32_t hist_words) {
    size_t b = 0;
    if (smem_tables) b += size_t(tk_pad) * 2 + size_t(t1_pad) * 2;
    b += size_t(hist_words) * 4;
    return b;
}

// Threads per CTA and resident CTAs per SM for this instantiation: 512-thread
// CTAs when several fit an SM, otherwise one 1024-thread CTA (big tables).
struct LaunchShape {
    int tpb;
    int per_sm;
};

LaunchShape launch_shape(ScanFn fn, size_t smem) {
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    LaunchShape best{512, 1};
    for (int tpb : {512, 1024}) {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, tpb, smem) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        if (n * tpb > best.tpb * best.per_sm) best = LaunchShape{tpb, n};
    }
    return best;
}

// --------------------------------------------------------------- helpers
__global__ void finalize_counts_kernel(const unsigned long long* visits, int32_t n_accept,
                                       const int32_t* off, const int32_t* ids,
                                       unsigned long long* counts, const uint16_t* exit_src,
                                       uint16_t* exit_dst) {
    if (exit_src && blockIdx.x == 0 && threadIdx.x == 0) *exit_dst = *exit_src;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_accept; s += gridDim.x * blockDim.x) {
        const unsigned long long v = visits[s];
        if (!v) continue;
        for (int k = off[s]; k < off[s + 1]; ++k) atomicAdd(&counts[ids[k]], v);
    }
}


}  // namespace

void chunk_geometry(int64_t begin, int64_t end, int64_t threads, int64_t* origin, int64_t* chunk_len,
                    int64_t* nchunks) {
    const int64_t o = (begin >> 6) << 6;
    const int64_t span = max64(end - o, 1);
    int64_t per = (span + threads - 1) / threads;
    per = ((per + 63) / 64) * 64;
    const char* force = std::getenv("KS_CHUNK_LEN");
    if (force && *force) per = max64(64, (std::atoll(force) + 63) / 64 * 64);
    *origin = o;
    *chunk_len = per;
    *nchunks = (span + per - 1) / per;
}

void scan_geometry(const ks_ctx* ctx, int64_t begin, int64_t end, int stride, bool smem_tables,
                   int32_t tk_pad, int32_t t1_pad, int32_t hist_words, int64_t* origin,
                   int64_t* chunk_len, int64_t* nchunks) {
    const size_t smem = scan_smem_bytes(smem_tables, tk_pad, t1_pad, hist_words);
    ScanFn fn = pick_kernel(kModeCount, stride, smem_tables);
    const LaunchShape sh = fn ? launch_shape(fn, smem) : LaunchShape{512, 1};
    chunk_geometry(begin, end, int64_t(ctx->num_sms) * sh.per_sm * sh.tpb, origin, chunk_len, nchunks);
}

int launch_scan(ks_ctx* ctx, ScanArgs a, int mode, int stride, bool smem_tables, int* launches) {
    if (a.end <= a.begin || a.nchunks <= 0) return KS_OK;
    if (!(mode == kModeCount || mode == kModeRows)) a.hist_smem = 0;
    const int32_t hist_words = a.hist_smem ? a.n_accept : 0;
    const size_t smem = scan_smem_bytes(smem_tables, a.tk_pad, a.t1_pad, hist_words);
    ScanFn fn = pick_kernel(mode, stride, smem_tables);
    if (!fn) return fail(KS_E_INVALID, "scan: bad mode/stride");
    const LaunchShape sh = launch_shape(fn, smem);
    const int64_t need_blocks = (a.nchunks + sh.tpb - 1) / sh.tpb;
    const int64_t max_blocks = int64_t(ctx->num_sms) * sh.per_sm;
    const int blocks = int(max64(1, std::min(need_blocks, max_blocks)));
    fn<<<blocks, sh.tpb, smem, ctx->stream>>>(a);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int launch_finalize_counts(ks_ctx* ctx, const unsigned long long* visits, int32_t n_accept,
                           const int32_t* acc_out_off, const int32_t* acc_out_ids,
                           unsigned long long* counts, const uint16_t* exit_src, uint16_t* exit_dst,
                           int* launches) {
    if (n_accept <= 0 && !exit_src) return KS_OK;
    const int threads = 256;
    const int blocks = std::max(1, std::min((n_accept + threads - 1) / threads, 1024));
    finalize_counts_kernel<<<blocks, threads, 0, ctx->stream>>>(visits, n_accept, acc_out_off,
                                                                  acc_out_ids, counts, exit_src, exit_dst);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int launch_scan_wide(ks_ctx* ctx, ScanArgs a, int mode, int* launches) {
    if (a.end <= a.begin || a.nchunks <= 0) return KS_OK;
    const char* hot_env = std::getenv("KS_WIDE_HOT");
    if (a.ht && a.hot_n > 0 && a.reset_state >= 0 && !(hot_env && *hot_env == '0')) {
        // count mode: the dynamic-task kernel (KS_WIDE_TASKS=0: one chunk per thread)
        const char* tk_env = std::getenv("KS_WIDE_TASKS");
        const bool tasks = mode == kModeCount && !(tk_env && *tk_env == '0');
        const size_t ht_need = (size_t(a.hot_n + 1) * 8 + 15) & ~size_t(15);
        const bool hsm = ht_need + size_t(a.n_accept) * 4 + 1024 <= ctx->smem_optin;
        ScanFn fn = tasks ? (hsm ? scan_wide_hot_ilp_kernel<true> : scan_wide_hot_ilp_kernel<false>)
                  : mode == kModeCount ? scan_wide_hot_kernel<kModeCount>
                  : mode == kModeRows  ? scan_wide_hot_kernel<kModeRows>
                  : mode == kModeEmit  ? scan_wide_hot_kernel<kModeEmit>
                                       : nullptr;
        if (!fn) return fail(KS_E_UNSUPPORTED, "wide automata: mode not supported");
        size_t smem = tasks ? ht_need : align16(size_t(a.hot_n) * 8);
        a.hist_smem = 0;
        if ((mode == kModeCount || mode == kModeRows) && smem + size_t(a.n_accept) * 4 + 1024 <= ctx->smem_optin) {
            a.hist_smem = 1;
            smem += size_t(a.n_accept) * 4;
        }
        KS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(smem)));
        const int threads = 1024;
        int blocks = int(max64(1, min64((a.nchunks + threads - 1) / threads, int64_t(ctx->num_sms))));
        if (tasks) {
            // runs of U blocks, tasks of 32 runs handed out by a counter:
            // about 6 tasks per warp (U in [2, 16]; 256 MiB: U = 3)
            const int64_t nB = ((a.end - 1) >> 6) - (a.begin >> 6) + 1;
            const int64_t warps = int64_t(ctx->num_sms) * (threads / 32);
            a.run_blocks = int32_t(std::max<int64_t>(2, std::min<int64_t>(16, nB / (32 * 6 * warps))));
            if (const char* e = std::getenv("KS_WIDE_RUN_BLOCKS"); e && *e) a.run_blocks = std::max(1, std::atoi(e));
            if (!ctx->wctr) KS_CUDA(cudaMalloc(&ctx->wctr, 256));
            KS_CUDA(cudaMemsetAsync(ctx->wctr, 0, 4, ctx->stream));
            a.work_ctr = ctx->wctr;
            const int64_t ntasks = (nB + int64_t(a.run_blocks) * 32 - 1) / (int64_t(a.run_blocks) * 32);
            blocks = int(max64(1, min64(int64_t(ctx->num_sms), (ntasks + 31) / 32)));
        }
        fn<<<blocks, threads, smem, ctx->stream>>>(a);
        if (launches) ++*launches;
        KS_CUDA(cudaGetLastError());
        return KS_OK;
    }
    ScanFn fn = mode == kModeCount ? scan_wide_kernel<kModeCount>
              : mode == kModeRows  ? scan_wide_kernel<kModeRows>
              : mode == kModeEmit  ? scan_wide_kernel<kModeEmit>
                                   : nullptr;
    if (!fn) return fail(KS_E_UNSUPPORTED, "wide automata: mode not supported");
    size_t smem = 0;
    a.hist_smem = 0;
    if ((mode == kModeCount || mode == kModeRows) && size_t(a.n_accept) * 4 <= 96 * 1024) {
        a.hist_smem = 1;
        smem = size_t(a.n_accept) * 4;
        if (smem > 48 * 1024)
            KS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    }
    const int threads = 256;
    const int blocks = int(max64(1, min64((a.nchunks + threads - 1) / threads, int64_t(ctx->num_sms) * 8)));
    fn<<<blocks, threads, smem, ctx->stream>>>(a);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}


}  // namespace ks
