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

template <class T>   // state id type of the tables: uint16_t, uint32_t for wide automata
__global__ void speculate_kernel(SeqView seq, const int64_t* cbeg, const int64_t* cend,
                                 const int64_t* pss_off, const T* pss, int32_t window,
                                 const SpecTask* tasks, int32_t ntasks, const T* t1,
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
        s = t1[size_t(s) * 5 + sym];
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
                     const int64_t* d_cend, const int64_t* d_pss_off, const void* d_pss, bool wide,
                     const int64_t* h_pss_off, int32_t window, const void* t1,
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
    if (wide)
        speculate_kernel<uint32_t><<<blocks, threads, 0, ctx->stream>>>(
            seq, d_cbeg, d_cend, d_pss_off, static_cast<const uint32_t*>(d_pss), window,
            static_cast<const SpecTask*>(d_tasks_buf), int32_t(tasks.size()), static_cast<const uint32_t*>(t1),
            n_accept, off, ids, ne, d_conv, d_delta);
    else
        speculate_kernel<uint16_t><<<blocks, threads, 0, ctx->stream>>>(
            seq, d_cbeg, d_cend, d_pss_off, static_cast<const uint16_t*>(d_pss), window,
            static_cast<const SpecTask*>(d_tasks_buf), int32_t(tasks.size()), static_cast<const uint16_t*>(t1),
            n_accept, off, ids, ne, d_conv, d_delta);
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

// ---------------------------------------------------------------- SPECULATE strategy
//
// Entry states for automata that neither synchronise nor have a small
// transition monoid.  Per chunk c >= 1 the candidate entry states are P_x,
// the image of the column of the symbol x before the chunk (the reference's
// possible_starting_states, engine.py:80-91).  One warp per chunk: lane 0
// walks R0 = P_x[0] through the chunk and leaves its trajectory in shared
// memory; then every other candidate walks until it meets R0's trajectory at
// the same step -- from there on it coincides with R0: the reference's
// reconciliation (_kernels.py:89-112) with the window widened to the whole
// chunk -- or until the chunk ends.  The chunk's map candidate -> exit state
// is stored; a chunk whose candidates all leave in one state is "constant".
// chunk_chain_kernel then resolves the entries: every run of non-constant
// chunks is walked by one thread, starting from the constant exit before it
// (or the segment's entry), through the stored maps.  Typical automata
// resolve in parallel; adversarial ones degrade to a sequential walk of the
// maps, never to a re-scan of the bases.  Segments bound the map memory.

namespace {

constexpr int kMapWarps = 4;

__global__ void __launch_bounds__(32 * kMapWarps) chunk_map_kernel(
    SeqView seq, int64_t begin, int64_t end, int64_t origin, int64_t L, int64_t c_lo, int64_t c_hi,
    const uint16_t* __restrict__ t1, const uint16_t* __restrict__ pss, const int32_t* __restrict__ pss_off,
    int32_t pss_max, int32_t entry_val, const uint16_t* entry_ptr, uint16_t* maps, uint8_t* flags,
    uint16_t* cval, uint8_t* psym) {
    extern __shared__ uint16_t traj_all[];   // kMapWarps x (L states + L symbols)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint16_t* traj = traj_all + size_t(warp) * size_t(L) * 3 / 2;
    uint8_t* syms = reinterpret_cast<uint8_t*>(traj + L);
    const int64_t c = c_lo + int64_t(blockIdx.x) * kMapWarps + warp;
    if (c >= c_hi) return;
    const int64_t cb = max64(begin, origin + c * L), ce = min64(end, origin + (c + 1) * L);
    const int64_t len = ce - cb;
    uint32_t first;
    const uint16_t* cand = nullptr;
    int ncand = 1;
    uint32_t x = 5;  // no symbol before the range's first chunk: its entry is given
    if (c == 0) {
        first = entry_val >= 0 ? uint32_t(entry_val) : uint32_t(*entry_ptr);
    } else {
        x = seq_sym(seq, cb - 1);
        cand = pss + pss_off[x];
        ncand = pss_off[x + 1] - pss_off[x];
        first = cand[0];
    }
    for (int64_t j = lane; j < len; j += 32) syms[j] = uint8_t(seq_sym(seq, cb + j));   // unpack once
    __syncwarp();
    if (lane == 0) {
        uint32_t s = first;
        for (int64_t j = 0; j < len; ++j) {
            s = __ldg(&t1[s * 5u + syms[j]]);
            traj[j] = uint16_t(s);
        }
    }
    __syncwarp();
    const uint32_t r0 = traj[len - 1];
    uint16_t* out = maps + size_t(c - c_lo) * size_t(pss_max);
    bool same = true;
    for (int i0 = 0; i0 < ncand; i0 += 32) {  // warp-uniform
        const int i = i0 + lane;
        uint32_t e = r0;
        if (i < ncand && i > 0) {
            uint32_t s = cand[i];
            int64_t j = 0;
            for (; j < len; ++j) {
                s = __ldg(&t1[s * 5u + syms[j]]);
                if (s == traj[j]) break;
            }
            if (j == len) e = s;
        }
        if (i < ncand) out[i] = uint16_t(e);
        same &= __all_sync(0xffffffffu, i >= ncand || e == r0);
    }
    if (lane == 0) {
        flags[c - c_lo] = same ? 1 : 0;
        cval[c - c_lo] = uint16_t(r0);
        psym[c - c_lo] = uint8_t(x);
    }
}

__global__ void chunk_chain_kernel(int64_t c_lo, int64_t c_hi, const uint16_t* __restrict__ maps, int32_t pss_max,
                                   const uint8_t* __restrict__ flags, const uint16_t* __restrict__ cval,
                                   const uint8_t* __restrict__ psym, const int16_t* __restrict__ inv, int32_t nq,
                                   int32_t seg_val, const uint16_t* seg_in, uint16_t* seg_out, uint16_t* centry) {
    for (int64_t c = c_lo + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < c_hi;
         c += int64_t(gridDim.x) * blockDim.x) {
        if (c != c_lo && !(flags[c - 1 - c_lo] & 1)) continue;  // not the start of a run
        uint32_t cur = c != c_lo ? cval[c - 1 - c_lo] : seg_val >= 0 ? uint32_t(seg_val) : uint32_t(*seg_in);
        for (int64_t v = c;; ++v) {
            centry[v] = uint16_t(cur);
            const int64_t k = v - c_lo;
            const bool cst = flags[k] & 1;
            const uint32_t nxt = cst ? cval[k] : maps[size_t(k) * size_t(pss_max) + inv[size_t(psym[k]) * nq + cur]];
            if (v + 1 == c_hi) {
                if (seg_out) *seg_out = uint16_t(nxt);
                break;
            }
            if (cst) break;
            cur = nxt;
        }
    }
}

}  // namespace

size_t speculate_entries_bytes(int64_t seg_chunks, int32_t pss_max) {
    return size_t(seg_chunks) * (size_t(pss_max) * 2 + 4) + 256;
}

int speculate_entries(ks_ctx* ctx, const SeqView& seq, int64_t begin, int64_t end, int64_t origin, int64_t L,
                      int64_t nch, const uint16_t* t1, int32_t nq, const uint16_t* pss, const int32_t* pss_off,
                      const int16_t* inv, int32_t pss_max, int32_t entry_val, const uint16_t* entry_ptr,
                      uint16_t* centry, uint16_t* d_exit, void* buf, int64_t seg_chunks, int* launches) {
    if (nch <= 0) return KS_OK;
    char* p = static_cast<char*>(buf);
    uint16_t* maps = reinterpret_cast<uint16_t*>(p);
    p += align16(size_t(seg_chunks) * size_t(pss_max) * 2);
    uint16_t* cval = reinterpret_cast<uint16_t*>(p);
    p += align16(size_t(seg_chunks) * 2);
    uint8_t* flags = reinterpret_cast<uint8_t*>(p);
    p += align16(size_t(seg_chunks));
    uint8_t* psym = reinterpret_cast<uint8_t*>(p);
    p += align16(size_t(seg_chunks));
    uint16_t* seg_state = reinterpret_cast<uint16_t*>(p);   // ping-pong pair
    const size_t smem = size_t(kMapWarps) * size_t(L) * 3;
    if (L % 2) return fail(KS_E_INVALID, "speculate: odd chunk length");
    if (smem > 48 * 1024)
        KS_CUDA(cudaFuncSetAttribute(chunk_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int k = 0;
    for (int64_t c0 = 0; c0 < nch; c0 += seg_chunks, ++k) {
        const int64_t c1 = min64(nch, c0 + seg_chunks);
        const int64_t n = c1 - c0;
        chunk_map_kernel<<<int((n + kMapWarps - 1) / kMapWarps), 32 * kMapWarps, smem, ctx->stream>>>(
            seq, begin, end, origin, L, c0, c1, t1, pss, pss_off, pss_max, entry_val, entry_ptr, maps, flags, cval,
            psym);
        KS_CUDA(cudaGetLastError());
        const uint16_t* in = c0 == 0 ? entry_ptr : seg_state + (k & 1);
        const int32_t in_val = c0 == 0 ? entry_val : -1;
        uint16_t* out = c1 == nch ? d_exit : seg_state + ((k + 1) & 1);
        const int threads = 256;
        chunk_chain_kernel<<<int(max64(1, min64((n + threads - 1) / threads, 4096))), threads, 0, ctx->stream>>>(
            c0, c1, maps, pss_max, flags, cval, psym, inv, nq, in_val, in, out, centry);
        KS_CUDA(cudaGetLastError());
        if (launches) *launches += 2;
    }
    return KS_OK;
}

}  // namespace ks
