// Exhaustive reconciliation sweep on the device (reference
// _kernels.py:116-179 reconciliation_sweep, oracle.py:94-116
// exhaustive_reconciliation_check).
//
// For every base word of one length (all 4^L of them) and every border
// symbol class b (candidate start states pss_data[pss_off[b] .. pss_off[b+1]),
// entry 0 = the full run R0), one thread runs the reference's chunk kernel
// on the word -- R0 records its first min(window, L) states and cumulative
// counts; every speculative run i >= 1 stops at the first step j where it
// meets R0's state, then takes counts_i + counts_0 - fr_counts_0[j] and R0's
// final state -- and checks each converged run against an independent full
// scan from its own start state.  Counters (speculative runs, converged
// runs, count mismatches, final-state mismatches) are reduced per block and
// added to four global words.  Tables are the reference Dfa arrays as
// uploaded (original state ids), staged in shared memory.
#include <algorithm>

#include "runtime.h"

namespace {

constexpr int kSweepMaxLen = 13;     // 4^13 words x borders per call
constexpr int kSweepMaxExpr = 16;    // per-thread count arrays
constexpr int kSweepThreads = 256;

struct SweepArgs {
    const int32_t* trans;     // nq x 5
    const int32_t* out_off;   // nq + 1
    const int32_t* out_ids;
    const int32_t* pss;       // candidate sets of all borders
    const int32_t* pss_off;   // n_borders + 1
    int32_t nq, ne, n_borders, length, window;
    int64_t n_words;
    unsigned long long* result;   // [4]
};

__device__ __forceinline__ int32_t step(const int32_t* __restrict__ t, int32_t s, int sym) {
    return __ldg(&t[s * 5 + sym]);
}

__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(const SweepArgs a) {
    extern __shared__ int32_t sm[];
    // stage the tables (small automata; the launcher checks the size)
    int32_t* trans = sm;
    int32_t* off = trans + a.nq * 5;
    int32_t* ids = off + a.nq + 1;
    const int n_ids = __ldg(&a.out_off[a.nq]);
    for (int i = threadIdx.x; i < a.nq * 5; i += blockDim.x) trans[i] = a.trans[i];
    for (int i = threadIdx.x; i <= a.nq; i += blockDim.x) off[i] = a.out_off[i];
    for (int i = threadIdx.x; i < n_ids; i += blockDim.x) ids[i] = a.out_ids[i];
    __syncthreads();

    unsigned long long runs = 0, conv_runs = 0, bad_c = 0, bad_s = 0;
    const int L = a.length;
    const int weff = min(a.window, L);
    const int64_t total = a.n_words * a.n_borders;
    for (int64_t task = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; task < total;
         task += int64_t(gridDim.x) * blockDim.x) {
        const int64_t wid = task / a.n_borders;
        const int b = int(task - wid * a.n_borders);
        const int lo = __ldg(&a.pss_off[b]), nr = __ldg(&a.pss_off[b + 1]) - lo;
        // word[p] = base p; the first position is the most significant digit
        // (the reference's odometer order -- the order does not change the sums)
        auto sym = [&](int p) { return int((wid >> (2 * (L - 1 - p))) & 3); };
        int32_t fr_state[kSweepMaxLen];
        int32_t fr_cnt[kSweepMaxLen][kSweepMaxExpr];
        int32_t c0[kSweepMaxExpr];
        for (int e = 0; e < a.ne; ++e) c0[e] = 0;
        int32_t s = __ldg(&a.pss[lo]);
        for (int j = 0; j < L; ++j) {   // R0: the full run with the recorded window
            s = trans[s * 5 + sym(j)];
            for (int k = off[s]; k < off[s + 1]; ++k) ++c0[ids[k]];
            if (j < weff) {
                fr_state[j] = s;
                for (int e = 0; e < a.ne; ++e) fr_cnt[j][e] = c0[e];
            }
        }
        const int32_t last0 = s;
        for (int i = 1; i < nr; ++i) {
            ++runs;
            const int32_t start = __ldg(&a.pss[lo + i]);
            int32_t ci[kSweepMaxExpr];
            for (int e = 0; e < a.ne; ++e) ci[e] = 0;
            int32_t x = start;
            int conv = -1;
            for (int j = 0; j < L; ++j) {   // the speculative run
                x = trans[x * 5 + sym(j)];
                for (int k = off[x]; k < off[x + 1]; ++k) ++ci[ids[k]];
                if (j < weff && x == fr_state[j]) {
                    conv = j;
                    for (int e = 0; e < a.ne; ++e) ci[e] += c0[e] - fr_cnt[j][e];
                    x = last0;
                    break;
                }
            }
            if (conv < 0) continue;
            ++conv_runs;
            int32_t full[kSweepMaxExpr];   // independent full scan from the run's own start
            for (int e = 0; e < a.ne; ++e) full[e] = 0;
            int32_t y = start;
            for (int j = 0; j < L; ++j) {
                y = trans[y * 5 + sym(j)];
                for (int k = off[y]; k < off[y + 1]; ++k) ++full[ids[k]];
            }
            bool diff = false;
            for (int e = 0; e < a.ne; ++e) diff |= full[e] != ci[e];
            bad_c += diff;
            bad_s += y != x;
        }
    }
    // block reduction of the four counters
    __shared__ unsigned long long red[4][kSweepThreads / 32];
    unsigned long long v[4] = {runs, conv_runs, bad_c, bad_s};
    for (int q = 0; q < 4; ++q) {
        unsigned long long x = v[q];
        for (int o = 16; o; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = x;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long x = 0;
        for (int w = 0; w < int(blockDim.x) / 32; ++w) x += red[threadIdx.x][w];
        if (x) atomicAdd(&a.result[threadIdx.x], x);
    }
}

}  // namespace

extern "C" int ks_reconciliation_sweep(ks_ctx* ctx, const int32_t* transitions, int32_t n_states,
                                       const int32_t* out_offsets, const int32_t* out_ids, int32_t n_expressions,
                                       const int32_t* pss_data, const int32_t* pss_off, int32_t n_borders,
                                       int32_t length, int32_t window, int64_t* result_out) {
    using namespace ks;
    CtxLock lock_(ctx);
    if (!ctx || !transitions || !out_offsets || !pss_data || !pss_off || !result_out || n_states < 1 ||
        n_borders < 1 || length < 0 || window < 0)
        return fail(KS_E_INVALID, "ks_reconciliation_sweep: bad argument");
    if (length > kSweepMaxLen || n_expressions > kSweepMaxExpr)
        return fail(KS_E_UNSUPPORTED, "ks_reconciliation_sweep: length <= 13 and <= 16 expressions");
    const int n_ids = out_offsets[n_states];
    for (int32_t b = 0; b < n_borders; ++b)
        if (pss_off[b + 1] <= pss_off[b]) return fail(KS_E_INVALID, "every border needs a candidate set");
    for (int32_t i = 0; i < pss_off[n_borders]; ++i)
        if (pss_data[i] < 0 || pss_data[i] >= n_states) return fail(KS_E_INVALID, "pss state out of range");
    for (int64_t i = 0; i < int64_t(n_states) * 5; ++i)
        if (transitions[i] < 0 || transitions[i] >= n_states) return fail(KS_E_INVALID, "transition out of range");
    for (int i = 0; i < n_ids; ++i)
        if (out_ids[i] < 0 || out_ids[i] >= n_expressions) return fail(KS_E_INVALID, "output id out of range");
    const size_t smem = (size_t(n_states) * 6 + 1 + size_t(std::max(n_ids, 1))) * 4;
    if (smem > 48 * 1024) return fail(KS_E_UNSUPPORTED, "ks_reconciliation_sweep: automaton too large");
    DeviceGuard guard(ctx->device);
    const size_t tb = size_t(n_states) * 20, ob = size_t(n_states + 1) * 4, ib = size_t(std::max(n_ids, 1)) * 4,
                 pb = size_t(pss_off[n_borders]) * 4, qb = size_t(n_borders + 1) * 4;
    Arena ar;
    int rc = ensure_scratch(ctx, tb + ob + ib + pb + qb + 32 + 8 * kAlign, &ar);
    if (rc) return rc;
    SweepArgs a{};
    a.trans = static_cast<int32_t*>(ar.take(tb));
    a.out_off = static_cast<int32_t*>(ar.take(ob));
    a.out_ids = static_cast<int32_t*>(ar.take(ib));
    a.pss = static_cast<int32_t*>(ar.take(pb));
    a.pss_off = static_cast<int32_t*>(ar.take(qb));
    a.result = static_cast<unsigned long long*>(ar.take(32));
    KS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(a.trans), transitions, tb, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(a.out_off), out_offsets, ob, cudaMemcpyHostToDevice, ctx->stream));
    if (n_ids) KS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(a.out_ids), out_ids, size_t(n_ids) * 4,
                                       cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(a.pss), pss_data, pb, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemcpyAsync(const_cast<int32_t*>(a.pss_off), pss_off, qb, cudaMemcpyHostToDevice, ctx->stream));
    KS_CUDA(cudaMemsetAsync(a.result, 0, 32, ctx->stream));
    a.nq = n_states;
    a.ne = n_expressions;
    a.n_borders = n_borders;
    a.length = length;
    a.window = window;
    a.n_words = int64_t(1) << (2 * length);
    const int64_t tasks = a.n_words * n_borders;
    const int blocks = int(std::max<int64_t>(1, std::min<int64_t>((tasks + kSweepThreads - 1) / kSweepThreads,
                                                                  int64_t(ctx->num_sms) * 16)));
    sweep_kernel<<<blocks, kSweepThreads, smem, ctx->stream>>>(a);
    KS_CUDA(cudaGetLastError());
    unsigned long long host[4];
    KS_CUDA(cudaMemcpyAsync(host, a.result, 32, cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int q = 0; q < 4; ++q) result_out[q] = int64_t(host[q]);
    return KS_OK;
}
