// Exclusive device-wide scans.
//
// * rows:   uint32 per-chunk row counts -> int64 exclusive offsets (locate
//           compaction: every chunk writes its rows at its offset, so the
//           concatenation is already sorted by (offset, id) -- no sort, unlike
//           the reference's np.lexsort in engine.py:176), and the kept-symbol
//           positions of the device compaction: one single-pass launch
//           (decoupled look-back, rows_scan_kernel);
// * max:    the FASTA line state's running maximum (the same single pass);
// * monoid: per-chunk transition-monoid elements -> each chunk's entry state,
//           the composition of chunk "start-state -> end-state" maps (the
//           reference's left-to-right chain walk, engine.py:155-163, done as
//           a scan).  The product is a dependent L2 lookup in the nm x nm
//           table, so depth is what costs: one single-pass launch with
//           decoupled look-back (tiles publish their product, then their
//           inclusive prefix; a tile composes its predecessors' words 32 at a
//           time) that also applies the prefix to the entry state.
#include <mutex>
#include <algorithm>
#include <cstdlib>

#include "scan_kernels.cuh"

namespace ks {
namespace {

constexpr int kThreads = 1024;
constexpr int kItems = 4;
constexpr int kTile = kThreads * kItems;

struct AddOp {
    using T = long long;
    __device__ __forceinline__ T identity() const { return 0; }
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};

struct MaxOp {   // last-terminator positions for FASTA line state (encode.cu)
    using T = long long;
    __device__ __forceinline__ T identity() const { return -1; }
    __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

struct MonoidOp {
    using T = unsigned int;
    const uint16_t* prod;
    int nm;
    __device__ __forceinline__ T identity() const { return 0u; }
    __device__ __forceinline__ T operator()(T a, T b) const {
        return __ldg(&prod[size_t(a) * nm + b]);
    }
};

// Block-wide exclusive scan of one value per thread (order = thread order).
template <class Op>
__device__ typename Op::T block_exclusive(typename Op::T v, const Op& op, typename Op::T* total) {
    using T = typename Op::T;
    __shared__ T warp_tot[kThreads / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x = op(y, x);
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        T w = lane < (kThreads / 32) ? warp_tot[lane] : op.identity();
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w = op(y, w);
        }
        warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    T before_warp = warp ? warp_tot[warp - 1] : op.identity();
    T excl_in_warp = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) excl_in_warp = op.identity();
    if (total) *total = warp_tot[kThreads / 32 - 1];
    T r = op(before_warp, excl_in_warp);
    __syncthreads();  // warp_tot reused by the next call
    return r;
}



// ---------------------------------------------------------------- single pass
// Status word of a tile: epoch << 32 | flag << 16 | element (flag 1: the
// tile's own product, 2: inclusive prefix through the tile).
constexpr unsigned kAgg = 1u, kIncl = 2u;
#ifndef KS_MITEMS   // build-time knob: elements per thread of the monoid scan
#define KS_MITEMS 2
#endif
constexpr int kMItems = KS_MITEMS;
constexpr int kMTile = kThreads * kMItems;

__device__ __forceinline__ unsigned long long status_word(uint32_t epoch, unsigned flag, unsigned v) {
    return (static_cast<unsigned long long>(epoch) << 32) | (flag << 16) | (v & 0xFFFFu);
}

__global__ void __launch_bounds__(kThreads) monoid_entry_scan_kernel(
    const uint16_t* __restrict__ in, int64_t n, MonoidOp op, const uint16_t* __restrict__ action, int32_t nq,
    int32_t entry_val, const uint16_t* entry_ptr, uint16_t* __restrict__ centry, uint16_t* d_total,
    unsigned long long* status, uint32_t epoch) {
    using T = unsigned int;
    __shared__ T s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = (n + kMTile - 1) / kMTile;
    const uint32_t q0 = entry_ptr ? uint32_t(*entry_ptr) : uint32_t(entry_val);
    // tiles in launch order: every tile a CTA waits for belongs to a CTA of
    // this (co-resident) grid that started it earlier
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t base = t * kMTile + int64_t(threadIdx.x) * kMItems;
        T items[kMItems];
        T acc = op.identity();
#pragma unroll
        for (int i = 0; i < kMItems; ++i) {
            items[i] = base + i < n ? T(in[base + i]) : op.identity();
            acc = op(acc, items[i]);
        }
        T total;
        const T ex = block_exclusive<MonoidOp>(acc, op, &total);
        if (warp == 0) {
            T prefix = op.identity();
            if (t == 0) {
                if (lane == 0) atomicExch(&status[0], status_word(epoch, kIncl, total));
            } else {
                if (lane == 0) atomicExch(&status[t], status_word(epoch, kAgg, total));
                // look back over windows of 32 predecessors (lane i: tile j - i)
                T run = op.identity();
                for (int64_t j = t - 1;; j -= 32) {
                    const int64_t k = j - lane;
                    unsigned flag = kIncl;
                    T v = op.identity();
                    if (k >= 0) {
                        unsigned long long w;
                        do {
                            w = atomicAdd(&status[k], 0ull);
                        } while (uint32_t(w >> 32) != epoch);
                        flag = unsigned(w >> 16) & 0xFFFFu;
                        v = T(w & 0xFFFFu);
                    }
                    const unsigned incl = __ballot_sync(0xffffffffu, flag == kIncl);
                    const int stop = incl ? __ffs(incl) - 1 : 32;
                    T x = lane <= stop ? v : op.identity();
                    // product in decreasing lane order (older tiles first)
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const T y = __shfl_down_sync(0xffffffffu, x, d);
                        if (lane + d < 32) x = op(y, x);
                    }
                    run = op(__shfl_sync(0xffffffffu, x, 0), run);
                    if (stop < 32) break;
                }
                prefix = run;
                if (lane == 0) atomicExch(&status[t], status_word(epoch, kIncl, op(prefix, total)));
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (t == ntiles - 1 && d_total) *d_total = uint16_t(op(prefix, total));
            }
        }
        __syncthreads();
        if (centry) {
            T run = op(s_prefix, ex);
#pragma unroll
            for (int i = 0; i < kMItems; ++i) {
                if (base + i < n) centry[base + i] = action[size_t(run) * nq + q0];
                run = op(run, items[i]);
            }
        }
        __syncthreads();   // s_prefix is rewritten by the next tile
    }
}


// Single-pass exclusive sum of uint32 counts into int64 offsets (decoupled
// look-back; replaces three launches on the locate and compaction paths).
// Tile t publishes its sum (flag 1) and then its inclusive prefix (flag 2);
// the flag word carries the call's epoch, values sit in separate arrays
// written before the flag.
template <class Op, class In>   // Op: commutative (sum, max) over long long
__global__ void __launch_bounds__(kThreads) rows_scan_kernel(const In* __restrict__ in, int64_t n,
                                                              long long* __restrict__ out, long long* total,
                                                              unsigned long long* flag, long long* agg,
                                                              long long* inc, uint32_t epoch) {
    using T = long long;
    Op op;
    __shared__ T s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t ntiles = (n + kTile - 1) / kTile;
    const unsigned long long e2 = (unsigned long long)epoch << 2;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t base = t * kTile + int64_t(threadIdx.x) * kItems;
        T items[kItems];
        T acc = op.identity();
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            items[i] = base + i < n ? T(in[base + i]) : op.identity();
            acc = op(acc, items[i]);
        }
        T tot;
        const T ex = block_exclusive<Op>(acc, op, &tot);
        if (warp == 0) {
            T prefix = op.identity();
            if (t == 0) {
                if (lane == 0) {
                    inc[0] = tot;
                    __threadfence();
                    atomicExch(&flag[0], e2 | 2ull);
                }
            } else {
                if (lane == 0) {
                    agg[t] = tot;
                    __threadfence();
                    atomicExch(&flag[t], e2 | 1ull);
                }
                T run = op.identity();
                for (int64_t j = t - 1;; j -= 32) {
                    const int64_t k = j - lane;
                    unsigned f = 2;
                    T v = op.identity();
                    if (k >= 0) {
                        unsigned long long w;
                        do {
                            w = atomicAdd(&flag[k], 0ull);
                        } while ((w >> 2) != (unsigned long long)epoch);
                        f = unsigned(w & 3ull);
                        __threadfence();
                        v = f == 2 ? __ldcg(&inc[k]) : __ldcg(&agg[k]);
                    }
                    const unsigned incl = __ballot_sync(0xffffffffu, f == 2);
                    const int stop = incl ? __ffs(incl) - 1 : 32;
                    T x = lane <= stop ? v : op.identity();
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) x = op(x, __shfl_down_sync(0xffffffffu, x, d));
                    run = op(run, __shfl_sync(0xffffffffu, x, 0));
                    if (stop < 32) break;
                }
                prefix = run;
                if (lane == 0) {
                    inc[t] = op(prefix, tot);
                    __threadfence();
                    atomicExch(&flag[t], e2 | 2ull);
                }
            }
            if (lane == 0) {
                s_prefix = prefix;
                if (t == ntiles - 1 && total) *total = op(prefix, tot);
            }
        }
        __syncthreads();
        T run = op(s_prefix, ex);
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            if (base + i < n) out[base + i] = run;
            run = op(run, items[i]);
        }
        __syncthreads();
    }
}

}  // namespace

size_t exclusive_scan_rows_tmp_bytes(int64_t n) {
    return size_t(std::max<int64_t>(1, (n + kTile - 1) / kTile)) * sizeof(long long) + 256;
}

template <class Op, class In>
int single_pass_scan(ks_ctx* ctx, const In* in, int64_t n, int64_t* out_excl, int64_t* d_total, int* launches) {
    Op op;
    if (n <= 0) {
        if (d_total) {
            const long long id = op.identity();
            KS_CUDA(cudaMemcpyAsync(d_total, &id, 8, cudaMemcpyHostToDevice, ctx->stream));
            KS_CUDA(cudaStreamSynchronize(ctx->stream));   // `id` lives on this stack frame
        }
        return KS_OK;
    }
    const int64_t ntiles = (n + kTile - 1) / kTile;
    if (ctx->rowstat_cap < ntiles) {
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->rowstat) KS_CUDA(cudaFree(ctx->rowstat));
        ctx->rowstat = nullptr;
        ctx->rowstat_cap = 0;
        const int64_t cap = std::max<int64_t>(ntiles, 1024);
        KS_CUDA(cudaMalloc(&ctx->rowstat, size_t(cap) * 24));
        KS_CUDA(cudaMemsetAsync(ctx->rowstat, 0, size_t(cap) * 24, ctx->stream));   // stream-ordered before the scan
        ctx->rowstat_cap = cap;
    }
    if (++ctx->rowepoch == 0) ctx->rowepoch = 1;
    unsigned long long* flag = static_cast<unsigned long long*>(ctx->rowstat);
    long long* agg = reinterpret_cast<long long*>(flag + ctx->rowstat_cap);
    long long* inc = agg + ctx->rowstat_cap;
    int per_sm = 0;
    KS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rows_scan_kernel<Op, In>, kThreads, 0));
    const int64_t grid = std::min<int64_t>(ntiles, int64_t(std::max(per_sm, 1)) * ctx->num_sms);
    rows_scan_kernel<Op, In><<<int(grid), kThreads, 0, ctx->stream>>>(
        in, n, reinterpret_cast<long long*>(out_excl), reinterpret_cast<long long*>(d_total), flag, agg, inc,
        ctx->rowepoch);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int exclusive_scan_rows(ks_ctx* ctx, const uint32_t* in, int64_t n, int64_t* out_excl,
                        int64_t* d_total, void* tmp, int* launches) {
    (void)tmp;
    return single_pass_scan<AddOp, uint32_t>(ctx, in, n, out_excl, d_total, launches);
}

int exclusive_scan_max(ks_ctx* ctx, const int64_t* in, int64_t n, int64_t* out_excl, int64_t* d_total,
                       void* tmp, int* launches) {
    (void)tmp;
    return single_pass_scan<MaxOp, int64_t>(ctx, in, n, out_excl, d_total, launches);
}


}  // namespace ks

namespace ks {

// The persisting-L2 set-aside is a device-wide limit: it is only ever raised
// here (read first, never lowered under another context's window), and the
// value found before the first raise is restored when the last context of the
// device closes (l2_persist_release, called by ks_close).
namespace {
std::mutex g_l2_mu;
struct L2Dev {
    int refs = 0;
    size_t orig = 0;
    bool saved = false;
};
L2Dev g_l2[64];
}  // namespace

void l2_persist_acquire(int device) {
    std::lock_guard<std::mutex> g(g_l2_mu);
    if (device >= 0 && device < 64) ++g_l2[device].refs;
}

void l2_persist_release(ks_ctx* ctx) {
    std::lock_guard<std::mutex> g(g_l2_mu);
    const int dev = ctx->device;
    if (dev < 0 || dev >= 64) return;
    L2Dev& d = g_l2[dev];
    if (--d.refs > 0 || !d.saved) return;
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, d.orig);
    cudaGetLastError();
    d.saved = false;
}

bool l2_persist_attr(ks_ctx* ctx, const void* base, size_t bytes, cudaLaunchAttribute* attr) {
    if (!bytes || !ctx->l2_persist_max || std::getenv("KS_NO_L2_PERSIST")) return false;
    {
        std::lock_guard<std::mutex> g(g_l2_mu);
        size_t cur = 0;
        if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) == cudaSuccess) {
            L2Dev* d = ctx->device >= 0 && ctx->device < 64 ? &g_l2[ctx->device] : nullptr;
            const size_t want = std::min(ctx->l2_persist_max, std::max(cur, bytes));
            if (want > cur && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
                if (d && !d->saved) {
                    d->orig = cur;
                    d->saved = true;
                }
                cur = want;
            }
            ctx->l2_persist = cur;
        }
        cudaGetLastError();
    }
    if (!ctx->l2_persist) return false;
    attr->id = cudaLaunchAttributeAccessPolicyWindow;
    attr->val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr->val.accessPolicyWindow.num_bytes = bytes;
    attr->val.accessPolicyWindow.hitRatio = float(std::min(1.0, double(ctx->l2_persist) / double(bytes)));
    attr->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    return true;
}

int monoid_scan_entries(ks_ctx* ctx, const uint16_t* in, int64_t n, const uint16_t* prod, int32_t nm,
                        const uint16_t* action, int32_t nq, int32_t entry_val, const uint16_t* entry_ptr,
                        uint16_t* centry, uint16_t* d_total, size_t window_bytes, int* launches) {
    if (n <= 0) return KS_OK;
    const int64_t ntiles = (n + kMTile - 1) / kMTile;
    if (ctx->mstat_cap < ntiles) {
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (ctx->mstat) KS_CUDA(cudaFree(ctx->mstat));
        ctx->mstat = nullptr;
        ctx->mstat_cap = 0;
        const int64_t cap = std::max<int64_t>(ntiles, 1024);
        KS_CUDA(cudaMalloc(&ctx->mstat, size_t(cap) * 8));
        KS_CUDA(cudaMemsetAsync(ctx->mstat, 0, size_t(cap) * 8, ctx->stream));   // stream-ordered before the scan
        ctx->mstat_cap = cap;
    }
    if (++ctx->mepoch == 0) ctx->mepoch = 1;   // epoch 0 marks never-written words
    int per_sm = 0;
    KS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, monoid_entry_scan_kernel, kThreads, 0));
    const int64_t grid = std::min<int64_t>(ntiles, int64_t(std::max(per_sm, 1)) * ctx->num_sms);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    if (l2_persist_attr(ctx, prod, window_bytes, &attr[0])) {
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    KS_CUDA(cudaLaunchKernelEx(&cfg, monoid_entry_scan_kernel, in, n, MonoidOp{prod, nm}, action, nq, entry_val,
                               entry_ptr, centry, d_total, ctx->mstat, ctx->mepoch));
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

}  // namespace ks
