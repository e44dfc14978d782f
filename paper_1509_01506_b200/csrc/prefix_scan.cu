// Exclusive device-wide scans (reduce-then-scan, three launches).
//
// * rows:   uint32 per-chunk row counts -> int64 exclusive offsets (locate
//           compaction: every chunk writes its rows at its offset, so the
//           concatenation is already sorted by (offset, id) -- no sort, unlike
//           the reference's np.lexsort in engine.py:176);
// * monoid: per-chunk transition-monoid elements -> exclusive prefix
//           elements under the (non-commutative) product table.  This is the
//           composition of chunk "start-state -> end-state" maps that fixes
//           every chunk's true start state (the reference's left-to-right
//           chain walk, engine.py:155-163, done as a scan).
#include <algorithm>

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

template <class Op>
__device__ typename Op::T load_item(const void* in, int64_t i, int64_t n, const Op& op);

template <>
__device__ long long load_item<AddOp>(const void* in, int64_t i, int64_t n, const AddOp& op) {
    return i < n ? (long long)static_cast<const uint32_t*>(in)[i] : op.identity();
}
template <>
__device__ long long load_item<MaxOp>(const void* in, int64_t i, int64_t n, const MaxOp& op) {
    return i < n ? static_cast<const long long*>(in)[i] : op.identity();
}
template <>
__device__ unsigned int load_item<MonoidOp>(const void* in, int64_t i, int64_t n, const MonoidOp& op) {
    return i < n ? (unsigned int)static_cast<const uint16_t*>(in)[i] : op.identity();
}

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

template <class Op>
__global__ void __launch_bounds__(kThreads) tile_reduce(const void* in, int64_t n, Op op,
                                                        typename Op::T* agg) {
    using T = typename Op::T;
    const int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
    T acc = op.identity();
#pragma unroll
    for (int i = 0; i < kItems; ++i) acc = op(acc, load_item<Op>(in, base + i, n, op));
    T total;
    block_exclusive<Op>(acc, op, &total);
    if (threadIdx.x == 0) agg[blockIdx.x] = total;
}

// One block: exclusive scan of the tile aggregates in place, total to *d_total.
template <class Op>
__global__ void __launch_bounds__(kThreads) agg_scan(typename Op::T* agg, int64_t ntiles, Op op,
                                                     typename Op::T* d_total) {
    using T = typename Op::T;
    T carry = op.identity();
    for (int64_t b0 = 0; b0 < ntiles; b0 += kThreads) {
        const int64_t i = b0 + threadIdx.x;
        T v = i < ntiles ? agg[i] : op.identity();
        T total;
        T ex = block_exclusive<Op>(v, op, &total);
        if (i < ntiles) agg[i] = op(carry, ex);
        carry = op(carry, total);
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

template <class Op, class Out>
__global__ void __launch_bounds__(kThreads) tile_scan(const void* in, int64_t n, Op op,
                                                      const typename Op::T* agg_excl, Out* out) {
    using T = typename Op::T;
    const int64_t base = int64_t(blockIdx.x) * kTile + int64_t(threadIdx.x) * kItems;
    T items[kItems];
    T acc = op.identity();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        items[i] = load_item<Op>(in, base + i, n, op);
        acc = op(acc, items[i]);
    }
    T ex = block_exclusive<Op>(acc, op, nullptr);
    T run = op(agg_excl[blockIdx.x], ex);
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if (base + i < n) out[base + i] = Out(run);
        run = op(run, items[i]);
    }
}

template <class Op, class Out>
int run_scan(ks_ctx* ctx, const void* in, int64_t n, const Op& op, Out* out, typename Op::T* d_total,
             void* tmp, int* launches) {
    using T = typename Op::T;
    const int64_t ntiles = std::max<int64_t>(1, (n + kTile - 1) / kTile);
    T* agg = static_cast<T*>(tmp);
    tile_reduce<Op><<<int(ntiles), kThreads, 0, ctx->stream>>>(in, n, op, agg);
    agg_scan<Op><<<1, kThreads, 0, ctx->stream>>>(agg, ntiles, op, d_total);
    if (n > 0) tile_scan<Op, Out><<<int(ntiles), kThreads, 0, ctx->stream>>>(in, n, op, agg, out);
    if (launches) *launches += n > 0 ? 3 : 2;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

}  // namespace

size_t exclusive_scan_rows_tmp_bytes(int64_t n) {
    return size_t(std::max<int64_t>(1, (n + kTile - 1) / kTile)) * sizeof(long long) + 256;
}
size_t exclusive_scan_monoid_tmp_bytes(int64_t n) {
    return size_t(std::max<int64_t>(1, (n + kTile - 1) / kTile)) * sizeof(unsigned int) + 256;
}

int exclusive_scan_rows(ks_ctx* ctx, const uint32_t* in, int64_t n, int64_t* out_excl,
                        int64_t* d_total, void* tmp, int* launches) {
    AddOp op;
    return run_scan<AddOp, long long>(ctx, in, n, op, reinterpret_cast<long long*>(out_excl),
                                      reinterpret_cast<long long*>(d_total), tmp, launches);
}

int exclusive_scan_max(ks_ctx* ctx, const int64_t* in, int64_t n, int64_t* out_excl, int64_t* d_total,
                       void* tmp, int* launches) {
    MaxOp op;
    return run_scan<MaxOp, long long>(ctx, in, n, op, reinterpret_cast<long long*>(out_excl),
                                      reinterpret_cast<long long*>(d_total), tmp, launches);
}

// d_total receives the product of all n elements (as uint16 via a uint32 slot).
int exclusive_scan_monoid(ks_ctx* ctx, const uint16_t* in, int64_t n, const uint16_t* prod,
                          int32_t nm, uint16_t* out_excl, uint16_t* d_total, void* tmp,
                          int* launches) {
    MonoidOp op{prod, nm};
    // the total goes through a 32-bit slot placed after the tile aggregates
    const int64_t ntiles = std::max<int64_t>(1, (n + kTile - 1) / kTile);
    unsigned int* total32 = static_cast<unsigned int*>(tmp) + ntiles;
    int rc = run_scan<MonoidOp, uint16_t>(ctx, in, n, op, out_excl, total32, tmp, launches);
    if (rc != KS_OK) return rc;
    if (d_total) {
        KS_CUDA(cudaMemcpyAsync(d_total, total32, sizeof(uint16_t), cudaMemcpyDeviceToDevice,
                                ctx->stream));
    }
    return KS_OK;
}

}  // namespace ks
