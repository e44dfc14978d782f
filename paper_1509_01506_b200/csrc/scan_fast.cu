// Fast chunked DFA scan for automata with |Q| < 4096 (every config C1-C5).
//
// Layout (all in shared memory, one 1024-thread CTA per SM):
//   * 128 KiB column-major K-stride table: entry for (word w, state s) at
//     byte address (w << LC) | (s << 1), LC = 17 - 2K, value
//     (next << 1) | (hit << 15) where hit = "a state with outputs was entered
//     during these K bases".  Bit 15 lies inside the field [LC, 17) that the
//     next K bases overwrite, so the next lookup address is a single LOP3
//     bit-select of the previous entry and the funnel-shifted input word:
//     per K bases the critical path is SHF -> LOP3 -> LDS.
//   * the 1-base table (|Q|+1) x 5, row-major (x 4 when OTHER resets every
//     state: the column is not stored) for re-walks, OTHER blocks and the
//     lookback;
//   * a per-lane ring of deferred hits, as deep as the shared memory left
//     allows (C3: 15): a flagged step only stores its table address (K = 2:
//     address | entry << 17) with a predicated STS, no divergence; every
//     chk_steps(K) steps the warp votes whether some lane's ring is nearly
//     full and only then calls the out-of-line drain, which resolves every
//     lane's entries (K = 2: the final state from the stored entry, the
//     intermediate one by one 1-base lookup; K > 2: a re-walk) into a
//     shared-memory histogram of accepting-state visits (shared atomics).
//     This replaces the reference's per-symbol CSR output loop
//     (_kernels.py:26-28, 80-84).
//   * lanes of a warp that have no work for a block (N-run blocks, finished
//     chunks) ride the fast path with their hit mask cleared instead of
//     diverging (no sink state: |Q| = 1024 keeps K = 3).
//   * rare-hit automata (LEAN instantiations, chosen from the compile-time
//     hit-rate estimate) scan blocks with no hit bookkeeping at all -- one OR
//     of the entries per step -- and re-run a block only when a lane's OR
//     shows the accept flag (C4: 0.61 -> 0.53 ms).
//   * the fused count of a K = 2 automaton (C3) runs on the visit-class table
//     instead of the ring (CLS instantiation, "visit-class count" below): an
//     accepting step names one histogram slot, hits are queued in registers
//     as 32-bit pairs and flushed by batched shared adds.
//   * items whose 32 lanes scan whole blocks of rows without OTHER (per-tile
//     row flags, SeqView::rowmask) take a plain `load block; scan block` loop
//     in every count and map kernel; the general block loop handles range
//     ends, N runs and sequences without flags (streamed pieces).
// Count mode: the last CTA turns the visit histogram into counts and writes
// them straight into pinned host memory; the kernel is launched with
// programmatic stream serialisation (table staging before
// griddepcontrol.wait), so back-to-back counts overlap.
// The lane/chunk/entry-state logic is the one of scan.cu (lookback, uniform
// or per-chunk entry states).
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cstdlib>

#include "scan_kernels.cuh"

namespace ks {
namespace {

constexpr int kRing = 8;      // minimum ring depth (deferred hits per lane)
constexpr int kRingMax = 32;  // the ring takes what shared memory is left, up to this
// steps between ring-fill checks: every 4th step at K = 2 (high hit rates),
// every 8th otherwise (the vote is pure overhead when hits are rare)
#ifndef KS_CHK2   // build-time tuning knob (make EXTRA=-DKS_CHK2=n)
#define KS_CHK2 4
#endif
__host__ __device__ constexpr int chk_steps(int k) { return k == 2 ? KS_CHK2 : 8; }
constexpr int kFastThreads = 1024;
constexpr int kTileCtrs = 32;   // dynamic-item counters of the count kernel, 128 B apart (ks_ctx::tctr)
constexpr uint32_t kRingStride = 4u * kFastThreads;  // bytes between ring slots

__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// d = (f & m) | (e & ~m) in one LOP3 (the compiler splits it otherwise).
template <uint32_t M>
__device__ __forceinline__ uint32_t bitsel(uint32_t f, uint32_t e) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(f), "r"(e), "n"(M));
    return d;
}
__device__ __forceinline__ void red_shared_add(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Keep a value in a register (stops the compiler from re-deriving shared
// window bases / reloading constants inside the drain loops).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
// K input bases of step j shifted so they start at bit LC; bits outside
// [LC, LC + 2K) are garbage (removed by the bit-select).  x0..x3 are the
// block's 128 bits; compile-time j makes this one SHF (funnel) or nothing.
template <int K>
__device__ __forceinline__ uint32_t field(const uint4& x, int j) {
    constexpr int LC = 17 - 2 * K;
    const int sh = 2 * K * j - LC;  // right shift of the 128-bit stream
    if (sh < 0) return x.x << (-sh);
    const int q = sh >> 5, r = sh & 31;
    const uint32_t lo = q == 0 ? x.x : q == 1 ? x.y : q == 2 ? x.z : x.w;
    const uint32_t hi = q == 0 ? x.y : q == 1 ? x.z : q == 2 ? x.w : 0u;
    if (r == 0) return lo;
    return __funnelshift_r(lo, hi, r);
}

// K >= 3 tables are row-swizzled: (state s, word w) lives at row s ^ (w & 31)
// of column w, so lanes sitting in the same (hot, shallow) state with
// different words hit different banks -- hot states are common for short
// literal sets (C4: 3.98 -> 3.49 simulated wavefronts per warp lookup).
// K = 2 automata are large and flat (C3: no gain), they stay unswizzled.
__host__ __device__ constexpr bool swizzled(int k) { return k >= 3; }

// The K input bases of step j shifted to start at bit AT (bits outside
// [AT, AT + 2K) are garbage).
template <int K, int AT>
__device__ __forceinline__ uint32_t field_at(const uint4& x, int j) {
    const int sh = 2 * K * j - AT;
    if (sh < 0) return x.x << (-sh);
    const int q = sh >> 5, r = sh & 31;
    const uint32_t lo = q == 0 ? x.x : q == 1 ? x.y : q == 2 ? x.z : x.w;
    const uint32_t hi = q == 0 ? x.y : q == 1 ? x.z : q == 2 ? x.w : 0u;
    if (r == 0) return lo;
    return __funnelshift_r(lo, hi, r);
}

// KS_KTIME=1 (diagnostic): per-phase device timestamps of the fast scan,
// min/max over CTAs (globaltimer ns), printed by launch_scan_fast.
__device__ unsigned long long g_ktime[10];
__device__ unsigned long long g_kcta[1024];   // KS_KTIME=2: per CTA: smid << 48 | (flush time - kernel-wide min start) ns
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void kt_mark(int on, int slot, bool is_min, bool per_warp = false) {
    if (on && (per_warp ? (threadIdx.x & 31) == 0 : threadIdx.x == 0)) {
        const unsigned long long t = gtimer();
        if (is_min) atomicMin(&g_ktime[slot], t);
        else atomicMax(&g_ktime[slot], t);
    }
}

struct Ctx {
    uint32_t tk;        // shared address of the K-stride table
    uint32_t t1;        // shared address of the 1-base table
    uint32_t hist;      // shared address of the visit histogram (count/rows)
    const uint16_t* outcnt;
    const int32_t* off;
    const int32_t* ids;
    int64_t* rows;
    int64_t row_base;
    uint32_t n_accept;
    uint32_t ring_thr;  // drain when a lane holds this many ring bytes (depth - chk_steps(K) entries)
    uint32_t t1_cols;   // 4 or 5
    uint32_t reset;     // OTHER target when t1_cols == 4
    uint32_t one;       // ScanArgs::one
    uint32_t hist2;     // class count: hist - 0x10000 (cls_flush)
    LogEntry* log;       // this CTA's segment of the visit log
    uint32_t log_slot;   // shared address of the CTA's visit counter
    uint32_t log_part;   // entries per segment
};

template <int MODE>
struct Lane {
    uint32_t nrows = 0;
    int64_t cur = 0;
    uint32_t ch = 0;
};

template <int MODE>
__device__ __forceinline__ void record(const Ctx& c, Lane<MODE>& L, int64_t pos, uint32_t s) {
    if constexpr (MODE == kModeCount || MODE == kModeRows) {
        red_shared_add(c.hist + 4u * s, 1u);
        if constexpr (MODE == kModeRows) L.nrows += __ldg(&c.outcnt[s]);
    } else if constexpr (MODE == kModeEmit) {
        const int k1 = __ldg(&c.off[s + 1]);
        for (int k = __ldg(&c.off[s]); k < k1; ++k, ++L.cur) {
            longlong2 r;
            r.x = c.row_base + pos + 1;
            r.y = __ldg(&c.ids[k]);
            reinterpret_cast<longlong2*>(c.rows)[L.cur] = r;
        }
    } else if constexpr (MODE == kModeLog) {
        red_shared_add(c.hist + 4u * s, 1u);
        const uint32_t local = L.nrows;
        L.nrows += __ldg(&c.outcnt[s]);
        // a slot in this CTA's segment (a shared-memory counter: one global
        // counter serialised every visit of the grid)
        uint32_t i;
        asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(i) : "r"(c.log_slot) : "memory");
        if (i < c.log_part) {
            LogEntry e;
            e.pos1 = c.row_base + pos + 1;
            e.chunk = L.ch;
            e.local = local;
            e.state = s;
            e.pad = 0;
            c.log[i] = e;
        }
    }
}

__device__ __forceinline__ uint32_t step1(const Ctx& c, uint32_t s, uint32_t sym) {
    if (sym == 4u && c.t1_cols == 4u) return c.reset;   // OTHER column not stored
    return lds16(c.t1 + (s * c.t1_cols + sym) * 2u);
}

// Re-walk one deferred K-step (ring value = its table byte address).
template <int K, int MODE>
__device__ __forceinline__ void rewalk(const Ctx& c, Lane<MODE>& L, uint32_t v, int64_t pos) {
    constexpr int LC = 17 - 2 * K;
    uint32_t s = (v >> 1) & ((1u << (LC - 1)) - 1u);
    if constexpr (swizzled(K)) s ^= (v >> LC) & 31u;   // undo the row swizzle
    const uint32_t w = v >> LC;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        s = step1(c, s, (w >> (2 * i)) & 3u);
        if (s < c.n_accept) record<MODE>(c, L, pos + i, s);
    }
}

// Count/rows resolution of one deferred step.  For K = 2 the ring value is
// address | entry << 17 and the entry's bits 13/14 say which of the two
// states accepts: the final state comes straight from the entry, the
// intermediate one is re-derived (one 1-base lookup) only when it accepts.
template <int K, int MODE>
__device__ __forceinline__ void resolve(const Ctx& c, Lane<MODE>& L, uint32_t a) {
    if constexpr (K == 2) {
        const uint32_t e = a >> 17;
        if (e & 0x2000u) record<MODE>(c, L, 0, step1(c, (a >> 1) & 0xFFFu, (a >> 13) & 3u));
        if (e & 0x4000u) record<MODE>(c, L, 0, (e >> 1) & 0xFFFu);
    } else {
        rewalk<K, MODE>(c, L, a, 0);
    }
}

// Predicated (branch-free) shared-memory helpers for the count drain.
__device__ __forceinline__ uint32_t lds32_if(uint32_t p, uint32_t addr) {
    uint32_t v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q ld.shared.u32 %0, [%2];\n\t}"
                 : "+r"(v) : "r"(p), "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds16_if(uint32_t p, uint32_t addr) {
    unsigned short v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q ld.shared.u16 %0, [%2];\n\t}"
                 : "+h"(v) : "r"(p), "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void red_if(uint32_t p, uint32_t addr) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %0, 0;\n\t@q red.shared.add.u32 [%1], 1;\n\t}"
                 :: "r"(p), "r"(addr) : "memory");
}

#ifndef KS_PDL   // build-time knob: programmatic dependent launch of the fast scan
#define KS_PDL 1
#endif
#ifndef KS_PRED_DRAIN
#define KS_PRED_DRAIN 1
#endif
// Count-mode drain of 2-base ring entries without divergent branches: every
// lane runs every row, the loads and the histogram adds are predicated.
__device__ __forceinline__ void drain_count2(const Ctx& c, uint32_t rp0, uint32_t cnt, uint32_t kmax) {
    for (uint32_t k = 0; k < kmax; ++k) {
        const uint32_t v = lds32_if(k < cnt, rp0 + k * kRingStride);
        const uint32_t e = v >> 17;
        const uint32_t h1 = e & 0x2000u, h2 = e & 0x4000u;
        const uint32_t s1 = lds16_if(h1, c.t1 + (((v >> 1) & 0xFFFu) * c.t1_cols + ((v >> 13) & 3u)) * 2u);
        red_if(h1, c.hist + 4u * s1);
        red_if(h2, c.hist + 4u * ((e >> 1) & 0xFFFu));
    }
}

template <int K, int MODE>
__device__ __forceinline__ void drain(const Ctx& c, Lane<MODE>& L, unsigned am, uint32_t rp0,
                                      uint32_t& rp, uint32_t ring_stride) {
    const uint32_t cnt = (rp - rp0) / kRingStride;
    const uint32_t kmax = __reduce_max_sync(am, cnt);  // warp-uniform trip count
    if constexpr (K == 2 && MODE == kModeCount && KS_PRED_DRAIN) {
        drain_count2(c, rp0, cnt, kmax);
    } else {
        for (uint32_t k = 0; k < kmax; ++k)
            if (k < cnt) resolve<K, MODE>(c, L, lds32(rp0 + k * ring_stride));
    }
    rp = rp0;
}

// Out-of-line drain for the adaptive drain sites inside the unrolled block
// loop (one copy of the resolve code instead of one per site).
template <int K, int MODE>
__device__ __noinline__ uint32_t drain_out(const Ctx c, uint32_t rp0, uint32_t cnt) {
    if constexpr (K == 2 && MODE == kModeCount && KS_PRED_DRAIN) {
        drain_count2(c, rp0, cnt, __reduce_max_sync(0xffffffffu, cnt));
        return 0u;
    }
    Lane<MODE> L;
    const uint32_t kmax = __reduce_max_sync(0xffffffffu, cnt);
    for (uint32_t k = 0; k < kmax; ++k)
        if (k < cnt) resolve<K, MODE>(c, L, lds32(rp0 + k * kRingStride));
    return L.nrows;
}

// A block without hit bookkeeping: the state after it, and in `hm` the OR of
// the entries (bit 15: some state on the way accepts).
template <int K>
__device__ __forceinline__ uint32_t fast_block_lean(const Ctx& c, uint32_t s, const uint4& xb, uint32_t& hm) {
    constexpr int NL = 64 / K;
    constexpr int LC = 17 - 2 * K;
    constexpr uint32_t FM = ((1u << (2 * K)) - 1u) << LC;
    uint32_t e = s << 1, acc = 0;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        uint32_t a = bitsel<FM>(field<K>(xb, j), e);
        if constexpr (swizzled(K)) a ^= field_at<K, 1>(xb, j) & 0x3Eu;
        e = lds16(c.tk + a);
        acc |= e;
    }
    s = (e >> 1) & ((1u << (LC - 1)) - 1u);
    const uint64_t w0 = (uint64_t(xb.y) << 32) | xb.x;
    const uint64_t w1 = (uint64_t(xb.w) << 32) | xb.z;
#pragma unroll
    for (int r = NL * K; r < 64; ++r) {
        s = step1(c, s, uint32_t(r < 32 ? w0 >> (2 * r) : w1 >> (2 * (r - 32))) & 3u);
        acc |= s < c.n_accept ? 0x8000u : 0u;
    }
    hm = acc;
    return s;
}

// One full, OTHER-free 64-base block.  Live lanes (lm = 0x8000) record
// hits; the others (lm = 0: no work for this block) ride along from any
// state without recording, so the warp never diverges.
template <int K, int MODE>
__device__ __forceinline__ uint32_t fast_block(const Ctx& c, Lane<MODE>& L, uint32_t s, uint32_t lm,
                                               const uint4& xb, int64_t p0, unsigned am, uint32_t rp0,
                                               uint32_t& rp, uint32_t ring_stride) {
    const uint64_t w0 = (uint64_t(xb.y) << 32) | xb.x;
    const uint64_t w1 = (uint64_t(xb.w) << 32) | xb.z;
    constexpr int NL = 64 / K;
    constexpr int LC = 17 - 2 * K;
    constexpr uint32_t FM = ((1u << (2 * K)) - 1u) << LC;  // field mask
    constexpr bool RING = MODE == kModeCount || MODE == kModeRows;
    uint32_t e = s << 1;  // entry form of the current state (no flag)
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        uint32_t a = bitsel<FM>(field<K>(xb, j), e);
        if constexpr (swizzled(K)) a ^= field_at<K, 1>(xb, j) & 0x3Eu;   // row = s ^ (w & 31)
        e = lds16(c.tk + a);
        if constexpr (RING) {
            if (e & lm) {
                sts32(rp, K == 2 ? a + (e << 17) : a);
                rp += ring_stride;
            }
            // drain only when some lane's ring is nearly full (checked every
            // chk_steps(K) steps): drains then run with full lanes, and ring entries
            // (table addresses) are position-free, so they may cross blocks
            constexpr int CHK = chk_steps(K);
            // (also after the block's last step: K = 3 has 21 steps, and the
            // 5 after the vote at step 15 plus the next block's first 8 would
            // be 13 pushes between two votes -- with dense hits a lane at the
            // threshold wrote past its ring, into the histogram)
            if (((j % CHK) == CHK - 1 || (NL % CHK != 0 && j == NL - 1)) &&
                __any_sync(am, rp - rp0 >= c.ring_thr)) {
                L.nrows += drain_out<K, MODE>(c, rp0, (rp - rp0) / kRingStride);
                rp = rp0;
            }
        } else if constexpr (MODE == kModeEmit || MODE == kModeLog) {
            if (e & lm) rewalk<K, MODE>(c, L, a, p0 + K * j);
        }
    }
    s = (e >> 1) & ((1u << (LC - 1)) - 1u);
#pragma unroll
    for (int r = NL * K; r < 64; ++r) {  // K == 3 leaves one base
        const uint32_t sym = uint32_t(r < 32 ? w0 >> (2 * r) : w1 >> (2 * (r - 32))) & 3u;
        s = step1(c, s, sym);
        if constexpr (MODE != kModeMap) {
            if (lm && s < c.n_accept) record<MODE>(c, L, p0 + r, s);
        }
    }
    return s;
}


// ---- visit-class count (K = 2, CompiledTable::cls_*) ----------------------
// An accepting K-step's entry is itself the record: (row << 1) | (sub << 13)
// | 0x8000 names the histogram slot (sub << 12) | row that stands for both
// visits of the step.  The entries of two consecutive K-steps make one
// 32-bit pair (e0 | e1 << 16, one multiply-add); a pair in which either step
// accepts (one LOP3 test per two steps) is pushed into a queue of
// KS_CLS_REGS registers per lane by predicated register moves -- nothing is
// stored to shared memory and the ALU pipe, which the scan's shifts,
// bit-selects and tests fill, sees one instruction per two steps (the
// 16-bit shift register of the first version cost three per step).  Every
// two pairs the warp votes whether some lane could overflow before the next
// vote, and only then the lanes add their KS_CLS_FLUSH newest pairs into the
// shared-memory histogram (cls_flush): per flushed slot one red for the
// lanes that hold a pair there (its first accepting half) and a second one
// for the few pairs whose both halves accept; older pairs stay queued.  The
// data pipe then carries the table gathers, the block loads and about one
// red wavefront per five accepting steps -- no ring
// stores, ring loads or intermediate re-walks.  Idle lanes ride along in
// the padding row (state nq), whose entries never accept.
#ifndef KS_CLS_REGS
#define KS_CLS_REGS 6
#endif
#ifndef KS_PLAIN_ALL   // plain items for every count / map kernel (0: the class count only)
#define KS_PLAIN_ALL 1
#endif
#ifndef KS_CLS_UNROLL   // 0: the block's word loop rolled (measured 1.2% slower)
#define KS_CLS_UNROLL 1
#endif
#ifndef KS_CLS_FLUSH   // newest slots flushed when a queue fills (KS_CLS_REGS: all)
#define KS_CLS_FLUSH 2
#endif
constexpr int kClsRegs = KS_CLS_REGS;
constexpr int kClsFlush = KS_CLS_FLUSH < KS_CLS_REGS ? KS_CLS_FLUSH : KS_CLS_REGS;
static_assert(kClsFlush >= 2, "class queue: a flush must make room for the two pushes before the next vote");
static_assert(kClsRegs >= 3, "class queue: two pushes between votes need a spare slot");

struct ClsBuf {
    uint32_t r[kClsRegs];
};
// The class kernel keeps its K-stride table at this absolute shared address
// (the dynamic window is shifted to it): the table base is then an
// instruction immediate, not a uniform register the compiler re-derives
// after every divergent flush.
constexpr uint32_t kClsTkAbs = 0x800;
constexpr size_t kClsSmemPad = 1024;   // room for the shift (launch_scan_fast)
__device__ __forceinline__ uint32_t lds16_tk(uint32_t off) {
    unsigned short v;
    asm("ld.shared.u16 %0, [%1+2048];" : "=h"(v) : "r"(off));
    return v;
}
static_assert(kClsTkAbs == 2048, "lds16_tk's immediate");
// d = s when t != 0, as a predicated multiply-add by the kernel-parameter 1:
// the move runs on the FMA pipe (a plain conditional move compiles to SEL,
// on the ALU pipe the scan saturates).
__device__ __forceinline__ void move_if(uint32_t& d, uint32_t s, uint32_t t, uint32_t one) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p mad.lo.u32 %0, %1, %3, 0;\n\t}"
        : "+r"(d) : "r"(s), "r"(t), "r"(one));
}
// Push `pair` when t != 0 (the newest pair in r[0]).
__device__ __forceinline__ void cls_push_if(ClsBuf& b, uint32_t pair, uint32_t t, uint32_t one) {
#pragma unroll
    for (int i = kClsRegs - 1; i > 0; --i) move_if(b.r[i], b.r[i - 1], t, one);
    move_if(b.r[0], pair, t, one);
}
// hist2: the histogram's shared address - 0x10000 (an accepting entry e has
// bit 15, its slot's byte offset is 2 * (e & 0x7FFF)); one: a
// kernel-parameter 1 (an immediate would become an aggregated increment).
// One queue slot into the histogram: the first accepting half of the pair
// (low when it accepts, else high), then the high half when both accept.
__device__ __forceinline__ void cls_flush_slot(uint32_t hist2, uint32_t x, uint32_t one) {
    asm volatile(
        "{\n\t"
        ".reg .pred p, lo, both;\n\t"
        ".reg .u32 t, h;\n\t"
        "and.b32 t, %0, 0x80008000;\n\t"
        "setp.eq.u32 p, t, 0;\n\t"
        "@p bra DONE;\n\t"
        "and.b32 t, %0, 0x8000;\n\t"
        "setp.ne.u32 lo, t, 0;\n\t"
        "shr.u32 h, %0, 15;\n\t"
        "shl.b32 t, %0, 1;\n\t"
        "selp.u32 t, t, h, lo;\n\t"
        "and.b32 t, t, 0x1FFFC;\n\t"
        "add.u32 t, t, %1;\n\t"
        "red.shared.add.u32 [t], %2;\n\t"
        "setp.lt.and.s32 both, %0, 0, lo;\n\t"
        "@!both bra DONE;\n\t"
        "and.b32 h, h, 0x1FFFC;\n\t"
        "add.u32 h, h, %1;\n\t"
        "red.shared.add.u32 [h], %2;\n\t"
        "DONE:\n\t"
        "}"
        :: "r"(x), "r"(hist2), "r"(one) : "memory");
}
// Flush the NF newest slots of every lane and move the older ones down.  In
// the scan NF = KS_CLS_FLUSH (2): the deep slots are held by a few lanes only
// (24 / 13 / 5 / 1.4 lanes in slots 0..3 when a queue fills), so their adds
// would run nearly empty; kept, they become slots 0 and 1 of a later flush.
template <int NF>
__device__ __forceinline__ void cls_flush(uint32_t hist2, ClsBuf& b, uint32_t one) {
#pragma unroll
    for (int i = 0; i < NF; ++i) cls_flush_slot(hist2, b.r[i], one);
#pragma unroll
    for (int i = 0; i < kClsRegs; ++i) b.r[i] = i + NF < kClsRegs ? b.r[i + NF] : 0u;
}
// One full, OTHER-free 64-base block on the class table: a loop over the
// block's four words (8 steps each; rolled, so the kernel's hot code stays
// small), two votes per word.  The 2 bases of a step reach bits [13, 17) by
// left shifts only (multiplies on the FMA pipe): the upper half of a word is
// shifted down once (y) instead of one funnel shift per step.
__device__ __forceinline__ uint32_t fast_block_cls(const Ctx& c, uint32_t s, const uint4& xb, ClsBuf& b) {
    constexpr int LC = 13;
    constexpr uint32_t FM = 0xFu << LC;
    uint32_t w0 = xb.x, w1 = xb.y, w2 = xb.z, w3 = xb.w;
    uint32_t e = s << 1;
    const uint32_t one = opaque(c.one);   // in a register: no constant-bank load per red
#if KS_CLS_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int q = 0; q < 4; ++q) {
        const uint32_t x = w0, y = w0 >> 16;
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
            const uint32_t f0 = j < 4 ? x << (13 - 4 * j) : y << (29 - 4 * j);
            const uint32_t f1 = j + 1 < 4 ? x << (13 - 4 * (j + 1)) : y << (29 - 4 * (j + 1));
            const uint32_t e0 = lds16_tk(bitsel<FM>(f0, e));
            e = lds16_tk(bitsel<FM>(f1, e0));
            uint32_t pair;
            asm("mad.lo.u32 %0, %1, 65536, %2;" : "=r"(pair) : "r"(e), "r"(e0));
            cls_push_if(b, pair, pair & 0x80008000u, one);
            if ((j & 2) && __any_sync(0xffffffffu, b.r[kClsRegs - 2] != 0u)) cls_flush<kClsFlush>(c.hist2, b, one);
        }
        w0 = w1;
        w1 = w2;
        w2 = w3;
    }
    return (e >> 1) & 0xFFFu;
}

extern __shared__ __align__(128) unsigned char f_smem[];

template <int K, int MODE, bool LEAN = false, bool CLS = false>
__global__ void __launch_bounds__(1024, 1) scan_fast_kernel(const ScanArgs a) {
    static_assert(!CLS || (K == 2 && MODE == kModeCount && !LEAN), "class table: K = 2 count only");
    constexpr bool RING = (MODE == kModeCount || MODE == kModeRows) && !CLS;
    constexpr bool HIST = RING || MODE == kModeLog || CLS;
    const int n_hist = CLS ? a.n_hist : a.n_accept;   // histogram slots
    constexpr int TK_BYTES = 1 << 17;
    // layout: table | t1 | ring (count/rows) | hist (count/rows/log)
    unsigned char* const smem0 = CLS ? f_smem + (kClsTkAbs - smem_addr(f_smem)) : f_smem;
    if constexpr (CLS) {
        if (smem_addr(f_smem) > kClsTkAbs) __trap();   // static shared memory outgrew the fixed table address
    }
    unsigned char* p_t1 = smem0 + TK_BYTES;
    unsigned char* p_ring = p_t1 + size_t(a.t1_pad) * 2;
    unsigned int* s_hist = reinterpret_cast<unsigned int*>(
        p_ring + (RING ? size_t(a.ring_depth) * 4 * kFastThreads : 0));
    // stage the tables with bulk copies (TMA engine, UBLKCP) completing on an
    // mbarrier, while the threads clear the histogram
    __shared__ __align__(8) unsigned long long tables_ready;
    const uint32_t mbar = smem_addr(&tables_ready);
    kt_mark(a.ktime, 0, true);
    kt_mark(a.ktime, 1, false);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t t1_bytes = uint32_t(a.t1_pad) * 2u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(mbar), "r"(uint32_t(TK_BYTES) + t1_bytes) : "memory");
        constexpr uint32_t kPart = 32768;   // bytes per bulk copy
        for (uint32_t o = 0; o < uint32_t(TK_BYTES); o += kPart)
            bulk_copy_g2s(smem_addr(smem0) + o, reinterpret_cast<const char*>(a.tk) + o, kPart, mbar);
        for (uint32_t o = 0; o < t1_bytes; o += kPart)
            bulk_copy_g2s(smem_addr(p_t1) + o, reinterpret_cast<const char*>(a.t1) + o, min(kPart, t1_bytes - o), mbar);
    }
    if constexpr (HIST)
        for (int i = threadIdx.x; i < n_hist; i += blockDim.x) s_hist[i] = 0u;
    // Launched with programmatic stream serialisation: let the next kernel of
    // the stream start as our CTAs retire, and wait for the previous one only
    // before touching memory it may still use -- nothing above reads memory a
    // preceding kernel writes (the tables come from a synchronous upload).
    // A fused count whose chunks are entered by lookback from constants reads
    // only the sequence and the tables while it scans, so it defers the wait
    // to the first write of state shared between calls (chunk exits, the
    // work counter, the visit flush): its CTAs scan while the previous
    // call's last CTA still finalizes and its other CTAs drain.
    // (the map pass of MAPSCAN likewise: every chunk starts from the identity)
    const bool late_wait = KS_PDL && !a.early_wait && !a.chunk_entry && !a.base_state_ptr &&
                           ((MODE == kModeCount && a.fin_counts && a.uniform_entry < 0) ||
                            (MODE == kModeMap && a.uniform_entry >= 0));
    bool waited = !late_wait;
    if constexpr (KS_PDL) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (!late_wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    mbarrier_wait0(mbar);
    __syncthreads();
    kt_mark(a.ktime, 2, true);
    kt_mark(a.ktime, 3, false);

    Ctx c;
    c.tk = smem_addr(smem0);
    c.t1 = opaque(smem_addr(p_t1));
    c.hist = opaque(smem_addr(s_hist));
    c.outcnt = a.acc_outcnt;
    c.off = a.acc_out_off;
    c.ids = a.acc_out_ids;
    c.rows = a.rows;
    c.row_base = a.row_base;
    c.n_accept = opaque(uint32_t(a.n_accept));
    c.ring_thr = uint32_t(a.ring_depth - chk_steps(K)) * kRingStride;
    c.t1_cols = opaque(uint32_t(a.t1_cols));
    c.reset = uint32_t(a.reset_state);
    c.one = a.one;
    c.hist2 = c.hist - 0x10000u;
    c.log = a.log;
    __shared__ unsigned int s_logn;
    c.log = a.log ? a.log + size_t(blockIdx.x) * uint32_t(a.log_part) : nullptr;
    c.log_slot = smem_addr(&s_logn);
    c.log_part = uint32_t(a.log_part);
    if (MODE == kModeLog && threadIdx.x == 0) s_logn = 0u;
    __syncthreads();
    // state of lanes without work: 0 with their hits masked; the class table's
    // padding row, which never accepts
    const uint32_t idle = CLS ? uint32_t(a.nq) : 0u;
    const uint32_t ring_stride = kRingStride;
    const uint32_t rp0 = smem_addr(p_ring) + 4u * threadIdx.x;
    uint32_t rp = rp0;
    ClsBuf cbuf;
#pragma unroll
    for (int i = 0; i < kClsRegs; ++i) cbuf.r[i] = 0u;

    const uint4* bases4 = reinterpret_cast<const uint4*>(a.seq.bases);
    const uint64_t* nmask = a.seq.nmask;
    const int lb = a.seq.lb;
    const int lane = threadIdx.x & 31;
    // Warp w scans tiles t0 + w, t0 + w + nwarps, ...: lane l takes unit
    // 32 t + l, so each block load of the warp is one contiguous 512 B run.
    const int64_t u0 = a.origin / a.chunk_len;
    const int64_t t0 = u0 >> 5;
    const int64_t t1 = (u0 + a.nchunks - 1) >> 5;
    // item bookkeeping in 32 bits (tiles of >= 2048 bases: < 2^31 items for
    // any sequence this library addresses) -- the 64-register budget is tight
    const int nwarps = int((gridDim.x * blockDim.x) >> 5);
    constexpr unsigned am = 0xffffffffu;
    // Work items.  Static: warp w takes tiles t0 + w, t0 + w + nwarps, ...
    // Dynamic (count mode with a tile counter): items are whole tiles, then
    // the last split_tiles tiles cut into split_parts block ranges (lane
    // chunks entered by lookback mid-unit, so the tail is a fraction of a
    // tile); items below static_items go round-robin, the rest come from
    // the counter (fetched one item ahead) -- faster SMs take more of the
    // last rounds.
    const bool dyn = MODE == kModeCount && a.tile_ctr != nullptr;
    const int ntiles = int(t1 - t0 + 1);
    const int whole = dyn ? ntiles - a.split_tiles : ntiles;
    const int n_split1 = (a.split_tiles - a.split2_tiles) * a.split_parts;   // items of the coarser split
    const int n_items = dyn ? whole + n_split1 + a.split2_tiles * a.split2_parts : ntiles;
    const int static_items = int(a.static_items);
    const int ublocks = int(a.chunk_len >> 6);
    const int wid = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    unsigned int* const my_ctr = dyn ? a.tile_ctr + (wid % kTileCtrs) * 32u : nullptr;
    int item = wid;
    for (; item < n_items;) {
        int next = item + nwarps;
        // dynamic items come from kTileCtrs counters 128 B apart (warp w asks
        // counter w % kTileCtrs, which hands out every kTileCtrs-th item): a
        // single counter serialised thousands of warps' first requests.  The
        // request goes out at the start of an item and is read at its end
        // once the preceding kernel is known to be done (the counters are
        // reset by its finalizing CTA); the first one waits for that at the end.
        const bool fetch = dyn && next >= static_items;
        const bool ask_now = fetch && waited;
        unsigned int g = 0;
        if (ask_now && lane == 0) g = atomicAdd(my_ctr, 1u);
        int64_t t;
        int pl = 0, ph = ublocks;   // blocks [pl, ph) of each lane's unit
        if (item < whole) {
            t = t0 + item;
        } else {
            const int j = item - whole;
            const bool fine = j >= n_split1;
            const int jj = fine ? j - n_split1 : j;
            const int parts = fine ? a.split2_parts : a.split_parts;
            t = t0 + whole + (fine ? a.split_tiles - a.split2_tiles : 0) + jj / parts;
            const int q = jj % parts;
            pl = q * ublocks / parts;
            ph = (q + 1) * ublocks / parts;
        }
        const int64_t u = (t << 5) + lane;
        const int64_t ch = u - u0;
        const int64_t cend = min64(a.end, (u + 1) * a.chunk_len);   // the chunk's end
        const int64_t cb0 = max64(a.begin, u * a.chunk_len + (int64_t(pl) << 6));
        const int64_t ce0 = ph == ublocks ? cend : min64(cend, u * a.chunk_len + (int64_t(ph) << 6));
        const bool active = ch >= 0 && ch < a.nchunks && cb0 < ce0;
        const int64_t cb = active ? cb0 : 0;
        const int64_t ce = active ? ce0 : 0;

        uint32_t s = idle;
        if (!active) {
        } else if (a.chunk_entry) {
            s = a.chunk_entry[ch];
        } else if (a.uniform_entry >= 0) {
            s = uint32_t(a.uniform_entry);
        } else {
            int64_t lbp = max64(a.base_pos, cb - a.lookback);
            s = uint32_t(lbp == a.base_pos ? (a.base_state_ptr ? int32_t(*a.base_state_ptr) : a.base_state) : a.any_state);
            if (lbp > a.base_pos && (cb & 63) == 0 && a.lookback <= 64 && a.lookback % K == 0) {
                // whole K-steps over the tail of the previous block, when it has no OTHER there
                const int64_t slot = blk_slot((cb >> 6) - 1, lb);
                const uint64_t xm = __ldg(nmask + slot);
                if (a.lookback == 0 || (xm >> (64 - a.lookback)) == 0) {
                    const uint4 xb = __ldg(bases4 + slot);
                    const uint64_t w0 = (uint64_t(xb.y) << 32) | xb.x, w1 = (uint64_t(xb.w) << 32) | xb.z;
                    constexpr int LC = 17 - 2 * K;
                    for (int q = 64 - a.lookback; q < 64; q += K) {
                        const uint64_t v = q == 0 ? w0 : q < 32 ? (w0 >> (2 * q)) | (w1 << (64 - 2 * q))
                                                               : w1 >> (2 * (q - 32));
                        const uint32_t wv = uint32_t(v) & ((1u << (2 * K)) - 1u);
                        const uint32_t row = swizzled(K) ? (s ^ (wv & 31u)) : s;
                        s = (lds16(c.tk + ((wv << LC) | (row << 1))) >> 1) & ((1u << (LC - 1)) - 1u);
                    }
                    lbp = cb;   // done
                }
            }
            int64_t lbk = -1;
            uint4 xb = make_uint4(0, 0, 0, 0);
            uint64_t xm = 0;
            for (int64_t p = lbp; p < cb; ++p) {  // <= 64 positions, <= 2 blocks
                if ((p >> 6) != lbk) {
                    lbk = p >> 6;
                    const int64_t slot = blk_slot(lbk, lb);
                    xb = __ldg(bases4 + slot);
                    xm = __ldg(nmask + slot);
                }
                const int q = int(p & 63);
                const uint32_t word = q < 16 ? xb.x : q < 32 ? xb.y : q < 48 ? xb.z : xb.w;
                const uint32_t sym = ((xm >> q) & 1ull) ? 4u : (word >> (2 * (q & 15))) & 3u;
                s = step1(c, s, sym);
            }
        }
        Lane<MODE> L;
        if constexpr (MODE == kModeEmit) L.cur = active ? a.chunk_row_off[ch] : 0;
        L.ch = uint32_t(ch);

        // block k of this unit sits at slot ubase + 32 k
        const int64_t ubase = (t << (5 + lb)) | lane;
        const int64_t gfirst = u << lb;  // global block index of the unit's first block
        const int k0 = active ? int((cb >> 6) - gfirst) : 0;
        const int nblk = active ? int(((ce + 63) >> 6) - (cb >> 6)) : 0;
        const int nmax = __reduce_max_sync(am, nblk);  // warp-uniform trip count
        // full (uncut) blocks of this unit are [kfl, kfh)
        const int kfl = k0 + ((cb & 63) != 0);
        const int kfh = active ? int((ce >> 6) - gfirst) : 0;
        const bool resets = a.reset_state >= 0;
        bool dirty = false;   // kModeMap over the submonoid: OTHER inside the chunk
        const uint4* pb = bases4 + ubase + (int64_t(k0) << 5);
        const uint64_t* pm = nmask + ubase + (int64_t(k0) << 5);
        uint4 wb = __ldg(pb);
        // rows of the tile without OTHER (SeqView::rowmask) skip the bitmap loads
        const uint64_t tmask = a.seq.rowmask ? __ldg(a.seq.rowmask + t) : ~0ull;
        uint64_t wm = ((tmask >> (k0 & 63)) & 1ull) ? __ldg(pm) : 0ull;
        // The common item of a count or map pass: whole, aligned block ranges
        // in every lane and no OTHER in any of its rows (SeqView::rowmask) -- a
        // loop of block load + scan, none of the per-lane range and bitmap
        // tests, no votes.  Everything else takes the general loop below.
        bool plain = false;
        if constexpr (KS_PLAIN_ALL ? (MODE == kModeCount || MODE == kModeMap) : CLS) {
            const uint64_t rows = nmax >= 64 ? ~0ull : ((1ull << nmax) - 1ull) << (k0 & 63);
            const int k0u = __shfl_sync(am, k0, 0);
            const bool mine = active & ((cb & 63) == 0) & ((ce & 63) == 0) & (nblk == nmax) & (k0 == k0u) &
                              ((tmask & rows) == 0ull);
            plain = __all_sync(am, mine) && a.seq.rowmask != nullptr;
            if (plain) {
#pragma unroll 1
                for (int i = 0; i < nmax; ++i) {
                    pb += 32;
                    const uint4 nb = __ldg(pb);   // the slot exists: arrays are padded by a whole tile
                    if constexpr (CLS) {
                        s = fast_block_cls(c, s, wb, cbuf);
                    } else if constexpr (LEAN && MODE != kModeMap) {
                        uint32_t hm;
                        uint32_t s2 = fast_block_lean<K>(c, s, wb, hm);
                        if (__any_sync(am, (hm & 0x8000u) != 0u))   // rare: re-run the block recording
                            s2 = fast_block<K, MODE>(c, L, s, 0x8000u, wb, (gfirst + k0 + i) << 6, am, rp0, rp,
                                                     ring_stride);
                        s = s2;
                    } else {
                        s = fast_block<K, MODE>(c, L, s, 0x8000u, wb, (gfirst + k0 + i) << 6, am, rp0, rp,
                                                ring_stride);
                    }
                    wb = nb;
                }
            }
        }
        if (!plain)
        for (int i = 0; i < nmax; ++i) {
            const bool has = i < nblk;
            const int k = k0 + (has ? i : 0);
            // the next slot exists: arrays are padded by a whole tile
            if (has) {
                pb += 32;
                pm += 32;
            }
            const uint4 nb = __ldg(pb);
            const uint64_t nm = ((tmask >> ((k + (has ? 1 : 0)) & 63)) & 1ull) ? __ldg(pm) : 0ull;
            const int64_t p0 = (gfirst + k) << 6;
            const uint64_t w0 = (uint64_t(wb.y) << 32) | wb.x;
            const uint64_t w1 = (uint64_t(wb.w) << 32) | wb.z;
            const uint32_t mlo = uint32_t(wm), mhi = uint32_t(wm >> 32);
            const bool alln = (mlo & mhi) == ~0u;
            const bool clean = (mlo | mhi) == 0u;
            const bool fast = !has || (k >= kfl && k < kfh && (clean || (alln && resets)));
            if constexpr (MODE == kModeMap) {
                if (has && !clean && a.map_dirty) {
                    const int lo = int(max64(cb - p0, 0)), hi = int(min64(ce - p0, 64));
                    const uint64_t rm = (hi >= 64 ? ~0ull : ((1ull << hi) - 1ull)) & (~0ull << lo);
                    dirty |= (wm & rm) != 0ull;
                }
            }
            if (__all_sync(am, fast)) {
                const bool live = has && !alln;
                uint32_t s2;
                // rare-hit automata (a compile-time variant: one path per kernel
                // keeps the registers of the other untouched)
                if constexpr (LEAN && MODE != kModeMap) {
                    uint32_t hm;
                    s2 = fast_block_lean<K>(c, live ? s : idle, wb, hm);
                    if constexpr (MODE == kModeLog) {
                        // rare: the lanes that hit re-walk the block base by base
                        // (a compact loop: the unrolled recording block would not
                        // fit the log mode into 64 registers)
                        if (live && (hm & 0x8000u)) {
                            const uint64_t b0 = (uint64_t(wb.y) << 32) | wb.x, b1 = (uint64_t(wb.w) << 32) | wb.z;
                            uint32_t x = s;
#pragma unroll 1
                            for (int q = 0; q < 64; ++q) {
                                x = step1(c, x, uint32_t(q < 32 ? b0 >> (2 * q) : b1 >> (2 * (q - 32))) & 3u);
                                if (x < c.n_accept) record<MODE>(c, L, p0 + q, x);
                            }
                        }
                    } else if (__any_sync(am, live && (hm & 0x8000u))) {   // rare: re-run the block recording
                        s2 = fast_block<K, MODE>(c, L, live ? s : idle, live ? 0x8000u : 0u, wb, p0, am, rp0, rp,
                                                 ring_stride);
                    }
                } else if constexpr (CLS) {
                    s2 = fast_block_cls(c, live ? s : idle, wb, cbuf);
                } else {
                    s2 = fast_block<K, MODE>(c, L, live ? s : idle, live ? 0x8000u : 0u, wb, p0, am, rp0, rp,
                                             ring_stride);
                }
                if (live) {
                    s = s2;
                } else if (has) {
                    s = uint32_t(a.reset_state);
                    if constexpr (MODE != kModeMap) {
                        if (s < c.n_accept) {
                            if constexpr (MODE == kModeEmit || MODE == kModeLog) {
                                for (int q = 0; q < 64; ++q) record<MODE>(c, L, p0 + q, s);
                            } else {  // count / rows / direct
                                red_shared_add(c.hist + 4u * s, 64u);
                                if constexpr (MODE == kModeRows) L.nrows += 64u * __ldg(&c.outcnt[s]);
                            }
                        }
                    }
                }
            } else if (has) {
                const int lo = int(max64(cb - p0, 0));
                const int hi = int(min64(ce - p0, 64));
                for (int q = lo; q < hi; ++q) {
                    const uint32_t sym = ((wm >> q) & 1ull)
                                             ? 4u
                                             : uint32_t((q < 32 ? w0 >> (2 * q) : w1 >> (2 * (q - 32)))) & 3u;
                    s = step1(c, s, sym);
                    if constexpr (MODE != kModeMap) {
                        if (s < c.n_accept) record<MODE>(c, L, p0 + q, s);
                    }
                }
            }
            if (has) {
                wb = nb;
                wm = nm;
            }
        }
        if constexpr (MODE == kModeRows) drain<K, MODE>(c, L, am, rp0, rp, ring_stride);   // rows are per chunk
        if (active) {
            if constexpr (MODE == kModeMap) {
                if (dirty) s = __ldg(&a.map_dirty[s]);
            }
            if (!waited) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            if (a.chunk_exit && ce == cend) {
                uint32_t sx = s;
                if constexpr (CLS) {
                    if (sx > uint32_t(a.nq)) sx = __ldg(&a.cls_prim[sx]);   // a row copy -> its state
                }
                a.chunk_exit[ch] = uint16_t(sx);
            }
            if constexpr (MODE == kModeRows || MODE == kModeLog) a.chunk_rows[ch] = L.nrows;
            if constexpr (MODE == kModeEmit) {
                if (L.cur != a.chunk_row_off[ch + 1]) atomicExch(a.error, 1);
            }
        }
        if (fetch) {
            if (!ask_now) {
                if (!waited) {
                    asm volatile("griddepcontrol.wait;" ::: "memory");
                    waited = true;
                }
                if (lane == 0) g = atomicAdd(my_ctr, 1u);
            }
            item = static_items + wid % kTileCtrs + kTileCtrs * int(__shfl_sync(am, g, 0));
        } else {
            item = next;
        }
    }

    kt_mark(a.ktime, 4, true, true);
    kt_mark(a.ktime, 5, false, true);
    if constexpr (CLS) {
        cls_flush<kClsRegs>(c.hist2, cbuf, c.one);   // the class queue's leftovers
    } else if constexpr (MODE == kModeCount) {   // the ring's leftovers
        Lane<MODE> L;
        drain<K, MODE>(c, L, am, rp0, rp, ring_stride);
    }
    if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
    if constexpr (HIST) {
        __syncthreads();
        for (int i = threadIdx.x; i < n_hist; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&a.visits[i], (unsigned long long)s_hist[i]);
    }
    __syncthreads();
    if constexpr (MODE == kModeLog) {
        if (threadIdx.x == 0) {   // the segment's length; an overflowing segment poisons the total
            const unsigned int nlog = s_logn;
            a.log_cta_n[blockIdx.x] = nlog;
            atomicAdd(a.log_n, nlog <= uint32_t(a.log_part) ? (unsigned long long)nlog
                                                             : (unsigned long long)a.log_cap + 1ull);
        }
    }
    kt_mark(a.ktime, 6, true);
    kt_mark(a.ktime, 7, false);
    if (a.ktime == 2 && threadIdx.x == 0 && blockIdx.x < 1024) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_kcta[blockIdx.x] = (static_cast<unsigned long long>(smid) << 48) | (gtimer() & 0xFFFFFFFFFFFFull);
    }
    if constexpr (MODE == kModeCount) {
        if (a.fin_counts) {   // fused finalize: the last CTA to finish converts visits to counts
            __shared__ unsigned int is_last;
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) is_last = atomicAdd(a.fin_done, 1u) == gridDim.x - 1;
            __syncthreads();
            if (is_last) {
                kt_mark(a.ktime, 9, false);
                __threadfence();
                if (threadIdx.x == 0 && a.fin_exit_src) *a.fin_exit_dst = __ldcg(a.fin_exit_src);
                // counts accumulate in the (drained) ring's shared memory when they fit
                // (class tables: in the flushed histogram)
                const bool in_smem = CLS ? size_t(a.n_expr) * 8 <= size_t(n_hist) * 4
                                         : size_t(a.n_expr) * 8 <= size_t(a.ring_depth) * 4 * blockDim.x;
                unsigned long long* acc = in_smem ? reinterpret_cast<unsigned long long*>(CLS ? (unsigned char*)s_hist : p_ring)
                                                  : a.fin_counts;
                for (int e = threadIdx.x; e < a.n_expr; e += blockDim.x) acc[e] = 0ull;
                __syncthreads();
                // (class tables: only the slots that can be counted, a compact list)
                const int n_fin = CLS ? a.n_used : n_hist;
                // four slots per thread at a time, their loads issued together
                // (the chain slot id -> visits -> CSR bounds -> ids is 4 dependent
                // L2 round trips per slot)
                constexpr int FB = 4;
                for (int k0 = threadIdx.x; k0 < n_fin; k0 += FB * blockDim.x) {
                    int st[FB], o0[FB], o1[FB];
                    unsigned long long v[FB];
#pragma unroll
                    for (int j = 0; j < FB; ++j) {
                        const int k = k0 + j * int(blockDim.x);
                        st[j] = k < n_fin ? (CLS ? __ldg(&a.cls_used[k]) : k) : -1;
                    }
#pragma unroll
                    for (int j = 0; j < FB; ++j) {
                        v[j] = st[j] >= 0 ? __ldcg(&a.visits[st[j]]) : 0ull;
                        o0[j] = st[j] >= 0 ? __ldg(&a.acc_out_off[st[j]]) : 0;
                        o1[j] = st[j] >= 0 ? __ldg(&a.acc_out_off[st[j] + 1]) : 0;
                    }
#pragma unroll
                    for (int j = 0; j < FB; ++j) {
                        if (!v[j]) continue;
                        a.visits[st[j]] = 0ull;   // clean for the next call
                        for (int k = o0[j]; k < o1[j]; ++k) atomicAdd(&acc[__ldg(&a.acc_out_ids[k])], v[j]);
                    }
                }
                if (!in_smem) __threadfence();
                __syncthreads();
                for (int e = threadIdx.x; e < a.n_expr; e += blockDim.x) {
                    const unsigned long long v = in_smem ? acc[e] : __ldcg(&acc[e]);
                    if (in_smem) a.fin_counts[e] = v;
                    if (a.fin_host) a.fin_host[e] = v;   // pinned host memory: visible once the kernel completes
                }
                if (threadIdx.x == 0) *a.fin_done = 0u;
                if (a.tile_ctr && threadIdx.x < kTileCtrs) a.tile_ctr[threadIdx.x * 32u] = 0u;   // all items taken
                if (a.fin_signal) {   // the counts are final: release them to a stream waiting on the flag
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        __threadfence_system();
                        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.fin_signal), "r"(a.fin_signal_value)
                                     : "memory");
                    }
                }
                kt_mark(a.ktime, 8, false);
            }
        }
    }
}

using FastFn = void (*)(const ScanArgs);

template <int K>
FastFn pick_mode(int mode, bool lean, bool cls) {
    if constexpr (K == 2) {
        if (cls) return mode == kModeCount && !lean ? scan_fast_kernel<2, kModeCount, false, true> : nullptr;
    } else {
        if (cls) return nullptr;
    }
    switch (mode) {
        case kModeCount: return lean ? scan_fast_kernel<K, kModeCount, true> : scan_fast_kernel<K, kModeCount, false>;
        case kModeRows: return lean ? scan_fast_kernel<K, kModeRows, true> : scan_fast_kernel<K, kModeRows, false>;
        case kModeEmit: return lean ? scan_fast_kernel<K, kModeEmit, true> : scan_fast_kernel<K, kModeEmit, false>;
        case kModeMap: return scan_fast_kernel<K, kModeMap>;
        case kModeLog: return lean ? scan_fast_kernel<K, kModeLog, true> : scan_fast_kernel<K, kModeLog, false>;
    }
    return nullptr;
}

// One block per log segment (one per scan CTA): entry i < seg_n[b] of
// segment b; nothing when the log overflowed (*n_dev > cap).
__global__ void log_scatter_kernel(const LogEntry* __restrict__ log, int64_t part, const unsigned int* seg_n,
                                   const unsigned long long* n_dev, int64_t cap, const int64_t* __restrict__ row_off,
                                   const int32_t* __restrict__ off, const int32_t* __restrict__ ids,
                                   int64_t* __restrict__ rows) {
    if (*n_dev > (unsigned long long)cap) return;
    const int64_t n = seg_n[blockIdx.x];
    const LogEntry* seg = log + int64_t(blockIdx.x) * part;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const LogEntry e = seg[i];
        const int64_t base = row_off[e.chunk] + e.local;
        const int k0 = off[e.state], k1 = off[e.state + 1];
        for (int k = k0; k < k1; ++k) {
            longlong2 r;
            r.x = e.pos1;
            r.y = ids[k];
            reinterpret_cast<longlong2*>(rows)[base + (k - k0)] = r;
        }
    }
}

FastFn pick(int mode, int k, bool lean, bool cls) {
    switch (k) {
        case 2: return pick_mode<2>(mode, lean, cls);
        case 3: return pick_mode<3>(mode, lean, cls);
        case 4: return pick_mode<4>(mode, lean, cls);
    }
    return nullptr;
}

int ring_depth_for(size_t fixed, size_t optin, int threads) {
    fixed += 256;   // the static mbarrier of the table staging (+ alignment of the dynamic region)
    if (optin <= fixed) return 0;
    return int(std::min<size_t>(kRingMax, (optin - fixed) / (size_t(4) * threads)));
}

}  // namespace

// Shared memory without the hit ring (the ring takes what is left).
size_t fast_fixed_bytes(int32_t t1_pad, int32_t hist_words) {
    return size_t(1 << 17) + size_t(t1_pad) * 2 + size_t((hist_words + 3) & ~3) * 4;
}

// Smallest configuration the fast kernel accepts (ring of kRing entries).
size_t fast_smem_bytes(int mode, int32_t t1_pad, int32_t hist_words, int threads) {
    const bool ring = mode == kModeCount || mode == kModeRows;
    return fast_fixed_bytes(t1_pad, ring ? hist_words : 0) + (ring ? size_t(kRing) * 4 * threads : 0);
}

int fast_threads() { return kFastThreads; }

int fast_warps_per_cta(int64_t tiles, int num_sms) {
    if (const char* e = std::getenv("KS_FAST_WARPS"); e && *e)   // tuning knob (16..32)
        return std::min(kFastThreads / 32, std::max(16, std::atoi(e)));
    int warps = kFastThreads / 32;
    if (tiles >= int64_t(num_sms) * 24) {
        double best = -1.0;
        for (int w = kFastThreads / 32; w >= 24; --w) {
            const int64_t slots = int64_t(num_sms) * w;
            const int64_t rounds = (tiles + slots - 1) / slots;
            const double eff = double(tiles) / double(rounds * slots);
            if (eff > best + 0.02) {   // fewer warps only when clearly better balanced
                best = eff;
                warps = w;
            }
        }
    }
    return warps;
}

int launch_log_scatter(ks_ctx* ctx, const LogEntry* log, const unsigned int* seg_n, int32_t segs, int64_t part,
                       const unsigned long long* n_dev, int64_t cap, const int64_t* row_off, const int32_t* acc_out_off,
                       const int32_t* acc_out_ids, int64_t* rows, int* launches) {
    if (segs <= 0) return KS_OK;
    log_scatter_kernel<<<segs, 256, 0, ctx->stream>>>(log, part, seg_n, n_dev, cap, row_off, acc_out_off, acc_out_ids,
                                                      rows);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int launch_scan_fast(ks_ctx* ctx, ScanArgs a, int mode, int k, int* launches) {
    if (a.end <= a.begin || a.nchunks <= 0) return KS_OK;
    const bool cls = a.cls != 0;
    const bool ring = (mode == kModeCount || mode == kModeRows) && !cls;
    const bool hist = ring || mode == kModeLog || cls;
    a.hist_smem = hist ? 1 : 0;
    FastFn fn = pick(mode, k, a.lean != 0, cls);
    if (!fn) return fail(KS_E_INVALID, "fast scan: bad mode/stride");
    size_t smem = fast_fixed_bytes(a.t1_pad, cls ? a.n_hist : hist ? a.n_accept : 0);
    if (cls) {
        a.ring_depth = 0;
        smem += kClsSmemPad;   // the window shift to kClsTkAbs
    }
    if (ring) {
        a.ring_depth = ring_depth_for(smem, ctx->smem_optin, kFastThreads);
        if (const char* env = std::getenv("KS_RING_DEPTH"))   // tuning knob
            a.ring_depth = std::min(a.ring_depth, std::max(chk_steps(k) + 1, std::atoi(env)));
        if (a.ring_depth < chk_steps(k) + 1) return fail(KS_E_UNSUPPORTED, "fast scan: no room for the hit ring");
        smem += size_t(a.ring_depth) * 4 * kFastThreads;
    }
    if (smem + 256 > ctx->smem_optin) return fail(KS_E_UNSUPPORTED, "fast scan: shared memory budget exceeded");
    {  // the attribute is per function and device; set it once per size
        static thread_local const void* last_fn[16];
        static thread_local size_t last_smem[16];
        static thread_local int last_dev[16];
        const int slot = int((reinterpret_cast<uintptr_t>(fn) >> 4) & 15);
        if (last_fn[slot] != reinterpret_cast<const void*>(fn) || last_smem[slot] < smem ||
            last_dev[slot] != ctx->device) {
            KS_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
            last_fn[slot] = reinterpret_cast<const void*>(fn);
            last_smem[slot] = smem;
            last_dev[slot] = ctx->device;
        }
    }
    const int64_t u0 = a.origin / a.chunk_len;
    const int64_t tiles = ((u0 + a.nchunks - 1) >> 5) - (u0 >> 5) + 1;
    // one tile (32 units) per warp at a time: when the tiles do not divide
    // into whole rounds over 148 x 32 warps, fewer warps per CTA can (e.g.
    // 4096 tiles: 28 warps x 148 = 4144 slots, one round, instead of 128
    // CTAs with 20 SMs idle); the shared-memory layout stays the 1024-thread one
    const int warps = fast_warps_per_cta(tiles, ctx->num_sms);
    if (const char* e = std::getenv("KS_EARLY_WAIT"); e && *e == '1') a.early_wait = 1;
    // dynamic work items (count mode, fused finalize: its last CTA resets the
    // counter); the last round of tiles is cut into block ranges when lane
    // chunks are entered by lookback (per-chunk or uniform entry states hold
    // only at chunk starts)
    // (seven or more rounds of tiles: with fewer, the extra items' restarts
    // and lookbacks cost more than the balance gains -- isolated C4 shards of
    // 400 M / 800 M bases (3 / 6 rounds) ran 7-9% slower dynamic, C1/C2 (one
    // round) 5-20%; C3 (7 rounds) and C4 (10) gain 1.5-4%)
    const int64_t nw = int64_t(warps) * std::max<int64_t>(1, std::min<int64_t>((tiles + warps - 1) / warps,
                                                                               ctx->num_sms));
    a.tile_ctr = nullptr;
    int64_t dyn_min_rounds = 6;
    if (const char* e = std::getenv("KS_DYN_MIN_ROUNDS"); e && *e) dyn_min_rounds = std::max(1, std::atoi(e));
    if (mode == kModeCount && a.fin_counts && a.dyn_items && tiles > dyn_min_rounds * nw &&
        !(std::getenv("KS_STATIC_TILES") && *std::getenv("KS_STATIC_TILES") == '1')) {
        if (!ctx->tctr) {   // zero once; every fused count's finalizing CTA leaves them zero
            KS_CUDA(cudaMalloc(&ctx->tctr, size_t(kTileCtrs) * 128));
            KS_CUDA(cudaMemsetAsync(ctx->tctr, 0, size_t(kTileCtrs) * 128, ctx->stream));
        }
        a.tile_ctr = ctx->tctr;
        const int ub = int(a.chunk_len >> 6);
        const bool entered_by_lookback = !a.chunk_entry && a.uniform_entry < 0;
        int parts = entered_by_lookback ? std::min(ub, 2) : 1;
        if (const char* e = std::getenv("KS_SPLIT_PARTS"); e && *e && entered_by_lookback)
            parts = std::max(1, std::min(ub, std::atoi(e)));
        a.split_parts = parts;
        a.split_tiles = parts > 1 ? int32_t(std::min<int64_t>(tiles, nw)) : 0;
        // round-robin for all but the last two rounds of items
        // (KS_SPLIT2_PARTS=n: the last half of the split tiles in n ranges; experiment)
        int parts2 = parts;
        if (const char* e = std::getenv("KS_SPLIT2_PARTS"); e && *e && parts > 1) parts2 = std::max(parts, std::min(ub, std::atoi(e)));
        a.split2_parts = parts2;
        a.split2_tiles = parts2 > parts ? a.split_tiles / 2 : 0;
        const int64_t items = tiles - a.split_tiles + int64_t(a.split_tiles - a.split2_tiles) * parts +
                              int64_t(a.split2_tiles) * parts2;
        int64_t dyn_rounds = 2;
        if (const char* e = std::getenv("KS_DYN_ROUNDS"); e && *e) dyn_rounds = std::max(1, std::atoi(e));
        a.static_items = std::max<int64_t>(nw, (items / nw - dyn_rounds) * nw);
    }
    if (const char* e = std::getenv("KS_KTIME"); e && (*e == '1' || *e == '2')) {
        unsigned long long h[10] = {~0ull, 0, ~0ull, 0, ~0ull, 0, ~0ull, 0, 0, 0};
        KS_CUDA(cudaMemcpyToSymbolAsync(g_ktime, h, sizeof(h), 0, cudaMemcpyHostToDevice, ctx->stream));
        a.ktime = *e - '0';
    }
    const int64_t need = (tiles + warps - 1) / warps;
    const int blocks = int(max64(1, min64(need, int64_t(ctx->num_sms))));
    if (mode == kModeLog) {   // the visit log: one segment per CTA
        a.log_part = a.log_cap / blocks;
        ctx->log_segs = blocks;
        ctx->log_part = a.log_part;
    }
    if constexpr (KS_PDL) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(blocks));
        cfg.blockDim = dim3(unsigned(warps * 32));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        // the staged tables (stride table, then the 1-base table) in persisting L2
        const size_t tbytes = size_t(reinterpret_cast<const char*>(a.t1) - reinterpret_cast<const char*>(a.tk)) +
                              size_t(a.t1_pad) * 2;
        if (a.t1 > a.tk && tbytes <= (size_t(1) << 20) && l2_persist_attr(ctx, a.tk, tbytes, &attr[1]))
            cfg.numAttrs = 2;
        KS_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
    } else {
        fn<<<blocks, warps * 32, smem, ctx->stream>>>(a);
    }
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    if (a.ktime) {
        unsigned long long h[10];
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        KS_CUDA(cudaMemcpyFromSymbol(h, g_ktime, sizeof(h)));
        auto us = [&](int i) { return h[i] ? (double(h[i]) - double(h[0])) * 1e-3 : -1.0; };
        std::fprintf(stderr,
                     "[ks ktime] grid %d x %d: CTA start 0..%.2f | tables ready %.2f..%.2f | warp scan end "
                     "%.2f..%.2f | CTA flushed %.2f..%.2f | last CTA found %.2f | finalized %.2f us\n",
                     blocks, warps * 32, us(1), us(2), us(3), us(4), us(5), us(6), us(7), us(9), us(8));
        if (a.ktime == 2) {
            std::vector<unsigned long long> c(size_t(std::min(blocks, 1024)));
            KS_CUDA(cudaMemcpyFromSymbol(c.data(), g_kcta, c.size() * 8));
            std::fprintf(stderr, "[ks ktime cta] smid:us");
            for (size_t i = 0; i < c.size(); ++i)
                std::fprintf(stderr, " %u:%.1f", unsigned(c[i] >> 48),
                             (double(c[i] & 0xFFFFFFFFFFFFull) - double(h[0] & 0xFFFFFFFFFFFFull)) * 1e-3);
            std::fprintf(stderr, "\n");
        }
    }
    return KS_OK;
}

}  // namespace ks
