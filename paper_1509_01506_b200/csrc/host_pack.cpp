// Host ASCII -> packed tile-slot format (see host_pack.h).  Symbol rules are
// the device encoder's (encode.cu classify(), reference alphabet.py:20-37):
// a/c/g/t either case -> 0..3 via ((x>>1)^(x>>2))&3, SP/TAB/CR/LF whitespace,
// anything else OTHER.  AVX-512BW does one 64-byte block per iteration;
// other CPUs take a table-driven scalar loop.
#include "host_pack.h"

#include <sched.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <immintrin.h>

#include "ks_internal.h"

namespace ks {

// ------------------------------------------------------------ thread pool

HostPool::HostPool(int threads) {
    for (int i = 1; i < threads; ++i) workers_.emplace_back([this] { worker(); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> lk(m_);
        stop_ = true;
        gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
}

void HostPool::drain() {
    const auto& fn = *fn_;
    for (;;) {
        const int64_t t = next_.fetch_add(1, std::memory_order_relaxed);
        if (t >= ntasks_) break;
        fn(t);
    }
}

void HostPool::worker() {
    uint64_t seen = 0;
    for (;;) {
        // spin ~20-50 us for the next generation, then sleep
        for (int i = 0; i < 20000 && gen_.load(std::memory_order_acquire) == seen; ++i) _mm_pause();
        {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_.load() != seen; });
            if (stop_) return;
            seen = gen_.load();
        }
        drain();
        std::lock_guard<std::mutex> lk(m_);
        if (--active_ == 0) done_.notify_all();
    }
}

void HostPool::run(int64_t ntasks, const std::function<void(int64_t)>& fn) {
    if (ntasks <= 0) return;
    if (workers_.empty() || ntasks == 1) {
        for (int64_t t = 0; t < ntasks; ++t) fn(t);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(m_);
        fn_ = &fn;
        ntasks_ = ntasks;
        next_.store(0);
        active_ = int(workers_.size());
        gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m_);
    done_.wait(lk, [&] { return active_ == 0; });
}

int host_pack_threads() {
    if (const char* s = std::getenv("KS_HOST_THREADS")) {
        const int v = std::atoi(s);
        if (v >= 1) return std::min(v, 256);
    }
    cpu_set_t set;
    int n = 0;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
    if (n < 1) n = int(std::thread::hardware_concurrency());
    return std::max(1, std::min(n, 32));
}

// ------------------------------------------------------------ packing

namespace {

// bit 0-1 code, bit 2 OTHER, bit 3 whitespace
struct Lut {
    uint8_t v[256];
    Lut() {
        for (int x = 0; x < 256; ++x) {
            const int lx = x | 0x20;
            const bool base = lx == 'a' || lx == 'c' || lx == 'g' || lx == 't';
            const bool ws = x == ' ' || x == '\t' || x == '\r' || x == '\n';
            v[x] = uint8_t(base ? (((x >> 1) ^ (x >> 2)) & 3) : ws ? 8 : 4);
        }
    }
};
const Lut kLut;

// Scalar block: `lim` valid bytes (< 64 only for the tail block).
inline void pack_block_scalar(const uint8_t* p, int lim, uint64_t* w, uint64_t* nm, PackFlags* f) {
    uint64_t w0 = 0, w1 = 0, n = 0;
    uint8_t acc = 0;
    for (int i = 0; i < lim; ++i) {
        const uint8_t c = kLut.v[p[i]];
        acc |= c;
        const uint64_t code = c & 3u;
        if (i < 32) w0 |= code << (2 * i);
        else w1 |= code << (2 * (i - 32));
        n |= uint64_t((c >> 2) & 1u) << i;
    }
    w[0] = w0;
    w[1] = w1;
    *nm = n;
    if (acc & 8) f->whitespace = true;
    if (acc & 4) f->other = true;
}

// Classification by nibble lookup: byte x (either case) is a base iff
// LUT_BASE[lo(x)] == hi(x) | 2, its code is LUT_CODE[lo(x)] (= the device
// rule ((x>>1)^(x>>2))&3, which only reads bits 1..3), and it is whitespace
// iff LUT_WS[lo(x)] == hi(x).  Non-base bytes are rare, so zeroing their
// codes and the whitespace test sit behind a branch; pure acgt costs two
// shuffles and one compare per 64 bytes.  Slots advance by 32 within a unit.
__attribute__((target("avx512f,avx512bw"))) PackFlags pack_avx512(const uint8_t* in, int64_t b0, int64_t b1,
                                                                   int lb, uint64_t* bases, uint64_t* nmask,
                                                                   int64_t sbase) {
    const __m512i kf = _mm512_set1_epi8(0x0f), k2 = _mm512_set1_epi8(0x02);
    //                                                        0   1   2   3   4   5   6   7   8   9   a   b   c   d   e   f
    const __m512i lut_base = _mm512_broadcast_i32x4(_mm_setr_epi8(-1, 6, -1, 6, 7, -1, -1, 6, -1, -1, -1, -1, -1, -1, -1, -1));
    const __m512i lut_code = _mm512_broadcast_i32x4(_mm_setr_epi8(0, 0, 1, 1, 3, 3, 2, 2, 2, 2, 3, 3, 1, 1, 0, 0));
    const __m512i lut_ws = _mm512_broadcast_i32x4(_mm_setr_epi8(2, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1, 0, -1, -1));
    const __m512i m16 = _mm512_set1_epi16(0x0401), m32 = _mm512_set1_epi32(0x00100001);
    const int64_t umask = (int64_t(1) << lb) - 1;
    __mmask64 any_ws = 0, any_other = 0;
    int64_t s = blk_slot(b0, lb) - sbase;
    // software prefetch 8 KiB ahead: crosses 4 KiB pages, which the hardware
    // streamer does not (measured on the B200 hosts: 104 -> 145 GB/s, 16 threads)
    static const int pf = std::getenv("KS_PACK_PREFETCH") ? std::atoi(std::getenv("KS_PACK_PREFETCH")) : 8192;
    for (int64_t b = b0; b < b1; ++b) {
        if (pf) _mm_prefetch(reinterpret_cast<const char*>(in + (b << 6) + pf), _MM_HINT_T0);
        const __m512i x = _mm512_loadu_si512(in + (b << 6));
        const __m512i lo = _mm512_and_si512(x, kf);
        const __m512i hi4 = _mm512_and_si512(_mm512_srli_epi16(x, 4), kf);
        const __mmask64 base =
            _mm512_cmpeq_epi8_mask(_mm512_shuffle_epi8(lut_base, lo), _mm512_or_si512(hi4, k2));
        __m512i code = _mm512_shuffle_epi8(lut_code, lo);
        __mmask64 other = ~base;
        if (other) {
            const __mmask64 ws = _mm512_cmpeq_epi8_mask(_mm512_shuffle_epi8(lut_ws, lo), hi4);
            code = _mm512_maskz_mov_epi8(base, code);
            other &= ~ws;
            any_ws |= ws;
            any_other |= other;
        }
        // 4 codes per byte: c0 + 4 c1 (16-bit), then + 16 (c2 + 4 c3) (32-bit)
        const __m512i p32 = _mm512_madd_epi16(_mm512_maddubs_epi16(code, m16), m32);
        _mm_storeu_si128(reinterpret_cast<__m128i*>(bases + 2 * s), _mm512_cvtepi32_epi8(p32));
        nmask[s] = uint64_t(other);
        s = ((b + 1) & umask) ? s + 32 : blk_slot(b + 1, lb) - sbase;
    }
    PackFlags f;
    f.whitespace = any_ws != 0;
    f.other = any_other != 0;
    return f;
}

bool has_avx512bw() {
    static const bool v = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
                          !std::getenv("KS_HOST_SCALAR");
    return v;
}

}  // namespace

namespace {

inline bool pack_codes_block_scalar(const uint8_t* p, int lim, uint64_t* w, uint64_t* nm) {
    uint64_t w0 = 0, w1 = 0, n = 0;
    bool ok = true;
    for (int i = 0; i < lim; ++i) {
        const uint8_t c = p[i];
        ok &= c <= 4;
        const uint64_t code = c & 3u;
        if (i < 32) w0 |= code << (2 * i);
        else w1 |= code << (2 * (i - 32));
        n |= uint64_t(c == 4) << i;
    }
    w[0] = w0;
    w[1] = w1;
    *nm = n;
    return ok;
}

// 64 codes -> 16 B of bases (code & 3; OTHER = 4 packs as 0) + the OTHER mask;
// the same madd packing as the ASCII path after its classification.
__attribute__((target("avx512f,avx512bw"))) bool pack_codes_avx512(const uint8_t* in, int64_t b0, int64_t b1,
                                                                    int lb, uint64_t* bases, uint64_t* nmask,
                                                                    int64_t sbase) {
    const __m512i k3 = _mm512_set1_epi8(3), k4 = _mm512_set1_epi8(4);
    const __m512i m16 = _mm512_set1_epi16(0x0401), m32 = _mm512_set1_epi32(0x00100001);
    const int64_t umask = (int64_t(1) << lb) - 1;
    __mmask64 bad = 0;
    int64_t s = blk_slot(b0, lb) - sbase;
    static const int pf = std::getenv("KS_PACK_PREFETCH") ? std::atoi(std::getenv("KS_PACK_PREFETCH")) : 8192;
    for (int64_t b = b0; b < b1; ++b) {
        if (pf) _mm_prefetch(reinterpret_cast<const char*>(in + (b << 6) + pf), _MM_HINT_T0);
        const __m512i x = _mm512_loadu_si512(in + (b << 6));
        bad |= _mm512_cmpgt_epu8_mask(x, k4);
        const __mmask64 other = _mm512_cmpeq_epi8_mask(x, k4);
        const __m512i code = _mm512_and_si512(x, k3);
        const __m512i p32 = _mm512_madd_epi16(_mm512_maddubs_epi16(code, m16), m32);
        _mm_storeu_si128(reinterpret_cast<__m128i*>(bases + 2 * s), _mm512_cvtepi32_epi8(p32));
        nmask[s] = uint64_t(other);
        s = ((b + 1) & umask) ? s + 32 : blk_slot(b + 1, lb) - sbase;
    }
    return bad == 0;
}

}  // namespace

bool pack_codes_blocks(const uint8_t* codes, int64_t n, int64_t b0, int64_t b1, int lb, uint64_t* bases,
                       uint64_t* nmask, int64_t sbase) {
    bool ok = true;
    const int64_t full = std::min(b1, n >> 6);
    int64_t b = b0;
    if (b < full) {
        if (has_avx512bw()) {
            ok = pack_codes_avx512(codes, b, full, lb, bases, nmask, sbase);
        } else {
            for (int64_t k = b; k < full; ++k) {
                const int64_t s = blk_slot(k, lb) - sbase;
                ok &= pack_codes_block_scalar(codes + (k << 6), 64, bases + 2 * s, nmask + s);
            }
        }
        b = full;
    }
    for (; b < b1; ++b) {
        const int64_t s = blk_slot(b, lb) - sbase;
        const int lim = int(std::max<int64_t>(0, std::min<int64_t>(64, n - (b << 6))));
        ok &= pack_codes_block_scalar(codes + (b << 6), lim, bases + 2 * s, nmask + s);
    }
    return ok;
}

PackFlags pack_ascii_blocks(const uint8_t* in, int64_t n_bytes, int64_t b0, int64_t b1, int lb,
                            uint64_t* bases, uint64_t* nmask, int64_t sbase) {
    PackFlags f;
    const int64_t full = std::min(b1, n_bytes >> 6);   // blocks with all 64 bytes present
    int64_t b = b0;
    if (b < full) {
        if (has_avx512bw()) {
            f = pack_avx512(in, b, full, lb, bases, nmask, sbase);
        } else {
            for (int64_t k = b; k < full; ++k) {
                const int64_t s = blk_slot(k, lb) - sbase;
                pack_block_scalar(in + (k << 6), 64, bases + 2 * s, nmask + s, &f);
            }
        }
        b = full;
    }
    for (; b < b1; ++b) {  // tail block (partial), or blocks past the end
        const int64_t s = blk_slot(b, lb) - sbase;
        const int lim = int(std::max<int64_t>(0, std::min<int64_t>(64, n_bytes - (b << 6))));
        pack_block_scalar(in + (b << 6), lim, bases + 2 * s, nmask + s, &f);
    }
    return f;
}

namespace {

// dst/src 64-byte aligned, bytes a multiple of 64
__attribute__((target("avx512f"))) void stream_copy_avx512(void* dst, const void* src, size_t bytes) {
    char* d = static_cast<char*>(dst);
    const char* s = static_cast<const char*>(src);
    for (size_t i = 0; i < bytes; i += 64)
        _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), _mm512_load_si512(s + i));
}

void stream_copy(void* dst, const void* src, size_t bytes) {
    static const bool nt = !std::getenv("KS_PACK_NT") || std::atoi(std::getenv("KS_PACK_NT")) != 0;
    if (nt && has_avx512bw()) {
        stream_copy_avx512(dst, src, bytes);
    } else {
        std::memcpy(dst, src, bytes);
    }
}

}  // namespace

// ------------------------------------------------------------ wire format for compaction on the device

namespace {

struct BlockMasks {
    uint64_t w0, w1;   // 2-bit codes of all 64 bytes (non-bases 0)
    uint64_t base, ws, term, gt;
};

inline void block_masks_scalar(const uint8_t* p, int lim, BlockMasks* m) {
    uint64_t w0 = 0, w1 = 0, base = 0, ws = 0, term = 0, gt = 0;
    for (int i = 0; i < lim; ++i) {
        const uint8_t x = p[i];
        const uint8_t c = kLut.v[x];
        const uint64_t bit = uint64_t(1) << i;
        if (!(c & 12)) {
            base |= bit;
            if (i < 32) w0 |= uint64_t(c & 3) << (2 * i);
            else w1 |= uint64_t(c & 3) << (2 * (i - 32));
        }
        if (c & 8) ws |= bit;
        if (x == '\n' || x == '\r') term |= bit;
        if (x == '>') gt |= bit;
    }
    *m = BlockMasks{w0, w1, base, ws, term, gt};
}

// Spread the 32 bits of v to the even bit positions of a 64-bit word.
inline uint64_t spread_even(uint32_t v) {
    uint64_t x = v;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

// Mark dropped positions: code 01 and the special bit.
inline void mark_dropped(uint64_t d, uint64_t* w0, uint64_t* w1, uint64_t* sp) {
    const uint64_t m0 = spread_even(uint32_t(d)), m1 = spread_even(uint32_t(d >> 32));
    *w0 = (*w0 & ~(m0 * 3)) | m0;
    *w1 = (*w1 & ~(m1 * 3)) | m1;
    *sp |= d;
}

// Header bytes of a block: from each line start holding '>' up to the next
// line terminator -- one carry chain per header run (F + S).  Updates the
// line state across the block.
inline uint64_t header_mask(const BlockMasks& m, uint64_t valid, int lim, bool* at_ls, bool* in_hdr) {
    const uint64_t F = ~m.term & valid;
    const uint64_t ls = (m.term << 1) | (*at_ls ? 1u : 0u);
    const uint64_t S = (ls & m.gt & F) | (*in_hdr ? 1u : 0u);
    const uint64_t hdr = ((F + S) ^ F) & F;
    *at_ls = (m.term >> (lim - 1)) & 1;
    *in_hdr = (hdr >> (lim - 1)) & 1;
    return hdr;
}

inline int popc64(uint64_t v) { return __builtin_popcountll(v); }

// Per-block bookkeeping shared by both task loops: returns the drop mask.
struct WireLoop {
    WireTask t;
    bool at_ls, in_hdr;
    bool fasta;
    explicit WireLoop(bool fa, int start_state) : at_ls(start_state == 0), in_hdr(start_state == 2), fasta(fa) {
        t.exact = start_state >= 0;
    }
    inline uint64_t drop_of(const BlockMasks& m, int lim) {
        const uint64_t valid = lim == 64 ? ~uint64_t(0) : (uint64_t(1) << lim) - 1;
        const uint64_t hdr = fasta && lim > 0 ? header_mask(m, valid, lim, &at_ls, &in_hdr) : 0;
        return m.ws | hdr | ~valid;
    }
    inline void account(const BlockMasks& m, uint64_t d, int64_t b) {
        const int k = 64 - popc64(d);
        t.kept += k;
        if (fasta && !t.exact && t.first_term < 0) {
            if (m.term) {
                const int ft = __builtin_ctzll(m.term);
                t.first_term = (b << 6) + ft;
                t.prefix_kept += popc64(~d & ((uint64_t(1) << ft) - 1));
            } else {
                t.prefix_kept += k;
            }
        }
    }
    inline WireTask finish() {
        t.end_state = at_ls ? 0 : in_hdr ? 2 : 1;
        return t;
    }
};

WireTask wire_task_scalar(const uint8_t* in, int64_t n_bytes, int64_t b0, int64_t b1, bool fasta, int start_state,
                          uint64_t* bases, uint64_t* special) {
    WireLoop L(fasta, start_state);
    for (int64_t b = b0; b < b1; ++b) {
        const int lim = int(std::max<int64_t>(0, std::min<int64_t>(64, n_bytes - (b << 6))));
        BlockMasks m;
        block_masks_scalar(in + (b << 6), lim, &m);
        const uint64_t d = L.drop_of(m, lim);
        uint64_t w0 = m.w0, w1 = m.w1, sp = ~m.base;
        if (d) mark_dropped(d, &w0, &w1, &sp);
        bases[2 * b] = w0;
        bases[2 * b + 1] = w1;
        special[b] = sp;
        L.account(m, d, b);
    }
    return L.finish();
}

// AVX-512 classification (the nibble LUTs of pack_avx512), BMI2 pdep to
// mark dropped codes, streaming stores (the staging is only read by the DMA).
__attribute__((target("avx512f,avx512bw,bmi2"))) WireTask wire_task_avx512(const uint8_t* in, int64_t n_bytes,
                                                                            int64_t b0, int64_t b1, bool fasta,
                                                                            int start_state, uint64_t* bases,
                                                                            uint64_t* special) {
    WireLoop L(fasta, start_state);
    const __m512i kf = _mm512_set1_epi8(0x0f), k2 = _mm512_set1_epi8(0x02);
    const __m512i lut_base = _mm512_broadcast_i32x4(_mm_setr_epi8(-1, 6, -1, 6, 7, -1, -1, 6, -1, -1, -1, -1, -1, -1, -1, -1));
    const __m512i lut_code = _mm512_broadcast_i32x4(_mm_setr_epi8(0, 0, 1, 1, 3, 3, 2, 2, 2, 2, 3, 3, 1, 1, 0, 0));
    const __m512i lut_ws = _mm512_broadcast_i32x4(_mm_setr_epi8(2, -1, -1, -1, -1, -1, -1, -1, -1, 0, 0, -1, -1, 0, -1, -1));
    const __m512i m16 = _mm512_set1_epi16(0x0401), m32 = _mm512_set1_epi32(0x00100001);
    const __m512i klf = _mm512_set1_epi8('\n'), kcr = _mm512_set1_epi8('\r'), kgt = _mm512_set1_epi8('>');
    for (int64_t b = b0; b < b1; ++b) {
        const int lim = int(std::max<int64_t>(0, std::min<int64_t>(64, n_bytes - (b << 6))));
        BlockMasks m;
        if (lim == 64) {
            const uint8_t* p = in + (b << 6);
            _mm_prefetch(reinterpret_cast<const char*>(p + 8192), _MM_HINT_T0);
            const __m512i x = _mm512_loadu_si512(p);
            const __m512i lo = _mm512_and_si512(x, kf);
            const __m512i hi4 = _mm512_and_si512(_mm512_srli_epi16(x, 4), kf);
            const __mmask64 base = _mm512_cmpeq_epi8_mask(_mm512_shuffle_epi8(lut_base, lo), _mm512_or_si512(hi4, k2));
            const __mmask64 ws = _mm512_cmpeq_epi8_mask(_mm512_shuffle_epi8(lut_ws, lo), hi4);
            const __mmask64 term = _mm512_cmpeq_epi8_mask(x, klf) | _mm512_cmpeq_epi8_mask(x, kcr);
            const __mmask64 gt = _mm512_cmpeq_epi8_mask(x, kgt);
            const __m512i code = _mm512_maskz_mov_epi8(base, _mm512_shuffle_epi8(lut_code, lo));
            const __m128i packed = _mm512_cvtepi32_epi8(_mm512_madd_epi16(_mm512_maddubs_epi16(code, m16), m32));
            m = BlockMasks{uint64_t(_mm_cvtsi128_si64(packed)), uint64_t(_mm_extract_epi64(packed, 1)),
                           uint64_t(base), uint64_t(ws), uint64_t(term), uint64_t(gt)};
        } else {
            block_masks_scalar(in + (b << 6), lim, &m);
        }
        const uint64_t d = L.drop_of(m, lim);
        uint64_t w0 = m.w0, w1 = m.w1, sp = ~m.base;
        if (d) {
            const uint64_t m0 = _pdep_u64(d, 0x5555555555555555ull);
            const uint64_t m1 = _pdep_u64(d >> 32, 0x5555555555555555ull);
            w0 = (w0 & ~(m0 * 3)) | m0;
            w1 = (w1 & ~(m1 * 3)) | m1;
            sp |= d;
        }
        _mm_stream_si64(reinterpret_cast<long long*>(bases + 2 * b), (long long)w0);
        _mm_stream_si64(reinterpret_cast<long long*>(bases + 2 * b + 1), (long long)w1);
        _mm_stream_si64(reinterpret_cast<long long*>(special + b), (long long)sp);
        L.account(m, d, b);
    }
    _mm_sfence();
    return L.finish();
}

}  // namespace

WireTask pack_wire_task(const uint8_t* in, int64_t n_bytes, int64_t b0, int64_t b1, bool fasta, int start_state,
                        uint64_t* bases, uint64_t* special) {
    static const bool simd = has_avx512bw() && __builtin_cpu_supports("bmi2");
    return simd ? wire_task_avx512(in, n_bytes, b0, b1, fasta, start_state, bases, special)
                : wire_task_scalar(in, n_bytes, b0, b1, fasta, start_state, bases, special);
}

void wire_drop_prefix(int64_t b0, int64_t b1, int64_t first_term, uint64_t* bases, uint64_t* special) {
    const int64_t end = first_term < 0 ? (b1 << 6) : first_term;
    for (int64_t b = b0; b < b1 && (b << 6) < end; ++b) {
        const int64_t upto = std::min<int64_t>(64, end - (b << 6));
        const uint64_t d = upto == 64 ? ~uint64_t(0) : (uint64_t(1) << upto) - 1;
        mark_dropped(d, &bases[2 * b], &bases[2 * b + 1], &special[b]);
    }
}

PackFlags pack_ascii_tiles(const uint8_t* in, int64_t n_bytes, int64_t t0, int64_t t1, int lb,
                           uint64_t* bases, uint64_t* nm_compact, int32_t* tile_ids,
                           std::atomic<int32_t>* n_compact) {
    const int64_t tb = int64_t(32) << lb;
    thread_local std::vector<uint64_t> local;
    if (local.size() < size_t(3 * tb + 8)) local.assign(size_t(3 * tb + 8), 0);
    uint64_t* lb_bases = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(local.data()) + 63) & ~uintptr_t(63));
    uint64_t* lb_nm = lb_bases + 2 * tb;
    PackFlags all;
    for (int64_t t = t0; t < t1; ++t) {
        const PackFlags f = pack_ascii_blocks(in, n_bytes, t * tb, (t + 1) * tb, lb, lb_bases, lb_nm, t * tb);
        stream_copy(bases + 2 * t * tb, lb_bases, size_t(tb) * 16);
        if (f.other) {
            const int32_t j = n_compact->fetch_add(1, std::memory_order_relaxed);
            stream_copy(nm_compact + size_t(j) * tb, lb_nm, size_t(tb) * 8);
            tile_ids[j] = int32_t(t);
        }
        all.whitespace |= f.whitespace;
        all.other |= f.other;
    }
    _mm_sfence();   // streaming stores visible before the DMA reads them
    return all;
}

}  // namespace ks
