// Device encode: ASCII / symbol codes -> packed device sequence (K1).
//
// Reference semantics (alphabet.py:20-37, ingest.py:67-69): a/c/g/t in either
// case -> 0..3 (lowercase soft-masking does not change matching); SP, TAB,
// CR, LF dropped; any other byte -> OTHER.  Device form (ks_seq):
//   bases : uint64[], 2 bits per base (base i at bits 2*(i%32) of word i/32)
//   nmask : uint64[], OTHER bitmap (bit i%64 of word i/64)
//   soft  : uint64[], lowercase-letter bitmap (informational, never scanned)
// One thread packs one 64-base block: 64 input bytes -> 16 B + 8 B + 8 B.
// Whitespace-free input (the common case) is written in place in a single
// pass; otherwise per-block kept counts are scanned and a compaction pass
// ORs each block's bits into their shifted output position.  FASTA input
// (ingest.py:65-66: lines starting with '>' dropped, CR/LF/CRLF line ends)
// adds one pass: each block's last line terminator, an exclusive running-max
// scan of those, and from it the line state at every block start.
#include <algorithm>

#include "scan_kernels.cuh"

namespace ks {
namespace {

struct Packed {
    uint64_t w0, w1, n, soft;
    uint32_t kept;
};

// Classify one ASCII byte: code bits, OTHER, lowercase, whitespace.
__device__ __forceinline__ void classify(uint32_t x, uint32_t& code, bool& other, bool& lower,
                                         bool& ws) {
    const uint32_t lx = x | 0x20u;
    const bool base = (lx == 'a') | (lx == 'c') | (lx == 'g') | (lx == 't');
    // a->0 c->1 g->2 t->3 from bits 1..3 of the byte, either case
    code = ((x >> 1) ^ (x >> 2)) & 3u;
    ws = (x == ' ') | (x == '\t') | (x == '\r') | (x == '\n');
    other = !base && !ws;
    lower = (x >= 'a') & (x <= 'z');
    if (!base) code = 0;
}

// FASTA line state (reference ingest.py:65-66 via bytes.splitlines: CR, LF
// and CRLF end lines; a line whose first byte is '>' is dropped whole).
// `carry` codes the state before the first byte of a piece: 0 = at a line
// start, 1 = inside a sequence line, 2 = inside a header line.
struct LineState {
    bool at_ls;   // the previous byte ended a line (or input start)
    bool in_hdr;  // inside a header line
};

__device__ __forceinline__ bool is_term(uint32_t x) { return x == '\n' || x == '\r'; }

// State at the start of block b: from the last line terminator before the
// block (lt_excl[b], exclusive running max) or, when the piece has none, the
// carry.
__device__ __forceinline__ LineState block_start_state(const uint8_t* in, int64_t b, const int64_t* lt_excl,
                                                       int carry) {
    LineState st;
    if (b == 0) {
        st.at_ls = carry == 0;
        st.in_hdr = carry == 2;
        return st;
    }
    const int64_t t = lt_excl[b];
    st.at_ls = t == (b << 6) - 1;
    if (st.at_ls) st.in_hdr = false;
    else if (t >= 0) st.in_hdr = in[t + 1] == '>';
    else st.in_hdr = carry == 0 ? in[0] == '>' : carry == 2;
    return st;
}

__device__ __forceinline__ int carry_of(const LineState& st) { return st.at_ls ? 0 : st.in_hdr ? 2 : 1; }

// Load the 64 bytes of block b as 16 words; bytes past n_bytes read as SP.
__device__ __forceinline__ void load_block(const uint8_t* in, int64_t n_bytes, int64_t b, uint32_t words[16]) {
    const int64_t p0 = b << 6;
    const int lim = int(min64(64, n_bytes - p0));
    if (lim == 64 && ((reinterpret_cast<uintptr_t>(in) & 15) == 0)) {
        const uint4* src = reinterpret_cast<const uint4*>(in + p0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 v = __ldg(src + q);
            words[4 * q] = v.x;
            words[4 * q + 1] = v.y;
            words[4 * q + 2] = v.z;
            words[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            uint32_t w = 0;
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * q + k;
                // pad bytes past the end with SP: dropped, contributes nothing
                const uint32_t byte = i < lim ? in[p0 + i] : uint32_t(' ');
                w |= byte << (8 * k);
            }
            words[q] = w;
        }
    }
}

// Encode the 64 bytes of block b (bytes past n_bytes are treated as dropped).
// FASTA: `st` enters as the line state at the block start and leaves as the
// state after its last real byte.
template <bool FASTA = false>
__device__ __forceinline__ Packed pack_block(const uint8_t* in, int64_t n_bytes, int64_t b, bool compact,
                                             LineState* st = nullptr) {
    Packed r{0, 0, 0, 0, 0};
    uint32_t words[16];
    load_block(in, n_bytes, b, words);
    const int lim = int(min64(64, n_bytes - (b << 6)));
    bool at_ls = false, in_hdr = false;
    if constexpr (FASTA) {
        at_ls = st->at_ls;
        in_hdr = st->in_hdr;
    }
    int o = 0;  // output slot within the block (== i when nothing is dropped)
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        const uint32_t x = (words[i >> 2] >> (8 * (i & 3))) & 0xffu;
        uint32_t code;
        bool other, lower, ws;
        classify(x, code, other, lower, ws);
        if constexpr (FASTA) {
            if (i < lim) {
                if (is_term(x)) {
                    at_ls = true;
                    in_hdr = false;
                } else {
                    if (at_ls) in_hdr = x == '>';
                    at_ls = false;
                    ws |= in_hdr;   // header bytes are dropped like whitespace
                }
            }
        }
        const int slot = compact ? o : i;
        if (!ws) {
            if (slot < 32) r.w0 |= uint64_t(code) << (2 * slot);
            else r.w1 |= uint64_t(code) << (2 * (slot - 32));
            r.n |= uint64_t(other) << slot;
            r.soft |= uint64_t(lower) << slot;
            ++o;
        }
    }
    if constexpr (FASTA) {
        st->at_ls = at_ls;
        st->in_hdr = in_hdr;
    }
    r.kept = uint32_t(o);
    return r;
}

// Last line terminator of each block (global position, -1 if none).
__global__ void last_term_kernel(const uint8_t* in, int64_t n_bytes, int64_t n_blocks, int64_t* lt) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        uint32_t words[16];
        load_block(in, n_bytes, b, words);
        int last = -1;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
            const uint32_t x = (words[i >> 2] >> (8 * (i & 3))) & 0xffu;
            if (is_term(x)) last = i;   // SP padding past the end never matches
        }
        lt[b] = last < 0 ? -1 : (b << 6) + last;
    }
}

// Kept (retained) symbols per block; the last block also records the line
// state after the input (FASTA carry out).
template <bool FASTA>
__global__ void kept_kernel(const uint8_t* in, int64_t n_bytes, int64_t n_blocks, const int64_t* lt_excl,
                            const int* carry, uint32_t* kept, int* carry_out) {
    const int c = FASTA && carry ? *carry : 0;
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        LineState st{};
        if constexpr (FASTA) st = block_start_state(in, b, lt_excl, c);
        const Packed r = pack_block<FASTA>(in, n_bytes, b, true, &st);
        kept[b] = r.kept;
        if constexpr (FASTA) {
            if (b == n_blocks - 1) *carry_out = carry_of(st);
        }
    }
}

// In-place encode (no whitespace expected), four lanes per 64-byte block:
// each lane classifies 16 bytes with byte-SIMD compares (__vcmpeq4 & co.),
// the quad assembles the block with two xor-shuffles, lane 0 stores it.  A
// warp reads 512 contiguous bytes per iteration.  Any whitespace sets
// *any_ws (the caller then takes the compacting path).
__device__ __forceinline__ uint32_t msb4(uint32_t m) {   // 4 byte masks (0x00 / 0xFF) -> 4 bits
    return (((m >> 7) & 0x01010101u) * 0x01020408u) >> 24;
}
__device__ __forceinline__ uint32_t pack4(uint32_t code) {   // 4 bytes holding 0..3 -> 8 bits
    const uint32_t c = (code | (code >> 6)) & 0x000F000Fu;
    return (c | (c >> 12)) & 0xFFu;
}

__global__ void encode_inplace_kernel(const uint8_t* in, int64_t n_bytes, int64_t n_blocks, int lb,
                                      uint64_t* bases, uint64_t* nmask, uint64_t* soft, int* any_ws) {
    const int lane = threadIdx.x & 31, q = lane & 3;
    const int64_t stride = (int64_t(gridDim.x) * blockDim.x) >> 2;
    bool saw_ws = false;
    for (int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + (threadIdx.x & ~31)) >> 2; b0 < n_blocks; b0 += stride) {
        const int64_t b = b0 + (lane >> 2);   // warp-uniform loop; b may pass the end
        const int64_t p = (b << 6) + 16 * q;
        uint32_t x[4] = {0x20202020u, 0x20202020u, 0x20202020u, 0x20202020u};   // SP padding
        uint32_t valid = 0;
        if (b < n_blocks) {
            if (p + 16 <= n_bytes && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(in + p));
                x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
                valid = 0xFFFFu;
            } else {
                for (int i = 0; i < 16 && p + i < n_bytes; ++i) {
                    x[i >> 2] = (x[i >> 2] & ~(0xFFu << (8 * (i & 3)))) | (uint32_t(in[p + i]) << (8 * (i & 3)));
                    valid |= 1u << i;
                }
            }
        }
        uint32_t codes = 0, oth = 0, ws = 0, low = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t w = x[k], lw = w | 0x20202020u;
            const uint32_t base = __vcmpeq4(lw, 0x61616161u) | __vcmpeq4(lw, 0x63636363u) |
                                  __vcmpeq4(lw, 0x67676767u) | __vcmpeq4(lw, 0x74747474u);
            const uint32_t wsm = __vcmpeq4(w, 0x20202020u) | __vcmpeq4(w, 0x09090909u) |
                                 __vcmpeq4(w, 0x0D0D0D0Du) | __vcmpeq4(w, 0x0A0A0A0Au);
            const uint32_t lower = __vcmpgeu4(w, 0x61616161u) & __vcmpleu4(w, 0x7A7A7A7Au);
            codes |= pack4(((w >> 1) ^ (w >> 2)) & 0x03030303u & base) << (8 * k);
            oth |= msb4(~base & ~wsm) << (4 * k);
            ws |= msb4(wsm) << (4 * k);
            low |= msb4(lower) << (4 * k);
        }
        saw_ws |= (ws & valid) != 0;
        // quad assembly: lane q holds bases 16q .. 16q + 15
        const uint64_t mine = uint64_t(codes) | (uint64_t(__shfl_down_sync(0xffffffffu, codes, 1, 4)) << 32);
        const uint64_t hi = __shfl_down_sync(0xffffffffu, mine, 2, 4);
        uint64_t n = uint64_t(oth & valid) << (16 * q), sm = uint64_t(low & valid) << (16 * q);
        n |= __shfl_xor_sync(0xffffffffu, n, 1, 4);
        n |= __shfl_xor_sync(0xffffffffu, n, 2, 4);
        sm |= __shfl_xor_sync(0xffffffffu, sm, 1, 4);
        sm |= __shfl_xor_sync(0xffffffffu, sm, 2, 4);
        if (q == 0 && b < n_blocks) {
            const int64_t slot = blk_slot(b, lb);
            reinterpret_cast<ulonglong2*>(bases)[slot] = make_ulonglong2(mine, hi);
            nmask[slot] = n;
            soft[slot] = sm;
        }
    }
    if (saw_ws) atomicOr(any_ws, 1);
}

// Storage word of linear 64-bit word w of a stream with `per_block` words
// per 64-base block (2 for bases, 1 for the bitmaps).
__device__ __forceinline__ int64_t word_slot(int64_t w, int per_block, int lb) {
    return per_block == 2 ? 2 * blk_slot(w >> 1, lb) + (w & 1) : blk_slot(w, lb);
}

// OR `nbits` bits (value v, nbits <= 64) at linear bit position `bit`.
__device__ __forceinline__ void or_bits(uint64_t* a, int64_t bit, uint64_t v, int nbits, int per_block,
                                        int lb) {
    if (nbits <= 0 || v == 0) return;
    const int64_t w = bit >> 6;
    const int sh = int(bit & 63);
    atomicOr(reinterpret_cast<unsigned long long*>(&a[word_slot(w, per_block, lb)]),
             (unsigned long long)(v << sh));
    if (sh && sh + nbits > 64)
        atomicOr(reinterpret_cast<unsigned long long*>(&a[word_slot(w + 1, per_block, lb)]),
                 (unsigned long long)(v >> (64 - sh)));
}

template <bool FASTA>
__global__ void encode_compact_kernel(const uint8_t* in, int64_t n_bytes, int64_t n_blocks, int lb,
                                      const int64_t* out_pos, const int64_t* lt_excl, const int* carry,
                                      uint64_t* bases, uint64_t* nmask, uint64_t* soft) {
    const int c = FASTA && carry ? *carry : 0;
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        LineState st{};
        if constexpr (FASTA) st = block_start_state(in, b, lt_excl, c);
        Packed r = pack_block<FASTA>(in, n_bytes, b, true, &st);
        const int64_t o = out_pos[b];
        const int k = int(r.kept);
        // bases: 2k bits starting at bit 2*o; split into the two 64-bit halves
        or_bits(bases, 2 * o, r.w0, std::min(64, 2 * k), 2, lb);
        if (k > 32) or_bits(bases, 2 * o + 64, r.w1, 2 * (k - 32), 2, lb);
        or_bits(nmask, o, r.n, k, 1, lb);
        or_bits(soft, o, r.soft, k, 1, lb);
    }
}

__global__ void pack_codes_kernel(const uint8_t* codes, int64_t n, int64_t n_blocks, int lb,
                                  uint64_t* bases, uint64_t* nmask, int* bad) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p0 = b << 6;
        uint64_t w0 = 0, w1 = 0, m = 0;
        const int lim = int(min64(64, n - p0));
        if (lim == 64) {
            const uint4* src = reinterpret_cast<const uint4*>(codes + p0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = __ldg(src + q);
                const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int t = 0; t < 4; ++t)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int i = 16 * q + 4 * t + k;
                        const uint32_t c = (ws[t] >> (8 * k)) & 0xffu;
                        if (c > 4u) atomicOr(bad, 1);
                        const uint64_t bits = c >= 4u ? 0ull : uint64_t(c);
                        if (i < 32) w0 |= bits << (2 * i);
                        else w1 |= bits << (2 * (i - 32));
                        m |= uint64_t(c >= 4u) << i;
                    }
            }
        } else {
            for (int i = 0; i < 64; ++i) {
                const uint32_t c = i < lim ? codes[p0 + i] : 4u;
                if (i < lim && c > 4u) atomicOr(bad, 1);
                const uint64_t bits = c >= 4u ? 0ull : uint64_t(c);
                if (i < 32) w0 |= bits << (2 * i);
                else w1 |= bits << (2 * (i - 32));
                m |= uint64_t(c >= 4u) << i;
            }
        }
        const int64_t slot = blk_slot(b, lb);
        reinterpret_cast<ulonglong2*>(bases)[slot] = make_ulonglong2(w0, w1);
        nmask[slot] = m;
    }
}

__global__ void unpack_codes_kernel(SeqView q, uint8_t* out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < q.n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = uint8_t(seq_sym(q, i));
}

__global__ void linear_mask_kernel(const uint64_t* mask, int64_t n_words, int lb, uint64_t* out) {
    for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n_words;
         g += int64_t(gridDim.x) * blockDim.x)
        out[g] = mask[blk_slot(g, lb)];
}

int grid_for(const ks_ctx* ctx, int64_t items, int threads) {
    return int(max64(1, min64((items + threads - 1) / threads,
                                                      int64_t(ctx->num_sms) * 16)));
}

}  // namespace

// Scratch of encode_compact_device for n_bytes of input.
size_t encode_scratch_bytes(int64_t n_bytes) {
    const int64_t nb = (n_bytes + 63) / 64 + 1;
    return align16(size_t(nb) * 4) + 3 * align16(size_t(nb) * 8) + exclusive_scan_rows_tmp_bytes(nb) + 128;
}

// Compacting encode of n_bytes of device ASCII into seq, no host sync: every
// block's retained count, an exclusive scan for its output position, then
// each block ORs its bits into place.  FASTA additionally drops header lines:
// the last line terminator before each block comes from an exclusive
// running-max scan, so every block knows its line state.  d_carry (FASTA,
// may be null = input start) holds the line state before d_in[0] and
// receives the state after the last byte.  *d_total = retained symbols.
int encode_compact_device(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, bool fasta, int* d_carry,
                          ks_seq* seq, void* scratch, int64_t* d_total, int* launches) {
    const int64_t nb = (n_bytes + 63) / 64;
    char* p = static_cast<char*>(scratch);
    uint32_t* kept = reinterpret_cast<uint32_t*>(p);
    p += align16(size_t(nb + 1) * 4);
    int64_t* pos = reinterpret_cast<int64_t*>(p);
    p += align16(size_t(nb + 1) * 8);
    int64_t* lt = reinterpret_cast<int64_t*>(p);
    p += align16(size_t(nb + 1) * 8);
    int64_t* lt_excl = reinterpret_cast<int64_t*>(p);
    p += align16(size_t(nb + 1) * 8);
    int* carry_next = reinterpret_cast<int*>(p);
    int64_t* lt_total = reinterpret_cast<int64_t*>(p + 16);
    p += 64;
    void* tmp = p;
    if (nb == 0) {
        KS_CUDA(cudaMemsetAsync(d_total, 0, sizeof(int64_t), ctx->stream));
        return KS_OK;
    }
    const int threads = 256;
    const int grid = grid_for(ctx, nb, threads);
    if (fasta) {
        last_term_kernel<<<grid, threads, 0, ctx->stream>>>(d_in, n_bytes, nb, lt);
        if (launches) ++*launches;
        KS_CUDA(cudaGetLastError());
        int rc = exclusive_scan_max(ctx, lt, nb, lt_excl, lt_total, tmp, launches);
        if (rc != KS_OK) return rc;
        kept_kernel<true><<<grid, threads, 0, ctx->stream>>>(d_in, n_bytes, nb, lt_excl, d_carry, kept, carry_next);
    } else {
        kept_kernel<false><<<grid, threads, 0, ctx->stream>>>(d_in, n_bytes, nb, nullptr, nullptr, kept, nullptr);
    }
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    int rc = exclusive_scan_rows(ctx, kept, nb, pos, d_total, tmp, launches);
    if (rc != KS_OK) return rc;
    const size_t words = size_t(seq->n_blocks);
    KS_CUDA(cudaMemsetAsync(seq->d_bases, 0, words * 16, ctx->stream));
    KS_CUDA(cudaMemsetAsync(seq->d_nmask, 0, words * 8, ctx->stream));
    if (seq->d_soft) KS_CUDA(cudaMemsetAsync(seq->d_soft, 0, words * 8, ctx->stream));
    if (fasta)
        encode_compact_kernel<true><<<grid, threads, 0, ctx->stream>>>(d_in, n_bytes, nb, seq->lb, pos, lt_excl, d_carry,
                                                                       seq->d_bases, seq->d_nmask, seq->d_soft);
    else
        encode_compact_kernel<false><<<grid, threads, 0, ctx->stream>>>(d_in, n_bytes, nb, seq->lb, pos, nullptr,
                                                                        nullptr, seq->d_bases, seq->d_nmask,
                                                                        seq->d_soft);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    if (fasta && d_carry)
        KS_CUDA(cudaMemcpyAsync(d_carry, carry_next, sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
    return KS_OK;
}

// Whitespace-free encode of a raw piece in place, no host sync: any
// whitespace sets *ws_flag (the caller then redoes the input on a compacting
// path).  Used for the raw pieces of the streamed count.
int encode_raw_piece(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, ks_seq* seq, uint32_t* kept, int* ws_flag,
                     int* launches) {
    const int64_t nb = (n_bytes + 63) / 64;
    seq->n = n_bytes;
    if (nb == 0) return KS_OK;
    const int threads = 256;
    encode_inplace_kernel<<<grid_for(ctx, nb * 4, threads), threads, 0, ctx->stream>>>(
        d_in, n_bytes, nb, seq->lb, seq->d_bases, seq->d_nmask, seq->d_soft, ws_flag);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

// Encode n_bytes of device ASCII into seq (whose arrays are sized for n_bytes
// bases).  Sets seq->n to the retained symbol count (host sync).  Raw input
// without whitespace is written in place in one pass; anything else takes
// the compacting path.  `scratch` holds encode_scratch_bytes(n_bytes).
int encode_ascii_device(ks_ctx* ctx, const uint8_t* d_in, int64_t n_bytes, bool fasta, ks_seq* seq,
                        void* scratch, int* launches) {
    const int64_t nb = (n_bytes + 63) / 64;
    if (nb == 0) {
        seq->n = 0;
        return KS_OK;
    }
    char* p = static_cast<char*>(scratch);
    uint32_t* kept = reinterpret_cast<uint32_t*>(p);
    int* flag = reinterpret_cast<int*>(static_cast<char*>(scratch) + encode_scratch_bytes(n_bytes) - 64);
    int64_t* d_total = reinterpret_cast<int64_t*>(flag + 4);
    int rc;
    if (!fasta) {
        KS_CUDA(cudaMemsetAsync(flag, 0, 64, ctx->stream));
        const int threads = 256;
        encode_inplace_kernel<<<grid_for(ctx, nb * 4, threads), threads, 0, ctx->stream>>>(
            d_in, n_bytes, nb, seq->lb, seq->d_bases, seq->d_nmask, seq->d_soft, flag);
        if (launches) ++*launches;
        KS_CUDA(cudaGetLastError());
        int any_ws = 0;
        KS_CUDA(cudaMemcpyAsync(&any_ws, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        KS_CUDA(cudaStreamSynchronize(ctx->stream));
        if (!any_ws) {
            seq->n = n_bytes;
            return KS_OK;
        }
    }
    rc = encode_compact_device(ctx, d_in, n_bytes, fasta, nullptr, seq, scratch, d_total, launches);
    if (rc != KS_OK) return rc;
    int64_t total = 0;
    KS_CUDA(cudaMemcpyAsync(&total, d_total, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    KS_CUDA(cudaStreamSynchronize(ctx->stream));
    seq->n = total;
    return KS_OK;
}

// Host wire form (host_pack.h pack_wire_task): per 64-byte block 2 words of
// 2-bit codes and a special mask; a special position with code 01 is
// dropped, with code 00 it is OTHER.  Blocks are compacted into the
// tile-slot layout like encode_compact_kernel does for ASCII.
__device__ __forceinline__ uint64_t even_bits(uint64_t w) {   // bit 2i of w -> bit i
    uint64_t x = w & 0x5555555555555555ull;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
    x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
    x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
    return x;
}

__device__ __forceinline__ uint64_t wire_drop(const uint64_t* lin, const uint64_t* special, int64_t b) {
    return special[b] & (even_bits(lin[2 * b]) | (even_bits(lin[2 * b + 1]) << 32));
}

__global__ void wire_kept_kernel(const uint64_t* __restrict__ lin, const uint64_t* __restrict__ special,
                                 int64_t n_blocks, uint32_t* kept) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x)
        kept[b] = 64u - uint32_t(__popcll(wire_drop(lin, special, b)));
}

__global__ void wire_compact_kernel(const uint64_t* __restrict__ lin, const uint64_t* __restrict__ special,
                                    int64_t n_blocks, const int64_t* pos, int lb, uint64_t* bases, uint64_t* nmask) {
    for (int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; b < n_blocks;
         b += int64_t(gridDim.x) * blockDim.x) {
        const uint64_t w0 = lin[2 * b], w1 = lin[2 * b + 1];
        const uint64_t drop = wire_drop(lin, special, b);
        const uint64_t oth = special[b] & ~drop;
        uint64_t keep = ~drop;
        uint64_t r0 = 0, r1 = 0, rn = 0;
        int o = 0;
        while (keep) {
            const int i = __ffsll(keep) - 1;
            keep &= keep - 1;
            const uint64_t code = ((oth >> i) & 1ull) ? 0ull : (i < 32 ? w0 >> (2 * i) : w1 >> (2 * (i - 32))) & 3u;
            if (o < 32) r0 |= code << (2 * o);
            else r1 |= code << (2 * (o - 32));
            rn |= ((oth >> i) & 1ull) << o;
            ++o;
        }
        const int64_t p = pos[b];
        or_bits(bases, 2 * p, r0, std::min(64, 2 * o), 2, lb);
        if (o > 32) or_bits(bases, 2 * p + 64, r1, 2 * (o - 32), 2, lb);
        or_bits(nmask, p, rn, o, 1, lb);
    }
}

// Compact n_blocks wire blocks into seq (bases + nmask; soft-mask untouched).
// `kept`/`pos`/`tmp` are scratch of n_blocks + 1 entries and the rows scan.
int wire_compact_device(ks_ctx* ctx, const uint64_t* d_lin, const uint64_t* d_special, int64_t n_blocks, ks_seq* seq,
                        uint32_t* kept, int64_t* pos, void* tmp, int64_t* d_total, int* launches) {
    if (n_blocks <= 0) return KS_OK;
    const int threads = 256;
    const int grid = grid_for(ctx, n_blocks, threads);
    wire_kept_kernel<<<grid, threads, 0, ctx->stream>>>(d_lin, d_special, n_blocks, kept);
    KS_CUDA(cudaGetLastError());
    int rc = exclusive_scan_rows(ctx, kept, n_blocks, pos, d_total, tmp, launches);
    if (rc != KS_OK) return rc;
    const size_t words = size_t(seq->n_blocks);
    KS_CUDA(cudaMemsetAsync(seq->d_bases, 0, words * 16, ctx->stream));
    KS_CUDA(cudaMemsetAsync(seq->d_nmask, 0, words * 8, ctx->stream));
    wire_compact_kernel<<<grid, threads, 0, ctx->stream>>>(d_lin, d_special, n_blocks, pos, seq->lb, seq->d_bases,
                                                           seq->d_nmask);
    KS_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
    return KS_OK;
}

// Host-packed wire format (host_pack.h): OTHER bitmaps arrive only for the
// tiles that hold OTHER, compacted; one CTA copies each into place.
__global__ void scatter_tile_masks_kernel(const uint64_t* __restrict__ compact, const int32_t* __restrict__ ids,
                                          int tile_words, uint64_t* __restrict__ nmask) {
    const uint64_t* src = compact + size_t(blockIdx.x) * tile_words;
    uint64_t* dst = nmask + size_t(ids[blockIdx.x]) * tile_words;
    for (int i = threadIdx.x; i < tile_words; i += blockDim.x) dst[i] = src[i];
}

int scatter_tile_masks_device(ks_ctx* ctx, const uint64_t* d_compact, const int32_t* d_ids, int n_tiles,
                              int tile_words, uint64_t* d_nmask, int* launches) {
    if (n_tiles <= 0) return KS_OK;
    scatter_tile_masks_kernel<<<n_tiles, 256, 0, ctx->stream>>>(d_compact, d_ids, tile_words, d_nmask);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int pack_codes_device(ks_ctx* ctx, const uint8_t* d_codes, int64_t n, ks_seq* seq, int* d_flag,
                      int* launches) {
    const int64_t nb = (n + 63) / 64;
    seq->n = n;
    if (nb == 0) return KS_OK;
    const int threads = 256;
    pack_codes_kernel<<<grid_for(ctx, nb, threads), threads, 0, ctx->stream>>>(
        d_codes, n, nb, seq->lb, seq->d_bases, seq->d_nmask, d_flag);
    if (launches) ++*launches;
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int unpack_codes_device(ks_ctx* ctx, const ks_seq* seq, uint8_t* d_out) {
    if (seq->n == 0) return KS_OK;
    const int threads = 256;
    SeqView q;
    q.bases = seq->d_bases;
    q.nmask = seq->d_nmask;
    q.n = seq->n;
    q.lb = seq->lb;
    unpack_codes_kernel<<<grid_for(ctx, seq->n, threads), threads, 0, ctx->stream>>>(q, d_out);
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

int linear_softmask_device(ks_ctx* ctx, const ks_seq* seq, uint64_t* d_out) {
    const int64_t words = (seq->n + 63) / 64;
    if (words == 0) return KS_OK;
    const int threads = 256;
    linear_mask_kernel<<<grid_for(ctx, words, threads), threads, 0, ctx->stream>>>(seq->d_soft, words, seq->lb,
                                                                                     d_out);
    KS_CUDA(cudaGetLastError());
    return KS_OK;
}

}  // namespace ks
