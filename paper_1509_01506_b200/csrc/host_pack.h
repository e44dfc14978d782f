// Host-side packing of ASCII input into the device sequence format, used as
// the H2D wire format of the streaming count (ks_count_host_ascii): 64 input
// bytes become 16 B of 2-bit bases + 8 B of OTHER bitmap (0.375 B/base, or
// 0.25 B/base when a piece holds no OTHER), written directly in tile-slot
// order so the device scans the copied buffer with no encode kernel.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ks {

// Fixed set of worker threads; run() blocks until every task has executed.
// Workers spin briefly before sleeping so back-to-back pieces wake fast.
class HostPool {
  public:
    explicit HostPool(int threads);
    ~HostPool();
    int threads() const { return int(workers_.size()) + 1; }
    void run(int64_t ntasks, const std::function<void(int64_t)>& fn);

  private:
    void worker();
    void drain();
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<void(int64_t)>* fn_ = nullptr;
    int64_t ntasks_ = 0;
    std::atomic<int64_t> next_{0};
    std::atomic<uint64_t> gen_{0};
    int active_ = 0;
    bool stop_ = false;
};

// Threads the host packer uses: $KS_HOST_THREADS, else the CPUs this process
// may run on (capped at 32).
int host_pack_threads();

struct PackFlags {
    bool whitespace = false;   // SP/TAB/CR/LF seen (positions would shift)
    bool other = false;        // a non-acgt, non-whitespace byte seen
};

// Pack blocks [b0, b1) of `in` (n_bytes long): block b -> slot
// blk_slot(b, lb) - sbase of bases (16 B per slot) and nmask (8 B per slot).
// Bytes past n_bytes encode as base 0, not OTHER.  Returns what the blocks
// contained.
PackFlags pack_ascii_blocks(const uint8_t* in, int64_t n_bytes, int64_t b0, int64_t b1, int lb,
                            uint64_t* bases, uint64_t* nmask, int64_t sbase = 0);

// Symbol codes (0..4, Sequence.symbols) instead of ASCII: code & 3 the base,
// 4 OTHER; blocks [b0, b1) -> slot blk_slot(b, lb) - sbase as above, codes
// past n encode as base 0.  Returns false when a code above 4 was seen.
bool pack_codes_blocks(const uint8_t* codes, int64_t n, int64_t b0, int64_t b1, int lb, uint64_t* bases,
                       uint64_t* nmask, int64_t sbase = 0);

// Streaming-path form, whole tiles [t0, t1) (tile = 32 << lb blocks): each
// tile is packed in a thread-local buffer, its bases streamed (non-temporal
// stores) to `bases` in slot order; a tile holding OTHER appends its OTHER
// bitmap (tile_blocks words) at index j = (*n_compact)++ of `nm_compact` and
// records tile_ids[j] = tile.  Tiles without OTHER write no bitmap at all: in
// real genomes OTHER comes in long N runs, so the bitmap is mostly zero.
PackFlags pack_ascii_tiles(const uint8_t* in, int64_t n_bytes, int64_t t0, int64_t t1, int lb,
                           uint64_t* bases, uint64_t* nm_compact, int32_t* tile_ids,
                           std::atomic<int32_t>* n_compact);

// Wire form for input with whitespace or FASTA headers (the device
// compacts, encode.cu wire_compact_kernel): blocks [b0, b1) of `in` in
// linear order, 24 B per 64 input bytes -- 2 words of 2-bit codes and a
// "special" mask.  A special position is OTHER when its code is 00 and
// dropped (whitespace, header line, past the end) when its code is 01.
// start_state: the line state before block b0 when known (0 line start,
// 1 sequence line, 2 header line), else -1: then the task assumes "sequence
// line" and reports what its first line contributed, so the caller can drop
// it once the true state is resolved.
struct WireTask {
    int64_t kept = 0;          // retained symbols
    int64_t prefix_kept = 0;   // of them, before the first line terminator (assumed start only)
    int64_t first_term = -1;   // byte index of the first line terminator (assumed start only), -1 none
    int end_state = 1;         // line state after the last byte
    bool exact = true;         // the start state was known
};
WireTask pack_wire_task(const uint8_t* in, int64_t n_bytes, int64_t b0, int64_t b1, bool fasta, int start_state,
                        uint64_t* bases, uint64_t* special);
// The assumed start was a header line after all: drop everything before the
// first terminator (or all of [b0, b1) when there is none).
void wire_drop_prefix(int64_t b0, int64_t b1, int64_t first_term, uint64_t* bases, uint64_t* special);

}  // namespace ks
