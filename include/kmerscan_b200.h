/*
 * kmerscan_b200.h -- C ABI of the B200-native chunked DFA scan.
 *
 * Drop-in native boundary for the reference's compiled hot path
 * (/root/reference/pkg/src/kmerscan/_kernels.py, numba @njit kernels) and the
 * engine entry points that call it (/root/reference/pkg/src/kmerscan/engine.py).
 * Plain C types only (pointers + sizes): no torch, no numpy, no C++ in the
 * signatures.  Every call returns 0 on success or a negative KS_E* status; the
 * message of the last failure on the calling thread is ks_last_error().  A
 * failing call never leaves partial results in caller buffers.
 *
 * Device memory is owned by the context and the dfa/seq handles (freed by
 * ks_*_free).  Handles are immutable after upload.  Thread safety: calls on
 * one context (and on its handles) take a per-context lock and run in order on
 * the context's CUDA stream; separate contexts run concurrently.
 */
#ifndef KMERSCAN_B200_H
#define KMERSCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KS_API __attribute__((visibility("default")))
#else
#define KS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define KS_OK 0
#define KS_E_INVALID (-1)   /* bad argument            -> Python ValueError            */
#define KS_E_CUDA (-2)      /* CUDA runtime failure    -> Python RuntimeError          */
#define KS_E_CHAIN (-3)     /* internal chain invariant-> Python ReductionChainError   */
#define KS_E_UNSUPPORTED (-4) /* outside the device limits (e.g. |Q| > 32767)        */
#define KS_E_NOMEM (-5)

typedef struct ks_ctx ks_ctx;
typedef struct ks_dfa ks_dfa;
typedef struct ks_seq ks_seq;

/* Scan strategy chosen by ks_dfa_upload (ks_dfa_info.strategy). */
#define KS_STRATEGY_LOOKBACK 1   /* definite DFA: state after D symbols is input-determined */
#define KS_STRATEGY_MAPSCAN 2    /* small transition monoid: chunk maps + exclusive scan     */
#define KS_STRATEGY_SPECULATE 3  /* generic: per-chunk speculative PSS maps + exclusive scan */

typedef struct ks_dfa_info {
    int32_t n_states;        /* |Q| */
    int32_t n_expressions;   /* ne */
    int32_t n_accepting;     /* states with a non-empty output multiset */
    int32_t strategy;        /* KS_STRATEGY_* */
    int32_t sync_depth;      /* D for LOOKBACK, -1 otherwise */
    int32_t stride;          /* bases per table lookup of the kernel that scans (1..4) */
    int32_t monoid_size;     /* |M| for MAPSCAN, 0 otherwise */
    int32_t other_resets;    /* 1 if every state goes to one state on OTHER */
    int64_t table_bytes;     /* bytes of the stride table staged per CTA */
    int32_t tables_in_smem;  /* 1: staged in shared memory, 0: read through L1/L2 */
    int32_t reserved;
} ks_dfa_info;

/* Per-call statistics of the last ks_count/ks_locate on a context. */
typedef struct ks_stats {
    float scan_ms;           /* device time of the dominant scan kernel(s)  */
    float total_ms;          /* device time of the whole call (events)      */
    int32_t kernel_launches; /* kernels launched by the call                */
    int32_t chunks;          /* lane chunks in the main scan                */
    int64_t chunk_len;       /* bases per lane chunk                        */
    int64_t rows;            /* locate rows produced                        */
    int64_t h2d_bytes;       /* host->device bytes the call copied          */
    int64_t d2h_bytes;       /* device->host bytes the call copied          */
} ks_stats;

/* ---- context ------------------------------------------------------------ */
/* Replaces the reference's ThreadPoolExecutor-per-call (engine.py:223-232). */
KS_API int ks_open(int device, ks_ctx** out);
KS_API int ks_close(ks_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the context's own stream. */
KS_API int ks_set_stream(ks_ctx* ctx, void* cuda_stream);
/* Size the scan grids for (SM count - n_sms) SMs, leaving n_sms free for
 * kernels on other streams (an NCCL collective overlapping the next scan: a
 * scan CTA fills its SM's shared memory and registers).  0 restores the
 * default; KS_RESERVE_SMS sets the initial value at ks_open. */
KS_API int ks_set_reserved_sms(ks_ctx* ctx, int32_t n_sms);
KS_API int ks_synchronize(ks_ctx* ctx);
KS_API int ks_get_stats(const ks_ctx* ctx, ks_stats* out);
KS_API const char* ks_last_error(void);
KS_API const char* ks_version(void);

/* ---- automaton ---------------------------------------------------------- */
/* Upload a Dfa (automaton.py:26-51 layout: transitions int32[nq][5] row-major,
 * columns a,c,g,t,OTHER; CSR out_offsets int32[nq+1], out_ids int32[...]).
 * Compiles the device form (renumbering, stride tables, synchronisation
 * analysis) natively.  Replaces the table arguments of match_chunk_kernel /
 * scan_from (_kernels.py:19,44). */
KS_API int ks_dfa_upload(ks_ctx* ctx, const int32_t* transitions, int32_t n_states,
                  const int32_t* out_offsets, const int32_t* out_ids,
                  int32_t n_expressions, ks_dfa** out);
/* Same, forcing a strategy (testing; KS_STRATEGY_* or 0 = automatic). */
KS_API int ks_dfa_upload_ex(ks_ctx* ctx, const int32_t* transitions, int32_t n_states,
                     const int32_t* out_offsets, const int32_t* out_ids,
                     int32_t n_expressions, int32_t force_strategy, ks_dfa** out);
KS_API int ks_dfa_info_get(const ks_dfa* dfa, ks_dfa_info* out);
KS_API int ks_dfa_free(ks_dfa* dfa);

/* ---- sequences ---------------------------------------------------------- */
/* A sequence is immutable once its upload call returns; the upload ends by
 * writing per-tile row flags (which block rows hold OTHER) that the scans of
 * a resident sequence use to skip OTHER-bitmap loads and per-lane tests. */
/* Symbol codes 0..4 (Sequence.symbols, ingest.py:20-32) -> packed device form. */
KS_API int ks_seq_upload_codes(ks_ctx* ctx, const uint8_t* codes, int64_t n, ks_seq** out);
/* Raw ASCII bytes -> device encode (alphabet.py:20-37 / ingest.py:67-69):
 * case fold, whitespace (SP,TAB,CR,LF) dropped, every other byte OTHER.
 * fasta != 0 additionally drops lines starting with '>' (ingest.py:65-66,
 * lines split at CR, LF, CRLF), on the device. */
KS_API int ks_seq_upload_ascii(ks_ctx* ctx, const uint8_t* bytes, int64_t n_bytes,
                        int32_t fasta, ks_seq** out);
/* Same, input already resident in device memory (not copied, not retained). */
KS_API int ks_seq_encode_device(ks_ctx* ctx, const uint8_t* d_bytes, int64_t n_bytes,
                         int32_t fasta, ks_seq** out);
KS_API int ks_seq_length(const ks_seq* seq, int64_t* n);
/* Decode back to codes 0..4 (tests); out has room for n bytes. */
KS_API int ks_seq_download_codes(ks_ctx* ctx, const ks_seq* seq, uint8_t* out);
/* Soft-mask bitmap (bit i of word i/64 = base i was lowercase). */
KS_API int ks_seq_download_softmask(ks_ctx* ctx, const ks_seq* seq, uint64_t* out, int64_t n_words);
KS_API int ks_seq_free(ks_seq* seq);

/* ---- scans -------------------------------------------------------------- */
/* Per-expression counts over the whole sequence from the start state:
 * the result of run(...).per_expression_counts (engine.py:207-237) and of
 * sequential_count (oracle.py:56-61 -> scan_from, _kernels.py:19-29).
 * counts_out: int64[n_expressions], caller-owned. */
KS_API int ks_count(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_out);

/* Counts plus match rows [exclusive end offset, expression id], sorted by
 * (offset, id), duplicates kept (engine.py:165-176).  *rows_out is
 * library-allocated (free with ks_free), int64[*n_rows][2]. */
KS_API int ks_locate(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_out,
              int64_t** rows_out, int64_t* n_rows);

/* Asynchronous ks_count on the device-resident sequence: enqueues the scan
 * (whose last CTA reduces the counts and writes them into `counts_pinned`,
 * page-locked host memory; a copy follows when that memory is not device-
 * visible) without waiting.  ks_async_wait synchronises and reports the calls
 * and kernel launches since the last wait; the summed scan-kernel time only
 * with KS_ASYNC_EVENTS=1 (per-call events, else 0: events between
 * back-to-back scans cost time and block their early launch). */
KS_API int ks_count_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t* counts_pinned);
KS_API int ks_async_wait(ks_ctx* ctx, float* scan_ms_total, int32_t* calls, int32_t* launches);

/* Counts straight from a HOST buffer of raw ASCII (the end-to-end call):
 * host worker threads pack each 64 MiB piece into the device tile-slot
 * format (2-bit bases + OTHER bitmap, 0.25-0.375 B/base on the wire) in
 * pinned staging, the copy stream moves it while the previous piece is
 * scanned, and each piece enters in the state the previous one left.  Same
 * result as ks_seq_upload_ascii + ks_count; input with whitespace falls back
 * to the device-encode stream of ks_count_host_bytes.  KS_HOST_THREADS caps
 * the packer threads; KS_DEVICE_ENCODE=1 copies raw ASCII and encodes on the
 * device instead. */
KS_API int ks_count_host_ascii(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes,
                               int64_t* counts_out);

/* Same for raw (fasta = 0) or FASTA (fasta != 0) file bytes: FASTA and
 * whitespace-bearing input stream raw bytes over PCIe into double device
 * buffers and are encoded + compacted there (header-line state carried
 * across pieces) while the next piece copies.  Replaces load_sequence +
 * run(count) (ingest.py:54-70, engine.py:207). */
KS_API int ks_count_host_bytes(ks_ctx* ctx, const ks_dfa* dfa, const uint8_t* bytes, int64_t n_bytes,
                               int32_t fasta, int64_t* counts_out);

/* The host packer on its own (CPU only, no context): blocks of `bytes` in
 * tile-slot order for units of 2^lb 64-base blocks, 32 units per tile --
 * block g lands in slot ((g>>lb)>>5 << (5+lb)) | (g & (2^lb-1)) << 5 | (g>>lb) & 31.
 * `bases` holds 2*slots words, `nmask` `slots` words, slots = ceil(n/64)
 * rounded up to whole tiles.  *flags gets bit0 = whitespace seen, bit1 =
 * OTHER seen. */
KS_API int ks_pack_host_ascii(const uint8_t* bytes, int64_t n_bytes, int32_t lb, uint64_t* bases,
                              uint64_t* nmask, int32_t* flags);

/* The host side of the FASTA / whitespace stream on its own (CPU only): the
 * whole buffer as one task starting at a line start.  Per 64-byte block g:
 * bases[2g..2g+1] 2-bit codes, special[g] a mask of non-base positions --
 * code 01 = dropped (whitespace, header line, past the end), code 00 =
 * OTHER.  *kept = retained symbols. */
/* The host side of the packed codes upload (ks_seq_upload_codes of >= 8 Mi
 * symbols) on its own: codes 0..4 -> the tile-slot layout of
 * ks_pack_host_ascii (no GPU needed); KS_E_INVALID for a code above 4. */
KS_API int ks_pack_host_codes(const uint8_t* codes, int64_t n, int32_t lb, uint64_t* bases, uint64_t* nmask);
KS_API int ks_pack_host_wire(const uint8_t* bytes, int64_t n_bytes, int32_t fasta, uint64_t* bases,
                             uint64_t* special, int64_t* kept);

/* Range form used by match_chunk (engine.py:94-134) and by sharded scans:
 * scan positions [begin, end) of seq entering at `entry_state` (original
 * state id; -1 = the true state of the sequence at `begin`, derived on
 * device).  Offsets in rows are seq positions + 1 + row_offset_base.
 * exit_state (may be NULL) receives the original id of the final state.
 * rows_out/n_rows may be NULL for count-only. */
KS_API int ks_scan_range(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin,
                  int64_t end, int32_t entry_state, int64_t row_offset_base,
                  int64_t* counts_out, int32_t* exit_state, int64_t** rows_out,
                  int64_t* n_rows);

/* Boundary map of a segment (the per-GPU "start-state -> end-state map"):
 * map_out[q] = original id of the state reached after scanning [begin,end)
 * from original state q, for all q < n_states. */
KS_API int ks_segment_map(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin,
                   int64_t end, int32_t* map_out);

/* Asynchronous multi-GPU building blocks (no host synchronisation; device
 * pointers).  ks_segment_map_async writes the shard's boundary map
 * (int32[n_states], original ids) into d_map_out -- the payload of the NCCL
 * all-gather.  ks_count_shard_async composes START through the gathered maps
 * d_maps[0..rank) (int32[world][n_states]) on the device, scans
 * [begin, end) from that state and writes the shard's per-expression counts
 * into d_counts (uint64[n_expressions], the NCCL all-reduce payload).
 * Halo mode (rank > 0, d_maps == NULL, definite automata only): the caller
 * loaded at least sync_depth bases of the previous shard in front of
 * `begin`, the entry state is recovered by lookback and no map exchange is
 * needed -- one all-reduce per step. */
KS_API int ks_segment_map_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin,
                                int64_t end, int32_t* d_map_out);
KS_API int ks_count_shard_async(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin,
                                int64_t end, const int32_t* d_maps, int32_t rank,
                                unsigned long long* d_counts);
/* The same, and once the counts are final the device writes signal_value to
 * *d_signal (uint32, device memory; raised by the scan kernel's finalizing
 * CTA, so the context's stream carries no extra operation between
 * back-to-back scans).  Another stream can then start the all-reduce of
 * d_counts after ks_stream_wait_value32(stream, d_signal, signal_value)
 * without the scan stream recording an event -- back-to-back scans keep
 * their programmatic overlap while the collectives run beside them. */
KS_API int ks_count_shard_async_signal(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int64_t begin,
                                       int64_t end, const int32_t* d_maps, int32_t rank,
                                       unsigned long long* d_counts, uint32_t* d_signal, uint32_t signal_value);
/* Make `cuda_stream` wait until *d_addr >= value (cuStreamWaitValue32, GEQ). */
KS_API int ks_stream_wait_value32(void* cuda_stream, const uint32_t* d_addr, uint32_t value);

/* Speculative-start convergence (match_chunk_kernel's speculative runs,
 * _kernels.py:91-112): for chunk k, candidate start states
 * pss_data[pss_off[k] .. pss_off[k+1]) (original ids; entry 0 is the full
 * run R0) scan seq[chunk_begin[k] ..) for at most min(window, chunk length)
 * steps; conv_out[i] = first step j where run i's state equals R0's, -1 if
 * none (always -1 for R0).  Warp lanes are the speculative runs;
 * convergence is detected with __match_any_sync.  delta_out (nullable,
 * int64[total_runs][n_expressions]) receives per-run prefix-count
 * corrections sum_{t<=conv} out(s_i(t)) - out(s_0(t)). */
KS_API int ks_speculate(ks_ctx* ctx, const ks_dfa* dfa, const ks_seq* seq, int32_t n_chunks,
                 const int64_t* chunk_begin, const int64_t* chunk_end,
                 const int64_t* pss_off, const int32_t* pss_data, int32_t window,
                 int32_t* conv_out, int64_t* delta_out);

/* Exhaustive reconciliation sweep (reference _kernels.py:116-179,
 * oracle.py:94-116): every base word of `length` (4^length words) x every
 * border class b (candidates pss_data[pss_off[b] .. pss_off[b+1]), entry 0 =
 * the full run) runs the chunk kernel's speculation with `window`, and each
 * converged speculative run is checked against a full scan from its own
 * start state -- one device thread per (word, border).  Tables are the
 * reference Dfa arrays (original ids).  result_out[4] = speculative runs,
 * converged runs, count mismatches, final-state mismatches.  length <= 13,
 * n_expressions <= 16 (else KS_E_UNSUPPORTED). */
KS_API int ks_reconciliation_sweep(ks_ctx* ctx, const int32_t* transitions, int32_t n_states,
                                   const int32_t* out_offsets, const int32_t* out_ids, int32_t n_expressions,
                                   const int32_t* pss_data, const int32_t* pss_off, int32_t n_borders,
                                   int32_t length, int32_t window, int64_t* result_out);

/* ---- multi-device (one process, several GPUs) -------------------------- */
/* One sequence sharded over devices dev_ids[0..n_dev) -- the reference's
 * run() spreading one call over all its workers (engine.py:207-237,
 * ingest.py:78-94 partition) with the workers being GPUs.  Distinct devices
 * exchange over NCCL (ncclCommInitAll; libnccl.so.2 loaded at run time:
 * all-gather of boundary maps, all-reduce of the counts); a device id may
 * repeat (tests on one GPU), or KS_MULTI_NCCL=0 be set, and the exchanges
 * then run as stream-ordered peer copies.  Results equal ks_count/ks_locate
 * of the whole sequence on one device. */
typedef struct ks_mctx ks_mctx;
typedef struct ks_mdfa ks_mdfa;
typedef struct ks_mseq ks_mseq;
KS_API int ks_open_multi(int32_t n_dev, const int32_t* dev_ids, ks_mctx** out);
KS_API int ks_close_multi(ks_mctx* m);
KS_API int ks_multi_info(const ks_mctx* m, int32_t* n_dev, int32_t* uses_nccl);
/* The automaton on every device (same arguments as ks_dfa_upload). */
KS_API int ks_mdfa_upload(ks_mctx* m, const int32_t* transitions, int32_t n_states,
                          const int32_t* out_offsets, const int32_t* out_ids, int32_t n_expressions,
                          ks_mdfa** out);
KS_API int ks_mdfa_free(ks_mdfa* d);
/* Codes 0..4: contiguous slices on 64-symbol boundaries, each slice with the
 * previous slice's last 2048 symbols in front (definite automata then need
 * no boundary-map exchange). */
KS_API int ks_mseq_upload_codes(ks_mctx* m, const uint8_t* codes, int64_t n, ks_mseq** out);
/* Raw / FASTA bytes cut into n_dev pieces (FASTA: at line starts), each
 * encoded on its device; slice offsets are the kept-symbol prefix sums. */
KS_API int ks_mseq_upload_ascii(ks_mctx* m, const uint8_t* bytes, int64_t n_bytes, int32_t fasta,
                                ks_mseq** out);
KS_API int ks_mseq_length(const ks_mseq* s, int64_t* n);
KS_API int ks_mseq_free(ks_mseq* s);
KS_API int ks_mcount(ks_mctx* m, const ks_mdfa* d, const ks_mseq* s, int64_t* counts_out);
/* Rows as ks_locate (library-allocated, ks_free), global offsets. */
KS_API int ks_mlocate(ks_mctx* m, const ks_mdfa* d, const ks_mseq* s, int64_t* counts_out,
                      int64_t** rows_out, int64_t* n_rows);

KS_API void ks_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* KMERSCAN_B200_H */
