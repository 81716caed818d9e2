/*
 * ngram_b200.h -- C-ABI of the B200-native N-gram Embedding hot path (libngram_b200.so).
 *
 * The reference (arXiv 2601.21204, /root/reference/proj) exposes only a C++ header API
 * (proj/include/ngram/*.hpp) and no FFI.  These entry points are what that API's hot
 * path binds to when it is backed by the GPU: include/ngram/*.hpp (the drop-in C++
 * headers) and the Python mirror (paper_2601_21204_b200/ngram.py) both call exactly
 * this surface.  Each entry cites the reference interface it replaces.
 *
 * Conventions
 *   - Plain pointers and sizes only.  "dev" pointers are CUDA device pointers on the
 *     bank's device; "host" pointers are host memory (pinned or pageable).
 *   - Every call returns an ngram_status.  On failure ngram_last_error() (thread-local)
 *     holds the message.  Status codes map 1:1 onto the reference's exceptions
 *     (include/ngram/errors.hpp): EINVAL -> std::invalid_argument, ERANGE ->
 *     std::out_of_range, EIO -> io_error, EPARSE -> parse_error, ECONFIG ->
 *     config_error, ENUMERIC -> numeric_error.
 *   - Device calls are stream-ordered (stream = cudaStream_t or NULL for the legacy
 *     stream) and never allocate on the hot path once ngram_bank_reserve() has sized
 *     the workspace.  Token-range errors detected on the device (token >= V0) are
 *     recorded in a device error word: every later kernel of the same call skips its
 *     writes (no output is produced, as the reference raises before writing) and the
 *     error surfaces as NGRAM_ERANGE from ngram_sync_errors() / any host-buffer call.
 *   - Threading: host-buffer entry points (*_host) may be called on one bank from many
 *     threads (serialised per bank, like the reference's read-only shared bank).  The
 *     stream-ordered device entry points share the bank's workspaces and error word:
 *     issue them for one bank on one stream at a time (as with a cuBLAS handle).
 *   - There is no CPU fallback: every compute entry point runs CUDA kernels.
 */
#ifndef NGRAM_B200_H
#define NGRAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum ngram_status {
    NGRAM_OK = 0,
    NGRAM_EINVAL = 1,   /* std::invalid_argument  */
    NGRAM_ERANGE = 2,   /* std::out_of_range      */
    NGRAM_EIO = 3,      /* ngram::io_error        */
    NGRAM_EPARSE = 4,   /* ngram::parse_error     */
    NGRAM_ECONFIG = 5,  /* ngram::config_error    */
    NGRAM_ENUMERIC = 6, /* ngram::numeric_error   */
    NGRAM_ECUDA = 7,    /* CUDA runtime / driver failure   */
    NGRAM_ENCCL = 8,    /* collective failure              */
    NGRAM_ENOMEM = 9    /* device allocation failure       */
} ngram_status;

typedef enum ngram_dtype { NGRAM_F32 = 0, NGRAM_BF16 = 1 } ngram_dtype;

typedef struct ngram_bank ngram_bank;     /* device-resident embedding_bank */
typedef struct ngram_decode ngram_decode; /* device-resident batch of sequence_cache */

/* ------------------------------------------------------------------ misc */
const char* ngram_last_error(void);
const char* ngram_version(void);
/* Number of kernels this process has launched through the library (bench evidence). */
uint64_t ngram_kernel_launches(void);

/* ------------------------------------------------------------------ config (host) */
/* Replaces ngram_config_from_json + validate (config.cpp:124-139, :32-77). */
int ngram_config_validate(const char* config_json);
/* Replaces make_default_config + to_json_string (config.cpp:163-183, :109-122). */
int ngram_make_default_config(uint32_t base_vocab, int dim, int max_order, int sub_tables, char* json_out,
                              size_t cap);

/* ------------------------------------------------------------------ banks */
/* Device bank for `config_json` (embedding_bank_t, embedding.hpp:31-70) on `device`.
 * Layout in HBM: sub-tables bf16, concatenated by branch, row pitch d;
 * E0 bf16 V0 x D; W_cat bf16 D x D with W_cat[i][b*d+j] = W_b[i*d+j] (K-major);
 * LayerNorm gain/bias f32.  shard_count > 1 keeps only rank shard_rank's contiguous
 * row block of every sub-table (owner(b,h) = floor(h * shard_count / V_b)). */
int ngram_bank_create(const char* config_json, int device, int shard_rank, int shard_count, ngram_bank** out);
/* As ngram_bank_create; flags: NGRAM_BANK_HASH_ONLY allocates no tables (hash_all_orders
 * needs only the config, hashing.cpp:61-81 -- e.g. moduli far beyond device memory). */
#define NGRAM_BANK_HASH_ONLY 1
int ngram_bank_create_ex(const char* config_json, int device, int shard_rank, int shard_count, int flags,
                         ngram_bank** out);
int ngram_bank_destroy(ngram_bank* bank);
/* Upload a reference-layout float bank (make_bank / load_bank output) from HOST memory,
 * converting to bf16 (round-to-nearest-even).  sub[b] / proj[b] indexed by branch_index;
 * proj ignored for averaged_v1; gain/bias only for layer_norm.  Replaces the implicit
 * "bank lives in host vectors" of embedding.hpp:31-38. */
int ngram_bank_upload_f32(ngram_bank* bank, const float* base, const float* const* sub, const float* const* proj,
                          const float* ln_gain, const float* ln_bias);
/* Fill the bank on device with the counter-based synthetic generator:
 * used for LongCat-scale tables that cannot exist on the host. */
int ngram_bank_generate(ngram_bank* bank, uint64_t seed, void* stream);
/* Stream a reference bank file (save_bank format, embedding.cpp:77-98 / SPEC.md:285)
 * straight into the device bank (f32 -> bf16 on device, chunked, no host bank). */
int ngram_bank_load_file(ngram_bank* bank, const char* path);
/* Size the per-bank workspace for calls of up to max_tokens tokens (no hot-path allocation). */
int ngram_bank_reserve(ngram_bank* bank, int64_t max_tokens);

typedef struct ngram_bank_info {
    int max_order, sub_tables, dim, branch_count, branch_dim, variant, amplification, merge_denominator;
    uint32_t base_vocab;
    int shard_rank, shard_count;
    int tensor_core_path; /* 1 if forward runs the tcgen05 projection GEMM */
    uint64_t device_bytes;
    uint64_t sub_vocab[64];   /* V_b in branch order */
    int64_t row_lo[64];       /* this shard's first row of table b */
    int64_t row_hi[64];       /* one past this shard's last row of table b */
    const void* sub_ptr;      /* dev: concatenated local sub-table rows (bf16) */
    const void* e0_ptr;       /* dev: E0 (bf16) */
    const void* wcat_ptr;     /* dev: W_cat (bf16), NULL for v1 */
} ngram_bank_info;
int ngram_bank_get_info(const ngram_bank* bank, ngram_bank_info* info);

/* ------------------------------------------------------------------ hashing */
/* rolling_hash over `count` windows (hashing.cpp:33-59).  windows: dev, count x stride
 * u32, window i = windows[i*stride .. i*stride+lengths[i]) oldest first; lengths (NULL =
 * orders), orders, bases, moduli: dev per-window hash_spec; out: dev u64.  status: dev
 * i32 per window: 0, NGRAM_EINVAL (hash_spec::validate or length != order) or
 * NGRAM_ERANGE (token >= base) -- the per-call exception of the reference. */
int ngram_rolling_hash_batch(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                             const uint64_t* bases, const uint64_t* moduli, int64_t count, uint64_t* out,
                             int32_t* status, void* stream);
/* hash_all_orders at every position of a batch of sequences (hashing.cpp:61-81 with the
 * windows of embed_sequence, embedding.hpp:391-405).
 *   tokens:      dev u32, total_tokens, sequences concatenated
 *   seq_offsets: dev i64, nseq+1 prefix offsets (seq s = tokens[off[s], off[s+1])); the
 *     device entry points trust them (0 = off[0] <= ... <= off[nseq] = total_tokens; the
 *     host entry points check) -- a malformed window is reported like a bad token
 *   prior:       dev u32 nseq x (N-1), the N-1 tokens preceding each sequence
 *                (prior_context, right-aligned, 0 = pad), or NULL for none
 *   ids_out:     dev, total_tokens x branch_count, u64 if ids_u64 else u32, entry
 *                [t][branch_index(n,k)] exactly as hash_all_orders' vector. */
int ngram_hash_ids(ngram_bank* bank, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                   int64_t total_tokens, const uint32_t* prior, void* ids_out, int ids_u64, void* stream);

/* ------------------------------------------------------------------ forward */
/* embed_sequence_cached over a batch (embedding.hpp:409-429): rows_out = amplify(merged),
 * merged_out = merged (either may be NULL), each total_tokens x D of out_dtype, dev. */
int ngram_embed_forward(ngram_bank* bank, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                        int64_t total_tokens, const uint32_t* prior, void* rows_out, void* merged_out,
                        int out_dtype, void* stream);
/* Which prefill kernel sequence ngram_embed_forward runs for a batch of total_tokens (for
 * benchmarks and logs): 0 fused K1+K2 -> X -> tcgen05 projection (or the small-T / CUDA-core
 * paths), 1 K1+K2 in the projection's producers, 2 the fused wide-tile kernel (D <= 768). */
int ngram_prefill_path(ngram_bank* bank, int64_t total_tokens, int* path);
/* embed_from_ids (embedding.hpp:163-201) for T tokens: ids dev u64 T x branch_count
 * (global bucket ids), merged_out dev T x D (pre-amplification, as the reference). */
int ngram_embed_from_ids(ngram_bank* bank, const uint32_t* tokens, const uint64_t* ids, int64_t T, void* merged_out,
                         int out_dtype, void* stream);
/* Synchronise `stream` and report (then clear) the bank's device error word:
 * NGRAM_ERANGE with the offending token when a token >= V0 was seen.  Decode steps and
 * verify + commit pairs do not reset the word per call: their last kernel moves a token error
 * into a reported word instead (so back-to-back steps need no reset node); this call reports
 * the earliest of both since the last sync. */
int ngram_sync_errors(ngram_bank* bank, void* stream);
/* Host-buffer entry (the drop-in embed_sequence path): copies tokens/prior from host,
 * runs the forward, copies rows/merged back to host (NULL to skip), overlapping the
 * copies with compute in chunks.  Synchronous; raises ERANGE before returning output. */
int ngram_embed_sequence_host(ngram_bank* bank, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                              const uint32_t* prior, void* rows_out, void* merged_out, int out_dtype);

/* Stage profiling: when enabled, every forward records CUDA events on its launch stream
 * around K1 (hash-index) and K2+K3 (gather + projection [+ LayerNorm]).
 * ngram_profile_read synchronises on the last event and returns the stage times (ms)
 * of the most recent forward: stage_ms[0] = hash, stage_ms[1] = gather (K2), stage_ms[2] = projection (K3). */
int ngram_profile_enable(ngram_bank* bank, int enable);
int ngram_profile_read(ngram_bank* bank, float* stage_ms, int n);

/* Host-buffer variants (synchronous) used by the C++ drop-in layer (include/ngram/*.hpp):
 * same semantics as the device entries above, all pointers host memory. */
int ngram_hash_ids_host(ngram_bank* bank, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                        const uint32_t* prior, uint64_t* ids_out);
int ngram_rolling_hash_host(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                            const uint64_t* bases, const uint64_t* moduli, int64_t count, uint64_t* out,
                            int32_t* status);
int ngram_embed_from_ids_host(ngram_bank* bank, const uint32_t* tokens, const uint64_t* ids, int64_t T,
                              float* merged_out);

/* ------------------------------------------------------------------ decode / verify */
/* A batch of `batch` decode streams (sequence_cache, cache.hpp:38-80): per-stream ring
 * of the trailing N-1 confirmed tokens (zero-initialised), length and last token,
 * resident on the device.  max_draft bounds verify blocks. */
int ngram_decode_create(ngram_bank* bank, int64_t batch, int max_draft, ngram_decode** out);
int ngram_decode_destroy(ngram_decode* st);
/* Reset every stream; prior (dev u32 batch x (N-1), may be NULL = zeros) seeds the ring
 * as if those tokens had been appended (prefill hand-off); lengths (dev u64 or NULL). */
int ngram_decode_reset(ngram_decode* st, const uint32_t* prior, const uint64_t* lengths, void* stream);
/* One decode step for every stream: sequence_cache::append(tokens[s]) (cache.cpp:37-57)
 * followed by embed_from_ids (cache.cpp:136): ids_out (dev u64 batch x branch_count, may
 * be NULL), merged_out (dev batch x D, pre-amplification, may be NULL). */
int ngram_decode_step(ngram_decode* st, const uint32_t* tokens, uint64_t* ids_out, void* merged_out, int out_dtype,
                      void* stream);
/* Speculative verification block (draft_verify, cache.cpp:152-195): for every stream s
 * and draft position i < L, the merged embedding of draft[s][i] given ring ++
 * draft[s][0..i) -- WITHOUT changing the state (the snapshot/rollback of the reference).
 * draft: dev u32 batch x L; merged_out: dev batch x L x D. */
int ngram_verify_block(ngram_decode* st, const uint32_t* draft, int L, void* merged_out, int out_dtype,
                       void* stream);
/* Accept the first accept[s] (0..L) draft tokens of every stream: the state afterwards
 * equals accept[s] sequential appends (cache.cpp:185-193); accept > L -> EINVAL. */
int ngram_commit(ngram_decode* st, const uint32_t* draft, int L, const int32_t* accept, void* stream);
/* Host-buffer variants of reset / step / verify+commit for the C++ sequence_cache / draft_verify. */
int ngram_decode_reset_host(ngram_decode* st, const uint32_t* prior, const uint64_t* lengths);
int ngram_decode_step_host(ngram_decode* st, const uint32_t* tokens, uint64_t* ids_out, float* merged_out);
int ngram_verify_commit_host(ngram_decode* st, const uint32_t* draft, int L, const int32_t* accept,
                             float* merged_out);
/* Overwrite the state (host buffers): ring batch x (N-1) (NULL = zeros), length (NULL = 0)
 * and last token (NULL = the ring's newest entry) -- an exact restore of ngram_decode_get_state
 * (sequence_cache::rollback, cache.cpp:78-87). */
int ngram_decode_set_state_host(ngram_decode* st, const uint32_t* ring, const uint64_t* length, const uint32_t* last);
/* Read back the state (host buffers): ring batch x (N-1), length, last token. */
int ngram_decode_get_state(ngram_decode* st, uint32_t* ring, uint64_t* length, uint32_t* last);
/* Device pointer of the rings [batch][max_order-1] (oldest first): the `prior` of a decode
 * step / verify block.  On a row-sharded bank a decode state holds only ring state
 * (create / reset / commit / get_state); its steps run through the shard group: all-gather
 * the step's tokens and the rings, ngram_shard_scatter_rows(all_prior = gathered rings),
 * barrier, ngram_shard_project (merged out), then ngram_commit on the local state. */
int ngram_decode_ring(ngram_decode* st, uint32_t** ring);
/* Stream-ordered copy of the rings [batch][max_order-1] into dst (device or host). */
int ngram_decode_copy_ring(ngram_decode* st, uint32_t* dst, void* stream);

/* ------------------------------------------------------------------ multi-GPU (row shards) */
/* Row-sharded exchange.  A process group of shard_count ranks, one GPU
 * each; rank r's bank holds its row block of every sub-table.  Each rank owns a
 * double-buffered X (home tokens x D, bf16).  Per step:
 *   1. all ranks hold the ALL-GATHERED token batch (4 B/token; the caller all-gathers);
 *   2. ngram_shard_scatter_rows: K1 over the whole batch, then a fused gather + NVLink
 *      peer-store kernel writes every locally owned row straight into its home rank's X;
 *   3. a cross-rank barrier on `stream` (e.g. a 1-element NCCL all-reduce);
 *   4. ngram_shard_project: K3 on this rank's X (its home tokens) -> rows / merged.
 * X is double-buffered (scatter i+1 writes the other buffer), so one barrier per step is
 * enough.  Peer buffers are CUDA IPC mappings: ngram_shard_export writes
 * NGRAM_SHARD_HANDLE_BYTES that the caller moves to every peer for ngram_shard_open.
 * ngram_shard_set_peer maps a peer's buffers by device pointer instead (all ranks in one
 * process: the single-GPU emulation used by the tests). */
#define NGRAM_SHARD_HANDLE_BYTES 128
/* Host-only: rank r's row block [lo, hi) of a table of V rows over `count` ranks,
 * lo = ceil(r*V/count) (owner(h) = floor(h*count/V)).  The partition every bank uses. */
int ngram_shard_rows(uint64_t V, int rank, int count, int64_t* lo, int64_t* hi);
typedef struct ngram_shard_group ngram_shard_group;
int ngram_shard_group_create(ngram_bank* bank, int64_t max_home_tokens, ngram_shard_group** out);
int ngram_shard_group_destroy(ngram_shard_group* g);
int ngram_shard_export(ngram_shard_group* g, void* handle_out);
int ngram_shard_open(ngram_shard_group* g, int peer_rank, const void* handle);
int ngram_shard_local_buffers(ngram_shard_group* g, void** x0, void** x1);
int ngram_shard_set_peer(ngram_shard_group* g, int peer_rank, void* x0, void* x1);
/* all_tokens/all_seq_offsets/all_prior: dev, the gathered batch (sequences of rank r are
 * [rank_seq_offsets[r], rank_seq_offsets[r+1]) of it); rank_token_offsets: HOST int64
 * shard_count+1 prefix offsets of each rank's home tokens in all_tokens. */
int ngram_shard_scatter_rows(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                             int64_t all_nseq, int64_t all_tokens_n, const int64_t* rank_token_offsets,
                             const uint32_t* all_prior, void* stream);
/* Projection + epilogue of this rank's home tokens (home_tokens: dev, home_T) from its X. */
int ngram_shard_project(ngram_shard_group* g, const uint32_t* home_tokens, int64_t home_T, void* rows_out,
                        void* merged_out, int out_dtype, void* stream);

/* NCCL exchange variants of step 2 (SURVEY.md 8(e) "all-to-all of rows" for large
 * batches, "reduce-scatter of the zero-padded X" for decode / verify).  The caller runs the
 * collective (NCCL through torch.distributed, or grouped ncclSend/ncclRecv); rows move raw, so
 * every variant leaves the same home X as the peer-store scatter, bit for bit.  Arguments of the
 * gathered batch as ngram_shard_scatter_rows.
 * All-to-all:
 *   1. ngram_shard_xchg_prepare: K1 over the gathered batch + the exchange counts; synchronises
 *      `stream`; send_rows[p] / recv_rows[p] (HOST, nranks) = d-wide bf16 rows this rank sends to /
 *      receives from rank p;
 *   2. ngram_shard_xchg_pack: the owned rows into `send` (dev, sum(send_rows) x d bf16), grouped
 *      by destination rank, (token, branch) order within a group;
 *   3. the all-to-all (send splits send_rows, receive splits recv_rows, rank order);
 *   4. ngram_shard_xchg_unpack: the received rows (dev, sum(recv_rows) x d) into this rank's home X
 *      (each row's slot follows from the ids this rank hashed: no index travels with the rows);
 *   5. ngram_shard_project.
 * Reduce-scatter:
 *   1. ngram_shard_pack_padded: `send` (dev, nranks x max_home_tokens x D bf16) = every rank's
 *      home X with only this rank's rows filled, -0.0 elsewhere (the additive identity, so the sum
 *      is exact);
 *   2. reduce-scatter (sum, bf16) of `send` into ngram_shard_home_x (max_home_tokens x D);
 *   3. ngram_shard_project. */
int ngram_shard_xchg_prepare(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                             int64_t all_nseq, int64_t all_tokens_n, const int64_t* rank_token_offsets,
                             const uint32_t* all_prior, int64_t* send_rows, int64_t* recv_rows, void* stream);
int ngram_shard_xchg_pack(ngram_shard_group* g, void* send, void* stream);
int ngram_shard_xchg_unpack(ngram_shard_group* g, const void* recv, void* stream);
int ngram_shard_pack_padded(ngram_shard_group* g, const uint32_t* all_tokens, const int64_t* all_seq_offsets,
                            int64_t all_nseq, int64_t all_tokens_n, const int64_t* rank_token_offsets,
                            const uint32_t* all_prior, void* send, void* stream);
/* Device pointer of the home X the next ngram_shard_project reads (max_home_tokens x D bf16). */
int ngram_shard_home_x(ngram_shard_group* g, void** x);

/* amplify (embedding.hpp:239-287) of `rows` HOST rows of width D on the current device:
 * amp_mode 0 none, 1 scale_sqrt_d, 2 layer_norm (gain / bias of size D). Synchronous. */
int ngram_amplify_host(int amp_mode, int D, int64_t rows, const float* gain, const float* bias, const float* in,
                       float* out);

/* Dense GEMM building block of the backward pass and PLNE (device buffers, stream-ordered):
 *   C[M][N] (fp32, pitch ldc) (+)= sum_k A(m, k) B(n, k)
 * A is logical [M][K], B logical [N][K]; each stored K-major (x_mn = 0: element (r, k) at
 * x[r * ldx + k]) or MN-major (x_mn = 1: at x[k * ldx + r]).  a_terms / b_terms: 3 = split the
 * fp32 operand into three bf16 terms (fp32-accurate tcgen05 products), 1 = one bf16 term (the
 * operand must be bf16-exact for an fp32-accurate result); a_terms = 0 = the fp32 CUDA-core
 * GEMM.  The embedding backward uses (3, 1), PLNE (3, 3) with NGRAM_PLNE_FAST and (0, -). */
int ngram_gemm_f32(int device, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda, int a_mn, const float* B,
                   int64_t ldb, int b_mn, float* C, int64_t ldc, int accumulate, int a_terms, int b_terms,
                   void* stream);

/* ------------------------------------------------------------------ fp64 instantiations */
/* The reference's double-precision templates (embedding_bank_t<double>, ple_params_t<double>)
 * evaluated on the device in double, in the reference's operation order -- the instantiations
 * its gradient checks use (proj/tests/gradcases.hpp).  Host buffers, synchronous, small
 * problems (tables uploaded per call).  Tables in the reference layout: base V0 x D,
 * sub[b] V_b x d, proj[b] D x d (branch order b = (n-2)K + (k-1)).  One sequence of T tokens
 * (+ prior context, right-aligned).  rows (amplified) may be NULL. */
int ngram_f64_forward(const char* config_json, const double* base, const double* const* sub,
                      const double* const* proj, const double* ln_gain, const double* ln_bias, const uint32_t* tokens,
                      int64_t T, const uint32_t* prior, int64_t prior_len, double* merged, double* rows);
/* embed_sequence_backward (merged != NULL: through amplify) / embed_backward (merged == NULL:
 * upstream is d(merged)); gradients ACCUMULATED into the host tables g_*. */
int ngram_f64_backward(const char* config_json, const double* base, const double* const* sub,
                       const double* const* proj, const double* ln_gain, const double* ln_bias, const uint32_t* tokens,
                       int64_t T, const uint32_t* prior, int64_t prior_len, const double* merged,
                       const double* upstream, double* g_base, double* const* g_sub, double* const* g_proj,
                       double* g_gain, double* g_bias);
int ngram_f64_amplify(int amp_mode, int64_t D, const double* gain, const double* bias, const double* in, double* out);
int ngram_f64_amplify_backward(int amp_mode, int64_t D, const double* pre, const double* upstream, const double* gain,
                               double* d_pre, double* g_gain, double* g_bias);
/* gated FFN body of ffn_ple / ffn_plne (ple.hpp:77-146): y = W_d (SiLU(W_g x) (.) g); the
 * backward accumulates g_gate, g_down, dx and dg (+= dL/dg). */
int ngram_f64_gated_ffn(int d_model, int hidden, const double* gate, const double* down, const double* x,
                        const double* g, double* y);
int ngram_f64_gated_ffn_backward(int d_model, int hidden, const double* gate, const double* down, const double* x,
                                 const double* g, const double* upstream, double* g_gate, double* g_down, double* dx,
                                 double* dg);

/* ------------------------------------------------------------------ backward (training) */
/* embed_sequence_backward (embedding.hpp:438-459) batched on the device: gradients of the
 * embedding rows w.r.t. every bank parameter, ACCUMULATED (+=) into an fp32 gradient bank
 * with the device layout (E0 V0 x D, sub-tables concatenated by branch, projections as
 * W_cat D x D, LN gain / bias D).  amplify_backward (embedding.hpp:291-336) then
 * embed_backward (:338-376) per position; the dense products dW_cat += U^T X and
 * dX = U W_cat are fp32-accurate GEMMs on the tensor cores (U split into three bf16 terms,
 * X / W_cat bf16-exact; pedantic fp32 on CUDA-core-shaped banks; see the flags below);
 * scatters use fp32 atomics, so results match the reference within an fp32 tolerance (not
 * bit-exact).  Single-shard banks only. */
typedef struct ngram_grad ngram_grad;
int ngram_grad_create(ngram_bank* bank, ngram_grad** out); /* zero-initialised */
/* NGRAM_GRAD_SPARSE_ROWS: the sub-table gradient is kept row-sparse instead of dense -- every
 * backward call APPENDS its (storage row, d-wide gradient row) pairs for all T x B
 * (position, branch) rows (duplicates not merged: their sum is the dense gradient).  E0,
 * W_cat and LN gradients stay dense.  Needed at LongCat scale, where a dense fp32 copy of
 * the 31.5 B sub-table parameters (126 GB) does not fit beside the tables. */
#define NGRAM_GRAD_SPARSE_ROWS 1
/* Backward GEMM precision on tensor-core banks (X and W_cat are exact bf16 values; only the
 * fp32 U = d(merged) * 1/denom is split into bf16 terms, products accumulated in fp32):
 *   default              U in two bf16 terms (17-bit operand, ~2-3e-6 relL2 of pedantic fp32 at
 *                        D = 3072; the 1e-5 gradient contract holds)
 *   NGRAM_GRAD_EXACT     three terms (24-bit operand: fp32-accurate, 1.5x the default's MMAs)
 *   NGRAM_GRAD_TF32      one term (U rounded to bf16: ~1e-3 relative, training precision; the
 *                        name is kept from the TF32 form it replaces)
 *   NGRAM_GRAD_PEDANTIC  the fp32 CUDA-core GEMM (also every bank without a tensor-core shape) */
#define NGRAM_GRAD_TF32 2
#define NGRAM_GRAD_PEDANTIC 4
#define NGRAM_GRAD_EXACT 8
/* NGRAM_GRAD_SPARSE_BASE: the E0 (base-table) gradient is kept as COO pairs too -- each call
 * appends (token, u) per position (u = the D-wide merged-row gradient, duplicates unmerged) --
 * instead of scatter-adding into a dense V0 x D table: no per-step zeroing of that table and no
 * read-modify-write of its rows.  ngram_grad_sparse_base reads the pairs; ngram_grad_tensor(0) /
 * ngram_grad_download densify on request. */
#define NGRAM_GRAD_SPARSE_BASE 16
int ngram_grad_create_ex(ngram_bank* bank, int flags, ngram_grad** out);
/* Row-sparse gradient view: rows = dev int32 [count] storage rows (the device layout of
 * ngram_grad_tensor(1)), vals = dev f32 [count][branch_dim]; count resets on ngram_grad_zero. */
int ngram_grad_sparse_rows(ngram_grad* g, int32_t** rows, float** vals, int64_t* count);
/* Copy pairs [first, first + count) to caller buffers (host or device; stream-ordered).
 * Pairs appended by a call whose tokens were out of range carry row -1 (no gradient). */
int ngram_grad_sparse_read(ngram_grad* g, int64_t first, int64_t count, int32_t* rows, float* vals, void* stream);
/* NGRAM_GRAD_SPARSE_BASE: the base-table gradient pairs, tokens = dev int32 [count], vals = dev
 * f32 [count][D]; count resets on ngram_grad_zero. */
int ngram_grad_sparse_base(ngram_grad* g, int32_t** tokens, float** vals, int64_t* count);
int ngram_grad_destroy(ngram_grad* g);
int ngram_grad_zero(ngram_grad* g, void* stream);
#define NGRAM_BWD_SKIP_AMPLIFY 1 /* upstream is d(merged) already: embed_backward only */
/* tokens/seq_offsets/prior as ngram_embed_forward (device); merged: dev f32 [T][D], the
 * pre-amplification rows of the forward (needed for layer_norm, else may be null);
 * upstream: dev f32 [T][D], dL/d(rows). */
int ngram_embed_backward(ngram_grad* g, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                         int64_t total_tokens, const uint32_t* prior, const float* merged, const float* upstream,
                         int flags, void* stream);
/* Same with HOST buffers (tokens, seq_offsets, prior, merged, upstream); synchronous; an
 * out-of-range token returns NGRAM_ERANGE and leaves the gradients untouched. */
int ngram_embed_backward_host(ngram_grad* g, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                              const uint32_t* prior, const float* merged, const float* upstream, int flags);
/* amplify_backward (embedding.hpp:291-336) of `rows` HOST rows with the bank's amplification
 * and LN gain: d_pre = d(amplify)/d(pre) . upstream; layer_norm ACCUMULATES the gain / bias
 * gradients into g_gain / g_bias (host, size D; null skips). Synchronous. */
int ngram_amplify_backward_host(ngram_bank* bank, int64_t rows, const float* pre, const float* upstream, float* d_pre,
                                float* g_gain, float* g_bias);
/* Device view of one gradient tensor: which 0 = E0, 1 = sub-tables (device row layout),
 * 2 = W_cat, 3 = ln_gain, 4 = ln_bias. */
int ngram_grad_tensor(ngram_grad* g, int which, float** dev_ptr, int64_t* numel);
/* Host copy in the reference layout (embedding_bank_t): base V0 x D, sub[b] V_b x d,
 * proj[b] D x d (v2 only), gain / bias D (layer_norm only); null pointers are skipped. */
int ngram_grad_download(ngram_grad* g, float* base, float* const* sub, float* const* proj, float* gain, float* bias);

/* ------------------------------------------------------------------ PLNE (per-layer FFN) */
/* ffn_plne (ple.hpp:168-181) batched on the device: y = W_d (SiLU(W_g x) (.) g) with g the
 * layer bank's merged embedding of each position's window (layer bank: amplification none,
 * dim = hidden).  gate: dev f32 [hidden][d_model]; down: dev f32 [d_model][hidden];
 * x, y: dev f32 [T][d_model]; tokens / seq_offsets / prior as ngram_embed_forward.  fp32-
 * accurate GEMMs (the library's tcgen05 GEMMs on split-bf16 operands by default; CUDA-core
 * fp32 with NGRAM_PLNE_PEDANTIC, see ngram_plne_create_ex).  ffn_ple (table-row gate) = a
 * base-only layer bank (max_order 1).
 * Outputs are unspecified when a token is out of range (NGRAM_ERANGE at the next sync). */
typedef struct ngram_plne ngram_plne;
int ngram_plne_create(ngram_bank* layer_bank, int d_model, ngram_plne** out);
/* Default (flags 0, or NGRAM_PLNE_FAST): the GEMMs on the bf16 tensor cores with both operands
 * split into three bf16 terms (six products, K chunks folded into fp32 registers): relL2
 * ~3e-7 vs fp64 at K = 3072, ~7x faster than NGRAM_PLNE_PEDANTIC -- the CUDA-core fp32 GEMM
 * (relL2 ~4e-7 there). */
#define NGRAM_PLNE_FAST 1
#define NGRAM_PLNE_PEDANTIC 2
int ngram_plne_create_ex(ngram_bank* layer_bank, int d_model, int flags, ngram_plne** out);
int ngram_plne_destroy(ngram_plne* p);
int ngram_plne_forward(ngram_plne* p, const float* gate, const float* down, const float* x, const uint32_t* tokens,
                       const int64_t* seq_offsets, int64_t nseq, int64_t total_tokens, const uint32_t* prior, float* y,
                       void* stream);
/* ffn_plne_backward (ple.hpp:183-196): ACCUMULATES d_gate, d_down, dx (dev f32, shapes as
 * gate / down / x) and, when bank_grads is not null, the layer bank's gradients. */
int ngram_plne_backward(ngram_plne* p, ngram_grad* bank_grads, const float* gate, const float* down, const float* x,
                        const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, int64_t total_tokens,
                        const uint32_t* prior, const float* upstream, float* d_gate, float* d_down, float* dx,
                        void* stream);
/* Host-buffer variants (synchronous; total_tokens = seq_offsets[nseq]); a token out of range
 * returns NGRAM_ERANGE.  The backward accumulates into the host d_gate / d_down / dx. */
int ngram_plne_forward_host(ngram_plne* p, const float* gate, const float* down, const float* x,
                            const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, const uint32_t* prior,
                            float* y);
int ngram_plne_backward_host(ngram_plne* p, ngram_grad* bank_grads, const float* gate, const float* down,
                             const float* x, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                             const uint32_t* prior, const float* upstream, float* d_gate, float* d_down, float* dx);

/* ------------------------------------------------------------------ corpus analysis */
/* Replaces corpus_analyzer (analysis.hpp:45-93, analysis.cpp:44-176): every position of every
 * sequence contributes one zero-padded window per order; counts windows seen, distinct windows
 * (exact, by their 128-bit polynomial value) and distinct buckets per (order, modulus).
 * Create checks and messages follow analysis.cpp:47-85 (EINVAL).  A token >= base_vocab:
 * like add_sequence/add_corpus, the sequences up to and including the bad one are counted
 * (with their full length) and the positions before the bad token are analysed; the error is
 * NGRAM_ERANGE from ngram_analyzer_add_host, or from ngram_analyzer_sync_errors after the
 * device entry.  Not thread-safe across concurrent adds to one analyzer (serialised). */
typedef struct ngram_analyzer ngram_analyzer;
int ngram_analyzer_create(int device, uint64_t base_vocab, const int* orders, int n_orders, const uint64_t* moduli,
                          int n_moduli, ngram_analyzer** out);
void ngram_analyzer_destroy(ngram_analyzer* a);
/* tokens: dev u32 [T]; seq_offsets: dev i64 [nseq+1], 0 = off[0] <= ... <= off[nseq] = T. */
int ngram_analyzer_add(ngram_analyzer* a, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq, int64_t T,
                       void* stream);
/* Host tokens / offsets (checked), synchronous. */
int ngram_analyzer_add_host(ngram_analyzer* a, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq);
/* Set-union merge (analysis.cpp:125-141): same base / orders / moduli, same device. */
int ngram_analyzer_merge(ngram_analyzer* dst, ngram_analyzer* src, void* stream);
/* Pre-size every set for `windows` more positions (no rehash inside the next adds;
 * the reference's unordered_set::reserve).  Synchronous. */
int ngram_analyzer_reserve(ngram_analyzer* a, uint64_t windows);
int ngram_analyzer_sync_errors(ngram_analyzer* a);
/* Synchronous.  ngrams_seen / distinct_ngrams: [n_orders]; distinct_buckets: [n_orders][n_moduli]
 * (order-major, the reference's layout).  Any pointer may be NULL. */
int ngram_analyzer_stats(ngram_analyzer* a, uint64_t* sequences, uint64_t* tokens, uint64_t* ngrams_seen,
                         uint64_t* distinct_ngrams, uint64_t* distinct_buckets);

#ifdef __cplusplus
}
#endif
#endif /* NGRAM_B200_H */
