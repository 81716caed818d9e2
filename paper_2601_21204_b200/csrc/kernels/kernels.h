// kernels.h -- host-side launchers for the sm_100a kernels (implemented in *.cu).
// Used only by the C++ host layer (csrc/host/*.cpp); no torch types anywhere.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace ngk {

constexpr int kMaxBranches = 64;
constexpr int kMaxOrder = 16;

// Immutable shape + hashing constants of a bank, resident in device memory.
struct HashTables {
    uint64_t modulus[kMaxBranches];            // V_b
    uint64_t barrett[kMaxBranches];            // floor(2^64 / V_b) (fast path, V_b >= 2)
    uint64_t pow[kMaxBranches][kMaxOrder];     // V0^j mod V_b
    int64_t row_base[kMaxBranches];            // storage row of (local) bucket row_lo[b]
    int64_t row_lo[kMaxBranches];              // first bucket stored on this shard
    int64_t row_hi[kMaxBranches];              // one past the last bucket stored here
};

struct Shape {
    int N, K, B, D, d, variant, amp, denom;
    uint32_t V0;
    int fast_hash;  // all V_b <= 2^32
};

enum AmpMode { kAmpNone = 0, kAmpSqrt = 1, kAmpLN = 2 };

// Global launch counter (bench evidence: kernels launched by this library).
void count_launch(int n = 1);
uint64_t launches();

// ---- hashing (hash.cu)
// ids_tok: [T][B] (u32 or u64) or null; grow: [B][Tpad] int32 storage rows (or -1 when the
// row is not local to this shard) or null.  err: device u64, min bad token index.
void launch_hash_ids(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                     int64_t nseq, int64_t T, const uint32_t* prior, void* ids_tok, int ids_u64, int32_t* grow,
                     int64_t Tpad, unsigned long long* err, cudaStream_t st);
// K1+K2 fused (X path): hash every position (lane per branch) and gather its rows into X.
void launch_hash_gather(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                        int64_t nseq, int64_t T, const uint32_t* prior, const __nv_bfloat16* sub, __nv_bfloat16* X,
                        int32_t* grow, int64_t Tpad, unsigned long long* err, cudaStream_t st, int64_t t_begin = 0,
                        int64_t t_end = -1, int64_t x_row0 = 0);  // X row 0 holds position x_row0
// Same, one warp per (position, branch): the small-T (decode / verify) latency variant.
void launch_hash_gather_rows(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* seq_off,
                             int64_t nseq, int64_t T, const uint32_t* prior, const __nv_bfloat16* sub,
                             __nv_bfloat16* X, unsigned long long* err, cudaStream_t st, int64_t uniform_len = 0);
// Token range check only (tokens and used prior tokens < V0), min bad window -> err.
void launch_validate_tokens(const Shape& s, const uint32_t* tokens, int64_t T, const int64_t* seq_off, int64_t nseq,
                            const uint32_t* prior, unsigned long long* err, cudaStream_t st);
void launch_rolling_hash_batch(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                               const uint64_t* bases,
                               const uint64_t* moduli, int64_t count, uint64_t* out, int32_t* status,
                               cudaStream_t st);
// ids (u64 [T][B], global bucket ids) -> grow (branch-major storage rows); validates range.
void launch_ids_to_rows(const Shape& s, const HashTables* ht, const uint64_t* ids, const uint32_t* tokens, int64_t T,
                        int32_t* grow, int64_t Tpad, unsigned long long* err, cudaStream_t st);

// ---- bank (bank.cu)
void launch_synth_fill_bf16(__nv_bfloat16* dst, uint64_t seed, uint32_t table, int64_t row0, int64_t nrows, int ncols,
                            int64_t pitch, float scale, cudaStream_t st);
// W_cat[i][b*d + j] = synth(100+b, i, j)
void launch_synth_wcat(__nv_bfloat16* wcat, uint64_t seed, int D, int d, int B, float scale, cudaStream_t st);
void launch_f32_to_bf16(const float* src, __nv_bfloat16* dst, int64_t n, cudaStream_t st);
// proj_b (D x d f32, dev) -> W_cat columns [b*d, (b+1)*d)
void launch_pack_wcat(const float* proj_b, __nv_bfloat16* wcat, int D, int d, int b, cudaStream_t st);
void launch_fill_f32(float* dst, float v, int64_t n, cudaStream_t st);

// ---- forward
// ---- backward (backward.cu): embed_sequence_backward's scatter / elementwise parts
// dense[tok[i]][:] += vals[i][:] over n D-wide rows
void launch_coo_densify(const int32_t* tok, const float* vals, int64_t n, int D, float* dense, cudaStream_t st);
// U (fp32, may be null) and / or `nterms` bf16 split terms of u (terms + h * tstride, may be null);
// g_e0 null: no E0 scatter-add (the sparse base-table gradient keeps U as its values).
void launch_amp_backward(const Shape& s, const float* up, const float* pre, const uint32_t* tokens, int64_t T,
                         int amp, const float* gain, float* U, float* g_e0, float* g_gain, float* g_bias,
                         const unsigned long long* err, cudaStream_t st, __nv_bfloat16* terms = nullptr,
                         int nterms = 0, int64_t tstride = 0);
void launch_gather_rows_f32(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, const __nv_bfloat16* sub,
                            float* X, const unsigned long long* err, cudaStream_t st);
void launch_scatter_rows(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, int width, int src_stride,
                         int src_branch_step, const float* src, float* g_sub, const unsigned long long* err,
                         cudaStream_t st);
void launch_bf16_to_f32(const __nv_bfloat16* src, float* dst, int64_t n, cudaStream_t st);
// u <- TF32-rounded u (round to nearest), lo <- the fp32 remainder (two-term TF32 GEMMs)
void launch_split_tf32(float* u, float* lo, int64_t n, cudaStream_t st);
void launch_split_tf32_copy(const float* a, float* hi, float* lo, int64_t n, cudaStream_t st);
// u -> u1 + u2 + u3 in bf16 (three-term split for bf16 tensor-core GEMMs with fp32-level accuracy)
// ---- fp64 instantiations of the reference templates (f64.cu): one sequence, small banks
void launch_f64_forward(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* off, int64_t T,
                        const uint32_t* prior, const double* base, const double* sub, const double* proj,
                        const double* gain, const double* bias, int amp, double* merged, double* rows,
                        cudaStream_t st);
// ws: [T][D] d_pre + [T][2][D] zeroed LN scratch
void launch_f64_backward(const Shape& s, const HashTables* ht, const uint32_t* tokens, const int64_t* off, int64_t T,
                         const uint32_t* prior, const double* sub, const double* proj, const double* gain, int amp,
                         const double* merged, const double* upstream, double* ws, double* g_base, double* g_sub,
                         double* g_proj, double* g_gain, double* g_bias, cudaStream_t st);
void launch_f64_amplify(int amp, int D, const double* gain, const double* bias, const double* in, double* out,
                        cudaStream_t st);
void launch_f64_amplify_backward(int amp, int D, const double* pre, const double* up, const double* gain,
                                 double* d_pre, double* g_gain, double* g_bias, cudaStream_t st);
void launch_f64_gated_ffn(int Dm, int H, const double* gate, const double* down, const double* x, const double* g,
                          double* h_ws, double* y, cudaStream_t st);
void launch_f64_gated_ffn_backward(int Dm, int H, const double* gate, const double* down, const double* x,
                                   const double* g, const double* up, double* ws, double* g_gate, double* g_down,
                                   double* dx, double* dg, cudaStream_t st);

// ---- dense GEMMs (gemm_gen.cu): C[M][N] (fp32) (+)= sum of term-pair products A_i . B_j^T.
// Operands are logical [R][K] (R = M for A, N for B): K-major maps are (inner K, rows R, box
// 64 x 128), MN-major maps (inner R, rows K, box 64 x 64); na / nb in {1, 3} terms.
void launch_gemm_bf16_terms(const CUtensorMap* ma, int na, bool a_mn, const CUtensorMap* mb, int nb, bool b_mn,
                            int64_t M, int64_t N, int64_t K, float* C, int64_t ldc, bool accumulate, int num_sms,
                            cudaStream_t st);
// fp32 CUDA-core GEMM, same convention (pedantic mode), two-level (per 16-k block) accumulation.
void launch_gemm_f32(const float* A, int64_t lda, bool a_mn, const float* B, int64_t ldb, bool b_mn, int64_t M,
                     int64_t N, int64_t K, float* C, int64_t ldc, bool accumulate, cudaStream_t st);
// rows x cols fp32 (pitch ldx) -> up to three bf16 terms (pitch ldt; t1 / t2 may be null).
void launch_split3(const float* x, int64_t rows, int64_t cols, int64_t ldx, __nv_bfloat16* t0, __nv_bfloat16* t1,
                   __nv_bfloat16* t2, int64_t ldt, cudaStream_t st);
void launch_split_bf16x3(const float* u, __nv_bfloat16* u1, __nv_bfloat16* u2, __nv_bfloat16* u3, int64_t n,
                         cudaStream_t st);
void launch_rows_to_coo(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, int32_t* rows,
                        const unsigned long long* err, cudaStream_t st);

// ---- PLNE (plne.cu): SwiGLU gating by the layer bank's embedding
void launch_silu_gate(const float* U, const float* G, float* Hh, int64_t n, const unsigned long long* err,
                      cudaStream_t st);
void launch_silu_gate_backward(const float* dHh, const float* U, const float* G, float* dG, float* dU, int64_t n,
                               const unsigned long long* err, cudaStream_t st);

// standalone amplify (simt.cu): out = in * s
void launch_scale(const float* in, float* out, int64_t n, float s, cudaStream_t st);

struct FwdArgs {
    Shape s;
    const HashTables* ht;
    const uint32_t* tokens;  // [T] base token per row (E0 row)
    const int32_t* grow;     // [B][Tpad] storage rows
    const __nv_bfloat16* sub;
    const __nv_bfloat16* e0;
    const __nv_bfloat16* wcat;
    const float* ln_gain;
    const float* ln_bias;
    int64_t T, Tpad;     // rows of this call; grow row stride (>= round_up(T, 128))
    void* rows_out;    // amplified, may be null
    void* merged_out;  // pre-amplification, may be null
    int out_bf16;
    const unsigned long long* err;
    // tensor maps (tensor-core path)
    const CUtensorMap* tmap_sub;
    const CUtensorMap* tmap_w;
    const CUtensorMap* tmap_w2;  // W_cat with a 128-row box (2-CTA kernel), or null
    const CUtensorMap* tmap_w32;  // W_cat, 32-column x 128-row box, SWIZZLE_64B (gemm_wide.cu), or null
    // X (materialised gathered rows, T x D bf16) instead of sub-table gather, or null
    const CUtensorMap* tmap_x;
    // decode step: commit the decode state in the projection kernel's tail (or null)
    const struct DecodeCommit* commit;
    // TMA epilogue of the pair kernel: [T][D] output maps (32 x 32 box; SWIZZLE_128B fp32 /
    // SWIZZLE_64B bf16) and the E0 gather map ([V0][D] bf16, 32 x 1 box, SWIZZLE_64B), or null
    const CUtensorMap* tmap_rows_out;
    const CUtensorMap* tmap_merged_out;
    const CUtensorMap* tmap_e0;
    const CUtensorMap* tmap_e0w;  // E0 gather map with a 64-column box, SWIZZLE_128B (epilogue mode 4)
    // small-T split-K with the hash fused into the GEMM producer (MODE 2): the windows of
    // `tokens` (seq_off / nseq / prior as ngram_embed_forward); null seq_off = not used
    const int64_t* seq_off;
    int64_t nseq;
    const uint32_t* prior;
    // T that selects the split-K sub-regime (0 = T): a row-sharded projection of home_T rows
    // takes the regime of the gathered batch, so its rows are computed as the 1-GPU call's
    int64_t regime_T;
    // prefill with seq_off set: the fused wide-tile kernel (gemm_wide.cu) instead of the pair
    // kernel's hashing producers
    int wide;
};
// tcgen05 projection GEMM with fused gather + base add + scale + amplify (gemm_tc.cu).
// splitk_ws (fp32, splitk_workspace_floats() long, may be null): small-T split-K path.
void launch_forward_tc(const FwdArgs& a, int num_sms, cudaStream_t st, float* splitk_ws = nullptr);
size_t splitk_workspace_floats(const FwdArgs& a, int num_sms);
int splitk_factor(const FwdArgs& a, int num_sms);  // small-T split: depends on D and the regime of T only
// Small-T regime (split-K BN=128 GEMM + reduce, S from D only): T <= 256.  A row's
// arithmetic depends only on its own ids within a regime.
bool small_t_regime(int D, int64_t T, int num_sms);
// Fused K1+K2+K3 prefill kernel for D <= 768 (gemm_wide.cu): shapes it takes, launcher
// (a.seq_off / nseq / prior give the windows; tokens validated before the launch).
bool wide_prefill_shape(const Shape& s);
void launch_forward_wide(const FwdArgs& a, int num_sms, cudaStream_t st);
// generic CUDA-core path: any shape, v1 and v2, reference float op order (simt.cu).
void launch_forward_simt(const FwdArgs& a, cudaStream_t st);
// K2 standalone: materialise X (T x D bf16) from the storage rows (d % 8 == 0).
void launch_gather_rows(const Shape& s, const int32_t* grow, int64_t Tpad, int64_t T, const __nv_bfloat16* sub,
                        __nv_bfloat16* X, const unsigned long long* err, cudaStream_t st);
// LayerNorm amplification over merged rows (f32 merged -> rows) (simt.cu).
// merged_copy (may be null): also write the merged rows in the output dtype.
void launch_layernorm_rows(const Shape& s, const float* merged, const float* gain, const float* bias, void* rows,
                           void* merged_copy, int out_bf16, int64_t T, const unsigned long long* err,
                           cudaStream_t st);

// ---- decode (decode.cu)
// Arguments of the decode-state commit (decodedev.cuh); ring == null means "no commit".
struct DecodeCommit {
    int R;  // N - 1
    uint32_t* ring;
    uint64_t* length;
    uint32_t* last;
    const uint32_t* draft;  // [batch][L]
    int L;
    const int32_t* accept;  // [batch] or null (= L for every stream)
    int64_t batch;
    unsigned long long* derr;
    // decode step only (null otherwise): the chain's last kernel moves a token error of this
    // step into *err_reported and leaves the error word clear for the next step, so steady
    // decode needs no per-step reset node; ticket counts the finishing blocks (kept zeroed)
    unsigned long long* err_reported;
    unsigned int* ticket;
};
// Small-T projection (T <= 256, D % 128 == 0, tensor-core shape): split-K over a thread-
// block cluster with the cross-split reduction, epilogue and optional commit fused.
void launch_decode_commit_c(const DecodeCommit& c, const unsigned long long* err, cudaStream_t st);
// The hashing of a decode step / verify block is launch_hash_ids with prior = ring and
// seq_off = {0, L, 2L, ...}; these kernels move the ring.  derr: decode error word
// ((status << 32) | detail), ~0 when clear.  err_reported (or null): the commit releases the
// token-error word of the verify block it commits (DecodeCommit::err_reported).
void launch_decode_commit(const Shape& s, uint32_t* ring, uint64_t* length, uint32_t* last, const uint32_t* draft,
                          int L, const int32_t* accept, int64_t batch, unsigned long long* err,
                          unsigned long long* derr, cudaStream_t st,
                          unsigned long long* err_reported = nullptr);
void launch_decode_reset(const Shape& s, uint32_t* ring, uint64_t* length, uint32_t* last, const uint32_t* prior,
                         const uint64_t* lengths, int64_t batch, cudaStream_t st);

// ---- multi-GPU (shard.cu)
// For every (token, branch) of the all-gathered batch whose bucket row is local (grow >= 0),
// copy the row into X of the token's home rank (peer pointer) at [t_home][b*d .. b*d+d).
// rank_token_offsets: host, nranks+1 prefix offsets of each rank's home tokens.
void launch_shard_scatter(const Shape& s, const int32_t* grow_all, int64_t Tpad_all, const int64_t* rank_token_offsets,
                          int nranks, const __nv_bfloat16* sub, __nv_bfloat16* const* peer_x, int64_t T_all,
                          const unsigned long long* err, cudaStream_t st);
// NCCL exchange variants (shard.cu).  prepare: exclusive prefixes of the exchange counts
// (column 0: this rank's owned pairs over the gathered batch; column 1+o: home-token pairs owned
// by rank o) into pref [1+nranks][pref_stride]; bounds_out (dev, 2*nranks+1): column-0 prefix at
// each rank's first home token (+ the total), then the rows received from each rank.
void launch_xchg_prepare(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks,
                         const int64_t* rank_token_offsets, int64_t all_T, const uint64_t* ids_all,
                         int64_t* tot, int64_t* chunk_off, int64_t* col_tot, int64_t* pref, int64_t pref_stride,
                         int64_t* bounds_out, const unsigned long long* err, cudaStream_t st);
void launch_xchg_pack(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks, int64_t all_T,
                      const uint64_t* ids_all, const int32_t* grow_all, int64_t Tpad, const int64_t* pref0,
                      const __nv_bfloat16* sub, __nv_bfloat16* send, const unsigned long long* err, cudaStream_t st);
void launch_xchg_unpack(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks,
                        const int64_t* rank_token_offsets, const uint64_t* ids_all, const int64_t* pref,
                        int64_t pref_stride, const int64_t* recv_rows, const __nv_bfloat16* recv, __nv_bfloat16* X,
                        const unsigned long long* err, cudaStream_t st);
void launch_xchg_pack_padded(const Shape& s, const int32_t* grow_all, int64_t Tpad_all,
                             const int64_t* rank_token_offsets, int nranks, int64_t max_home,
                             const __nv_bfloat16* sub, __nv_bfloat16* send, int64_t T_all,
                             const unsigned long long* err, cudaStream_t st);
constexpr int kXchgChunkTokens = 1024;

// ---- corpus analysis (analysis.cu; corpus_analyzer, analysis.cpp:93-121)
// Open-addressing set of 128-bit keys (x = low word); all-ones = empty slot; mask = slots - 1.
struct AnSet {
    ulonglong2* slots;
    uint64_t mask;
};
// Distinct-bucket store of one (order, modulus): a bitmap of m bits, or (bits == null) a set.
struct AnBucket {
    unsigned long long* bits;
    AnSet set;
};
struct AnDev {
    uint64_t V0;
    int n_orders, n_moduli;
    const int* orders;              // [n_orders]
    const ulonglong2* vpow;         // [max_order] V0^j as 128-bit (x = low word)
    const uint64_t* moduli;         // [n_moduli]
    const uint64_t* barrett;        // floor(2^64 / m) for 2 <= m <= 2^32, else 0
    const uint64_t* c64;            // 2^64 mod m (Barrett path)
    const AnSet* ngram_sets;        // [n_orders]
    const AnBucket* buckets;        // [n_orders * n_moduli], order-major (analysis.hpp:92)
    unsigned long long* counts;     // [n_orders] distinct windows, then [n_orders * n_moduli] buckets
    unsigned long long* err;        // set to 1 if a set overflowed (host load bound violated)
};
// validate -> account (counters, insert limit, first error) -> insert.  first_bad: device
// scratch word, preset to ~0 by the caller.  meta: [sequences, tokens, ngrams_seen per order].
// err_pos: [position, token] of the analyzer's first bad token (~0 when clear).
void launch_an_add(const AnDev& a, const uint32_t* tokens, const int64_t* off, int64_t nseq, int64_t T,
                   unsigned long long* first_bad, unsigned long long* meta, unsigned long long* err_pos,
                   int num_sms, cudaStream_t st);
void launch_an_rehash(const ulonglong2* old_slots, uint64_t old_n, const AnSet& dst, unsigned long long* err,
                      int num_sms, cudaStream_t st);
void launch_an_merge_set(const ulonglong2* src, uint64_t n, const AnSet& dst, unsigned long long* counter,
                         unsigned long long* err, int num_sms, cudaStream_t st);
void launch_an_merge_bits(const unsigned long long* src, uint64_t nwords, unsigned long long* dst,
                          unsigned long long* counter, int num_sms, cudaStream_t st);
void launch_an_merge_meta(const unsigned long long* src, unsigned long long* dst, int n, cudaStream_t st);

}  // namespace ngk
