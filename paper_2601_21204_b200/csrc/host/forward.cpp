// forward.cpp -- C-ABI entry points of the prefill hot path: misc / config, hashing,
// embed forward (device buffers), embed_from_ids, and the host-buffer pipeline.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"

namespace ngh {

namespace {
thread_local std::string g_last_error;
}

int set_error(int status, const char* msg) {
    g_last_error = msg ? msg : "";
    return status;
}

// Validate the per-sequence offsets on the host side of the boundary (cheap, nseq+1).
static void check_offsets(const int64_t* off, int64_t nseq, int64_t T) {
    if (off[0] != 0 || off[nseq] != T) throw Error(NGRAM_EINVAL, "seq_offsets must start at 0 and end at total_tokens");
    for (int64_t i = 0; i < nseq; ++i)
        if (off[i + 1] < off[i]) throw Error(NGRAM_EINVAL, "seq_offsets must be non-decreasing");
}

// Fused gather (TMA gather4 straight into the GEMM's smem) vs K1+K2 -> X -> K3.  Measured
// on B200 (profiles/README.md): with the block K1+K2 kernel and the all-TMA epilogue the X
// path wins at every width (config A 56 vs 53 M tok/s, B 399 vs 375 M, C 64 vs 42 M: the
// gather4 stream cannot keep the K-blocks fed).  NGRAM_FUSED_GATHER=1 selects the fused path.
static bool fused_gather(int D) {
    static const int env = [] {
        const char* e = getenv("NGRAM_FUSED_GATHER");
        return e ? atoi(e) : 0;
    }();
    (void)D;
    return env != 0;
}

// Prefill path (tensor-core banks, D % 256 == 0, T beyond the split-K regime):
//   "x"    fused K1+K2 kernel writes X, K3 (pair kernel) reads it: two launches, X round trip
//   "wide" (gemm_wide.cu; D <= 768, d % 64 == 0) token validation, then ONE kernel: the
//          producers hash + gather an m-block's rows into shared memory once, the MMA warp
//          sweeps every N-tile over them -- no X.  Bit-identical to "x".  DEFAULT for its
//          shapes once the batch fills a wave of CTA pairs (T >= 256 x num_sms / 2): config B
//          129-131 vs 140-142 us; at T = 2048 (config A) the X path stays (23.1-24.2 vs
//          24.1-24.8 us) -- profiles/README.md
//   "lsu"  token validation, then K3 alone with K1+K2 in its producers (hash + cp.async rows
//          into shared memory; the peer CTA's stages relayed to the leader): no X, no
//          storage-row array.  Bit-identical, but measured slower (profiles/README.md):
//          config B 205 vs 150 us, C 1.30 vs 1.02 ms -- every n-tile pair re-gathers its
//          m-block's rows as 128-byte L2 requests (12x at D = 3072) where the X path moves the
//          same bytes as 16 KB TMA tiles; tensor pipe 33 % active vs 66 % (ncu).
// NGRAM_PREFILL_PATH=x|wide|lsu forces one; read per call, so one process can A/B the paths.
// Returns 0 (x), 1 (lsu) or 2 (wide).
static int prefill_path(const ngram_bank* b, int64_t T) {
    const char* e = getenv("NGRAM_PREFILL_PATH");
    const std::string v(e ? e : "");
    const int env = v == "lsu" ? 1 : v == "wide" ? 2 : v == "x" ? 0 : -1;
    const auto& s = b->shape;
    if (!b->tc_path || s.D % 256 != 0 || s.N > 8 || s.variant != 1 || s.B < 1) return 0;
    const bool wide_ok = ngk::wide_prefill_shape(s);
    if (env == 2) return wide_ok ? 2 : 0;
    if (env >= 0) return env;
    return (wide_ok && T >= 256 * int64_t(b->num_sms / 2)) ? 2 : 0;
}

// Entry points that gather rows themselves need every row on this device: a row-sharded bank
// (shard_count > 1) holds only its row block, its forward runs through the shard group.
static void require_unsharded(const ngram_bank* b, const char* what) {
    if (b->shard_count != 1)
        throw Error(NGRAM_EINVAL, std::string(what) + ": the bank is row-sharded (shard_count " +
                                      std::to_string(b->shard_count) +
                                      "); its forward runs through the shard group (ngram_shard_scatter_rows + "
                                      "ngram_shard_project)");
}

static bool small_t(const ngram_bank* b, int64_t T) { return ngk::small_t_regime(b->shape.D, T, b->num_sms); }

// Small-T split-K GEMM with the hash in its producers (MODE 2), opt-in NGRAM_DECODE_HASH_IN_GEMM=1:
// measured 2x slower than gather kernel + GEMM on X (every split's 24 n-tile CTAs re-gather
// the same rows through L2 one K-block at a time, behind a window-load + hash prologue).
static bool hash_in_gemm(const ngram_bank* b) {
    static const bool env = getenv("NGRAM_DECODE_HASH_IN_GEMM") && atoi(getenv("NGRAM_DECODE_HASH_IN_GEMM")) != 0;
    if (!env || b->shape.N > 8 || b->shape.variant != 1) return false;
    ngk::FwdArgs a{};
    a.s = b->shape;
    return ngk::splitk_factor(a, b->num_sms) > 1;
}

// One forward over T rows whose storage rows are already in `grow` (stride gstride).
// Tensor-core path: K2 gathers X (T x D bf16) into `xb`, K3 projects it.  Writes
// merged/rows per the amplification; LayerNorm via a third kernel.
void run_projection(ngram_bank* b, const uint32_t* tokens, const int32_t* grow, int64_t gstride, int64_t T,
                    void* rows, void* merged, int out_bf16, float* ln_scratch, const CUtensorMap* tmap_x,
                    cudaStream_t st, int amp, XBuf* xb, bool allow_splitk, const ngk::DecodeCommit* commit,
                    const HashCtx* hc, int64_t regime_T) {
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only (NGRAM_BANK_HASH_ONLY)");
    if (b->tc_path && ((reinterpret_cast<uintptr_t>(rows) | reinterpret_cast<uintptr_t>(merged)) & 15) != 0)
        throw Error(NGRAM_EINVAL, "output buffers must be 16-byte aligned (tensor-core path: vector / TMA stores)");
    if (T <= 0) return;
    ngk::FwdArgs a{};
    a.s = b->shape;
    if (amp >= 0) a.s.amp = amp;
    a.ht = b->ht.p;
    a.tokens = tokens;
    a.grow = grow;
    a.sub = b->sub.p;
    a.e0 = b->e0.p;
    a.wcat = b->wcat.p;
    a.ln_gain = b->ln_gain.p;
    a.ln_bias = b->ln_bias.p;
    a.T = T;
    a.Tpad = gstride;
    a.err = b->err.p;
    a.tmap_sub = &b->tmap_sub;
    a.tmap_w = &b->tmap_w;
    a.tmap_w2 = &b->tmap_w2;
    a.tmap_w32 = &b->tmap_w32;
    a.tmap_x = tmap_x;
    a.commit = commit;
    const int64_t rT = regime_T > 0 ? regime_T : T;  // the T whose kernel regime this call follows
    a.regime_T = rT;
    const bool ln = a.s.amp == 2;
    float* ln_merged = nullptr;
    if (ln) {
        ln_merged = (merged && !out_bf16) ? static_cast<float*>(merged) : ln_scratch;
        a.merged_out = ln_merged;
        a.rows_out = nullptr;
        a.out_bf16 = 0;
    } else {
        a.merged_out = merged;
        a.rows_out = rows;
        a.out_bf16 = out_bf16;
    }
    if (hc) {  // the GEMM producers hash and gather the rows themselves
        a.seq_off = hc->seq_off;
        a.nseq = hc->nseq;
        a.prior = hc->prior;
        a.wide = hc->wide ? 1 : 0;
    } else if (b->tc_path && !tmap_x && ((allow_splitk && small_t(b, rT)) || !fused_gather(b->shape.D))) {
        if (!xb) xb = &b->ws.xbuf;
        xb->ensure(round_up(T, kRowPad), b->shape.D);
        ngk::launch_gather_rows(a.s, grow, gstride, T, b->sub.p, xb->x.p, b->err.p, st);
        a.tmap_x = &xb->map;
    }
    b->prof_record(2, st);
    // output maps for the pair kernel's TMA epilogue (prefill tiling: not the split-K path)
    CUtensorMap map_rows, map_merged;
    if (b->tc_path && b->shape.D % 256 == 0 && (!small_t(b, rT) || !allow_splitk)) {
        const uint64_t D = uint64_t(b->shape.D);
        const bool f32 = !a.out_bf16;
        const uint64_t pitch = D * (f32 ? 4 : 2);
        if (a.rows_out) {
            make_tensor_map_2d(&map_rows, a.rows_out, D, uint64_t(T), pitch, 32, 32, f32, f32 ? 128 : 64);
            a.tmap_rows_out = &map_rows;
        }
        if (a.merged_out) {
            make_tensor_map_2d(&map_merged, a.merged_out, D, uint64_t(T), pitch, 32, 32, f32, f32 ? 128 : 64);
            a.tmap_merged_out = &map_merged;
        }
        a.tmap_e0 = &b->tmap_e0;
        if (b->shape.D % 64 == 0) a.tmap_e0w = &b->tmap_e0w;
    }
    if (b->tc_path) {
        float* ws = nullptr;
        const size_t need = allow_splitk ? ngk::splitk_workspace_floats(a, b->num_sms) : 0;
        if (need) {
            b->ws.splitk.ensure(need);
            ws = b->ws.splitk.p;
        }
        ngk::launch_forward_tc(a, b->num_sms, st, ws);
    } else {
        ngk::launch_forward_simt(a, st);
    }
    if (ln)
        ngk::launch_layernorm_rows(a.s, ln_merged, b->ln_gain.p, b->ln_bias.p, rows,
                                   (merged && ln_merged != merged) ? merged : nullptr, out_bf16, T, b->err.p, st);
    NGH_CUDA(cudaGetLastError());
}

// Hash + gather + project T positions given by (tokens, seq_off, prior).  X path: the
// fused K1+K2 kernel writes X directly; otherwise K1 writes storage rows for the fused-
// gather GEMM or the CUDA-core kernels.
// Returns true when `commit` was fused into the projection (decode GEMM path).
bool forward_tokens(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_off, int64_t nseq, int64_t T,
                    const uint32_t* prior, void* rows, void* merged, int out_bf16, cudaStream_t st, int amp,
                    XBuf* xb, int32_t* grow, bool allow_splitk, const ngk::DecodeCommit* commit,
                    int64_t uniform_len) {
    bool fused_commit = false;
    const int64_t Tpad = round_up(std::max<int64_t>(T, 1), kRowPad);
    b->prof_record(0, st);
    if (b->tc_path && allow_splitk && T <= 256 && hash_in_gemm(b)) {  // MODE 2: T <= 256 only
        // decode / verify: K1 fused into the split-K GEMM's producers (2 launches per step)
        b->prof_record(1, st);
        fused_commit = commit != nullptr;
        const HashCtx hc{seq_off, nseq, prior};
        run_projection(b, tokens, nullptr, Tpad, T, rows, merged, out_bf16, b->ws.merged_f32.p, nullptr, st, amp,
                       nullptr, true, fused_commit ? commit : nullptr, &hc);
    } else if (!(allow_splitk && small_t(b, T)) && prefill_path(b, T) != 0 && !fused_gather(b->shape.D)) {
        // K1+K2 fused into the projection's producers; a bad token must still abort the call
        // before any output, so the range check runs first (the kernel returns on the error word)
        ngk::launch_validate_tokens(b->shape, tokens, T, seq_off, nseq, prior, b->err.p, st);
        b->prof_record(1, st);
        const HashCtx hc{seq_off, nseq, prior, prefill_path(b, T) == 2};
        fused_commit = commit != nullptr;
        run_projection(b, tokens, nullptr, Tpad, T, rows, merged, out_bf16, b->ws.merged_f32.p, nullptr, st, amp,
                       nullptr, allow_splitk, fused_commit ? commit : nullptr, &hc);
    } else if (b->tc_path && ((allow_splitk && small_t(b, T)) || !fused_gather(b->shape.D))) {
        if (!xb) xb = &b->ws.xbuf;
        xb->ensure(Tpad, b->shape.D);
        if (T <= 1024)
            ngk::launch_hash_gather_rows(b->shape, b->ht.p, tokens, seq_off, nseq, T, prior, b->sub.p, xb->x.p,
                                         b->err.p, st, uniform_len);
        else
            ngk::launch_hash_gather(b->shape, b->ht.p, tokens, seq_off, nseq, T, prior, b->sub.p, xb->x.p, nullptr,
                                    Tpad, b->err.p, st);
        b->prof_record(1, st);
        fused_commit = commit != nullptr;  // every tensor-core projection path consumes it
        run_projection(b, tokens, nullptr, Tpad, T, rows, merged, out_bf16, b->ws.merged_f32.p, &xb->map, st, amp,
                       nullptr, allow_splitk, fused_commit ? commit : nullptr);
    } else {
        ngk::launch_hash_ids(b->shape, b->ht.p, tokens, seq_off, nseq, T, prior, nullptr, 0, grow, Tpad, b->err.p, st);
        b->prof_record(1, st);
        run_projection(b, tokens, grow, Tpad, T, rows, merged, out_bf16, b->ws.merged_f32.p, nullptr, st, amp, xb,
                       allow_splitk, nullptr);
    }
    b->prof_record(3, st);
    return fused_commit;
}

void reset_error_word(ngram_bank* b, cudaStream_t st) {
    NGH_CUDA(cudaMemsetAsync(b->err.p, 0xff, sizeof(unsigned long long), st));
    b->err_clean = false;  // this call's kernels may leave an error in it
}

}  // namespace ngh

using namespace ngh;

extern "C" {

const char* ngram_last_error(void) { return g_last_error.c_str(); }
const char* ngram_version(void) { return "ngram_b200 0.1 (sm_100a)"; }
uint64_t ngram_kernel_launches(void) { return ngk::launches(); }

// amplify (embedding.hpp:239-287) of `rows` host rows of width D on the current device.
int ngram_amplify_host(int amp_mode, int D, int64_t rows, const float* gain, const float* bias, const float* in,
                       float* out) {
    NGRAM_API_BEGIN
    if (D < 1 || rows < 0 || amp_mode < 0 || amp_mode > 2 || (rows > 0 && (!in || !out)))
        throw Error(NGRAM_EINVAL, "ngram_amplify_host: bad argument");
    if (amp_mode == 2 && (!gain || !bias)) throw Error(NGRAM_EINVAL, "amplify: layer_norm needs gain/bias of size D");
    if (rows == 0) return NGRAM_OK;
    const size_t n = size_t(rows) * size_t(D);
    DevBuf<float> din, dout, g, b;
    DevBuf<unsigned long long> err;
    din.alloc(n);
    dout.alloc(n);
    NGH_CUDA(cudaMemcpy(din.p, in, n * 4, cudaMemcpyHostToDevice));
    if (amp_mode == 2) {
        g.alloc(size_t(D));
        b.alloc(size_t(D));
        err.alloc(1);
        NGH_CUDA(cudaMemcpy(g.p, gain, size_t(D) * 4, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(b.p, bias, size_t(D) * 4, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemset(err.p, 0xff, sizeof(unsigned long long)));
        ngk::Shape s{};
        s.D = D;
        ngk::launch_layernorm_rows(s, din.p, g.p, b.p, dout.p, nullptr, 0, rows, err.p, nullptr);
    } else {
        ngk::launch_scale(din.p, dout.p, int64_t(n), amp_mode == 1 ? float(std::sqrt(double(D))) : 1.0f, nullptr);
    }
    NGH_CUDA(cudaMemcpy(out, dout.p, n * 4, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_prefill_path(ngram_bank* b, int64_t total_tokens, int* path) {
    NGRAM_API_BEGIN
    if (!b || !path || total_tokens < 0) throw Error(NGRAM_EINVAL, "ngram_prefill_path: bad argument");
    *path = (b->tc_path && !small_t(b, total_tokens)) ? prefill_path(b, total_tokens) : 0;
    NGRAM_API_END
}

int ngram_config_validate(const char* config_json) {
    NGRAM_API_BEGIN
    if (!config_json) throw Error(NGRAM_EINVAL, "null config");
    parse_config(config_json);
    NGRAM_API_END
}

int ngram_make_default_config(uint32_t base_vocab, int dim, int max_order, int sub_tables, char* json_out,
                              size_t cap) {
    NGRAM_API_BEGIN
    const std::string s = to_json(default_config(base_vocab, dim, max_order, sub_tables));
    if (!json_out || cap < s.size() + 1) throw Error(NGRAM_EINVAL, "output buffer too small");
    std::memcpy(json_out, s.c_str(), s.size() + 1);
    NGRAM_API_END
}

int ngram_rolling_hash_batch(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                             const uint64_t* bases, const uint64_t* moduli, int64_t count, uint64_t* out,
                             int32_t* status, void* stream) {
    NGRAM_API_BEGIN
    if (count < 0 || (count > 0 && (!windows || !orders || !bases || !moduli || !out || !status)))
        throw Error(NGRAM_EINVAL, "ngram_rolling_hash_batch: bad argument");
    ngk::launch_rolling_hash_batch(windows, stride, lengths, orders, bases, moduli, count, out, status,
                                   static_cast<cudaStream_t>(stream));
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_hash_ids(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                   int64_t total_tokens, const uint32_t* prior, void* ids_out, int ids_u64, void* stream) {
    NGRAM_API_BEGIN
    if (!b || nseq < 1 || total_tokens < 0 || !seq_offsets || (total_tokens > 0 && (!tokens || !ids_out)))
        throw Error(NGRAM_EINVAL, "ngram_hash_ids: bad argument");
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    reset_error_word(b, st);
    ngk::launch_hash_ids(b->shape, b->ht.p, tokens, seq_offsets, nseq, total_tokens, prior, ids_out, ids_u64, nullptr,
                         0, b->err.p, st);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_embed_forward(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                        int64_t total_tokens, const uint32_t* prior, void* rows_out, void* merged_out, int out_dtype,
                        void* stream) {
    NGRAM_API_BEGIN
    if (!b || nseq < 1 || total_tokens < 0 || !seq_offsets || (total_tokens > 0 && !tokens))
        throw Error(NGRAM_EINVAL, "ngram_embed_forward: bad argument");
    if (out_dtype != NGRAM_F32 && out_dtype != NGRAM_BF16) throw Error(NGRAM_EINVAL, "bad out_dtype");
    require_unsharded(b, "ngram_embed_forward");
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ensure_workspace(b, total_tokens);
    const int64_t Tpad = round_up(std::max<int64_t>(total_tokens, 1), kRowPad);
    reset_error_word(b, st);
    if (total_tokens == 0) return NGRAM_OK;
    (void)Tpad;
    forward_tokens(b, tokens, seq_offsets, nseq, total_tokens, prior, rows_out, merged_out, out_dtype == NGRAM_BF16,
                   st, -1, nullptr, b->ws.grow.p, true, nullptr);
    NGRAM_API_END
}

int ngram_embed_from_ids(ngram_bank* b, const uint32_t* tokens, const uint64_t* ids, int64_t T, void* merged_out,
                         int out_dtype, void* stream) {
    NGRAM_API_BEGIN
    if (!b || T < 0 || (T > 0 && (!tokens || !ids || !merged_out)))
        throw Error(NGRAM_EINVAL, "ngram_embed_from_ids: bad argument");
    require_unsharded(b, "ngram_embed_from_ids");
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ensure_workspace(b, T);
    const int64_t Tpad = round_up(std::max<int64_t>(T, 1), kRowPad);
    reset_error_word(b, st);
    if (T == 0) return NGRAM_OK;
    ngk::launch_ids_to_rows(b->shape, b->ht.p, ids, tokens, T, b->ws.grow.p, Tpad, b->err.p, st);
    // embed_from_ids returns the merged (pre-amplification) vector: run with amp = none.
    run_projection(b, tokens, b->ws.grow.p, Tpad, T, nullptr, merged_out, out_dtype == NGRAM_BF16, nullptr, nullptr,
                   st, 0, nullptr, true, nullptr);
    NGRAM_API_END
}

int ngram_sync_errors(ngram_bank* b, void* stream) {
    NGRAM_API_BEGIN
    if (!b) throw Error(NGRAM_EINVAL, "null bank");
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned long long e = 0, r = 0;
    NGH_CUDA(cudaMemcpyAsync(&e, b->err.p, sizeof(e), cudaMemcpyDeviceToHost, st));
    NGH_CUDA(cudaMemcpyAsync(&r, b->err_rep.p, sizeof(r), cudaMemcpyDeviceToHost, st));
    NGH_CUDA(cudaStreamSynchronize(st));
    e = std::min(e, r);  // errors of decode steps are released into err_rep
    b->err_clean = true;
    if (e != ~0ull) {
        NGH_CUDA(cudaMemsetAsync(b->err.p, 0xff, sizeof(e), st));
        NGH_CUDA(cudaMemsetAsync(b->err_rep.p, 0xff, sizeof(r), st));
        NGH_CUDA(cudaStreamSynchronize(st));
        throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                      std::to_string(b->cfg.base_vocab) + " (first bad window at position " +
                                      std::to_string(e) + ")");
    }
    NGRAM_API_END
}

int ngram_embed_sequence_host(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                              const uint32_t* prior, void* rows_out, void* merged_out, int out_dtype) {
    NGRAM_API_BEGIN
    if (!b || nseq < 1 || !seq_offsets) throw Error(NGRAM_EINVAL, "ngram_embed_sequence_host: bad argument");
    if (out_dtype != NGRAM_F32 && out_dtype != NGRAM_BF16) throw Error(NGRAM_EINVAL, "bad out_dtype");
    require_unsharded(b, "ngram_embed_sequence_host");
    const int64_t T = seq_offsets[nseq];
    check_offsets(seq_offsets, nseq, T);
    std::lock_guard<std::mutex> host_lock(b->host_mu);
    DeviceGuard g(b->device);
    for (int i = 0; i < 2; ++i)
        if (!b->host_streams[i]) NGH_CUDA(cudaStreamCreateWithFlags(&b->host_streams[i], cudaStreamNonBlocking));
    cudaStream_t s0 = b->host_streams[0], s1 = b->host_streams[1];
    const int N1 = std::max(b->cfg.max_order - 1, 0);
    ensure_workspace(b, T);
    const int64_t Tpad = round_up(std::max<int64_t>(T, 1), kRowPad);
    b->ws.tokens.ensure(size_t(std::max<int64_t>(T, 1)));
    b->ws.offsets.ensure(size_t(nseq + 1));
    if (prior && N1 > 0) b->ws.prior.ensure(size_t(nseq) * size_t(N1));
    if (T > 0) NGH_CUDA(cudaMemcpyAsync(b->ws.tokens.p, tokens, size_t(T) * 4, cudaMemcpyHostToDevice, s0));
    NGH_CUDA(cudaMemcpyAsync(b->ws.offsets.p, seq_offsets, size_t(nseq + 1) * 8, cudaMemcpyHostToDevice, s0));
    if (prior && N1 > 0)
        NGH_CUDA(cudaMemcpyAsync(b->ws.prior.p, prior, size_t(nseq) * size_t(N1) * 4, cudaMemcpyHostToDevice, s0));
    reset_error_word(b, s0);
    if (T == 0) {
        NGH_CUDA(cudaStreamSynchronize(s0));
        return NGRAM_OK;
    }
    // The reference raises before producing any output: every token is checked first.  Tensor-
    // core banks past the small-T regime then run the device entry's kernels chunk by chunk
    // (the fused K1+K2 block kernel -> X -> projection); the other shapes hash the whole batch
    // into storage rows here and gather per chunk.
    const uint32_t* dprior = (prior && N1 > 0) ? b->ws.prior.p : nullptr;
    const bool xpath = b->tc_path && !small_t(b, T) && !fused_gather(b->shape.D);
    if (xpath)
        ngk::launch_validate_tokens(b->shape, b->ws.tokens.p, T, b->ws.offsets.p, nseq, dprior, b->err.p, s0);
    else
        ngk::launch_hash_ids(b->shape, b->ht.p, b->ws.tokens.p, b->ws.offsets.p, nseq, T, dprior, nullptr, 0,
                             b->ws.grow.p, Tpad, b->err.p, s0);
    unsigned long long e = 0;
    NGH_CUDA(cudaMemcpyAsync(&e, b->err.p, sizeof(e), cudaMemcpyDeviceToHost, s0));
    NGH_CUDA(cudaStreamSynchronize(s0));
    if (e != ~0ull)
        throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                      std::to_string(b->cfg.base_vocab) + " (first bad window at position " +
                                      std::to_string(e) + ")");
    // Chunked projection on two streams: chunk i's D2H overlaps chunk i+1's kernels.
    const size_t esz = out_dtype == NGRAM_BF16 ? 2 : 4;
    const int64_t D = b->cfg.dim;
    const int64_t chunk = std::min<int64_t>(Tpad, 8192);
    const size_t cbytes = size_t(chunk) * size_t(D) * esz;
    cudaPointerAttributes pa{};
    auto is_pinned = [&](const void* p) {
        if (!p) return true;
        if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return pa.type == cudaMemoryTypeHost;
    };
    const bool direct = is_pinned(rows_out) && is_pinned(merged_out);
    for (int i = 0; i < 2; ++i) {
        if (rows_out) b->host_out[i].ensure(cbytes);
        if (merged_out) b->host_merged[i].ensure(cbytes);
    }
    if (!direct && b->pinned_bytes < cbytes * 2) {
        for (int i = 0; i < 2; ++i) {
            if (b->pinned[i]) cudaFreeHost(b->pinned[i]);
            b->pinned[i] = nullptr;
            NGH_CUDA(cudaMallocHost(&b->pinned[i], cbytes * 2));
        }
        b->pinned_bytes = cbytes * 2;
    }
    cudaEvent_t hashed;
    NGH_CUDA(cudaEventCreateWithFlags(&hashed, cudaEventDisableTiming));
    NGH_CUDA(cudaEventRecord(hashed, s0));
    NGH_CUDA(cudaStreamWaitEvent(s1, hashed, 0));
    int64_t nchunks = (T + chunk - 1) / chunk;
    std::vector<int64_t> pending(2, -1);  // chunk index whose staged copy awaits a host memcpy
    auto drain = [&](int slot) {
        const int64_t c = pending[size_t(slot)];
        if (c < 0) return;
        NGH_CUDA(cudaStreamSynchronize(b->host_streams[slot]));
        const int64_t c0 = c * chunk, n = std::min(chunk, T - c0);
        const size_t bytes = size_t(n) * size_t(D) * esz;
        uint8_t* pin = static_cast<uint8_t*>(b->pinned[slot]);
        if (rows_out) std::memcpy(static_cast<uint8_t*>(rows_out) + size_t(c0) * size_t(D) * esz, pin, bytes);
        if (merged_out)
            std::memcpy(static_cast<uint8_t*>(merged_out) + size_t(c0) * size_t(D) * esz, pin + cbytes, bytes);
        pending[size_t(slot)] = -1;
    };
    for (int64_t c = 0; c < nchunks; ++c) {
        const int slot = int(c & 1);
        cudaStream_t st = b->host_streams[slot];
        const int64_t c0 = c * chunk, n = std::min(chunk, T - c0);
        if (!direct) drain(slot);
        void* drows = rows_out ? b->host_out[slot].p : nullptr;
        void* dmerged = merged_out ? b->host_merged[slot].p : nullptr;
        float* ln = b->ws.merged_f32.p ? b->ws.merged_f32.p + size_t(c0) * size_t(D) : nullptr;
        if (xpath) {
            XBuf& xc = b->host_x[slot];
            xc.ensure(round_up(chunk, kRowPad), int(D));
            // positions [c0, c0 + n) into rows [0, n) of the chunk's X
            ngk::launch_hash_gather(b->shape, b->ht.p, b->ws.tokens.p, b->ws.offsets.p, nseq, T, dprior, b->sub.p,
                                    xc.x.p, nullptr, Tpad, b->err.p, st, c0, c0 + n, c0);
            run_projection(b, b->ws.tokens.p + c0, nullptr, Tpad, n, drows, dmerged, out_dtype == NGRAM_BF16, ln,
                           &xc.map, st, -1, nullptr, false, nullptr);
        } else {
            run_projection(b, b->ws.tokens.p + c0, b->ws.grow.p + c0, Tpad, n, drows, dmerged, out_dtype == NGRAM_BF16,
                           ln, nullptr, st, -1, &b->host_x[slot], small_t(b, T), nullptr);  // chunks keep the batch's regime
        }
        const size_t bytes = size_t(n) * size_t(D) * esz;
        if (direct) {
            if (rows_out)
                NGH_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(rows_out) + size_t(c0) * size_t(D) * esz, drows, bytes,
                                         cudaMemcpyDeviceToHost, st));
            if (merged_out)
                NGH_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(merged_out) + size_t(c0) * size_t(D) * esz, dmerged,
                                         bytes, cudaMemcpyDeviceToHost, st));
        } else {
            uint8_t* pin = static_cast<uint8_t*>(b->pinned[slot]);
            if (rows_out) NGH_CUDA(cudaMemcpyAsync(pin, drows, bytes, cudaMemcpyDeviceToHost, st));
            if (merged_out) NGH_CUDA(cudaMemcpyAsync(pin + cbytes, dmerged, bytes, cudaMemcpyDeviceToHost, st));
            pending[size_t(slot)] = c;
        }
    }
    if (!direct) {
        drain(0);
        drain(1);
    }
    NGH_CUDA(cudaStreamSynchronize(s0));
    NGH_CUDA(cudaStreamSynchronize(s1));
    cudaEventDestroy(hashed);
    NGRAM_API_END
}


}  // extern "C"

// ---------------------------------------------------------------- host-buffer variants
namespace {
// One small host call on the bank's I/O arena (bank.hpp): inputs packed into the pinned block
// and copied in ONE H2D transfer, outputs and the two error words copied back in ONE D2H
// transfer, ONE stream synchronisation; a token error raises as ngram_sync_errors does.
class Staged {
  public:
    explicit Staged(ngram_bank* b) : b_(b) {}
    size_t in(size_t bytes) { return take(in_, bytes); }
    size_t out(size_t bytes) { return take(out_, bytes) | kOut; }
    void ready() {
        words_ = al(in_ + out_);
        total_ = words_ + 16;
        b_->io_pin.ensure(total_);
        b_->io_dev.ensure(total_);
        if (!b_->io_stream) NGH_CUDA(cudaStreamCreateWithFlags(&b_->io_stream, cudaStreamNonBlocking));
    }
    void put(size_t off, const void* src, size_t bytes) { std::memcpy(b_->io_pin.p + at(off), src, bytes); }
    void upload() { NGH_CUDA(cudaMemcpyAsync(b_->io_dev.p, b_->io_pin.p, in_, cudaMemcpyHostToDevice, stream())); }
    template <typename T>
    T* dev(size_t off) { return reinterpret_cast<T*>(b_->io_dev.p + at(off)); }
    const uint8_t* host(size_t off) const { return b_->io_pin.p + at(off); }
    cudaStream_t stream() const { return b_->io_stream; }
    void finish() {
        cudaStream_t st = stream();
        if (out_) NGH_CUDA(cudaMemcpyAsync(b_->io_pin.p + in_, b_->io_dev.p + in_, out_, cudaMemcpyDeviceToHost, st));
        auto* w = reinterpret_cast<unsigned long long*>(b_->io_pin.p + words_);
        NGH_CUDA(cudaMemcpyAsync(&w[0], b_->err.p, 8, cudaMemcpyDeviceToHost, st));
        NGH_CUDA(cudaMemcpyAsync(&w[1], b_->err_rep.p, 8, cudaMemcpyDeviceToHost, st));
        NGH_CUDA(cudaStreamSynchronize(st));
        const unsigned long long e = std::min(w[0], w[1]);
        b_->err_clean = true;
        if (e != ~0ull) {
            NGH_CUDA(cudaMemsetAsync(b_->err.p, 0xff, 8, st));
            NGH_CUDA(cudaMemsetAsync(b_->err_rep.p, 0xff, 8, st));
            NGH_CUDA(cudaStreamSynchronize(st));
            throw Error(NGRAM_ERANGE, "embedding: token out of range for base vocabulary " +
                                          std::to_string(b_->cfg.base_vocab) + " (first bad window at position " +
                                          std::to_string(e) + ")");
        }
    }

  private:
    static constexpr size_t kOut = size_t(1) << 62;  // tag: offset in the output region
    static size_t al(size_t x) { return (x + 15) & ~size_t(15); }
    static size_t take(size_t& region, size_t bytes) {
        const size_t off = region;
        region = al(region + bytes);
        return off;
    }
    size_t at(size_t off) const { return (off & kOut) ? in_ + (off & ~kOut) : off; }
    ngram_bank* b_;
    size_t in_ = 0, out_ = 0, words_ = 0, total_ = 0;
};

template <typename T>
struct HostStage {  // device copy of a host array, freed on scope exit
    DevBuf<T> d;
    T* put(const T* h, size_t n) {
        if (!h || n == 0) return nullptr;
        d.alloc(n);
        NGH_CUDA(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
        return d.p;
    }
};
}  // namespace

extern "C" {

int ngram_hash_ids_host(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_offsets, int64_t nseq,
                        const uint32_t* prior, uint64_t* ids_out) {
    NGRAM_API_BEGIN
    if (!b || nseq < 1 || !seq_offsets) throw Error(NGRAM_EINVAL, "ngram_hash_ids_host: bad argument");
    const int64_t T = seq_offsets[nseq];
    check_offsets(seq_offsets, nseq, T);
    std::lock_guard<std::mutex> host_lock(b->host_mu);
    if (T == 0) NGRAM_API_RETURN_OK;
    DeviceGuard g(b->device);
    const int N1 = std::max(b->cfg.max_order - 1, 0);
    const size_t nb = size_t(std::max(b->shape.B, 1));
    Staged io(b);
    const size_t o_tok = io.in(size_t(T) * 4), o_off = io.in(size_t(nseq + 1) * 8);
    const size_t o_pri = (prior && N1 > 0) ? io.in(size_t(nseq) * size_t(N1) * 4) : 0;
    const size_t o_ids = io.out(size_t(T) * nb * 8);
    io.ready();
    io.put(o_tok, tokens, size_t(T) * 4);
    io.put(o_off, seq_offsets, size_t(nseq + 1) * 8);
    if (prior && N1 > 0) io.put(o_pri, prior, size_t(nseq) * size_t(N1) * 4);
    io.upload();
    int rc = ngram_hash_ids(b, io.dev<uint32_t>(o_tok), io.dev<int64_t>(o_off), nseq, T,
                            (prior && N1 > 0) ? io.dev<uint32_t>(o_pri) : nullptr, io.dev<uint64_t>(o_ids), 1,
                            io.stream());
    if (rc) return rc;
    io.finish();  // one D2H of outputs + error words, one sync; raises a token error
    if (b->shape.B > 0) std::memcpy(ids_out, io.host(o_ids), size_t(T) * size_t(b->shape.B) * 8);
    NGRAM_API_END
}

int ngram_rolling_hash_host(const uint32_t* windows, int64_t stride, const int32_t* lengths, const int32_t* orders,
                            const uint64_t* bases, const uint64_t* moduli, int64_t count, uint64_t* out,
                            int32_t* status) {
    NGRAM_API_BEGIN
    if (count <= 0) NGRAM_API_RETURN_OK;
    // a bank-free entry: a per-thread staging arena on the current device
    thread_local PinBuf pin;
    thread_local DevBuf<uint8_t> dev;
    thread_local cudaStream_t st = nullptr;
    thread_local int st_dev = -1;
    int cur = 0;
    NGH_CUDA(cudaGetDevice(&cur));
    if (!st || st_dev != cur) {
        NGH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        dev.release();
        st_dev = cur;
    }
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    const size_t s_w = size_t(count) * size_t(stride) * 4, s_c = size_t(count) * 4, s_8 = size_t(count) * 8;
    const size_t o_w = 0, o_l = al(o_w + s_w), o_o = al(o_l + s_c), o_b = al(o_o + s_c), o_m = al(o_b + s_8);
    const size_t o_out = al(o_m + s_8), o_st = al(o_out + s_8), total = al(o_st + s_c);
    pin.ensure(total);
    dev.ensure(total);
    std::memcpy(pin.p + o_w, windows, s_w);
    if (lengths) std::memcpy(pin.p + o_l, lengths, s_c);
    std::memcpy(pin.p + o_o, orders, s_c);
    std::memcpy(pin.p + o_b, bases, s_8);
    std::memcpy(pin.p + o_m, moduli, s_8);
    NGH_CUDA(cudaMemcpyAsync(dev.p, pin.p, o_out, cudaMemcpyHostToDevice, st));
    int rc = ngram_rolling_hash_batch(reinterpret_cast<const uint32_t*>(dev.p + o_w), stride,
                                      lengths ? reinterpret_cast<const int32_t*>(dev.p + o_l) : nullptr,
                                      reinterpret_cast<const int32_t*>(dev.p + o_o),
                                      reinterpret_cast<const uint64_t*>(dev.p + o_b),
                                      reinterpret_cast<const uint64_t*>(dev.p + o_m), count,
                                      reinterpret_cast<uint64_t*>(dev.p + o_out),
                                      reinterpret_cast<int32_t*>(dev.p + o_st), st);
    if (rc) return rc;
    NGH_CUDA(cudaMemcpyAsync(pin.p + o_out, dev.p + o_out, total - o_out, cudaMemcpyDeviceToHost, st));
    NGH_CUDA(cudaStreamSynchronize(st));
    std::memcpy(out, pin.p + o_out, s_8);
    std::memcpy(status, pin.p + o_st, s_c);
    NGRAM_API_END
}

int ngram_embed_from_ids_host(ngram_bank* b, const uint32_t* tokens, const uint64_t* ids, int64_t T,
                              float* merged_out) {
    NGRAM_API_BEGIN
    if (!b || T < 0 || (T > 0 && (!tokens || !ids || !merged_out)))
        throw Error(NGRAM_EINVAL, "ngram_embed_from_ids_host: bad argument");
    std::lock_guard<std::mutex> host_lock(b->host_mu);
    if (T == 0) NGRAM_API_RETURN_OK;
    DeviceGuard g(b->device);
    const size_t nb = size_t(std::max(b->shape.B, 1)), D = size_t(b->cfg.dim);
    Staged io(b);
    const size_t o_tok = io.in(size_t(T) * 4), o_ids = io.in(size_t(T) * nb * 8);
    const size_t o_out = io.out(size_t(T) * D * 4);
    io.ready();
    io.put(o_tok, tokens, size_t(T) * 4);
    io.put(o_ids, ids, size_t(T) * nb * 8);
    io.upload();
    int rc = ngram_embed_from_ids(b, io.dev<uint32_t>(o_tok), io.dev<uint64_t>(o_ids), T, io.dev<float>(o_out),
                                  NGRAM_F32, io.stream());
    if (rc) return rc;
    io.finish();
    std::memcpy(merged_out, io.host(o_out), size_t(T) * D * 4);
    NGRAM_API_END
}

}  // extern "C"

