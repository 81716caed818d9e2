// bank.hpp -- the device-resident bank (ngram_bank) and decode state (ngram_decode)
// behind the C-ABI.  Host C++: allocation, layout, tensor maps, workspaces; every
// computation is a kernel in csrc/kernels.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../kernels/kernels.h"
#include "config.hpp"

namespace ngh {

void check_cuda(cudaError_t e, const char* what);
#define NGH_CUDA(x) ::ngh::check_cuda((x), #x)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev);
    ~DeviceGuard();
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        release();
        if (count == 0) return;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw Error(NGRAM_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed: " +
                                          cudaGetErrorString(e));
        }
        n = count;
    }
    void ensure(size_t count) {
        if (count > n) alloc(count);
    }
};

// Page-locked host staging (cudaMallocHost), grown on demand.
struct PinBuf {
    unsigned char* p = nullptr;
    size_t n = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    PinBuf& operator=(const PinBuf&) = delete;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t bytes) {
        if (bytes <= n) return;
        if (p) cudaFreeHost(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&p), bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw Error(NGRAM_ENOMEM, "cudaMallocHost of " + std::to_string(bytes) + " bytes failed");
        }
        n = bytes;
    }
};

// A materialised X buffer (T x D bf16) with its TMA descriptor (box 64 x 128 rows).
struct XBuf {
    DevBuf<__nv_bfloat16> x;
    CUtensorMap map{};
    int64_t rows = 0;
    void ensure(int64_t nrows, int D);
};

struct Workspace {
    int64_t tokens_cap = 0;
    DevBuf<int32_t> grow;           // [B][Tpad]
    DevBuf<float> merged_f32;       // [T][D] (LayerNorm staging)
    DevBuf<uint32_t> tokens;        // host-API staging / decode tokens
    DevBuf<int64_t> offsets;
    DevBuf<uint32_t> prior;
    XBuf xbuf;                      // K2 output / K3 A operand
    DevBuf<float> splitk;           // small-T split-K partial sums
};

}  // namespace ngh

struct ngram_bank {
    ngh::Config cfg;
    ngk::Shape shape{};
    int device = 0;
    int num_sms = 148;
    int shard_rank = 0, shard_count = 1;
    std::vector<int64_t> row_lo, row_hi, row_base;
    int64_t local_rows = 0;
    bool tc_path = false;
    bool hash_only = false;  // NGRAM_BANK_HASH_ONLY: no tables, hashing entry points only

    ngh::DevBuf<__nv_bfloat16> sub, e0, wcat;
    ngh::DevBuf<float> ln_gain, ln_bias;
    ngh::DevBuf<ngk::HashTables> ht;
    ngh::DevBuf<unsigned long long> err;
    // decode steps release the error word themselves (DecodeCommit::err_reported): token errors
    // of such steps land in err_rep; err_clean = the error word is known clear at the stream's
    // tail, so the next decode step needs no reset
    ngh::DevBuf<unsigned long long> err_rep;
    ngh::DevBuf<unsigned int> err_ticket;
    bool err_clean = true;

    CUtensorMap tmap_sub{}, tmap_w{}, tmap_w2{}, tmap_w32{}, tmap_e0{}, tmap_e0w{};
    ngh::Workspace ws;

    // Serialises the host-buffer entry points (the reference's bank is shareable across
    // threads; this bank's workspaces and error word are not)
    std::mutex host_mu;
    // host-buffer pipeline (ngram_embed_sequence_host)
    cudaStream_t host_streams[2] = {nullptr, nullptr};
    ngh::DevBuf<uint8_t> host_out[2];
    ngh::DevBuf<uint8_t> host_merged[2];
    ngh::DevBuf<int64_t> host_off[2];
    ngh::DevBuf<uint32_t> host_prior[2];
    ngh::XBuf host_x[2];
    void* pinned[2] = {nullptr, nullptr};
    size_t pinned_bytes = 0;
    // small host calls (ngram_hash_ids_host, ngram_embed_from_ids_host): one pinned staging block
    // and one device block, reused -- inputs in one H2D copy, outputs + error words in one D2H
    // copy, one synchronisation, no allocation after the first call
    ngh::PinBuf io_pin;
    ngh::DevBuf<uint8_t> io_dev;
    cudaStream_t io_stream = nullptr;

    // stage profiling (ngram_profile_enable)
    bool prof = false;
    cudaEvent_t prof_ev[4] = {nullptr, nullptr, nullptr, nullptr};
    void prof_record(int i, cudaStream_t st) {
        if (prof) cudaEventRecord(prof_ev[i], st);
    }

    uint64_t device_bytes() const;
    ~ngram_bank();
};

struct ngram_decode {
    ngram_bank* bank = nullptr;
    int64_t batch = 0;
    int max_draft = 0;
    ngh::DevBuf<uint32_t> ring;             // [batch][N-1] trailing confirmed tokens, oldest first
    ngh::DevBuf<uint64_t> length;           // [batch]
    ngh::DevBuf<uint32_t> last;             // [batch]
    ngh::DevBuf<int64_t> seq_off;           // [max_draft][batch+1] = s * L
    ngh::DevBuf<int32_t> grow;              // [B][round_up(batch*max_draft, 128)]
    ngh::DevBuf<unsigned long long> derr;   // decode error word
    ngh::XBuf xbuf;                         // gathered block rows
    // host-buffer entries (ngram_decode_step_host / ngram_verify_commit_host): persistent device
    // buffers + one pinned staging block, so a call is H2D -> kernels -> D2H with one sync and
    // no allocation after the first call
    ngh::DevBuf<uint32_t> io_tok;           // [batch][max_draft]
    ngh::DevBuf<int32_t> io_acc;            // [batch]
    ngh::DevBuf<uint64_t> io_ids;           // [batch][B]
    ngh::DevBuf<float> io_out;              // [batch][max_draft][D]
    ngh::PinBuf io_pin;                     // error words | ids | out, then tokens | accept
    cudaStream_t io_stream = nullptr;
    // ngram_decode_step_host in steady state (merged out, no ids, released error word): the
    // whole H2D -> 3 kernels -> D2H sequence captured once and replayed (one launch per step);
    // keyed by the staging block it was captured on
    cudaGraphExec_t step_exec = nullptr;
    // staging in / out / ids, device token / output / ids buffers, X, split-K workspace, variant
    const void* step_key[9] = {};
    uint64_t step_launches = 0;
    int64_t host_steps = 0;        // eager host steps so far (the first sizes every workspace)
    ~ngram_decode() {
        if (step_exec) cudaGraphExecDestroy(step_exec);
        if (io_stream) cudaStreamDestroy(io_stream);
    }
};

namespace ngh {
// Build the TMA descriptors of a bank (driver entry point, no libcuda link).
void make_tensor_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint64_t row_pitch_bytes,
                        uint32_t box_inner, uint32_t box_rows, bool f32 = false, int swizzle_bytes = 128);
void ensure_workspace(ngram_bank* b, int64_t T);

// Forward building blocks shared by forward.cpp / decode.cpp / shard.cpp.
void reset_error_word(ngram_bank* b, cudaStream_t st);
// Windows of the call's tokens for kernels that hash on the fly (small-T MODE 2 GEMM).
struct HashCtx {
    const int64_t* seq_off;
    int64_t nseq;
    const uint32_t* prior;
    bool wide = false;  // fused wide-tile kernel (gemm_wide.cu) instead of the pair kernel's LSU producers
};
void run_projection(ngram_bank* b, const uint32_t* tokens, const int32_t* grow, int64_t gstride, int64_t T,
                    void* rows, void* merged, int out_bf16, float* ln_scratch, const CUtensorMap* tmap_x,
                    cudaStream_t st, int amp, XBuf* xb, bool allow_splitk, const ngk::DecodeCommit* commit,
                    const HashCtx* hc = nullptr, int64_t regime_T = 0);
bool forward_tokens(ngram_bank* b, const uint32_t* tokens, const int64_t* seq_off, int64_t nseq, int64_t T,
                    const uint32_t* prior, void* rows, void* merged, int out_bf16, cudaStream_t st, int amp,
                    XBuf* xb, int32_t* grow, bool allow_splitk, const ngk::DecodeCommit* commit,
                    int64_t uniform_len = 0);
inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
// Row padding of every per-token workspace: the 2-CTA GEMM tile is 256 tokens.
constexpr int64_t kRowPad = 256;
ngram_bank* grad_bank(ngram_grad* g);  // backward.cpp
}  // namespace ngh
