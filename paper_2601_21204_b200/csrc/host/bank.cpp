// bank.cpp -- ngram_bank: creation (layout + hashing constants + TMA descriptors),
// upload of reference float banks, device-side synthetic generation, streaming of
// reference bank files, and workspace sizing.
#include "bank.hpp"

#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>

#include <json.hpp>

#include "api_util.hpp"

namespace ngh {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw Error(NGRAM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

DeviceGuard::DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) NGH_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Error(NGRAM_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    return fn;
}

// ceil(r * V / P) without overflow.
int64_t shard_lo(uint64_t V, int r, int P) {
    const unsigned __int128 x = (unsigned __int128)V * (unsigned)r + (unsigned)(P - 1);
    return (int64_t)(x / (unsigned)P);
}

}  // namespace

void make_tensor_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t rows, uint64_t row_pitch_bytes,
                        uint32_t box_inner, uint32_t box_rows, bool f32, int swizzle_bytes) {
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {row_pitch_bytes};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                   const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(NGRAM_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

void XBuf::ensure(int64_t nrows, int D) {
    if (nrows <= rows) return;
    x.alloc(size_t(nrows) * size_t(D));
    make_tensor_map_2d(&map, x.p, uint64_t(D), uint64_t(nrows), uint64_t(D) * 2, 64, 128);
    rows = nrows;
}

void ensure_workspace(ngram_bank* b, int64_t T) {
    if (T <= b->ws.tokens_cap) return;
    const int64_t Tpad = round_up(std::max<int64_t>(T, 1), kRowPad);
    b->ws.grow.ensure(size_t(std::max(b->shape.B, 1)) * size_t(Tpad));
    if (b->cfg.amp == 2) b->ws.merged_f32.ensure(size_t(Tpad) * size_t(b->cfg.dim));
    if (b->tc_path) b->ws.xbuf.ensure(Tpad, b->cfg.dim);
    b->ws.tokens_cap = Tpad;
}

}  // namespace ngh

using namespace ngh;

uint64_t ngram_bank::device_bytes() const {
    return sub.n * 2 + e0.n * 2 + wcat.n * 2 + (ln_gain.n + ln_bias.n) * 4;
}

ngram_bank::~ngram_bank() {
    // no DeviceGuard (it throws): a bank may be released after the driver has shut down
    int prev = -1;
    if (cudaGetDevice(&prev) == cudaSuccess && prev != device) cudaSetDevice(device);
    for (auto& e : prof_ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (host_streams[i]) cudaStreamDestroy(host_streams[i]);
        if (pinned[i]) cudaFreeHost(pinned[i]);
    }
    if (io_stream) cudaStreamDestroy(io_stream);
    cudaGetLastError();
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
}

extern "C" {

int ngram_bank_create(const char* config_json, int device, int shard_rank, int shard_count, ngram_bank** out) {
    return ngram_bank_create_ex(config_json, device, shard_rank, shard_count, 0, out);
}

int ngram_bank_create_ex(const char* config_json, int device, int shard_rank, int shard_count, int flags,
                         ngram_bank** out) {
    NGRAM_API_BEGIN
    if (!config_json || !out) throw Error(NGRAM_EINVAL, "ngram_bank_create: null argument");
    *out = nullptr;
    Config cfg = parse_config(config_json);
    if (shard_count < 1 || shard_rank < 0 || shard_rank >= shard_count)
        throw Error(NGRAM_EINVAL, "ngram_bank_create: bad shard rank/count");
    if (cfg.branch_count() > ngk::kMaxBranches) throw Error(NGRAM_EINVAL, "more than 64 (n,k) branches");
    if (cfg.max_order > ngk::kMaxOrder) throw Error(NGRAM_EINVAL, "max_order above 16 is not supported");
    DeviceGuard g(device);
    auto b = std::make_unique<ngram_bank>();
    b->cfg = cfg;
    b->device = device;
    b->shard_rank = shard_rank;
    b->shard_count = shard_count;
    NGH_CUDA(cudaDeviceGetAttribute(&b->num_sms, cudaDevAttrMultiProcessorCount, device));

    const int B = cfg.branch_count();
    const int D = cfg.dim;
    const int d = cfg.branch_dim();
    ngk::Shape& s = b->shape;
    s.N = cfg.max_order;
    s.K = cfg.sub_tables;
    s.B = B;
    s.D = D;
    s.d = d;
    s.variant = cfg.variant;
    s.amp = cfg.amp;
    s.denom = cfg.merge_denominator();
    s.V0 = cfg.base_vocab;
    s.fast_hash = 1;

    auto ht = std::make_unique<ngk::HashTables>();
    std::memset(ht.get(), 0, sizeof(ngk::HashTables));
    b->row_lo.resize(size_t(B));
    b->row_hi.resize(size_t(B));
    b->row_base.resize(size_t(B));
    int64_t rows = 0;
    for (int i = 0; i < B; ++i) {
        const uint64_t m = cfg.sub_vocab[size_t(i)];
        if (m > (uint64_t(1) << 32)) s.fast_hash = 0;
        ht->modulus[i] = m;
        ht->barrett[i] = m >= 2 ? (uint64_t)(((unsigned __int128)1 << 64) / m) : 0;
        uint64_t pw = 1 % m;
        const uint64_t base_mod = uint64_t(cfg.base_vocab) % m;
        for (int j = 0; j < ngk::kMaxOrder; ++j) {  // V0^j mod V_b, the reference's running `power`
            ht->pow[i][j] = pw;
            pw = (uint64_t)(((unsigned __int128)pw * base_mod) % m);
        }
        const int64_t lo = shard_lo(m, shard_rank, shard_count);
        const int64_t hi = shard_lo(m, shard_rank + 1, shard_count);
        b->row_lo[size_t(i)] = lo;
        b->row_hi[size_t(i)] = hi;
        b->row_base[size_t(i)] = rows;
        ht->row_lo[i] = lo;
        ht->row_hi[i] = hi;
        ht->row_base[i] = rows;
        rows += hi - lo;
    }
    b->local_rows = rows;
    b->hash_only = (flags & NGRAM_BANK_HASH_ONLY) != 0;
    b->tc_path = !b->hash_only && cfg.variant == 1 && B > 0 && d % 64 == 0 && D % 128 == 0 &&
                 rows < (int64_t(1) << 31) && cfg.base_vocab < (1u << 31);
    if (!b->hash_only) {
        const double bytes = double(rows) * d * 2 + double(cfg.base_vocab) * D * 2 + double(D) * D * 2;
        if (bytes > 1.0e15) throw Error(NGRAM_ENOMEM, "bank tables too large for a device");
        b->sub.alloc(size_t(rows) * size_t(d));
        b->e0.alloc(size_t(cfg.base_vocab) * size_t(D));
        if (cfg.variant == 1 && B > 0) b->wcat.alloc(size_t(D) * size_t(D));
    }
    if (cfg.amp == 2 && !b->hash_only) {
        b->ln_gain.alloc(size_t(D));
        b->ln_bias.alloc(size_t(D));
        ngk::launch_fill_f32(b->ln_gain.p, 1.0f, D, nullptr);
        ngk::launch_fill_f32(b->ln_bias.p, 0.0f, D, nullptr);
    }
    b->ht.alloc(1);
    NGH_CUDA(cudaMemcpy(b->ht.p, ht.get(), sizeof(ngk::HashTables), cudaMemcpyHostToDevice));
    b->err.alloc(1);
    NGH_CUDA(cudaMemset(b->err.p, 0xff, sizeof(unsigned long long)));
    b->err_rep.alloc(1);
    NGH_CUDA(cudaMemset(b->err_rep.p, 0xff, sizeof(unsigned long long)));
    b->err_ticket.alloc(1);
    NGH_CUDA(cudaMemset(b->err_ticket.p, 0, sizeof(unsigned int)));
    if (b->tc_path) {
        make_tensor_map_2d(&b->tmap_sub, b->sub.p, uint64_t(d), uint64_t(std::max<int64_t>(rows, 1)),
                           uint64_t(d) * 2, 64, 1);
        make_tensor_map_2d(&b->tmap_w, b->wcat.p, uint64_t(D), uint64_t(D), uint64_t(D) * 2, 64,
                           D % 256 == 0 ? 256 : 128);
        make_tensor_map_2d(&b->tmap_w2, b->wcat.p, uint64_t(D), uint64_t(D), uint64_t(D) * 2, 64, 128);
        // gemm_wide: 32-column x 128-row W stages, SWIZZLE_64B
        make_tensor_map_2d(&b->tmap_w32, b->wcat.p, uint64_t(D), uint64_t(D), uint64_t(D) * 2, 32, 128, false, 64);
        // E0 rows gathered by token id (tile::gather4) into the pair kernel's TMA epilogue
        make_tensor_map_2d(&b->tmap_e0, b->e0.p, uint64_t(D), uint64_t(b->cfg.base_vocab), uint64_t(D) * 2, 32, 1,
                           false, 64);
        if (D % 64 == 0)
            make_tensor_map_2d(&b->tmap_e0w, b->e0.p, uint64_t(D), uint64_t(b->cfg.base_vocab), uint64_t(D) * 2, 64,
                               1, false, 128);
    }
    NGH_CUDA(cudaDeviceSynchronize());
    *out = b.release();
    NGRAM_API_END
}

int ngram_shard_rows(uint64_t V, int rank, int count, int64_t* lo, int64_t* hi) {
    NGRAM_API_BEGIN
    if (!lo || !hi || count < 1 || rank < 0 || rank >= count) throw Error(NGRAM_EINVAL, "bad shard rank/count");
    *lo = shard_lo(V, rank, count);
    *hi = shard_lo(V, rank + 1, count);
    NGRAM_API_END
}

int ngram_bank_destroy(ngram_bank* bank) {
    NGRAM_API_BEGIN
    delete bank;
    NGRAM_API_END
}

int ngram_bank_get_info(const ngram_bank* b, ngram_bank_info* info) {
    NGRAM_API_BEGIN
    if (!b || !info) throw Error(NGRAM_EINVAL, "null argument");
    std::memset(info, 0, sizeof(*info));
    info->max_order = b->cfg.max_order;
    info->sub_tables = b->cfg.sub_tables;
    info->dim = b->cfg.dim;
    info->branch_count = b->shape.B;
    info->branch_dim = b->shape.d;
    info->variant = b->cfg.variant;
    info->amplification = b->cfg.amp;
    info->merge_denominator = b->shape.denom;
    info->base_vocab = b->cfg.base_vocab;
    info->shard_rank = b->shard_rank;
    info->shard_count = b->shard_count;
    info->tensor_core_path = b->tc_path ? 1 : 0;
    info->device_bytes = b->device_bytes();
    for (int i = 0; i < b->shape.B; ++i) {
        info->sub_vocab[i] = b->cfg.sub_vocab[size_t(i)];
        info->row_lo[i] = b->row_lo[size_t(i)];
        info->row_hi[i] = b->row_hi[size_t(i)];
    }
    info->sub_ptr = b->sub.p;
    info->e0_ptr = b->e0.p;
    info->wcat_ptr = b->wcat.p;
    NGRAM_API_END
}

int ngram_bank_upload_f32(ngram_bank* b, const float* base, const float* const* sub, const float* const* proj,
                          const float* ln_gain, const float* ln_bias) {
    NGRAM_API_BEGIN
    if (!b || !base) throw Error(NGRAM_EINVAL, "ngram_bank_upload_f32: null argument");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only");
    DeviceGuard g(b->device);
    const int B = b->shape.B, D = b->shape.D, d = b->shape.d;
    const size_t chunk = size_t(16) << 20;  // floats per staging chunk (64 MB)
    DevBuf<float> stage;
    stage.alloc(chunk);
    auto put = [&](const float* src, __nv_bfloat16* dst, size_t n) {
        for (size_t o = 0; o < n; o += chunk) {
            const size_t c = std::min(chunk, n - o);
            NGH_CUDA(cudaMemcpy(stage.p, src + o, c * 4, cudaMemcpyHostToDevice));
            ngk::launch_f32_to_bf16(stage.p, dst + o, int64_t(c), nullptr);
            NGH_CUDA(cudaDeviceSynchronize());
        }
    };
    put(base, b->e0.p, size_t(b->cfg.base_vocab) * size_t(D));
    for (int i = 0; i < B; ++i) {
        if (!sub || !sub[i]) throw Error(NGRAM_EINVAL, "ngram_bank_upload_f32: missing sub-table");
        const int64_t lo = b->row_lo[size_t(i)], hi = b->row_hi[size_t(i)];
        put(sub[i] + size_t(lo) * size_t(d), b->sub.p + size_t(b->row_base[size_t(i)]) * size_t(d),
            size_t(hi - lo) * size_t(d));
    }
    if (b->cfg.variant == 1) {
        for (int i = 0; i < B; ++i) {
            if (!proj || !proj[i]) throw Error(NGRAM_EINVAL, "ngram_bank_upload_f32: missing projection");
            NGH_CUDA(cudaMemcpy(stage.p, proj[i], size_t(D) * size_t(d) * 4, cudaMemcpyHostToDevice));
            ngk::launch_pack_wcat(stage.p, b->wcat.p, D, d, i, nullptr);
            NGH_CUDA(cudaDeviceSynchronize());
        }
    }
    if (b->cfg.amp == 2) {
        if (!ln_gain || !ln_bias) throw Error(NGRAM_EINVAL, "ngram_bank_upload_f32: layer_norm needs gain/bias");
        NGH_CUDA(cudaMemcpy(b->ln_gain.p, ln_gain, size_t(D) * 4, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(b->ln_bias.p, ln_bias, size_t(D) * 4, cudaMemcpyHostToDevice));
    }
    NGH_CUDA(cudaDeviceSynchronize());
    NGRAM_API_END
}

int ngram_bank_generate(ngram_bank* b, uint64_t seed, void* stream) {
    NGRAM_API_BEGIN
    if (!b) throw Error(NGRAM_EINVAL, "null bank");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only");
    DeviceGuard g(b->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = b->shape.B, D = b->shape.D, d = b->shape.d;
    const float s_tab = float(0.02 / 37837.2328);
    const float s_proj = float((0.02 / std::sqrt(double(d))) / 37837.2328);
    ngk::launch_synth_fill_bf16(b->e0.p, seed, 0, 0, int64_t(b->cfg.base_vocab), D, D, s_tab, st);
    for (int i = 0; i < B; ++i) {
        const int64_t lo = b->row_lo[size_t(i)], hi = b->row_hi[size_t(i)];
        ngk::launch_synth_fill_bf16(b->sub.p + size_t(b->row_base[size_t(i)]) * size_t(d), seed, uint32_t(1 + i), lo,
                                    hi - lo, d, d, s_tab, st);
    }
    if (b->cfg.variant == 1 && B > 0) ngk::launch_synth_wcat(b->wcat.p, seed, D, d, B, s_proj, st);
    NGH_CUDA(cudaGetLastError());
    NGRAM_API_END
}

int ngram_profile_enable(ngram_bank* b, int enable) {
    NGRAM_API_BEGIN
    if (!b) throw Error(NGRAM_EINVAL, "null bank");
    DeviceGuard g(b->device);
    if (enable && !b->prof_ev[0])
        for (auto& e : b->prof_ev) NGH_CUDA(cudaEventCreate(&e));
    b->prof = enable != 0;
    NGRAM_API_END
}

int ngram_profile_read(ngram_bank* b, float* stage_ms, int n) {
    NGRAM_API_BEGIN
    if (!b || !stage_ms || n < 2 || !b->prof_ev[0]) throw Error(NGRAM_EINVAL, "ngram_profile_read: not enabled");
    DeviceGuard g(b->device);
    NGH_CUDA(cudaEventSynchronize(b->prof_ev[3]));
    NGH_CUDA(cudaEventElapsedTime(&stage_ms[0], b->prof_ev[0], b->prof_ev[1]));
    NGH_CUDA(cudaEventElapsedTime(&stage_ms[1], b->prof_ev[1], b->prof_ev[2]));
    if (n >= 3) NGH_CUDA(cudaEventElapsedTime(&stage_ms[2], b->prof_ev[2], b->prof_ev[3]));
    NGRAM_API_END
}

int ngram_bank_reserve(ngram_bank* b, int64_t max_tokens) {
    NGRAM_API_BEGIN
    if (!b || max_tokens < 0) throw Error(NGRAM_EINVAL, "ngram_bank_reserve: bad argument");
    DeviceGuard g(b->device);
    ensure_workspace(b, max_tokens);
    NGRAM_API_END
}

// save_bank format (embedding.cpp:77-98): u32 LE header length, JSON config echo, then
// raw LE f32: base, sub-tables by branch, projections by branch, [LN gain, bias].
int ngram_bank_load_file(ngram_bank* b, const char* path) {
    NGRAM_API_BEGIN
    if (!b || !path) throw Error(NGRAM_EINVAL, "null argument");
    if (b->hash_only) throw Error(NGRAM_EINVAL, "bank was created hash-only");
    DeviceGuard g(b->device);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), &std::fclose);
    if (!f) throw Error(NGRAM_EIO, std::string("cannot open bank file: ") + path);
    unsigned char lenbuf[4];
    if (std::fread(lenbuf, 1, 4, f.get()) != 4)
        throw Error(NGRAM_EPARSE, std::string("bank file too short for header: ") + path + " (line 0, offset 0)");
    const uint32_t len = uint32_t(lenbuf[0]) | (uint32_t(lenbuf[1]) << 8) | (uint32_t(lenbuf[2]) << 16) |
                         (uint32_t(lenbuf[3]) << 24);
    std::string header(len, '\0');
    if (std::fread(header.data(), 1, len, f.get()) != len)
        throw Error(NGRAM_EPARSE, std::string("bank file truncated in header: ") + path + " (line 0, offset 4)");
    Config fc;
    try {
        fc = parse_config(header);
    } catch (const Error& e) {
        if (e.status == NGRAM_EPARSE) throw Error(NGRAM_EPARSE, std::string("bad bank header JSON: ") + e.what());
        throw;
    }
    if (to_json(fc) != to_json(b->cfg))
        throw Error(NGRAM_ECONFIG, std::string("bank file config does not match the device bank: ") + path);
    const int B = b->shape.B, D = b->shape.D, d = b->shape.d;
    const size_t chunk = size_t(16) << 20;
    void* pinned = nullptr;
    NGH_CUDA(cudaMallocHost(&pinned, chunk * 4));
    std::unique_ptr<void, cudaError_t (*)(void*)> pin_guard(pinned, &cudaFreeHost);
    DevBuf<float> stage;
    stage.alloc(chunk);
    float* hbuf = static_cast<float*>(pinned);
    auto read_f32 = [&](size_t n, auto&& sink) {
        for (size_t o = 0; o < n; o += chunk) {
            const size_t c = std::min(chunk, n - o);
            const size_t got = std::fread(hbuf, 4, c, f.get());
            if (got != c)
                throw Error(NGRAM_EPARSE, std::string("bank file truncated: ") + path + " (line 0, offset " +
                                              std::to_string(got * 4) + ")");
            NGH_CUDA(cudaMemcpy(stage.p, hbuf, c * 4, cudaMemcpyHostToDevice));
            sink(o, c);
            NGH_CUDA(cudaDeviceSynchronize());
        }
    };
    auto skip_f32 = [&](size_t n) {
        if (n && std::fseek(f.get(), long(n * 4), SEEK_CUR) != 0)
            throw Error(NGRAM_EPARSE, std::string("bank file truncated: ") + path + " (line 0, offset 0)");
    };
    read_f32(size_t(b->cfg.base_vocab) * size_t(D),
             [&](size_t o, size_t c) { ngk::launch_f32_to_bf16(stage.p, b->e0.p + o, int64_t(c), nullptr); });
    for (int i = 0; i < B; ++i) {
        const size_t V = size_t(b->cfg.sub_vocab[size_t(i)]);
        const size_t lo = size_t(b->row_lo[size_t(i)]), hi = size_t(b->row_hi[size_t(i)]);
        __nv_bfloat16* dst = b->sub.p + size_t(b->row_base[size_t(i)]) * size_t(d);
        skip_f32(lo * size_t(d));
        read_f32((hi - lo) * size_t(d),
                 [&](size_t o, size_t c) { ngk::launch_f32_to_bf16(stage.p, dst + o, int64_t(c), nullptr); });
        skip_f32((V - hi) * size_t(d));
    }
    if (b->cfg.variant == 1) {
        for (int i = 0; i < B; ++i) {
            const size_t n = size_t(D) * size_t(d);
            if (n > chunk) throw Error(NGRAM_EINVAL, "projection larger than the staging chunk");
            read_f32(n, [&](size_t, size_t) { ngk::launch_pack_wcat(stage.p, b->wcat.p, D, d, i, nullptr); });
        }
    }
    if (b->cfg.amp == 2) {
        read_f32(size_t(D), [&](size_t, size_t) {
            NGH_CUDA(cudaMemcpy(b->ln_gain.p, stage.p, size_t(D) * 4, cudaMemcpyDeviceToDevice));
        });
        read_f32(size_t(D), [&](size_t, size_t) {
            NGH_CUDA(cudaMemcpy(b->ln_bias.p, stage.p, size_t(D) * 4, cudaMemcpyDeviceToDevice));
        });
    }
    char extra;
    if (std::fread(&extra, 1, 1, f.get()) == 1)
        throw Error(NGRAM_EPARSE, std::string("bank file longer than its header declares: ") + path +
                                      " (line 0, offset 0)");
    NGRAM_API_END
}

}  // extern "C"
