// f64.cpp -- C-ABI of the double-precision instantiations (f64.cu): the drop-in's
// embedding_bank_t<double> / ple_params_t<double> templates run on the device through these
// (the reference uses them for its gradient checks, tests/gradcases.hpp).  Host buffers,
// synchronous, small problems: the tables are uploaded per call (a gradient check edits them
// in place between calls), the hash constants come from a hash-only bank cached per config.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "api_util.hpp"
#include "bank.hpp"

using namespace ngh;

namespace {

struct F64Ctx {
    std::shared_ptr<ngram_bank> hasher;  // HashTables + Shape of the config
    DevBuf<double> tables, work, grads;
    DevBuf<uint32_t> toks;
    DevBuf<int64_t> off;
};

// One context per config (hash-only bank + reusable device buffers); never destroyed (the
// buffers must not be released after the driver shut down at exit).
F64Ctx& ctx_for(const char* cfg_json) {
    static std::mutex mu;
    static auto& m = *new std::map<std::string, std::unique_ptr<F64Ctx>>();
    std::lock_guard<std::mutex> g(mu);
    auto& slot = m[cfg_json];
    if (!slot) {
        ngram_bank* h = nullptr;
        int dev = 0;
        NGH_CUDA(cudaGetDevice(&dev));
        const int rc = ngram_bank_create_ex(cfg_json, dev, 0, 1, NGRAM_BANK_HASH_ONLY, &h);
        if (rc) throw Error(rc, ngram_last_error());
        auto c = std::make_unique<F64Ctx>();
        c->hasher.reset(h, [](ngram_bank* b) { ngram_bank_destroy(b); });
        slot = std::move(c);
    }
    return *slot;
}

struct Layout {  // offsets (doubles) of the flattened tables
    size_t base = 0, sub = 0, proj = 0, gain = 0, bias = 0, total = 0;
};

Layout layout(const ngram_bank* b) {
    const auto& s = b->shape;
    Layout L;
    L.base = 0;
    L.sub = size_t(b->cfg.base_vocab) * size_t(s.D);
    L.proj = L.sub + size_t(b->local_rows) * size_t(s.d);
    L.gain = L.proj + (s.variant == 1 ? size_t(s.B) * size_t(s.D) * size_t(s.d) : 0);
    L.bias = L.gain + size_t(s.D);
    L.total = L.bias + size_t(s.D);
    return L;
}

// host tables (reference layout) -> one flattened host vector in the device layout
std::vector<double> flatten(const ngram_bank* b, const double* base, const double* const* sub,
                            const double* const* proj, const double* gain, const double* bias) {
    const auto& s = b->shape;
    const Layout L = layout(b);
    std::vector<double> h(L.total, 0.0);
    std::memcpy(h.data() + L.base, base, size_t(b->cfg.base_vocab) * size_t(s.D) * 8);
    for (int i = 0; i < s.B; ++i)
        std::memcpy(h.data() + L.sub + size_t(b->row_base[size_t(i)]) * size_t(s.d), sub[i],
                    size_t(b->row_hi[size_t(i)] - b->row_lo[size_t(i)]) * size_t(s.d) * 8);
    if (s.variant == 1)
        for (int i = 0; i < s.B; ++i)
            std::memcpy(h.data() + L.proj + size_t(i) * size_t(s.D) * size_t(s.d), proj[i],
                        size_t(s.D) * size_t(s.d) * 8);
    if (gain) std::memcpy(h.data() + L.gain, gain, size_t(s.D) * 8);
    if (bias) std::memcpy(h.data() + L.bias, bias, size_t(s.D) * 8);
    return h;
}

// windows of one sequence (+ prior) to the device; validates tokens (the reference raises
// out_of_range before any output, hashing.cpp:49-54)
void put_sequence(F64Ctx& c, const ngram_bank* b, const uint32_t* tokens, int64_t T, const uint32_t* prior,
                  int64_t prior_len, const uint32_t** d_prior) {
    const int R = std::max(b->cfg.max_order - 1, 0);
    std::vector<uint32_t> h(size_t(T) + size_t(R), 0u);
    std::memcpy(h.data(), tokens, size_t(T) * 4);
    const int64_t n = std::min<int64_t>(prior_len, R);
    for (int64_t i = 0; i < n; ++i) h[size_t(T) + size_t(R - n + i)] = prior[prior_len - n + i];  // right-aligned
    for (size_t i = 0; i < h.size(); ++i)
        if (h[i] >= b->cfg.base_vocab && (i < size_t(T) || n > 0))
            throw Error(NGRAM_ERANGE, "embedding: token " + std::to_string(h[i]) + " out of range for base vocabulary " +
                                          std::to_string(b->cfg.base_vocab));
    c.toks.ensure(h.size());
    NGH_CUDA(cudaMemcpy(c.toks.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    const int64_t off[2] = {0, T};
    c.off.ensure(2);
    NGH_CUDA(cudaMemcpy(c.off.p, off, 16, cudaMemcpyHostToDevice));
    *d_prior = (R > 0 && n > 0) ? c.toks.p + T : nullptr;
}

}  // namespace

extern "C" {

int ngram_f64_forward(const char* cfg_json, const double* base, const double* const* sub, const double* const* proj,
                      const double* ln_gain, const double* ln_bias, const uint32_t* tokens, int64_t T,
                      const uint32_t* prior, int64_t prior_len, double* merged, double* rows) {
    NGRAM_API_BEGIN
    if (!cfg_json || T < 0 || (T > 0 && (!tokens || !base || !merged))) throw Error(NGRAM_EINVAL, "ngram_f64_forward: bad argument");
    F64Ctx& c = ctx_for(cfg_json);
    const ngram_bank* b = c.hasher.get();
    if (T == 0) return NGRAM_OK;
    if (b->shape.amp == ngk::kAmpLN && rows && (!ln_gain || !ln_bias))
        throw Error(NGRAM_EINVAL, "amplify: layer_norm needs gain/bias of size D");
    const Layout L = layout(b);
    const auto h = flatten(b, base, sub, proj, ln_gain, ln_bias);
    c.tables.ensure(L.total);
    NGH_CUDA(cudaMemcpy(c.tables.p, h.data(), L.total * 8, cudaMemcpyHostToDevice));
    const uint32_t* d_prior = nullptr;
    put_sequence(c, b, tokens, T, prior, prior_len, &d_prior);
    const size_t TD = size_t(T) * size_t(b->shape.D);
    c.work.ensure(2 * TD);
    ngk::launch_f64_forward(b->shape, b->ht.p, c.toks.p, c.off.p, T, d_prior, c.tables.p + L.base, c.tables.p + L.sub,
                            c.tables.p + L.proj, c.tables.p + L.gain, c.tables.p + L.bias, b->shape.amp, c.work.p,
                            rows ? c.work.p + TD : nullptr, nullptr);
    NGH_CUDA(cudaGetLastError());
    NGH_CUDA(cudaMemcpy(merged, c.work.p, TD * 8, cudaMemcpyDeviceToHost));
    if (rows) NGH_CUDA(cudaMemcpy(rows, c.work.p + TD, TD * 8, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_f64_backward(const char* cfg_json, const double* base, const double* const* sub, const double* const* proj,
                       const double* ln_gain, const double* ln_bias, const uint32_t* tokens, int64_t T,
                       const uint32_t* prior, int64_t prior_len, const double* merged, const double* upstream,
                       double* g_base, double* const* g_sub, double* const* g_proj, double* g_gain, double* g_bias) {
    NGRAM_API_BEGIN
    if (!cfg_json || T < 0 || (T > 0 && (!tokens || !upstream || !g_base || !g_sub)))
        throw Error(NGRAM_EINVAL, "ngram_f64_backward: bad argument");
    F64Ctx& c = ctx_for(cfg_json);
    const ngram_bank* b = c.hasher.get();
    if (T == 0) return NGRAM_OK;
    const auto& s = b->shape;
    const bool ln = merged && s.amp == ngk::kAmpLN;
    if (ln && (!ln_gain || !g_gain || !g_bias)) throw Error(NGRAM_EINVAL, "layer_norm gradients need gain and grads");
    const Layout L = layout(b);
    const auto h = flatten(b, base, sub, proj, ln_gain, ln_bias);
    const auto gh = flatten(b, g_base, const_cast<const double* const*>(g_sub),
                            s.variant == 1 ? const_cast<const double* const*>(g_proj) : nullptr, ln ? g_gain : nullptr,
                            ln ? g_bias : nullptr);
    c.tables.ensure(L.total);
    c.grads.ensure(L.total);
    NGH_CUDA(cudaMemcpy(c.tables.p, h.data(), L.total * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(c.grads.p, gh.data(), L.total * 8, cudaMemcpyHostToDevice));
    const uint32_t* d_prior = nullptr;
    put_sequence(c, b, tokens, T, prior, prior_len, &d_prior);
    const size_t TD = size_t(T) * size_t(s.D);
    c.work.ensure(5 * TD);  // upstream | merged | d_pre | LN scratch [T][2][D]
    NGH_CUDA(cudaMemcpy(c.work.p, upstream, TD * 8, cudaMemcpyHostToDevice));
    if (merged) NGH_CUDA(cudaMemcpy(c.work.p + TD, merged, TD * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemset(c.work.p + 3 * TD, 0, 2 * TD * 8));
    ngk::launch_f64_backward(s, b->ht.p, c.toks.p, c.off.p, T, d_prior, c.tables.p + L.sub, c.tables.p + L.proj,
                             c.tables.p + L.gain, merged ? s.amp : ngk::kAmpNone, merged ? c.work.p + TD : nullptr,
                             c.work.p, c.work.p + 2 * TD, c.grads.p + L.base, c.grads.p + L.sub, c.grads.p + L.proj,
                             c.grads.p + L.gain, c.grads.p + L.bias, nullptr);
    NGH_CUDA(cudaGetLastError());
    std::vector<double> out(L.total);
    NGH_CUDA(cudaMemcpy(out.data(), c.grads.p, L.total * 8, cudaMemcpyDeviceToHost));
    std::memcpy(g_base, out.data() + L.base, size_t(b->cfg.base_vocab) * size_t(s.D) * 8);
    for (int i = 0; i < s.B; ++i)
        std::memcpy(g_sub[i], out.data() + L.sub + size_t(b->row_base[size_t(i)]) * size_t(s.d),
                    size_t(b->row_hi[size_t(i)] - b->row_lo[size_t(i)]) * size_t(s.d) * 8);
    if (s.variant == 1 && g_proj)
        for (int i = 0; i < s.B; ++i)
            std::memcpy(g_proj[i], out.data() + L.proj + size_t(i) * size_t(s.D) * size_t(s.d),
                        size_t(s.D) * size_t(s.d) * 8);
    if (ln) {
        std::memcpy(g_gain, out.data() + L.gain, size_t(s.D) * 8);
        std::memcpy(g_bias, out.data() + L.bias, size_t(s.D) * 8);
    }
    NGRAM_API_END
}

int ngram_f64_amplify(int amp_mode, int64_t D, const double* gain, const double* bias, const double* in,
                      double* out) {
    NGRAM_API_BEGIN
    if (D < 0 || amp_mode < 0 || amp_mode > 2 || (D > 0 && (!in || !out)) || (amp_mode == 2 && D > 0 && (!gain || !bias)))
        throw Error(NGRAM_EINVAL, "ngram_f64_amplify: bad argument");
    if (D == 0) return NGRAM_OK;
    DevBuf<double> w;
    w.alloc(size_t(4 * D));
    NGH_CUDA(cudaMemcpy(w.p, in, size_t(D) * 8, cudaMemcpyHostToDevice));
    if (amp_mode == 2) {
        NGH_CUDA(cudaMemcpy(w.p + D, gain, size_t(D) * 8, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(w.p + 2 * D, bias, size_t(D) * 8, cudaMemcpyHostToDevice));
    }
    ngk::launch_f64_amplify(amp_mode, int(D), w.p + D, w.p + 2 * D, w.p, w.p + 3 * D, nullptr);
    NGH_CUDA(cudaGetLastError());
    NGH_CUDA(cudaMemcpy(out, w.p + 3 * D, size_t(D) * 8, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_f64_amplify_backward(int amp_mode, int64_t D, const double* pre, const double* upstream, const double* gain,
                               double* d_pre, double* g_gain, double* g_bias) {
    NGRAM_API_BEGIN
    if (D < 0 || amp_mode < 0 || amp_mode > 2 || (D > 0 && (!pre || !upstream || !d_pre)) ||
        (amp_mode == 2 && D > 0 && (!gain || !g_gain || !g_bias)))
        throw Error(NGRAM_EINVAL, "ngram_f64_amplify_backward: bad argument");
    if (D == 0) return NGRAM_OK;
    DevBuf<double> w;
    w.alloc(size_t(6 * D));
    NGH_CUDA(cudaMemcpy(w.p, pre, size_t(D) * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(w.p + D, upstream, size_t(D) * 8, cudaMemcpyHostToDevice));
    if (amp_mode == 2) {
        NGH_CUDA(cudaMemcpy(w.p + 2 * D, gain, size_t(D) * 8, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(w.p + 4 * D, g_gain, size_t(D) * 8, cudaMemcpyHostToDevice));
        NGH_CUDA(cudaMemcpy(w.p + 5 * D, g_bias, size_t(D) * 8, cudaMemcpyHostToDevice));
    }
    ngk::launch_f64_amplify_backward(amp_mode, int(D), w.p, w.p + D, w.p + 2 * D, w.p + 3 * D, w.p + 4 * D, w.p + 5 * D,
                                     nullptr);
    NGH_CUDA(cudaGetLastError());
    NGH_CUDA(cudaMemcpy(d_pre, w.p + 3 * D, size_t(D) * 8, cudaMemcpyDeviceToHost));
    if (amp_mode == 2) {
        NGH_CUDA(cudaMemcpy(g_gain, w.p + 4 * D, size_t(D) * 8, cudaMemcpyDeviceToHost));
        NGH_CUDA(cudaMemcpy(g_bias, w.p + 5 * D, size_t(D) * 8, cudaMemcpyDeviceToHost));
    }
    NGRAM_API_END
}

int ngram_f64_gated_ffn(int d_model, int hidden, const double* gate, const double* down, const double* x,
                        const double* g, double* y) {
    NGRAM_API_BEGIN
    if (d_model < 1 || hidden < 1 || !gate || !down || !x || !g || !y)
        throw Error(NGRAM_EINVAL, "ngram_f64_gated_ffn: bad argument");
    const size_t Dm = size_t(d_model), H = size_t(hidden);
    DevBuf<double> w;
    w.alloc(2 * H * Dm + Dm + H + H + Dm);
    double *dg = w.p, *dd = dg + H * Dm, *dx = dd + H * Dm, *gv = dx + Dm, *hw = gv + H, *dy = hw + H;
    NGH_CUDA(cudaMemcpy(dg, gate, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(dd, down, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(dx, x, Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(gv, g, H * 8, cudaMemcpyHostToDevice));
    ngk::launch_f64_gated_ffn(d_model, hidden, dg, dd, dx, gv, hw, dy, nullptr);
    NGH_CUDA(cudaGetLastError());
    NGH_CUDA(cudaMemcpy(y, dy, Dm * 8, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

int ngram_f64_gated_ffn_backward(int d_model, int hidden, const double* gate, const double* down, const double* x,
                                 const double* g, const double* upstream, double* g_gate, double* g_down, double* dx,
                                 double* dg) {
    NGRAM_API_BEGIN
    if (d_model < 1 || hidden < 1 || !gate || !down || !x || !g || !upstream || !g_gate || !g_down || !dx || !dg)
        throw Error(NGRAM_EINVAL, "ngram_f64_gated_ffn_backward: bad argument");
    const size_t Dm = size_t(d_model), H = size_t(hidden);
    DevBuf<double> w;
    w.alloc(4 * H * Dm + 3 * Dm + 6 * H);
    double *wg = w.p, *wd = wg + H * Dm, *gg = wd + H * Dm, *gd = gg + H * Dm, *xv = gd + H * Dm, *up = xv + Dm,
           *dxv = up + Dm, *gv = dxv + Dm, *dgv = gv + H, *ws = dgv + H;
    NGH_CUDA(cudaMemcpy(wg, gate, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(wd, down, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(gg, g_gate, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(gd, g_down, H * Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(xv, x, Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(up, upstream, Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(dxv, dx, Dm * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(gv, g, H * 8, cudaMemcpyHostToDevice));
    NGH_CUDA(cudaMemcpy(dgv, dg, H * 8, cudaMemcpyHostToDevice));
    ngk::launch_f64_gated_ffn_backward(d_model, hidden, wg, wd, xv, gv, up, ws, gg, gd, dxv, dgv, nullptr);
    NGH_CUDA(cudaGetLastError());
    NGH_CUDA(cudaMemcpy(g_gate, gg, H * Dm * 8, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(g_down, gd, H * Dm * 8, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(dx, dxv, Dm * 8, cudaMemcpyDeviceToHost));
    NGH_CUDA(cudaMemcpy(dg, dgv, H * 8, cudaMemcpyDeviceToHost));
    NGRAM_API_END
}

}  // extern "C"
