// ple.hpp -- drop-in for proj/include/ngram/ple.hpp: the per-layer embedding FFN blocks
//   y = W_d (SiLU(W_g x) (.) g),   g = E0l(t) (ffn_ple) or a layer bank's embedding (ffn_plne)
// ple_params_t stays the reference's host parameter store (same make_ple_params RNG order).
// The float forward / backward run on the GPU (ngram_plne_* in include/ngram_b200.h):
// ffn_plne over a device_bank; ffn_ple as ffn_plne over a base-only layer bank whose E0 is
// the table (test_ple.cpp:150-172).  Device tables are bf16: parity with the reference
// float path holds on bf16-representable tables.
#pragma once
#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "ngram/embedding.hpp"

namespace ngram {

template <typename T>
struct ple_params_t {
    int d_model = 0;
    int hidden = 0;
    std::uint32_t base_vocab = 0;
    std::vector<T> gate;   // hidden x d_model
    std::vector<T> down;   // d_model x hidden
    std::vector<T> table;  // base_vocab x hidden; empty for the n-gram form
};
using ple_params = ple_params_t<float>;

inline void ple_shape_check(int d_model, int hidden, std::uint32_t base_vocab) {  // ple.cpp:8-16
    if (d_model < 1 || hidden < 1) throw std::invalid_argument("ple: d_model and hidden must be >= 1");
    if (base_vocab < 2) throw std::invalid_argument("ple: base vocabulary must be >= 2");
}

// make_ple_params (ple.hpp:34-50): gate, down, table ~ N(0, 0.02^2) in that order.
template <typename T>
ple_params_t<T> make_ple_params(int d_model, int hidden, std::uint32_t base_vocab, std::uint64_t seed) {
    ple_shape_check(d_model, hidden, base_vocab);
    ple_params_t<T> p;
    p.d_model = d_model;
    p.hidden = hidden;
    p.base_vocab = base_vocab;
    rng64 rng(seed);
    p.gate.resize(std::size_t(hidden) * std::size_t(d_model));
    p.down.resize(std::size_t(d_model) * std::size_t(hidden));
    p.table.resize(std::size_t(base_vocab) * std::size_t(hidden));
    for (auto& x : p.gate) x = T(0.02 * gaussian(rng));
    for (auto& x : p.down) x = T(0.02 * gaussian(rng));
    for (auto& x : p.table) x = T(0.02 * gaussian(rng));
    return p;
}

template <typename T>
ple_params_t<T> ple_zeros_like(const ple_params_t<T>& p) {
    ple_params_t<T> g;
    g.d_model = p.d_model;
    g.hidden = p.hidden;
    g.base_vocab = p.base_vocab;
    g.gate.assign(p.gate.size(), T(0));
    g.down.assign(p.down.size(), T(0));
    g.table.assign(p.table.size(), T(0));
    return g;
}

// Plain per-layer form: gate the layer table row of the current token (ple.hpp:146-166).
std::vector<float> ffn_ple(std::span<const float> x, token_id token, const ple_params& p);
void ffn_ple_backward(std::span<const float> x, token_id token, const ple_params& p, std::span<const float> upstream,
                      ple_params& grads, std::span<float> dx);

// N-gram per-layer form: gate the layer bank's embedding of the trailing context
// (ple.hpp:168-196).  The layer bank's width must equal the gate width, amplification none.
std::vector<float> ffn_plne(std::span<const float> x, std::span<const token_id> context, const device_bank& layer_bank,
                            const ple_params& p);
std::vector<float> ffn_plne(std::span<const float> x, std::span<const token_id> context,
                            const embedding_bank& layer_bank, const ple_params& p);
void ffn_plne_backward(std::span<const float> x, std::span<const token_id> context, const device_bank& layer_bank,
                       const ple_params& p, std::span<const float> upstream, ple_params& grads,
                       embedding_bank& bank_grads, std::span<float> dx);
void ffn_plne_backward(std::span<const float> x, std::span<const token_id> context, const embedding_bank& layer_bank,
                       const ple_params& p, std::span<const float> upstream, ple_params& grads,
                       embedding_bank& bank_grads, std::span<float> dx);

// The reference's templates (ple.hpp:148-198): T = float -> the device float path above,
// T = double -> the device fp64 instantiation (ngram_f64_gated_ffn*, embed via ngram_f64_*).
template <typename T>
std::vector<T> ffn_ple(std::span<const T> x, token_id token, const ple_params_t<T>& p);
template <typename T>
void ffn_ple_backward(std::span<const T> x, token_id token, const ple_params_t<T>& p, std::span<const T> upstream,
                      ple_params_t<T>& grads, std::span<T> dx);
template <typename T>
std::vector<T> ffn_plne(std::span<const T> x, std::span<const token_id> context, const embedding_bank_t<T>& layer_bank,
                        const ple_params_t<T>& p);
template <typename T>
void ffn_plne_backward(std::span<const T> x, std::span<const token_id> context, const embedding_bank_t<T>& layer_bank,
                       const ple_params_t<T>& p, std::span<const T> upstream, ple_params_t<T>& grads,
                       embedding_bank_t<T>& bank_grads, std::span<T> dx);

}  // namespace ngram
