// shard.cu -- the row-sharded exchange: K1 + K2 fused with the
// collective.  Every rank hashes the ALL-GATHERED token batch (4 B/token of input, ids
// recomputed locally instead of exchanged) and, for every (token, branch) whose bucket row
// it owns, copies that d-wide row straight into the X buffer of the token's home rank --
// a peer pointer over NVLink (CUDA IPC), or a local pointer for its own tokens.  Each X
// row slice has exactly one owner, so after all ranks' scatters X is complete and
// bit-identical to the single-GPU gather.
#include <cstdint>

#include "kernels.h"

namespace ngk {

namespace {

struct PeerX {
    __nv_bfloat16* x[64];
    int64_t tok_off[65];  // rank r's home tokens = [tok_off[r], tok_off[r+1]) of the gathered batch
};

// Lane l of a warp checks pair (t = t0 + l, branch b) (coalesced reads of grow's [B][Tpad]
// rows); the rows this rank owns (~1/P of them) are then copied one after another by the
// whole warp (d/8 lanes x 16 B each), so no warp idles on a non-owned pair.
__global__ void __launch_bounds__(256) shard_scatter_kernel(int B, int d, int D, const int32_t* __restrict__ grow,
                                                            int64_t Tpad, int64_t T, int nranks, PeerX px,
                                                            const __nv_bfloat16* __restrict__ sub,
                                                            const unsigned long long* err) {
    if (*err != ~0ull) return;
    const int lane = threadIdx.x & 31;
    const int vec_per_row = d / 8;
    const int64_t tiles = ((T + 31) / 32) * B;  // (branch, 32-position group)
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; w < tiles; w += warps) {
        const int b = (int)(w % B);
        const int64_t t = (w / B) * 32 + lane;
        const int32_t row = t < T ? __ldg(grow + (int64_t)b * Tpad + t) : -1;  // -1: another rank owns it
        int home = 0;
        if (row >= 0)
            while (home + 1 < nranks && t >= px.tok_off[home + 1]) ++home;
        unsigned owned = __ballot_sync(0xffffffffu, row >= 0);
        while (owned) {
            const int l = __ffs(owned) - 1;
            owned &= owned - 1;
            const int32_t r = __shfl_sync(0xffffffffu, row, l);
            const int h = __shfl_sync(0xffffffffu, home, l);
            const int64_t tl = (w / B) * 32 + l;
            const uint4* src = reinterpret_cast<const uint4*>(sub + (int64_t)r * d);
            uint4* dst = reinterpret_cast<uint4*>(px.x[h] + (tl - px.tok_off[h]) * D + (int64_t)b * d);
            for (int c = lane; c < vec_per_row; c += 32) dst[c] = __ldg(src + c);
        }
    }
    __threadfence_system();  // peer stores visible system-wide before the barrier that follows
}

}  // namespace

void launch_shard_scatter(const Shape& s, const int32_t* grow_all, int64_t Tpad_all, const int64_t* rank_token_offsets,
                          int nranks, const __nv_bfloat16* sub, __nv_bfloat16* const* peer_x, int64_t T_all,
                          const unsigned long long* err, cudaStream_t st) {
    if (T_all <= 0) return;
    PeerX px{};
    for (int r = 0; r < nranks; ++r) px.x[r] = peer_x[r];
    for (int r = 0; r <= nranks; ++r) px.tok_off[r] = rank_token_offsets[r];
    const int64_t tiles = ((T_all + 31) / 32) * s.B;
    int64_t blocks = (tiles + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    shard_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(s.B, s.d, s.D, grow_all, Tpad_all, T_all, nranks, px, sub,
                                                           err);
    count_launch();
}

}  // namespace ngk
