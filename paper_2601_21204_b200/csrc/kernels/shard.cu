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

// ---------------------------------------------------------------- NCCL exchange variants
// The same exchange as the peer-store scatter, expressed as data for a collective the caller
// runs (NCCL through torch.distributed): rows are moved raw, so every variant produces the
// same home X, bit for bit.
//   * compact (all-to-all / grouped send-recv): each rank packs the rows it owns, per
//     destination rank in (token, branch) order; the receiver derives every row's slot from
//     the ids it hashes itself, so no index travels with the rows;
//   * padded (reduce-scatter): [nranks][max_home][D] with the owned rows in place and -0.0
//     everywhere else -- -0.0 is the identity of IEEE addition (x + -0 = x, also for x = +0),
//     so the summed home X is the owned rows exactly.

namespace {

// owner(b, h) = floor(h * P / V_b): the rank whose row block [ceil(rV/P), ceil((r+1)V/P)) holds h.
__device__ __forceinline__ int xchg_owner(uint64_t h, uint64_t V, int P) {
    if (V < (uint64_t(1) << 57)) return (int)((h * (uint64_t)P) / V);
    return (int)(((unsigned __int128)h * (unsigned)P) / V);
}

constexpr int kXchgChunk = 1024;  // tokens per scan block (256 threads x 4)

// Column c of the exchange counts, for token t: c = 0 -> pairs this rank owns (over the whole
// gathered batch); c = 1 + o -> pairs of a home token owned by rank o.
__device__ __forceinline__ int xchg_count(const uint64_t* __restrict__ ids, const uint64_t* __restrict__ V, int B,
                                          int P, int who, int64_t t) {
    int c = 0;
    for (int b = 0; b < B; ++b) c += xchg_owner(__ldg(ids + t * B + b), V[b], P) == who;
    return c;
}

struct XchgCols {
    uint64_t V[kMaxBranches];
    int B, P, rank;
    int64_t all_T, h0, h1;  // gathered batch size; this rank's home tokens [h0, h1)
};

__device__ __forceinline__ void xchg_range(const XchgCols& c, int col, int64_t* lo, int64_t* hi, int* who) {
    if (col == 0) {
        *lo = 0;
        *hi = c.all_T;
        *who = c.rank;
    } else {
        *lo = c.h0;
        *hi = c.h1;
        *who = col - 1;
    }
}

// Block-wide exclusive scan of one value per thread (256 threads); returns the block total.
__device__ __forceinline__ int block_excl_scan(int v, int* out_excl) {
    __shared__ int warp_tot[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    int base = 0, tot = 0;
    for (int i = 0; i < 8; ++i) {
        if (i < w) base += warp_tot[i];
        tot += warp_tot[i];
    }
    __syncthreads();
    *out_excl = base + x - v;
    return tot;
}

// phase 1 (tot != null, pref == null): chunk totals; phase 3: exclusive prefix per token.
__global__ void __launch_bounds__(256) xchg_scan_kernel(XchgCols c, const uint64_t* __restrict__ ids,
                                                        int64_t* __restrict__ tot, const int64_t* __restrict__ chunk_off,
                                                        int64_t* __restrict__ pref, int64_t pref_stride,
                                                        const unsigned long long* err) {
    if (*err != ~0ull) return;
    const int col = blockIdx.y;
    int64_t lo, hi;
    int who;
    xchg_range(c, col, &lo, &hi, &who);
    const int64_t t0 = lo + (int64_t)blockIdx.x * kXchgChunk;
    if (t0 >= hi) {  // past this column's range (home columns are shorter): contributes 0
        if (!pref && threadIdx.x == 0) tot[(int64_t)col * gridDim.x + blockIdx.x] = 0;
        return;
    }
    int v[4], sum = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t t = t0 + threadIdx.x * 4 + i;
        v[i] = t < hi ? xchg_count(ids, c.V, c.B, c.P, who, t) : 0;
        sum += v[i];
    }
    int excl;
    const int total = block_excl_scan(sum, &excl);
    if (!pref) {
        if (threadIdx.x == 0) tot[(int64_t)col * gridDim.x + blockIdx.x] = total;
        return;
    }
    int64_t run = chunk_off[(int64_t)col * gridDim.x + blockIdx.x] + excl;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t t = t0 + threadIdx.x * 4 + i;
        if (t < hi) pref[(int64_t)col * pref_stride + (t - lo)] = run;
        run += v[i];
    }
}

// phase 2: exclusive scan of the chunk totals of every column (one thread per column) and
// the column totals; `bounds`: col-0 prefix at every rank's first home token (send offsets).
__global__ void xchg_scan_tot_kernel(int ncols, int nchunks, const int64_t* __restrict__ tot,
                                     int64_t* __restrict__ chunk_off, int64_t* __restrict__ col_tot,
                                     const unsigned long long* err) {
    const int col = threadIdx.x;
    if (col >= ncols) return;
    int64_t run = 0;
    const bool bad = *err != ~0ull;
    for (int k = 0; k < nchunks; ++k) {
        chunk_off[(int64_t)col * nchunks + k] = run;
        if (!bad) run += tot[(int64_t)col * nchunks + k];
    }
    col_tot[col] = run;
}

__global__ void xchg_bounds_kernel(const int64_t* __restrict__ pref0, const int64_t* __restrict__ col_tot,
                                   XchgCols c, PeerX px, int64_t* __restrict__ out, const unsigned long long* err) {
    // out[0 .. P]: col-0 prefix at rank p's first home token (out[P] = total owned);
    // out[P+1 .. 2P]: rows received from each source rank.  All zero after a bad token (the
    // call reports ERANGE; no rows move).
    const int i = threadIdx.x;
    const bool bad = *err != ~0ull;
    if (i <= c.P) out[i] = bad ? 0 : (px.tok_off[i] < c.all_T ? pref0[px.tok_off[i]] : col_tot[0]);
    if (i < c.P) out[c.P + 1 + i] = bad ? 0 : col_tot[1 + i];
}

// warp per gathered token: the rows this rank owns -> send[pref0[t] + k] (k-th owned branch).
__global__ void __launch_bounds__(256) xchg_pack_kernel(XchgCols c, int d, const uint64_t* __restrict__ ids,
                                                        const int32_t* __restrict__ grow, int64_t Tpad,
                                                        const int64_t* __restrict__ pref0,
                                                        const __nv_bfloat16* __restrict__ sub,
                                                        __nv_bfloat16* __restrict__ send, const unsigned long long* err) {
    if (*err != ~0ull) return;
    const int lane = threadIdx.x & 31;
    const int vec = d / 8;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; t < c.all_T; t += warps) {
        int64_t pos = __ldg(pref0 + t);
        for (int b0 = 0; b0 < c.B; b0 += 32) {
            const int b = b0 + lane;
            const bool own = b < c.B && xchg_owner(__ldg(ids + t * c.B + b), c.V[b], c.P) == c.rank;
            unsigned m = __ballot_sync(0xffffffffu, own);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int32_t row = __ldg(grow + (int64_t)(b0 + l) * Tpad + t);
                const uint4* src = reinterpret_cast<const uint4*>(sub + (int64_t)row * d);
                uint4* dst = reinterpret_cast<uint4*>(send + pos * d);
                for (int v = lane; v < vec; v += 32) dst[v] = __ldg(src + v);
                ++pos;
            }
        }
    }
}

struct RecvBase {
    int64_t base[64];
};

// warp per home token: row (t, b) came from rank o = owner(b, h) at slot
// base[o] + pref_o[t] + #{b' < b : owner(b') = o}  ->  X[t - h0][b*d ..].
__global__ void __launch_bounds__(256) xchg_unpack_kernel(XchgCols c, int d, int D, const uint64_t* __restrict__ ids,
                                                          const int64_t* __restrict__ pref, int64_t pref_stride,
                                                          RecvBase rb, const __nv_bfloat16* __restrict__ recv,
                                                          __nv_bfloat16* __restrict__ X, const unsigned long long* err) {
    if (*err != ~0ull) return;
    __shared__ int cnt[8][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int vec = d / 8;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
    const int64_t home = c.h1 - c.h0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + w; i < home; i += warps) {
        const int64_t t = c.h0 + i;
        for (int o = lane; o < c.P; o += 32) cnt[w][o] = 0;
        __syncwarp();
        for (int b0 = 0; b0 < c.B; b0 += 32) {
            const int b = b0 + lane;
            const int o = b < c.B ? xchg_owner(__ldg(ids + t * c.B + b), c.V[b], c.P) : 64 + lane;  // unique if idle
            const unsigned peers = __match_any_sync(0xffffffffu, o);
            int64_t slot = 0;
            if (b < c.B)
                slot = rb.base[o] + __ldg(pref + (int64_t)(1 + o) * pref_stride + i) + cnt[w][o] +
                       __popc(peers & ((1u << lane) - 1u));
            __syncwarp();
            if (b < c.B && (peers & ((1u << lane) - 1u)) == 0) cnt[w][o] += __popc(peers);  // group leader
            __syncwarp();
            unsigned m = __ballot_sync(0xffffffffu, b < c.B);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int64_t sl = __shfl_sync(0xffffffffu, slot, l);
                const uint4* src = reinterpret_cast<const uint4*>(recv + sl * d);
                uint4* dst = reinterpret_cast<uint4*>(X + i * D + (int64_t)(b0 + l) * d);
                for (int v = lane; v < vec; v += 32) dst[v] = __ldg(src + v);
            }
        }
        __syncwarp();
    }
}

__global__ void fill_u16_kernel(uint16_t* __restrict__ p, uint16_t v, int64_t n) {
    const int64_t n8 = n / 8;
    const uint32_t v2 = (uint32_t)v | ((uint32_t)v << 16);
    const uint4 vv = make_uint4(v2, v2, v2, v2);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x)
        reinterpret_cast<uint4*>(p)[i] = vv;
    for (int64_t i = n8 * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

}  // namespace

void launch_xchg_prepare(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks,
                         const int64_t* rank_token_offsets, int64_t all_T, const uint64_t* ids_all,
                         int64_t* tot, int64_t* chunk_off, int64_t* col_tot, int64_t* pref, int64_t pref_stride,
                         int64_t* bounds_out, const unsigned long long* err, cudaStream_t st) {
    XchgCols c{};
    for (int b = 0; b < s.B; ++b) c.V[b] = sub_vocab[b];
    c.B = s.B;
    c.P = nranks;
    c.rank = rank;
    c.all_T = all_T;
    c.h0 = rank_token_offsets[rank];
    c.h1 = rank_token_offsets[rank + 1];
    PeerX px{};
    for (int r = 0; r <= nranks; ++r) px.tok_off[r] = rank_token_offsets[r];
    const int ncols = 1 + nranks;
    const int nchunks = (int)((all_T + kXchgChunk - 1) / kXchgChunk);
    const dim3 grid((unsigned)nchunks, (unsigned)ncols);
    xchg_scan_kernel<<<grid, 256, 0, st>>>(c, ids_all, tot, nullptr, nullptr, 0, err);
    xchg_scan_tot_kernel<<<1, 128, 0, st>>>(ncols, nchunks, tot, chunk_off, col_tot, err);
    xchg_scan_kernel<<<grid, 256, 0, st>>>(c, ids_all, tot, chunk_off, pref, pref_stride, err);
    xchg_bounds_kernel<<<1, 128, 0, st>>>(pref, col_tot, c, px, bounds_out, err);
    count_launch(4);
}

void launch_xchg_pack(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks, int64_t all_T,
                      const uint64_t* ids_all, const int32_t* grow_all, int64_t Tpad, const int64_t* pref0,
                      const __nv_bfloat16* sub, __nv_bfloat16* send, const unsigned long long* err, cudaStream_t st) {
    if (all_T <= 0) return;
    XchgCols c{};
    for (int b = 0; b < s.B; ++b) c.V[b] = sub_vocab[b];
    c.B = s.B;
    c.P = nranks;
    c.rank = rank;
    c.all_T = all_T;
    int64_t blocks = (all_T + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    xchg_pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(c, s.d, ids_all, grow_all, Tpad, pref0, sub, send, err);
    count_launch();
}

void launch_xchg_unpack(const Shape& s, const uint64_t* sub_vocab, int rank, int nranks,
                        const int64_t* rank_token_offsets, const uint64_t* ids_all, const int64_t* pref,
                        int64_t pref_stride, const int64_t* recv_rows, const __nv_bfloat16* recv, __nv_bfloat16* X,
                        const unsigned long long* err, cudaStream_t st) {
    XchgCols c{};
    for (int b = 0; b < s.B; ++b) c.V[b] = sub_vocab[b];
    c.B = s.B;
    c.P = nranks;
    c.rank = rank;
    c.h0 = rank_token_offsets[rank];
    c.h1 = rank_token_offsets[rank + 1];
    if (c.h1 <= c.h0) return;
    RecvBase rb{};
    int64_t run = 0;
    for (int o = 0; o < nranks; ++o) {
        rb.base[o] = run;
        run += recv_rows[o];
    }
    int64_t blocks = (c.h1 - c.h0 + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    xchg_unpack_kernel<<<(unsigned)blocks, 256, 0, st>>>(c, s.d, s.D, ids_all, pref, pref_stride, rb, recv, X, err);
    count_launch();
}

void launch_xchg_pack_padded(const Shape& s, const int32_t* grow_all, int64_t Tpad_all,
                             const int64_t* rank_token_offsets, int nranks, int64_t max_home,
                             const __nv_bfloat16* sub, __nv_bfloat16* send, int64_t T_all,
                             const unsigned long long* err, cudaStream_t st) {
    const int64_t n = (int64_t)nranks * max_home * s.D;
    int64_t blocks = (n / 8 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    fill_u16_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<uint16_t*>(send), 0x8000u, n);  // -0.0 bf16
    count_launch();
    __nv_bfloat16* dst[64];
    for (int r = 0; r < nranks; ++r) dst[r] = send + (int64_t)r * max_home * s.D;
    launch_shard_scatter(s, grow_all, Tpad_all, rank_token_offsets, nranks, sub, dst, T_all, err, st);
}

}  // namespace ngk
