// Local CSR SpMM  Y = Â_i T  (eq. 1; Alg. 1 L3).
//
// Row-group-per-row CSR: LPR lanes own one output row, each lane VPL float4
// column chunks, so every neighbour's feature row is one coalesced 16-byte-per-
// lane read (ld % 4 == 0, reading R24).  The group first loads LPR (col, val)
// pairs cooperatively (one coalesced load each) and broadcasts them with
// shuffles; UNR neighbours are in flight per lane before the FMAs.  The sum
// over a row's neighbours runs in CSR order, so results are run-to-run
// deterministic.
//
// Rows are visited in longest-first order (a degree-descending permutation built
// at init): power-law hubs start first and the short rows fill the tail, and the
// warps of a block get rows of similar length (ncu r1: long-scoreboard stalls with
// only 19 of 32 resident warps active under the identity order).
//
// Wide rows (ld > panel) can be processed in column panels, panel-major across the
// grid: while one panel is in flight its slice of T (n x panel x 4 B) stays
// resident in the 126 MB L2 instead of being streamed from HBM once per
// neighbour (profiles/r1: 52.7 GB of DRAM reads per unpanelled
// 256-wide launch on C3 vs 1.4 GB compulsory).
#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int kThreads = 256;

template <int LPR, int VPL, int UNR, int TAIL>
__global__ void __launch_bounds__(kThreads) spmm_kernel(int64_t n, const int32_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const float* __restrict__ val,
                                                        const float* __restrict__ T,
                                                        float* __restrict__ Y, int64_t ld, int pw,
                                                        int64_t blocks_per_panel,
                                                        const int32_t* __restrict__ order) {
    constexpr int GPW = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, gl = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const int64_t panel = blockIdx.x / blocks_per_panel;
    const int64_t blk = blockIdx.x - panel * blocks_per_panel;
    const int64_t slot = (blk * (kThreads / 32) + (threadIdx.x >> 5)) * GPW + g;
    if (slot >= n) return;
    const int64_t row = order ? __ldg(order + slot) : slot;
    const int col0 = (int)panel * pw;
    const int width = min((int64_t)pw, ld - col0);
    const float* Tp = T + col0;
    const int beg = __ldg(rowptr + row), end = __ldg(rowptr + row + 1);
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    bool colok[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) colok[v] = (gl + v * LPR) * 4 < width;
    for (int base = beg; base < end; base += LPR) {
        const int e = base + gl;
        const int c = e < end ? __ldg(colidx + e) : 0;
        const float w = e < end ? __ldg(val + e) : 0.f;
        const int cnt = min(LPR, end - base);
        if (TAIL == 0) {
            // full batches of UNR neighbours, then the remainder one at a time
            int k = 0;
            for (; k + UNR <= cnt; k += UNR) {
                int ck[UNR];
                float wk[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    ck[u] = __shfl_sync(gmask, c, k + u, LPR);
                    wk[u] = __shfl_sync(gmask, w, k + u, LPR);
                }
                float4 t[UNR][VPL];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const float* tr = Tp + (int64_t)ck[u] * ld;
#pragma unroll
                    for (int v = 0; v < VPL; ++v)
                        t[u][v] = colok[v] ? __ldg(reinterpret_cast<const float4*>(tr + (gl + v * LPR) * 4))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u)
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        acc[v].x = fmaf(wk[u], t[u][v].x, acc[v].x);
                        acc[v].y = fmaf(wk[u], t[u][v].y, acc[v].y);
                        acc[v].z = fmaf(wk[u], t[u][v].z, acc[v].z);
                        acc[v].w = fmaf(wk[u], t[u][v].w, acc[v].w);
                    }
            }
            for (; k < cnt; ++k) {
                const int ck = __shfl_sync(gmask, c, k, LPR);
                const float wk = __shfl_sync(gmask, w, k, LPR);
                const float* tr = Tp + (int64_t)ck * ld;
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    if (!colok[v]) continue;
                    const float4 t = __ldg(reinterpret_cast<const float4*>(tr + (gl + v * LPR) * 4));
                    acc[v].x = fmaf(wk, t.x, acc[v].x);
                    acc[v].y = fmaf(wk, t.y, acc[v].y);
                    acc[v].z = fmaf(wk, t.z, acc[v].z);
                    acc[v].w = fmaf(wk, t.w, acc[v].w);
                }
            }
        } else {
            // UNR neighbours per batch; the last, partial batch uses predicated loads so its
            // neighbours are still in flight together (dead slots add +0)
            for (int k = 0; k < cnt; k += UNR) {
                int ck[UNR];
                float wk[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    ck[u] = __shfl_sync(gmask, c, (k + u) & (LPR - 1), LPR);
                    wk[u] = __shfl_sync(gmask, w, (k + u) & (LPR - 1), LPR);
                    if (k + u >= cnt) wk[u] = 0.f;
                }
                float4 t[UNR][VPL];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const float* tr = Tp + (int64_t)ck[u] * ld;
                    const bool live = k + u < cnt;
#pragma unroll
                    for (int v = 0; v < VPL; ++v)
                        t[u][v] = (live && colok[v]) ? __ldg(reinterpret_cast<const float4*>(tr + (gl + v * LPR) * 4))
                                                     : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u)
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        acc[v].x = fmaf(wk[u], t[u][v].x, acc[v].x);
                        acc[v].y = fmaf(wk[u], t[u][v].y, acc[v].y);
                        acc[v].z = fmaf(wk[u], t[u][v].z, acc[v].z);
                        acc[v].w = fmaf(wk[u], t[u][v].w, acc[v].w);
                    }
            }
        }
    }
    float* yr = Y + row * ld + col0;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
        if (colok[v]) *reinterpret_cast<float4*>(yr + (gl + v * LPR) * 4) = acc[v];
}

template <int LPR, int VPL, int UNR>
void launch(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* val, const float* T, float* Y,
            int64_t ld, int pw, const int32_t* order, cudaStream_t s, int tail) {
    const int64_t rows_per_block = (kThreads / 32) * (32 / LPR);
    const int64_t bpp = (n + rows_per_block - 1) / rows_per_block;
    const int64_t panels = (ld + pw - 1) / pw;
    if (tail)
        spmm_kernel<LPR, VPL, UNR, 1><<<(unsigned)(bpp * panels), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y,
                                                                                    ld, pw, bpp, order);
    else
        spmm_kernel<LPR, VPL, UNR, 0><<<(unsigned)(bpp * panels), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y,
                                                                                    ld, pw, bpp, order);
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);    // tuning knobs for tools/spmm_bench.py
    return e ? atoi(e) : dflt;
}

}  // namespace

void launch_spmm(const int32_t* rowptr, const int32_t* colidx, const float* val, int64_t n,
                 const float* T, float* Y, int64_t ld, const int32_t* order, cudaStream_t s) {
    if (n <= 0) return;
    if (env_int("CDFGNN_SPMM_IDENTITY", 0)) order = nullptr;
    int pw = env_int("CDFGNN_SPMM_PANEL", 256);
    if (pw < 4 || pw % 4) pw = 256;
    pw = (int)std::min<int64_t>(pw, ld);
    const int nv = pw / 4;      // float4 per row within a panel
    const int unr = env_int("CDFGNN_SPMM_UNR", 0);
    const int tail = env_int("CDFGNN_SPMM_TAIL", ld > 64 ? 1 : 0);   // predicated tail for wide rows
    if (nv <= 2) launch<2, 1, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    else if (nv <= 4) launch<4, 1, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    else if (nv <= 8) launch<8, 1, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    else if (nv <= 16) {
        if (unr == 4) launch<16, 1, 4>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
        else launch<16, 1, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    } else if (nv <= 32) {
        if (unr == 4) launch<32, 1, 4>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
        else launch<32, 1, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    } else if (nv <= 64) {
        if (unr == 2) launch<32, 2, 2>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
        else if (unr == 8) launch<32, 2, 8>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
        else launch<32, 2, 4>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    } else if (nv <= 128) launch<32, 4, 4>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
    else launch<32, 8, 2>(n, rowptr, colidx, val, T, Y, ld, pw, order, s, tail);
}

}  // namespace cdfgnn
