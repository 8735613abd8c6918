// Local CSR SpMM  Y = Â_i T  (eq. 1; Alg. 1 L3).
//
// Row-group-per-row CSR: LPR lanes own one output row, each lane VPL float4
// column chunks, so every neighbour's feature row is one coalesced 16-byte-per-
// lane read (ld % 4 == 0, reading R24).  The group first loads LPR (col, val)
// pairs cooperatively (one coalesced load each) and broadcasts them with
// shuffles; four neighbours are in flight per lane before the FMAs.  The sum
// over a row's neighbours runs in CSR order, so results are run-to-run
// deterministic.  HBM/L2-bound; roofline and algorithmic bytes in DESIGN.md.
#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int kThreads = 256;

template <int LPR, int VPL>
__global__ void __launch_bounds__(kThreads) spmm_kernel(int64_t n, const int32_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const float* __restrict__ val,
                                                        const float* __restrict__ T,
                                                        float* __restrict__ Y, int64_t ld) {
    constexpr int GPW = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, gl = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const int64_t row = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * GPW + g;
    if (row >= n) return;
    const int beg = __ldg(rowptr + row), end = __ldg(rowptr + row + 1);
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    bool colok[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) colok[v] = (gl + v * LPR) * 4 < ld;
    for (int base = beg; base < end; base += LPR) {
        const int e = base + gl;
        const int c = e < end ? __ldg(colidx + e) : 0;
        const float w = e < end ? __ldg(val + e) : 0.f;
        const int cnt = min(LPR, end - base);
        int k = 0;
        for (; k + 4 <= cnt; k += 4) {
            int ck[4];
            float wk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                ck[u] = __shfl_sync(gmask, c, k + u, LPR);
                wk[u] = __shfl_sync(gmask, w, k + u, LPR);
            }
            float4 t[4][VPL];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float* tr = T + (int64_t)ck[u] * ld;
#pragma unroll
                for (int v = 0; v < VPL; ++v)
                    t[u][v] = colok[v] ? __ldg(reinterpret_cast<const float4*>(tr + (gl + v * LPR) * 4))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
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
            const float* tr = T + (int64_t)ck * ld;
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
    }
    float* yr = Y + row * ld;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
        if (colok[v]) *reinterpret_cast<float4*>(yr + (gl + v * LPR) * 4) = acc[v];
}

}  // namespace

void launch_spmm(const int32_t* rowptr, const int32_t* colidx, const float* val, int64_t n,
                 const float* T, float* Y, int64_t ld, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t nv = ld / 4;
    auto blocks = [&](int lpr) {
        const int64_t rows_per_block = (kThreads / 32) * (32 / lpr);
        return (unsigned)((n + rows_per_block - 1) / rows_per_block);
    };
    if (nv <= 2) spmm_kernel<2, 1><<<blocks(2), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 4) spmm_kernel<4, 1><<<blocks(4), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 8) spmm_kernel<8, 1><<<blocks(8), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 16) spmm_kernel<16, 1><<<blocks(16), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 32) spmm_kernel<32, 1><<<blocks(32), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 64) spmm_kernel<32, 2><<<blocks(32), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else if (nv <= 128) spmm_kernel<32, 4><<<blocks(32), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
    else spmm_kernel<32, 8><<<blocks(32), kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld);
}

}  // namespace cdfgnn
