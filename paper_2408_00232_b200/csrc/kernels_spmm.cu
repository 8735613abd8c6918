// Local CSR SpMM  Y = Â_i T  (eq. 1; Alg. 1 L3).
//
// Row-group-per-item CSR: LPR lanes own one work item, each lane VPL float4 column
// chunks, so every neighbour's feature row is one coalesced 16-byte-per-lane read
// (ld % 4 == 0, reading R24).  The group first loads LPR (col, val) pairs
// cooperatively (one coalesced load each) and broadcasts them with shuffles; UNR
// neighbours are in flight per lane before the FMAs.
//
// Work items (built once at init, SpmmItems): a row, or one segment of a split row.
// Segments are either fixed-length chunks (a power-law hub row is a chain of dependent
// L2 round trips whose latency can set a short launch's critical path) or column
// phases (all split rows' neighbours in column range k are visited before range k+1,
// so the slice of T being gathered is an L2-sized window).  Each segment writes its
// partial row to a scratch slot, and the group that completes a row's last segment
// (atomic counter) sums the partials in segment order, so results are bitwise
// run-to-run deterministic regardless of which warp finishes last.  Unsplit rows are
// visited longest-first (LPT).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int kThreads = 256;

#include "halo_common.cuh"

template <int LPR, int VPL, int UNR, int TAIL, bool FUSE>
__global__ void __launch_bounds__(kThreads) spmm_kernel(int64_t n_items, const int32_t* __restrict__ rowptr,
                                                        const int32_t* __restrict__ colidx,
                                                        const float* __restrict__ val,
                                                        const float* __restrict__ T,
                                                        float* __restrict__ Y, int64_t ld, int64_t width,
                                                        SpmmItems it, int stream,
                                                        const __grid_constant__ GatherFuse gf, int64_t relu_row0) {
    constexpr int GPW = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, gl = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const int64_t slot = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * GPW + g;
    if (slot >= n_items) return;
    int64_t row = slot;
    int chunk = -1;
    if (it.items) {
        const int2 w = __ldg(it.items + slot);
        row = w.x;
        chunk = w.y;
    }
    const int rb = __ldg(rowptr + row), re = __ldg(rowptr + row + 1);
    int beg = rb, end = re;
    int4 sp = make_int4(0, 0, 0, 0);
    if (chunk >= 0) {
        sp = __ldg(it.split + row);
        beg = __ldg(it.seg_beg + sp.z + chunk);
        end = __ldg(it.seg_beg + sp.z + chunk + 1);
    }
    float4 acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    bool colok[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) colok[v] = (gl + v * LPR) * 4 < width;
    for (int base = beg; base < end; base += LPR) {
        const int e = base + gl;
        const int c = e < end ? (stream ? __ldcs(colidx + e) : __ldg(colidx + e)) : 0;
        const float w = e < end ? (stream ? __ldcs(val + e) : __ldg(val + e)) : 0.f;
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
                    const float* tr = T + (int64_t)ck[u] * ld;
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
                    const float* tr = T + (int64_t)ck[u] * ld;
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
    if (chunk >= 0) {
        // split row: publish this chunk's partial; the last of the row's chunks to finish
        // sums all partials in chunk order (fixed order => deterministic bits)
        const int pbase = sp.x, nch = sp.y;
        float* pr = it.partial + (int64_t)(pbase + chunk) * width;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
            if (colok[v]) __stcg(reinterpret_cast<float4*>(pr + (gl + v * LPR) * 4), acc[v]);
        __threadfence();
        int last = 0;
        if (gl == 0) last = atomicAdd(it.counter + pbase, 1) == nch - 1;
        last = __shfl_sync(gmask, last, 0, LPR);
        if (!last) return;
        __threadfence();
        float4 sum[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) sum[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int cc = 0; cc < nch; ++cc) {
            const float* qr = it.partial + (int64_t)(pbase + cc) * width;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                if (!colok[v]) continue;
                const float4 q = cc == chunk ? acc[v] : __ldcg(reinterpret_cast<const float4*>(qr + (gl + v * LPR) * 4));
                if (cc == 0) {
                    sum[v] = q;
                } else {
                    sum[v].x = __fadd_rn(sum[v].x, q.x);
                    sum[v].y = __fadd_rn(sum[v].y, q.y);
                    sum[v].z = __fadd_rn(sum[v].z, q.z);
                    sum[v].w = __fadd_rn(sum[v].w, q.w);
                }
            }
        }
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = sum[v];
        if (gl == 0) it.counter[pbase] = 0;     // re-armed for the next launch
    }
    float* yr = Y + row * ld;
    const bool relu = row >= relu_row0;
#pragma unroll
    for (int v = 0; v < VPL; ++v)
        if (colok[v]) {
            float4* yp = reinterpret_cast<float4*>(yr + (gl + v * LPR) * 4);
            const float4 o = relu ? make_float4(fmaxf(acc[v].x, 0.f), fmaxf(acc[v].y, 0.f), fmaxf(acc[v].z, 0.f),
                                                fmaxf(acc[v].w, 0.f))
                                  : acc[v];
            if (stream) __stcs(yp, o); else *yp = o;
        }
    if constexpr (FUSE) {
        // a mirror row: the following synchronisation's gather (Alg. 2 L3-L9) from registers
        const int64_t mrow = row - gf.h.B;
        if (mrow >= 0 && mrow < gf.h.M) {
            const int q = find_seg(gf.h.moff, gf.h.p, mrow);
            uint8_t* slot = gf.dst.base[q] + (mrow - gf.h.moff[q]) * gf.a.stride;
            gather_row_fused<LPR, VPL>(gf.h, gf.a, slot, mrow, gmask, gl, acc);
        }
    }
}

__global__ void count_flags_kernel(const uint8_t* __restrict__ f, int64_t n, unsigned long long* out) {
    unsigned c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        c += f[i] ? 1u : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    __shared__ unsigned sc;
    if (threadIdx.x == 0) sc = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&sc, c);
    __syncthreads();
    if (threadIdx.x == 0 && sc) atomicAdd(out, (unsigned long long)sc);
}

template <int LPR, int VPL, int UNR>
void launch(int64_t n, const int32_t* rowptr, const int32_t* colidx, const float* val, const float* T, float* Y,
            int64_t ld, int64_t width, const SpmmItems& it, cudaStream_t s, int tail, int stream,
            const GatherFuse* gf, int64_t relu_row0) {
    const int64_t rows_per_block = (kThreads / 32) * (32 / LPR);
    const unsigned grid = (unsigned)((n + rows_per_block - 1) / rows_per_block);
    static const GatherFuse none{};
    const GatherFuse& g = gf ? *gf : none;
    if (gf) {
        if (tail)
            spmm_kernel<LPR, VPL, UNR, 1, true><<<grid, kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld, width, it, stream, g, relu_row0);
        else
            spmm_kernel<LPR, VPL, UNR, 0, true><<<grid, kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld, width, it, stream, g, relu_row0);
    } else {
        if (tail)
            spmm_kernel<LPR, VPL, UNR, 1, false><<<grid, kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld, width, it, stream, g, relu_row0);
        else
            spmm_kernel<LPR, VPL, UNR, 0, false><<<grid, kThreads, 0, s>>>(n, rowptr, colidx, val, T, Y, ld, width, it, stream, g, relu_row0);
    }
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);    // tuning knobs for tools/spmm_bench.py
    return e ? atoi(e) : dflt;
}

}  // namespace

// chunk length for the wide (ld > 64) and narrow row classes; 0 = no chunking.  Narrow rows:
// about the average work of one resident row group (148 SMs x 64 warps x 4 groups of the
// 8-lane shape), rounded to a power of two in [512, 4096] — C3 44-wide: 4096 at p=1
// (1.46 ms vs 2.08 unchunked), 1024 at p=4 (0.40 vs 0.47 ms at 2048; tools/spmm_bench.py)
int spmm_chunk(bool wide, int64_t nnz) {
    if (wide) return env_int("CDFGNN_SPMM_CHUNK_WIDE", 0);
    const double per_group = (double)std::max<int64_t>(nnz, 1) / (148.0 * 64.0 * 4.0);
    int c = 1 << (int)std::lround(std::log2(std::max(per_group, 1.0)));
    c = std::min(std::max(c, 512), 4096);
    return env_int("CDFGNN_SPMM_CHUNK", c);
}
int spmm_default_phases() { return env_int("CDFGNN_SPMM_PHASES", 1); }
int spmm_phase_min_degree() { return env_int("CDFGNN_SPMM_PHASE_MIN", 64); }

void launch_count_flags(const uint8_t* f, int64_t n, unsigned long long* out, cudaStream_t s) {
    if (n <= 0) return;
    count_flags_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4), 256, 0, s>>>(f, n, out);
}

void launch_spmm(const int32_t* rowptr, const int32_t* colidx, const float* val, int64_t n_items,
                 const SpmmItems& it, const float* T, float* Y, int64_t ld, cudaStream_t s, int64_t width,
                 const GatherFuse* gf, int64_t relu_row0) {
    if (n_items <= 0) return;
    if (width <= 0) width = ld;
    const int nv = (int)(width / 4);   // float4 per row (width % 4 == 0, width <= 1024)
    const int unr = env_int("CDFGNN_SPMM_UNR", 0);
    const int tail = env_int("CDFGNN_SPMM_TAIL", width > 64 ? 1 : 0);   // predicated tail for wide rows
    // narrow rows: stream the CSR arrays and the output past L2 (evict-first), keeping T's lines
    const int stream = env_int("CDFGNN_SPMM_STREAM", width <= 64 ? 1 : 0);
    if (nv <= 2) launch<2, 1, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    else if (nv <= 4) launch<4, 1, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    else if (nv <= 8) launch<8, 1, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    else if (nv <= 16) {
        // 8 lanes x 2 float4 per row, 8 neighbours in flight, predicated tail batch: at ld = 44
        // (C3's 41 classes) 1.75 -> 1.48 ms per launch vs 16 lanes x 1 (p = 1, tools/spmm_bench.py,
        // profiles/r1); 4x3 and 2x6 were slower (fewer neighbours in flight per lane)
        const int shape = env_int("CDFGNN_SPMM_SHAPE", 3);
        if (shape == 1 && nv <= 12) launch<4, 3, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (shape == 2 && nv <= 12) launch<2, 6, 2>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (shape == 3) launch<8, 2, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (shape == 4) launch<16, 1, 16>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (shape == 5) launch<4, 4, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (shape == 6) launch<8, 2, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, 1, stream, gf, relu_row0);
        else if (unr == 4) launch<16, 1, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else launch<16, 1, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    } else if (nv <= 32) {
        if (unr == 4) launch<32, 1, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else launch<32, 1, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    } else if (nv <= 64) {
        const int wshape = env_int("CDFGNN_SPMM_WSHAPE", 0);
        if (wshape == 1) launch<16, 4, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else if (wshape == 2) launch<16, 4, 2>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else if (wshape == 3) launch<32, 2, 6>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else if (unr == 2) launch<32, 2, 2>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else if (unr == 8) launch<32, 2, 8>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
        else launch<32, 2, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    } else if (nv <= 128) launch<32, 4, 4>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
    else launch<32, 8, 2>(n_items, rowptr, colidx, val, T, Y, ld, width, it, s, tail, stream, gf, relu_row0);
}

}  // namespace cdfgnn
