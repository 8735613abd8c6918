// Halo-exchange kernels: adaptive-cache test, quantise + pack, apply (sm_100a).
//
// One synchronisation (§3.2, Alg. 2, §5):
//   gather_pack   mirrors: d = z − s; send iff max|d| > RN(ε·max|s|) (Alg. 2 L4, reading R15);
//                 quantise d to uint8 codes per vertex (lo, hi header, §5), compact the
//                 senders per master peer (warp ballot + block prefix + one atomic range
//                 reservation per block), update the snapshot s += deq (reading R11)
//   map           received message -> row index tables
//   master        per boundary master: a += deq(Δ) in ascending source part (Alg. 2
//                 L11-L13, R13), own test + a += z − s (L14-L19), active flag, scatter
//                 delta q(a − b) staged once, b += deq (R12), Z row ← b
//   scatter_pack  per mirror peer: compact active masters, copy staged codes / a
//   mirror_apply  b += deq (or b ← a), Z row ← b
// Messages carry their halo-list position, every row receives at most one message per
// source and masters add sources in ascending order, so results do not depend on the
// order blocks reserve their ranges in a message buffer (bitwise-deterministic outputs).
// Every floating-point step of the cache test and the quantiser uses explicit
// round-to-nearest intrinsics (no FMA contraction) in the canonical order of
// reading R15, so masks and codes are bit-identical to oracle/cache.py's fp32 replay.
#include <cuda/atomic>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kScatterTile = 256;

#include "halo_common.cuh"

// ==================================================================================
// gather_pack: one tile = 8 warps x RPW x (32/LPR) mirror rows, all within one master
// peer.  Each warp tests RPW row groups back to back (loads of all of them in flight),
// the tile's senders are ranked in row order and the tile's offset inside its peer's
// message buffer comes from the decoupled look-back, so the buffer keeps halo-list order.
// ==================================================================================
template <int LPR, int VPL, int RPW>
__global__ void __launch_bounds__(kThreads, VPL <= 2 ? 2 : 1) gather_pack_kernel(HaloDev h, SyncArgs a) {
    constexpr int GPW = 32 / LPR;
    constexpr int TR = kWarps * GPW * RPW;
    __shared__ int s_wcnt[kWarps];
    __shared__ uint32_t s_excl;
    __shared__ int64_t s_moff[kMaxParts + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x <= h.p) s_moff[threadIdx.x] = h.moff[threadIdx.x];
    __syncthreads();
    const int tile = blockIdx.x;
    // segment (master peer) of this tile
    int seg = 0, tbase = 0;
    for (int j = 0; j < h.p; ++j) {
        int64_t len = s_moff[j + 1] - s_moff[j];
        int nt = (int)((len + TR - 1) / TR);
        if (tile < tbase + nt) { seg = j; break; }
        tbase += nt;
    }
    const int ltile = tile - tbase;
    const int64_t seg_len = s_moff[seg + 1] - s_moff[seg];
    const int g = lane / LPR, gl = lane % LPR;
    // all RPW rows' z and s chunks are loaded before any is used, so a warp keeps
    // RPW x VPL x 2 sixteen-byte loads in flight (they stay in registers for the pack below)
    float4 xs[RPW][VPL], ss[RPW][VPL];
    float lo[RPW], hi[RPW];
    bool flag[RPW];
    unsigned bal[RPW];
    int64_t ridx[RPW];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        ridx[r] = (int64_t)ltile * TR + (warp * RPW + r) * GPW + g;   // position in halo list
        const bool valid = ridx[r] < seg_len;
        const int64_t mrow = s_moff[seg] + (valid ? ridx[r] : 0);     // mirror index
        const float* xr = a.X + (h.B + mrow) * a.ld;
        const float* sr = a.nocache ? nullptr : a.c.s_mir + mrow * a.ld;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            xs[r][v] = make_float4(0.f, 0.f, 0.f, 0.f);
            ss[r][v] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (valid && c0 < a.ld) {
                xs[r][v] = __ldcs(reinterpret_cast<const float4*>(xr + c0));   // read once: evict-first
                if (sr) ss[r][v] = __ldcs(reinterpret_cast<const float4*>(sr + c0));
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const bool valid = ridx[r] < seg_len;
        float maxd = 0.f, maxs = 0.f;
        lo[r] = INFINITY;
        hi[r] = -INFINITY;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float dk = __fsub_rn(comp(xs[r][v], k), comp(ss[r][v], k));
                if (c0 + k < a.F) {
                    maxs = fmaxf(maxs, fabsf(comp(ss[r][v], k)));
                    lo[r] = fminf(lo[r], dk);
                    hi[r] = fmaxf(hi[r], dk);
                }
            }
        }
        maxs = gmax<LPR>(maxs);
        lo[r] = gmin<LPR>(lo[r]);
        hi[r] = gmax<LPR>(hi[r]);
        // ‖d‖∞ = max(|min d|, |max d|): exact, no separate reduction
        maxd = (ridx[r] < seg_len) ? fmaxf(fabsf(lo[r]), fabsf(hi[r])) : 0.f;
        flag[r] = valid && (a.nocache || maxd > __fmul_rn(a.eps, maxs));
        bal[r] = __ballot_sync(0xffffffffu, flag[r] && gl == 0);
        if (valid && gl == 0) h.gflag[s_moff[seg] + ridx[r]] = flag[r] ? 1 : 0;
    }
    int wcnt = 0;
#pragma unroll
    for (int r = 0; r < RPW; ++r) wcnt += __popc(bal[r]);
    if (lane == 0) s_wcnt[warp] = wcnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t cnt = 0;
        for (int w = 0; w < kWarps; ++w) cnt += s_wcnt[w];
        s_excl = cnt ? (uint32_t)atomicAdd(h.gsend->cnt[seg], (int32_t)cnt) : 0u;
        if (cnt) atomicAdd(&a.stats[0], (unsigned long long)cnt);
    }
    __syncthreads();
    int64_t m = (int64_t)s_excl;
    for (int w = 0; w < warp; ++w) m += s_wcnt[w];
    uint8_t* hdr = h.gsend->hdr[seg];
    uint8_t* pay = h.gsend->pay[seg];
    const int lead = g * LPR;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const int64_t mm = m + __popc(bal[r] & ((1u << lead) - 1u));
        m += __popc(bal[r]);
        if (!flag[r]) continue;
        const int64_t mrow = s_moff[seg] + ridx[r];
        float* sr = a.nocache ? nullptr : a.c.s_mir + mrow * a.ld;
        if (h.quant) {
            const QRow qr = qrow(lo[r], hi[r], h.quant);
            const float stp = stepq(lo[r], hi[r], h.quant);
            if (gl == 0) {
                uint32_t* hp = reinterpret_cast<uint32_t*>(hdr + mm * 12);
                hp[0] = (uint32_t)ridx[r];
                hp[1] = __float_as_uint(lo[r]);
                hp[2] = __float_as_uint(hi[r]);
            }
            uint8_t* codes = pay + mm * a.rowb;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t q[4];
                float4 snew = make_float4(0.f, 0.f, 0.f, 0.f);
                const float4 s4 = ss[r][v];
                float dd[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) dd[k] = __fsub_rn(comp(xs[r][v], k), comp(s4, k));
                qx4(dd, qr, q);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float sk = (c0 + k < a.F) ? __fadd_rn(comp(s4, k), dqv(q[k], lo[r], stp)) : 0.f;
                    setc(snew, k, sk);
                }
                store_codes4(codes, c0, a.F, q, h.quant);
                if (sr) __stcs(reinterpret_cast<float4*>(sr + c0), snew);   // reading R11: s ← s + deq(q(Δ))
            }
        } else {
            if (gl == 0) reinterpret_cast<uint32_t*>(hdr)[mm] = (uint32_t)ridx[r];
            float* prow = reinterpret_cast<float*>(pay) + mm * a.ld;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.ld) continue;
                float4 dv;
#pragma unroll
                for (int k = 0; k < 4; ++k) setc(dv, k, __fsub_rn(comp(xs[r][v], k), comp(ss[r][v], k)));
                st4(prow + c0, dv);
                if (sr) st4(sr + c0, xs[r][v]);   // Alg. 2 L6: s ← z
            }
        }
    }
    if (h.remote) __threadfence_system();   // pushed to a peer GPU: visible before the barrier
}

// ==================================================================================
// map: message -> row tables.  mirror_side = 0: idxmap[src*B + master row] = m;
// mirror_side = 1: mmap[mirror index] = m.
// ==================================================================================
__global__ void map_kernel(HaloDev h, const __grid_constant__ RegionTab t, int mirror_side) {
    const int q = blockIdx.y;
    if (q == h.me) return;
    const int32_t cnt = *t.cnt[q];
    const uint8_t* hdr = t.hdr[q];
    const int64_t len = mirror_side ? (h.moff[q + 1] - h.moff[q]) : (h.hoff[q + 1] - h.hoff[q]);
    if (cnt > len) { if (threadIdx.x == 0 && blockIdx.x == 0) atomicExch(h.err, 1); return; }
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < cnt;
         m += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t pos = *reinterpret_cast<const uint32_t*>(hdr + m * h.hdr_bytes);
        if (pos >= len) { atomicExch(h.err, 2); continue; }
        if (mirror_side) h.mmap[h.moff[q] + pos] = (int32_t)m;
        else h.idxmap[(int64_t)q * h.B + h.halo_local[h.hoff[q] + pos]] = (int32_t)m;
    }
}

// ==================================================================================
// master: one row group per boundary master row
// ==================================================================================
// Alg. 2 L10-L22 for one master row r whose aggregate, own value, snapshot and scatter base
// are already in registers (acc, x, s4v, b); shared by the two master kernels below.
template <int LPR, int VPL>
__device__ __forceinline__ void master_row(const HaloDev& h, const SyncArgs& a, const RegionTab& rt, int lane,
                                           int g, int gl, int64_t r, bool valid, float* xr, float* smr,
                                           float* bmr, float4 (&acc)[VPL], float4 (&x)[VPL],
                                           float4 (&s4v)[VPL], float4 (&b)[VPL]) {
    const int nsrc = a.no_msgs ? 0 : h.p;
    // lane gl of the row group holds source gl's message index (p <= LPR), and its header
    int32_t mine = -1;
    float mlo = 0.f, mhi = 0.f;
    if (nsrc <= LPR) {
        if (valid && gl < nsrc && gl != h.me) {
            mine = h.idxmap[(int64_t)gl * h.B + r];
            if (mine >= 0 && h.quant) {
                const uint32_t* hp = reinterpret_cast<const uint32_t*>(rt.hdr[gl] + (int64_t)mine * 12);
                mlo = __uint_as_float(__ldg(hp + 1));
                mhi = __uint_as_float(__ldg(hp + 2));
            }
        }
    }
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const unsigned have = (__ballot_sync(0xffffffffu, mine >= 0) & gmask) >> (g * LPR);
    bool any_msg = false;
    // Alg. 2 L11-L13: received Δ in ascending source part (R13)
    for (int s = 0; s < nsrc; ++s) {
        if (s == h.me) continue;
        int32_t m;
        float lo = 0.f, hi = 0.f;
        if (nsrc <= LPR) {
            if (!((have >> s) & 1u)) continue;
            m = __shfl_sync(gmask, mine, g * LPR + s);
            lo = __shfl_sync(gmask, mlo, g * LPR + s);
            hi = __shfl_sync(gmask, mhi, g * LPR + s);
        } else {
            m = valid ? h.idxmap[(int64_t)s * h.B + r] : -1;
            if (m < 0) continue;
            if (h.quant) {
                const uint32_t* hp = reinterpret_cast<const uint32_t*>(rt.hdr[s] + (int64_t)m * 12);
                lo = __uint_as_float(hp[1]);
                hi = __uint_as_float(hp[2]);
            }
        }
        any_msg = true;
        const uint8_t* pay = rt.pay[s];
        if (h.quant) {
            const float stp = stepq(lo, hi, h.quant);
            const uint8_t* codes = pay + (int64_t)m * a.rowb;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t q[4];
                load_codes4(codes, c0, h.quant, q);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F)
                        setc(acc[v], k, __fadd_rn(comp(acc[v], k), dqv(q[k], lo, stp)));
            }
        } else {
            const float* prow = reinterpret_cast<const float*>(pay) + (int64_t)m * a.ld;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.ld) continue;
                const float4 pv = ld4(prow + c0);
#pragma unroll
                for (int k = 0; k < 4; ++k) setc(acc[v], k, __fadd_rn(comp(acc[v], k), comp(pv, k)));
            }
        }
    }
    // Alg. 2 L14-L19: the master's own replica, unquantised
    float4 dd[VPL];
    float maxd = 0.f, maxs = 0.f;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dk = __fsub_rn(comp(x[v], k), comp(s4v[v], k));
            setc(dd[v], k, dk);
            if (c0 + k < a.F) {
                maxd = fmaxf(maxd, fabsf(dk));
                maxs = fmaxf(maxs, fabsf(comp(s4v[v], k)));
            }
        }
    }
    maxd = gmax<LPR>(maxd);
    maxs = gmax<LPR>(maxs);
    const bool fired = valid && (a.nocache || maxd > __fmul_rn(a.eps, maxs));
    if (fired) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 >= a.ld) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) setc(acc[v], k, __fadd_rn(comp(acc[v], k), comp(dd[v], k)));
            if (smr) st4(smr + c0, x[v]);
        }
    }
    const bool act = valid && (fired || any_msg);
    // aggregate store (the no-cache fp32 scatter reads it from stage_a)
    float* adst = a.nocache ? h.stage_a + r * a.ld : a.c.a + r * a.ld;
    if (act) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 < a.ld) st4(adst + c0, acc[v]);
        }
    }
    // Alg. 2 L20-L22 / R12: scatter delta staged once; every replica applies the same codes
    // scatter delta and its range, reduced by every lane of the warp (shuffles stay converged)
    float4 del[VPL];
    float lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dk = __fsub_rn(comp(acc[v], k), comp(b[v], k));
            setc(del[v], k, dk);
            if (c0 + k < a.F) { lo = fminf(lo, dk); hi = fmaxf(hi, dk); }
        }
    }
    if (h.quant) {
        lo = gmin<LPR>(lo);
        hi = gmax<LPR>(hi);
    }
    if (act) {
        if (h.quant) {
            const QRow qr = qrow(lo, hi, h.quant);
            const float stp = stepq(lo, hi, h.quant);
            uint8_t* codes = h.stage_codes + r * a.rowb;
            if (gl == 0) { h.stage_lohi[2 * r] = lo; h.stage_lohi[2 * r + 1] = hi; }
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t q[4];
                const float dd[4] = {del[v].x, del[v].y, del[v].z, del[v].w};
                qx4(dd, qr, q);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F) setc(b[v], k, __fadd_rn(comp(b[v], k), dqv(q[k], lo, stp)));
                store_codes4(codes, c0, a.F, q, h.quant);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPL; ++v) b[v] = acc[v];
        }
        if (bmr) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) st4(bmr + c0, b[v]);
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 < a.ld) st4(xr + c0, b[v]);      // Z row from the cached value
        }
        if (gl == 0) {
            h.fired[r] = fired ? 1 : 0;
            h.active[r] = act ? 1 : 0;
        }
    }
    // counters
    const unsigned bf = __ballot_sync(0xffffffffu, fired && gl == 0);
    const unsigned ba = __ballot_sync(0xffffffffu, act && gl == 0);
    if (lane == 0) {
        if (bf) atomicAdd(&a.stats[1], (unsigned long long)__popc(bf));
        if (ba) atomicAdd(&a.stats[2], (unsigned long long)__popc(ba));
    }
}

template <int LPR, int VPL>
__global__ void __launch_bounds__(kThreads, VPL <= 2 ? 4 : 1) master_kernel(HaloDev h, SyncArgs a,
                                                                             const __grid_constant__ RegionTab rt) {
    constexpr int GPW = 32 / LPR;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, gl = lane % LPR;
    const int64_t row = ((int64_t)blockIdx.x * kWarps + warp) * GPW + g;
    const bool valid = row < h.B;
    const int64_t r = valid ? row : 0;
    // Independent loads first (aggregate, own value, snapshot, scatter base, and the message
    // index of every source), so a row costs ~3 dependent memory round trips, not ~3 per source.
    float* xr = a.X + r * a.ld;
    float* smr = a.nocache ? nullptr : a.c.s_mas + r * a.ld;
    float* bmr = a.nocache ? nullptr : a.c.b_mas + r * a.ld;
    const float* aold = a.nocache ? nullptr : a.c.a + r * a.ld;
    float4 acc[VPL], x[VPL], s4v[VPL], b[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        const bool in = valid && c0 < a.ld;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        acc[v] = (aold && in) ? ld4(aold + c0) : z4;
        x[v] = in ? ld4(xr + c0) : z4;
        s4v[v] = (smr && in) ? ld4(smr + c0) : z4;
        b[v] = (bmr && in) ? ld4(bmr + c0) : z4;
    }
    master_row<LPR, VPL>(h, a, rt, lane, g, gl, r, valid, xr, smr, bmr, acc, x, s4v, b);
}

// ==================================================================================
// scatter_pack: one tile = 256 halo-list entries of one mirror peer
// ==================================================================================
__global__ void __launch_bounds__(kThreads) scatter_pack_kernel(HaloDev h, SyncArgs a) {
    __shared__ int s_wcnt[kWarps];
    __shared__ uint32_t s_excl;
    __shared__ int32_t s_row[kScatterTile];
    __shared__ int32_t s_pos[kScatterTile];
    __shared__ int64_t s_hoff[kMaxParts + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x <= h.p) s_hoff[threadIdx.x] = h.hoff[threadIdx.x];
    __syncthreads();
    const int tile = blockIdx.x;
    int seg = 0, tbase = 0;
    for (int j = 0; j < h.p; ++j) {
        int64_t len = s_hoff[j + 1] - s_hoff[j];
        int nt = (int)((len + kScatterTile - 1) / kScatterTile);
        if (tile < tbase + nt) { seg = j; break; }
        tbase += nt;
    }
    const int ltile = tile - tbase;
    const int64_t seg_len = s_hoff[seg + 1] - s_hoff[seg];
    const int64_t pos = (int64_t)ltile * kScatterTile + threadIdx.x;
    const bool valid = pos < seg_len;
    const int32_t row = valid ? h.halo_local[s_hoff[seg] + pos] : 0;
    const bool flag = valid && h.active[row];
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) s_wcnt[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t cnt = 0;
        for (int w = 0; w < kWarps; ++w) cnt += s_wcnt[w];
        s_excl = cnt ? (uint32_t)atomicAdd(h.ssend->cnt[seg], (int32_t)cnt) : 0u;
        if (cnt) atomicAdd(&a.stats[3], (unsigned long long)cnt);
    }
    int woff = 0;
    for (int w = 0; w < warp; ++w) woff += s_wcnt[w];
    const int lrank = woff + __popc(bal & ((1u << lane) - 1u));
    if (flag) { s_row[lrank] = row; s_pos[lrank] = (int32_t)pos; }
    __syncthreads();
    int total = 0;
    for (int w = 0; w < kWarps; ++w) total += s_wcnt[w];
    uint8_t* hdr = h.ssend->hdr[seg];
    uint8_t* pay = h.ssend->pay[seg];
    const int64_t m0 = (int64_t)s_excl;       // this block's contiguous range of messages
    // headers: one thread per message
    for (int k = threadIdx.x; k < total; k += kThreads) {
        const int32_t rr = s_row[k];
        if (h.quant) {
            uint32_t* hp = reinterpret_cast<uint32_t*>(hdr + (m0 + k) * 12);
            hp[0] = (uint32_t)s_pos[k];
            hp[1] = __float_as_uint(h.stage_lohi[2 * rr]);
            hp[2] = __float_as_uint(h.stage_lohi[2 * rr + 1]);
        } else {
            reinterpret_cast<uint32_t*>(hdr)[m0 + k] = (uint32_t)s_pos[k];
        }
    }
    // payloads: the block's destination range is contiguous, so the copy is flattened over
    // (message, word) with coalesced stores
    // (4 independent loads in flight per thread before the stores: the copy is latency-bound)
    if (h.quant) {
        const int wpr = (int)(a.rowb >> 2);      // code rows are rowb bytes (multiple of 4)
        uint32_t* dst = reinterpret_cast<uint32_t*>(pay + m0 * a.rowb);
        const int nw = total * wpr;
        for (int i0 = threadIdx.x; i0 < nw; i0 += 4 * kThreads) {
            uint32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads;
                const int k = i / wpr, o = i - k * wpr;
                w[u] = i < nw ? __ldg(reinterpret_cast<const uint32_t*>(h.stage_codes + (int64_t)s_row[min(k, total - 1)] * a.rowb) + o) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * kThreads < nw) dst[i0 + u * kThreads] = w[u];
        }
    } else {
        const float* srcb = a.nocache ? h.stage_a : a.c.a;
        const int vpr = (int)(a.ld >> 2);
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(pay) + m0 * a.ld);
        const int nv = total * vpr;
        for (int i0 = threadIdx.x; i0 < nv; i0 += 4 * kThreads) {
            float4 w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * kThreads;
                const int k = i / vpr, o = i - k * vpr;
                w[u] = i < nv ? reinterpret_cast<const float4*>(srcb + (int64_t)s_row[min(k, total - 1)] * a.ld)[o]
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * kThreads < nv) dst[i0 + u * kThreads] = w[u];
        }
    }
    if (h.remote) __threadfence_system();
}

// ==================================================================================
// mirror_apply: one row group per mirror row
// ==================================================================================
template <int LPR, int VPL>
__global__ void __launch_bounds__(kThreads) mirror_apply_kernel(HaloDev h, SyncArgs a,
                                                                const __grid_constant__ RegionTab rt) {
    constexpr int GPW = 32 / LPR;
    __shared__ int64_t s_moff[kMaxParts + 1];
    if (threadIdx.x <= h.p) s_moff[threadIdx.x] = h.moff[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, gl = lane % LPR;
    const int64_t row = ((int64_t)blockIdx.x * kWarps + warp) * GPW + g;
    if (row >= h.M) return;
    const int q = find_seg(s_moff, h.p, row);
    const int32_t m = h.mmap[row];
    float* bmr = a.nocache ? nullptr : a.c.b_mir + row * a.ld;
    float4 b[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        b[v] = (bmr && c0 < a.ld) ? ld4(bmr + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (m >= 0) {
        const uint8_t* hdr = rt.hdr[q];
        const uint8_t* pay = rt.pay[q];
        if (h.quant) {
            const uint32_t* hp = reinterpret_cast<const uint32_t*>(hdr + (int64_t)m * 12);
            const float lo = __uint_as_float(__ldg(hp + 1)), hi = __uint_as_float(__ldg(hp + 2));
            const float stp = stepq(lo, hi, h.quant);
            const uint8_t* codes = pay + (int64_t)m * a.rowb;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t q[4];
                load_codes4(codes, c0, h.quant, q);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F)
                        setc(b[v], k, __fadd_rn(comp(b[v], k), dqv(q[k], lo, stp)));
            }
        } else {
            const float* prow = reinterpret_cast<const float*>(pay) + (int64_t)m * a.ld;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) b[v] = ld4(prow + c0);
            }
        }
        if (bmr) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) st4(bmr + c0, b[v]);
            }
        }
    }
    float* xr = a.X + (h.B + row) * a.ld;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        if (c0 < a.ld) st4(xr + c0, b[v]);
    }
}

// ==================================================================================
// put: bulk copy of compacted messages into peer GPUs (16-byte stores over NVLink)
// ==================================================================================
__device__ __forceinline__ void copy_bytes(uint8_t* dst, const uint8_t* src, int64_t n, int64_t tid,
                                           int64_t nthreads) {
    // both 256-byte aligned region starts; n arbitrary
    const int64_t n16 = n / 16;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    // 4 independent 16-byte loads in flight per thread before the (NVLink) stores
    for (int64_t i0 = tid; i0 < n16; i0 += 4 * nthreads) {
        int4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * nthreads;
            v[u] = i < n16 ? __ldcs(s4 + i) : make_int4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * nthreads;
            if (i < n16) d4[i] = v[u];
        }
    }
    for (int64_t i = n16 * 16 + tid; i < n; i += nthreads) dst[i] = src[i];
}

__global__ void put_kernel(const PutTab* __restrict__ tab, int64_t hdr_bytes, int64_t row_bytes) {
    const int q = blockIdx.y;
    uint8_t* dh = tab->dst_hdr[q];
    if (!dh) return;
    const int64_t cnt = *tab->src_cnt[q];
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    copy_bytes(dh, tab->src_hdr[q], cnt * hdr_bytes, tid, nth);
    copy_bytes(tab->dst_pay[q], tab->src_pay[q], cnt * row_bytes, tid, nth);
    if (tid == 0) *tab->dst_cnt[q] = (int32_t)cnt;
    __threadfence_system();
}

// ==================================================================================
// NVLink barrier (push transport): one thread per peer
// ==================================================================================
__global__ void nvl_barrier_kernel(const __grid_constant__ BarTab t, uint64_t seq, int32_t* err) {
    const int j = threadIdx.x;
    if (j >= t.p || j == t.me) return;
    // the put kernel's peer stores precede this kernel in stream order; fence, then publish
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(t.peer_slot[j]), "l"(seq) : "memory");
    const long long t0 = clock64();
    for (;;) {
        uint64_t v;
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(t.my_slots + j) : "memory");
        if (v >= seq) break;
        if (clock64() - t0 > 20000000000LL) {   // ~10 s at 2 GHz: report, do not hang
            atomicExch(err, 5);
            break;
        }
    }
    __threadfence_system();   // acquire: the peer's stores before its release are visible
}

// ==================================================================================
// Slot-addressed exchange (co-resident parts and the NVLink push transport; kernels.h
// SlotTab).  The message of the vertex at halo-list position pos travels in slot pos of
// the (source -> destination) region: a 16-byte header {u32 stamp, f32 lo, f32 hi, 0}
// followed by the code row (or the fp32 row).  stamp = the phase's sequence number, so the
// receiver tells this phase's messages from stale slots without counts, prefix sums, range
// reservations or index maps, and the sender stores straight into the receiver's region
// (through the CUDA-IPC mapping when it lives on a peer GPU: no local staging, no copy pass).
// ==================================================================================
// gather (Alg. 2 L3-L9): RPW row groups per warp pass, one mirror row per group
template <int LPR, int VPL, int RPW, int QB>
__global__ void __launch_bounds__(kThreads, VPL <= 2 ? 2 : 1)
gather_slot_kernel(HaloDev h, SyncArgs a, const __grid_constant__ SlotTab dst) {
    constexpr int GPW = 32 / LPR;
    __shared__ int64_t s_moff[kMaxParts + 1];
    __shared__ unsigned s_cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x <= h.p) s_moff[threadIdx.x] = h.moff[threadIdx.x];
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const int g = lane / LPR, gl = lane % LPR;
    unsigned sent = 0;
    // grid-stride over passes of RPW row groups per warp (one counter atomic per block)
    for (int64_t row0 = ((int64_t)blockIdx.x * kWarps + warp) * RPW * GPW; row0 < h.M;
         row0 += (int64_t)gridDim.x * kWarps * RPW * GPW) {
        float4 xs[RPW][VPL], ss[RPW][VPL];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int64_t row = row0 + r * GPW + g;
            const bool valid = row < h.M;
            const float* xr = a.X + (h.B + (valid ? row : 0)) * a.ld;
            const float* sr = a.nocache ? nullptr : a.c.s_mir + (valid ? row : 0) * a.ld;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                xs[r][v] = make_float4(0.f, 0.f, 0.f, 0.f);
                ss[r][v] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid && c0 < a.ld) {
                    xs[r][v] = __ldcs(reinterpret_cast<const float4*>(xr + c0));   // read once
                    if (sr) ss[r][v] = __ldcs(reinterpret_cast<const float4*>(sr + c0));
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
            const int64_t row = row0 + r * GPW + g;
            const bool valid = row < h.M;
            float maxs = 0.f, lo = INFINITY, hi = -INFINITY;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float dk = __fsub_rn(comp(xs[r][v], k), comp(ss[r][v], k));
                    if (c0 + k < a.F) {
                        maxs = fmaxf(maxs, fabsf(comp(ss[r][v], k)));
                        lo = fminf(lo, dk);
                        hi = fmaxf(hi, dk);
                    }
                }
            }
            maxs = gmax<LPR>(maxs);
            lo = gmin<LPR>(lo);
            hi = gmax<LPR>(hi);
            // ‖d‖∞ = max(|min d|, |max d|): exact; the test of Alg. 2 L4 (reading R15)
            const float maxd = valid ? fmaxf(fabsf(lo), fabsf(hi)) : 0.f;
            const bool flag = valid && (a.nocache || maxd > __fmul_rn(a.eps, maxs));
            sent += __popc(__ballot_sync(0xffffffffu, flag && gl == 0));
            if (valid && gl == 0) h.gflag[row] = flag ? 1 : 0;
            if (!flag) continue;
            const int q = find_seg(s_moff, h.p, row);
            uint8_t* slot = dst.base[q] + (row - s_moff[q]) * a.stride;
            float* sr = a.nocache ? nullptr : a.c.s_mir + row * a.ld;
            if constexpr (QB != 0) {
                const QRow qr = qrow(lo, hi, QB);
                const float stp = stepq(lo, hi, QB);
                if (gl == 0) st_hdr(slot, a.gstamp, lo, hi);
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    const int c0 = (gl + v * LPR) * 4;
                    if (c0 >= a.F) continue;
                    uint32_t qc[4];
                    float dd[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) dd[k] = __fsub_rn(comp(xs[r][v], k), comp(ss[r][v], k));
                    qx4(dd, qr, qc);
                    store_codes4(slot + 16, c0, a.F, qc, QB);
                    if (sr) {
                        float4 snew;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            setc(snew, k, (c0 + k < a.F) ? __fadd_rn(comp(ss[r][v], k), dqv(qc[k], lo, stp)) : 0.f);
                        __stcs(reinterpret_cast<float4*>(sr + c0), snew);   // reading R11: s ← s + deq(q(Δ))
                    }
                }
            } else {
                if (gl == 0) st_hdr(slot, a.gstamp, 0.f, 0.f);
                float* prow = reinterpret_cast<float*>(slot + 16);
#pragma unroll
                for (int v = 0; v < VPL; ++v) {
                    const int c0 = (gl + v * LPR) * 4;
                    if (c0 >= a.ld) continue;
                    float4 dv;
#pragma unroll
                    for (int k = 0; k < 4; ++k) setc(dv, k, __fsub_rn(comp(xs[r][v], k), comp(ss[r][v], k)));
                    st4(prow + c0, dv);
                    if (sr) st4(sr + c0, xs[r][v]);   // Alg. 2 L6: s ← z
                }
            }
        }
    }
    if (lane == 0 && sent) atomicAdd(&s_cnt, sent);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(&a.stats[0], (unsigned long long)s_cnt);
    if (h.remote) __threadfence_system();   // stored into peer GPUs: visible before the barrier
}

// master apply + scatter (Alg. 2 L10-L22): one row group per boundary master row.  Lane s of
// the group holds the row's slot in the halo list shared with part s (static, -1: no replica
// on s) — the slot its gather message arrives in and the slot its scatter message goes to.
template <int LPR, int VPL, int QB>
__device__ __forceinline__ void master_slot_row(const HaloDev& h, const SyncArgs& a, const SlotTab& src,
                                                const SlotTab& sdst, int64_t row, int g, int gl,
                                                unsigned& n_fired, unsigned& n_active, unsigned& n_msgs) {
    const bool valid = row < h.B;
    const int64_t r = valid ? row : 0;
    const int p = h.p;
    const bool lanes_hold = p <= LPR;
    // independent loads first: the row's slots, aggregate, own value, snapshot, scatter base
    int32_t hp = -1;
    if (lanes_hold && valid && gl < p && gl != h.me) hp = __ldg(h.hpos + r * p + gl);
    float* xr = a.X + r * a.ld;
    float* smr = a.nocache ? nullptr : a.c.s_mas + r * a.ld;
    float* bmr = a.nocache ? nullptr : a.c.b_mas + r * a.ld;
    float* ar = a.nocache ? nullptr : a.c.a + r * a.ld;
    float4 acc[VPL], x[VPL], s4v[VPL], b[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        const bool in = valid && c0 < a.ld;
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        acc[v] = (ar && in) ? ld4(ar + c0) : z4;
        x[v] = in ? ld4(xr + c0) : z4;
        s4v[v] = (smr && in) ? ld4(smr + c0) : z4;
        b[v] = (bmr && in) ? ld4(bmr + c0) : z4;
    }
    uint4 hd = make_uint4(0u, 0u, 0u, 0u);
    if (hp >= 0 && !a.no_msgs) hd = ld_hdr(src.base[gl] + (int64_t)hp * a.stride);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    const unsigned have = (__ballot_sync(0xffffffffu, hp >= 0 && !a.no_msgs && hd.x == a.gstamp) & gmask) >> (g * LPR);
    const unsigned peers = (__ballot_sync(0xffffffffu, hp >= 0) & gmask) >> (g * LPR);
    bool any_msg = false;
    // The code words of the first NSP sources' slots are loaded together with their headers
    // (the slot address only needs hpos): one dependent round trip less per message; a stale
    // slot's words are loaded and ignored.
    constexpr int NSP = 4, NW = QB == 16 ? 2 : 1;
    uint32_t pre[NSP][VPL][NW];
    if constexpr (QB != 0) {
#pragma unroll
        for (int s = 0; s < NSP; ++s) {
            const int32_t hps = __shfl_sync(gmask, hp, g * LPR + (s < LPR ? s : 0));
            const bool live = lanes_hold && s < p && s != h.me && hps >= 0 && !a.no_msgs;
            const uint8_t* pay = live ? src.base[s] + (int64_t)hps * a.stride + 16 : nullptr;
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                uint32_t w[2] = {0u, 0u};
                if (live && c0 < a.F) fetch_codes4(pay, c0, QB, w);
#pragma unroll
                for (int t = 0; t < NW; ++t) pre[s][v][t] = w[t];
            }
        }
    }
    // Alg. 2 L11-L13: received Δ in ascending source part (R13) — first the prefetched sources
#pragma unroll
    for (int s = 0; s < NSP; ++s) {
        if (!lanes_hold || s >= p || s == h.me || !((have >> s) & 1u)) continue;
        const float lo = __uint_as_float(__shfl_sync(gmask, hd.y, g * LPR + s));
        const float hi = __uint_as_float(__shfl_sync(gmask, hd.z, g * LPR + s));
        any_msg = true;
        if constexpr (QB != 0) {
            const float stp = stepq(lo, hi, QB);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t w[2] = {pre[s][v][0], NW == 2 ? pre[s][v][NW - 1] : 0u};
                uint32_t qc[4];
                unpack_codes4(w, QB, qc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F) setc(acc[v], k, __fadd_rn(comp(acc[v], k), dqv(qc[k], lo, stp)));
            }
        } else {
            const int32_t hps = __shfl_sync(gmask, hp, g * LPR + s);
            const float* prow = reinterpret_cast<const float*>(src.base[s] + (int64_t)hps * a.stride + 16);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.ld) continue;
                const float4 pv = ld4(prow + c0);
#pragma unroll
                for (int k = 0; k < 4; ++k) setc(acc[v], k, __fadd_rn(comp(acc[v], k), comp(pv, k)));
            }
        }
    }
    // ... then the rest (sources >= NSP, or every source when the group's lanes cannot hold p)
    for (int s = lanes_hold ? NSP : 0; s < p; ++s) {
        if (s == h.me) continue;
        int32_t hps;
        float lo = 0.f, hi = 0.f;
        if (lanes_hold) {
            if (!((have >> s) & 1u)) continue;
            hps = __shfl_sync(gmask, hp, g * LPR + s);
            lo = __uint_as_float(__shfl_sync(gmask, hd.y, g * LPR + s));
            hi = __uint_as_float(__shfl_sync(gmask, hd.z, g * LPR + s));
        } else {
            hps = (valid && !a.no_msgs) ? __ldg(h.hpos + r * p + s) : -1;
            if (hps < 0) continue;
            const uint4 hs = ld_hdr(src.base[s] + (int64_t)hps * a.stride);
            if (hs.x != a.gstamp) continue;
            lo = __uint_as_float(hs.y);
            hi = __uint_as_float(hs.z);
        }
        any_msg = true;
        const uint8_t* pay = src.base[s] + (int64_t)hps * a.stride + 16;
        if constexpr (QB != 0) {
            const float stp = stepq(lo, hi, QB);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t qc[4];
                load_codes4(pay, c0, QB, qc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F) setc(acc[v], k, __fadd_rn(comp(acc[v], k), dqv(qc[k], lo, stp)));
            }
        } else {
            const float* prow = reinterpret_cast<const float*>(pay);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.ld) continue;
                const float4 pv = ld4(prow + c0);
#pragma unroll
                for (int k = 0; k < 4; ++k) setc(acc[v], k, __fadd_rn(comp(acc[v], k), comp(pv, k)));
            }
        }
    }
    // Alg. 2 L14-L19: the master's own replica, unquantised
    float4 dd[VPL];
    float maxd = 0.f, maxs = 0.f;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dk = __fsub_rn(comp(x[v], k), comp(s4v[v], k));
            setc(dd[v], k, dk);
            if (c0 + k < a.F) {
                maxd = fmaxf(maxd, fabsf(dk));
                maxs = fmaxf(maxs, fabsf(comp(s4v[v], k)));
            }
        }
    }
    maxd = gmax<LPR>(maxd);
    maxs = gmax<LPR>(maxs);
    const bool fired = valid && (a.nocache || maxd > __fmul_rn(a.eps, maxs));
    if (fired) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 >= a.ld) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) setc(acc[v], k, __fadd_rn(comp(acc[v], k), comp(dd[v], k)));
            if (smr) st4(smr + c0, x[v]);
        }
    }
    const bool act = valid && (fired || any_msg);
    if (act && ar) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 < a.ld) st4(ar + c0, acc[v]);
        }
    }
    // Alg. 2 L20-L22 / R12: the scatter delta a − b quantised once; every replica applies the
    // same codes (range reduced by every lane of the warp: shuffles stay converged)
    float lo = INFINITY, hi = -INFINITY;
    float4 del[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dk = __fsub_rn(comp(acc[v], k), comp(b[v], k));
            setc(del[v], k, dk);
            if (c0 + k < a.F) { lo = fminf(lo, dk); hi = fmaxf(hi, dk); }
        }
    }
    if constexpr (QB != 0) {
        lo = gmin<LPR>(lo);
        hi = gmax<LPR>(hi);
    }
    int nmsg = 0;
    if (act) {
        uint32_t pk[VPL][2];
        if constexpr (QB != 0) {
            const QRow qr = qrow(lo, hi, QB);
            const float stp = stepq(lo, hi, QB);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                pk[v][0] = pk[v][1] = 0u;
                if (c0 >= a.F) continue;
                uint32_t qc[4];
                const float d4[4] = {del[v].x, del[v].y, del[v].z, del[v].w};
                qx4(d4, qr, qc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F) setc(b[v], k, __fadd_rn(comp(b[v], k), dqv(qc[k], lo, stp)));
                pack_codes4(qc, c0, a.F, QB, pk[v]);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VPL; ++v) b[v] = acc[v];
        }
        if (bmr) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) st4(bmr + c0, b[v]);
            }
        }
        // one message per mirror peer, stored straight into its slot
        if (!a.no_scatter) {
            for (int s = 0; s < p; ++s) {
                if (s == h.me) continue;
                int32_t hps;
                if (lanes_hold) {
                    if (!((peers >> s) & 1u)) continue;
                    hps = __shfl_sync(gmask, hp, g * LPR + s);
                } else {
                    hps = __ldg(h.hpos + r * p + s);
                    if (hps < 0) continue;
                }
                uint8_t* slot = sdst.base[s] + (int64_t)hps * a.stride;
                ++nmsg;
                if (gl == 0) st_hdr(slot, a.sstamp, lo, hi);
                if constexpr (QB != 0) {
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        const int c0 = (gl + v * LPR) * 4;
                        if (c0 < a.F) put_codes4(slot + 16, c0, QB, pk[v]);
                    }
                } else {
                    float* prow = reinterpret_cast<float*>(slot + 16);
#pragma unroll
                    for (int v = 0; v < VPL; ++v) {
                        const int c0 = (gl + v * LPR) * 4;
                        if (c0 < a.ld) st4(prow + c0, b[v]);
                    }
                }
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 < a.ld) st4(xr + c0, a.relu ? relu4(b[v]) : b[v]);   // Z row from the cached value
        }
        if (gl == 0) {
            h.fired[r] = fired ? 1 : 0;
            h.active[r] = act ? 1 : 0;
        }
    }
    if (gl == 0) {
        n_fired += fired ? 1u : 0u;
        n_active += act ? 1u : 0u;
        n_msgs += (unsigned)nmsg;
    }
}

// Grid-stride over warps of row groups (every lane of a warp runs the same iterations, so the
// full-warp shuffles stay converged); counters are reduced per block, one atomic each.
template <int LPR, int VPL, int QB>
__global__ void __launch_bounds__(kThreads, VPL <= 2 ? 3 : 1)
master_slot_kernel(HaloDev h, SyncArgs a, const __grid_constant__ SlotTab src, const __grid_constant__ SlotTab sdst) {
    constexpr int GPW = 32 / LPR;
    __shared__ unsigned s_cnt[3];
    if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, gl = lane % LPR;
    unsigned nf = 0, na = 0, nm = 0;
    const int64_t wstride = (int64_t)gridDim.x * kWarps * GPW;
    for (int64_t base = ((int64_t)blockIdx.x * kWarps + warp) * GPW; base < h.B; base += wstride)
        master_slot_row<LPR, VPL, QB>(h, a, src, sdst, base + g, g, gl, nf, na, nm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nf += __shfl_xor_sync(0xffffffffu, nf, o);
        na += __shfl_xor_sync(0xffffffffu, na, o);
        nm += __shfl_xor_sync(0xffffffffu, nm, o);
    }
    if (lane == 0) {
        if (nf) atomicAdd(&s_cnt[0], nf);
        if (na) atomicAdd(&s_cnt[1], na);
        if (nm) atomicAdd(&s_cnt[2], nm);
    }
    __syncthreads();
    if (threadIdx.x < 3 && s_cnt[threadIdx.x])
        atomicAdd(&a.stats[1 + threadIdx.x], (unsigned long long)s_cnt[threadIdx.x]);
    if (h.remote) __threadfence_system();
}

// mirrors receive the scatter: b += deq(q) (or b ← a), Z row ← b
template <int LPR, int VPL, int QB>
__global__ void __launch_bounds__(kThreads) mirror_slot_kernel(HaloDev h, SyncArgs a,
                                                               const __grid_constant__ SlotTab src) {
    constexpr int GPW = 32 / LPR;
    __shared__ int64_t s_moff[kMaxParts + 1];
    if (threadIdx.x <= h.p) s_moff[threadIdx.x] = h.moff[threadIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / LPR, gl = lane % LPR;
    const int64_t row = ((int64_t)blockIdx.x * kWarps + warp) * GPW + g;
    if (row >= h.M) return;
    const int q = find_seg(s_moff, h.p, row);
    const uint8_t* slot = src.base[q] + (row - s_moff[q]) * a.stride;
    const uint4 hd = ld_hdr(slot);
    float* bmr = a.nocache ? nullptr : a.c.b_mir + row * a.ld;
    float4 b[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        b[v] = (bmr && c0 < a.ld) ? ld4(bmr + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (hd.x == a.sstamp) {
        if constexpr (QB != 0) {
            const float lo = __uint_as_float(hd.y), hi = __uint_as_float(hd.z);
            const float stp = stepq(lo, hi, QB);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 >= a.F) continue;
                uint32_t qc[4];
                load_codes4(slot + 16, c0, QB, qc);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (c0 + k < a.F) setc(b[v], k, __fadd_rn(comp(b[v], k), dqv(qc[k], lo, stp)));
            }
        } else {
            const float* prow = reinterpret_cast<const float*>(slot + 16);
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) b[v] = ld4(prow + c0);
            }
        }
        if (bmr) {
#pragma unroll
            for (int v = 0; v < VPL; ++v) {
                const int c0 = (gl + v * LPR) * 4;
                if (c0 < a.ld) st4(bmr + c0, b[v]);
            }
        }
    }
    float* xr = a.X + (h.B + row) * a.ld;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        if (c0 < a.ld) st4(xr + c0, a.relu ? relu4(b[v]) : b[v]);
    }
}

// ---- dispatch by row width: LPR lanes x VPL float4 per lane cover ld columns ------
struct Shape { int lpr, vpl; };
Shape shape_of(int64_t ld) {
    const int64_t nv = ld / 4;
    if (nv <= 2) return {2, 1};
    if (nv <= 4) return {4, 1};
    if (nv <= 8) return {8, 1};
    if (nv <= 16) return {8, 2};      // 4 rows per warp (ld 36..64; C3's 41 classes: 11 float4)
    if (nv <= 32) return {32, 1};
    if (nv <= 64) return {32, 2};
    if (nv <= 128) return {32, 4};
    return {32, 8};   // ld <= 1024
}

// rows per warp pass of gather_pack (must match the launch dispatch below)
int gather_rpw(int lpr, int vpl) {
    if (lpr == 16 || (lpr == 8 && vpl == 2)) return 2;
    if (lpr < 32) return 1;
    return vpl <= 2 ? 4 : (vpl == 4 ? 2 : 1);
}

#define CDF_DISPATCH(LD, KERNEL, GRID, STREAM, ...)                                         \
    do {                                                                                    \
        Shape _s = shape_of(LD);                                                            \
        if (_s.lpr == 2) KERNEL<2, 1><<<GRID(2), kThreads, 0, STREAM>>>(__VA_ARGS__);       \
        else if (_s.lpr == 4) KERNEL<4, 1><<<GRID(4), kThreads, 0, STREAM>>>(__VA_ARGS__);  \
        else if (_s.lpr == 8 && _s.vpl == 1) KERNEL<8, 1><<<GRID(8), kThreads, 0, STREAM>>>(__VA_ARGS__); \
        else if (_s.lpr == 8) KERNEL<8, 2><<<GRID(8), kThreads, 0, STREAM>>>(__VA_ARGS__);  \
        else if (_s.lpr == 16) KERNEL<16, 1><<<GRID(16), kThreads, 0, STREAM>>>(__VA_ARGS__); \
        else if (_s.vpl == 1) KERNEL<32, 1><<<GRID(32), kThreads, 0, STREAM>>>(__VA_ARGS__); \
        else if (_s.vpl == 2) KERNEL<32, 2><<<GRID(32), kThreads, 0, STREAM>>>(__VA_ARGS__); \
        else if (_s.vpl == 4) KERNEL<32, 4><<<GRID(32), kThreads, 0, STREAM>>>(__VA_ARGS__); \
        else KERNEL<32, 8><<<GRID(32), kThreads, 0, STREAM>>>(__VA_ARGS__);                 \
    } while (0)

}  // namespace

int gather_tiles_host(const int64_t* moff, int p, int64_t ld) {
    const Shape sh = shape_of(ld);
    const int TR = kWarps * (32 / sh.lpr) * gather_rpw(sh.lpr, sh.vpl);
    int t = 0;
    for (int j = 0; j < p; ++j) t += (int)((moff[j + 1] - moff[j] + TR - 1) / TR);
    return t;
}
int scatter_tiles_host(const int64_t* hoff, int p) {
    int t = 0;
    for (int j = 0; j < p; ++j) t += (int)((hoff[j + 1] - hoff[j] + kScatterTile - 1) / kScatterTile);
    return t;
}

int launch_gather_pack_n(const HaloDev& h, const SyncArgs& a, int ntiles, cudaStream_t s) {
    if (ntiles <= 0) return 0;
    const Shape sh = shape_of(a.ld);
    if (sh.lpr == 2) gather_pack_kernel<2, 1, 1><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.lpr == 4) gather_pack_kernel<4, 1, 1><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.lpr == 8 && sh.vpl == 1) gather_pack_kernel<8, 1, 1><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.lpr == 8) gather_pack_kernel<8, 2, 2><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.lpr == 16) gather_pack_kernel<16, 1, 2><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.vpl == 1) gather_pack_kernel<32, 1, 4><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.vpl == 2) gather_pack_kernel<32, 2, 4><<<ntiles, kThreads, 0, s>>>(h, a);
    else if (sh.vpl == 4) gather_pack_kernel<32, 4, 2><<<ntiles, kThreads, 0, s>>>(h, a);
    else gather_pack_kernel<32, 8, 1><<<ntiles, kThreads, 0, s>>>(h, a);
    return 1;
}

int launch_put(const PutTab* tab, int p, int64_t hdr_bytes, int64_t row_bytes, int64_t max_count,
               cudaStream_t s) {
    if (p <= 1 || max_count <= 0) return 0;
    const int64_t bytes = max_count * (hdr_bytes + row_bytes);
    const unsigned bx = (unsigned)std::min<int64_t>(std::max<int64_t>((bytes / 16 + 255) / 256, 1), 592);
    put_kernel<<<dim3(bx, p), 256, 0, s>>>(tab, hdr_bytes, row_bytes);
    return 1;
}

int launch_nvl_barrier(const BarTab& t, uint64_t seq, int32_t* err, cudaStream_t s) {
    if (t.p <= 1) return 0;
    nvl_barrier_kernel<<<1, 32 * ((t.p + 31) / 32), 0, s>>>(t, seq, err);
    return 1;
}

int launch_map(const HaloDev& h, const RegionTab& rt, int mirror_side, int64_t max_count, cudaStream_t s) {
    if (max_count <= 0 || h.p <= 1) return 0;
    dim3 grid((unsigned)std::min<int64_t>((max_count + 255) / 256, 4096), h.p);
    map_kernel<<<grid, 256, 0, s>>>(h, rt, mirror_side);
    return 1;
}

int launch_master(const HaloDev& h, const SyncArgs& a, const RegionTab& rt, cudaStream_t s) {
    if (h.B <= 0) return 0;
    auto grid = [&](int lpr) {
        const int64_t rows_per_block = kWarps * (32 / lpr);
        return (unsigned)((h.B + rows_per_block - 1) / rows_per_block);
    };
    CDF_DISPATCH(a.ld, master_kernel, grid, s, h, a, rt);
    return 1;
}

int launch_scatter_pack_n(const HaloDev& h, const SyncArgs& a, int ntiles, cudaStream_t s) {
    if (ntiles <= 0) return 0;
    scatter_pack_kernel<<<ntiles, kThreads, 0, s>>>(h, a);
    return 1;
}

int launch_mirror_apply(const HaloDev& h, const SyncArgs& a, const RegionTab& rt, cudaStream_t s) {
    if (h.M <= 0) return 0;
    auto grid = [&](int lpr) {
        const int64_t rows_per_block = kWarps * (32 / lpr);
        return (unsigned)((h.M + rows_per_block - 1) / rows_per_block);
    };
    CDF_DISPATCH(a.ld, mirror_apply_kernel, grid, s, h, a, rt);
    return 1;
}

// the slot kernels are instantiated per message width B (QB): the code packing and the
// quantiser's branches fold at compile time
#define CDF_QB(QBV, ...)                                           \
    do {                                                           \
        if ((QBV) == 8) { constexpr int QB = 8; __VA_ARGS__; }     \
        else if ((QBV) == 4) { constexpr int QB = 4; __VA_ARGS__; } \
        else if ((QBV) == 16) { constexpr int QB = 16; __VA_ARGS__; } \
        else { constexpr int QB = 0; __VA_ARGS__; }                \
    } while (0)

template <int QB>
void gather_slot_q(const HaloDev& h, const SyncArgs& a, const SlotTab& dst, cudaStream_t s, const Shape& sh,
                   unsigned grid) {
    if (sh.lpr == 2) gather_slot_kernel<2, 1, 1, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.lpr == 4) gather_slot_kernel<4, 1, 1, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.lpr == 8 && sh.vpl == 1) gather_slot_kernel<8, 1, 1, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.lpr == 8) gather_slot_kernel<8, 2, 2, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.vpl == 1) gather_slot_kernel<32, 1, 4, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.vpl == 2) gather_slot_kernel<32, 2, 4, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else if (sh.vpl == 4) gather_slot_kernel<32, 4, 2, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
    else gather_slot_kernel<32, 8, 1, QB><<<grid, kThreads, 0, s>>>(h, a, dst);
}

int launch_gather_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& dst, cudaStream_t s) {
    if (h.M <= 0) return 0;
    const Shape sh = shape_of(a.ld);
    const int rpw = gather_rpw(sh.lpr, sh.vpl);
    const int64_t rpb = (int64_t)kWarps * (32 / sh.lpr) * rpw;
    const unsigned grid = (unsigned)std::min<int64_t>((h.M + rpb - 1) / rpb, 148 * 4);
    CDF_QB(h.quant, gather_slot_q<QB>(h, a, dst, s, sh, grid));
    return 1;
}

template <int LPR, int VPL>
struct MasterSlotQ {
    template <int QB>
    static void go(unsigned g, cudaStream_t s, const HaloDev& h, const SyncArgs& a, const SlotTab& src,
                   const SlotTab& sdst) {
        master_slot_kernel<LPR, VPL, QB><<<g, kThreads, 0, s>>>(h, a, src, sdst);
    }
};
template <int LPR, int VPL>
struct MirrorSlotQ {
    template <int QB>
    static void go(unsigned g, cudaStream_t s, const HaloDev& h, const SyncArgs& a, const SlotTab& src) {
        mirror_slot_kernel<LPR, VPL, QB><<<g, kThreads, 0, s>>>(h, a, src);
    }
};
// row-width shape x message width dispatch of a slot kernel family F (MasterSlotQ / MirrorSlotQ)
#define CDF_DISPATCH_SLOT(LD, QBV, F, GRID, STREAM, ...)                                          \
    do {                                                                                          \
        Shape _s = shape_of(LD);                                                                  \
        if (_s.lpr == 2) CDF_QB(QBV, F<2, 1>::template go<QB>(GRID(2), STREAM, __VA_ARGS__));      \
        else if (_s.lpr == 4) CDF_QB(QBV, F<4, 1>::template go<QB>(GRID(4), STREAM, __VA_ARGS__)); \
        else if (_s.lpr == 8 && _s.vpl == 1) CDF_QB(QBV, F<8, 1>::template go<QB>(GRID(8), STREAM, __VA_ARGS__)); \
        else if (_s.lpr == 8) CDF_QB(QBV, F<8, 2>::template go<QB>(GRID(8), STREAM, __VA_ARGS__)); \
        else if (_s.lpr == 16) CDF_QB(QBV, F<16, 1>::template go<QB>(GRID(16), STREAM, __VA_ARGS__)); \
        else if (_s.vpl == 1) CDF_QB(QBV, F<32, 1>::template go<QB>(GRID(32), STREAM, __VA_ARGS__)); \
        else if (_s.vpl == 2) CDF_QB(QBV, F<32, 2>::template go<QB>(GRID(32), STREAM, __VA_ARGS__)); \
        else if (_s.vpl == 4) CDF_QB(QBV, F<32, 4>::template go<QB>(GRID(32), STREAM, __VA_ARGS__)); \
        else CDF_QB(QBV, F<32, 8>::template go<QB>(GRID(32), STREAM, __VA_ARGS__));                \
    } while (0)

int launch_master_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& src, const SlotTab& sdst,
                       cudaStream_t s) {
    if (h.B <= 0) return 0;
    // grid-stride: 3 resident blocks per SM (148 SMs), fewer for short launches
    auto grid = [&](int lpr) {
        const int64_t rows_per_block = kWarps * (32 / lpr);
        return (unsigned)std::min<int64_t>((h.B + rows_per_block - 1) / rows_per_block, 148 * 3);
    };
    CDF_DISPATCH_SLOT(a.ld, h.quant, MasterSlotQ, grid, s, h, a, src, sdst);
    return 1;
}

int launch_mirror_slot(const HaloDev& h, const SyncArgs& a, const SlotTab& src, cudaStream_t s) {
    if (h.M <= 0) return 0;
    auto grid = [&](int lpr) {
        const int64_t rows_per_block = kWarps * (32 / lpr);
        return (unsigned)((h.M + rows_per_block - 1) / rows_per_block);
    };
    CDF_DISPATCH_SLOT(a.ld, h.quant, MirrorSlotQ, grid, s, h, a, src);
    return 1;
}

}  // namespace cdfgnn
