// Device helpers shared by the halo kernels (kernels_halo.cu) and the SpMM kernel's fused
// gather epilogue (kernels_spmm.cu): the R15 canonical quantiser, code-row packing, the slot
// header, and the per-row gather of Alg. 2 L3-L9 run by a row group.  Included inside
// `namespace cdfgnn { namespace { ... } }` of each translation unit.
#pragma once

// ---- R15 canonical quantiser (B = 4, 8 or 16 bits) ---------------------------
// code = min(floor(RN(RN(RN(RN(d − lo)·2^B) / rng) + 0.5)), 2^B − 1), 0 when rng = 0.
// Fast path (B <= 8): y = RN(t·RN(1/rng)) is within a few ulp(2^B) of t/rng (t/rng ∈ [0, 2^B]),
// so v = RN(y + 0.5) is within 2^-13 of the canonical RN(RN(t/rng) + 0.5); whenever v's
// fractional part is at least 2^-11 away from an integer both floors agree.  Closer to a
// boundary the canonical IEEE division decides, so every code is bit-identical to the
// oracle's fp32 replay (oracle/quant.py quantize_f32) — one reciprocal per row instead of one
// division per element.  B = 16: ulp(2^16) = 2^-7 leaves no such margin, every code divides.
struct QRow {
    float lo, rng;
    float rinv_s;          // RN(1/rng)·2^B (exact scaling); 0 when rng = 0: the fast path yields code 0
    float scale;           // 2^B (exact)
    float qmax;            // 2^B − 1
    int bits;
};
__device__ __forceinline__ QRow qrow(float lo, float hi, int bits) {
    QRow q;
    q.lo = lo;
    q.rng = __fsub_rn(hi, lo);
    q.scale = (float)(1u << bits);
    q.rinv_s = q.rng == 0.f ? 0.f : __fmul_rn(__frcp_rn(q.rng), q.scale);
    q.qmax = (float)((1u << bits) - 1u);
    q.bits = bits;
    return q;
}
// fast-path floor of RN(RN(t/rng) + 0.5); *slow is set when the canonical division must decide.
// t·RN(1/rng) = RN(d − lo)·2^B·RN(1/rng): the power-of-two factor is exact, so it is applied to
// the reciprocal once per row (one multiplication per element fewer, same bits).
__device__ __forceinline__ float q_fast(float d, const QRow& q, bool* slow) {
    const float v = __fadd_rn(__fmul_rn(__fsub_rn(d, q.lo), q.rinv_s), 0.5f);
    const float fl = floorf(v);
    *slow = fabsf(__fsub_rn(__fsub_rn(v, fl), 0.5f)) >= 0.49951171875f;   // within 2^-11 of an integer
    return fl;
}
__device__ __noinline__ float q_slow(float d, const QRow& q) {
    if (q.rng == 0.f) return 0.f;
    const float t = __fmul_rn(__fsub_rn(d, q.lo), q.scale);
    return floorf(__fadd_rn(__fdiv_rn(t, q.rng), 0.5f));
}
// 4 codes of one float4 chunk; the (rare) canonical division runs only for flagged elements
__device__ __forceinline__ void qx4(const float (&d)[4], const QRow& q, uint32_t (&c)[4]) {
    float fl[4];
    if (q.bits > 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k) fl[k] = q_slow(d[k], q);
    } else {
        bool sl[4], any = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            fl[k] = q_fast(d[k], q, &sl[k]);
            any |= sl[k];
        }
        if (any) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (sl[k]) fl[k] = q_slow(d[k], q);
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = (uint32_t)fminf(fl[k], q.qmax);
}
// dequantisation m̃ = RN(RN(step·q) + lo), step = RN((hi − lo)·2^-B)  (R15)
__device__ __forceinline__ float dqv(uint32_t q, float lo, float step) {
    return __fadd_rn(__fmul_rn(step, (float)q), lo);
}
__device__ __forceinline__ float stepq(float lo, float hi, int bits) {
    return __fmul_rn(__fsub_rn(hi, lo), 1.0f / (float)(1u << bits));   // 2^-B exact
}

// Code rows (kernels.h code_row_bytes): B = 8 one byte per code, B = 4 two codes per byte
// (code k in the low nibble of byte k/2 for even k), B = 16 one little-endian uint16 per code;
// the F codes are followed by zero padding.  Every group of 4 codes at column c0 (c0 % 4 = 0)
// is one aligned 16-, 32- or 64-bit access.
__device__ __forceinline__ void pack_codes4(const uint32_t (&q)[4], int c0, int F, int bits, uint32_t (&w)[2]) {
    uint32_t m[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) m[k] = (c0 + k < F) ? q[k] : 0u;
    if (bits == 8) { w[0] = m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24); w[1] = 0; }
    else if (bits == 4) { w[0] = m[0] | (m[1] << 4) | (m[2] << 8) | (m[3] << 12); w[1] = 0; }
    else { w[0] = m[0] | (m[1] << 16); w[1] = m[2] | (m[3] << 16); }
}
__device__ __forceinline__ void put_codes4(uint8_t* row, int c0, int bits, const uint32_t (&w)[2]) {
    if (bits == 8) *reinterpret_cast<uint32_t*>(row + c0) = w[0];
    else if (bits == 4) *reinterpret_cast<uint16_t*>(row + c0 / 2) = (uint16_t)w[0];
    else *reinterpret_cast<uint2*>(row + 2 * c0) = make_uint2(w[0], w[1]);
}
__device__ __forceinline__ void store_codes4(uint8_t* row, int c0, int F, const uint32_t (&q)[4], int bits) {
    uint32_t w[2];
    pack_codes4(q, c0, F, bits, w);
    put_codes4(row, c0, bits, w);
}
__device__ __forceinline__ void unpack_codes4(const uint32_t (&w)[2], int bits, uint32_t (&q)[4]) {
    if (bits == 8) { q[0] = w[0] & 0xFFu; q[1] = (w[0] >> 8) & 0xFFu; q[2] = (w[0] >> 16) & 0xFFu; q[3] = w[0] >> 24; }
    else if (bits == 4) { q[0] = w[0] & 0xFu; q[1] = (w[0] >> 4) & 0xFu; q[2] = (w[0] >> 8) & 0xFu; q[3] = (w[0] >> 12) & 0xFu; }
    else { q[0] = w[0] & 0xFFFFu; q[1] = w[0] >> 16; q[2] = w[1] & 0xFFFFu; q[3] = w[1] >> 16; }
}
__device__ __forceinline__ void fetch_codes4(const uint8_t* row, int c0, int bits, uint32_t (&w)[2]) {
    if (bits == 8) { w[0] = __ldg(reinterpret_cast<const uint32_t*>(row + c0)); w[1] = 0; }
    else if (bits == 4) { w[0] = __ldg(reinterpret_cast<const unsigned short*>(row + c0 / 2)); w[1] = 0; }
    else { const uint2 v = __ldg(reinterpret_cast<const uint2*>(row + 2 * c0)); w[0] = v.x; w[1] = v.y; }
}
__device__ __forceinline__ void load_codes4(const uint8_t* row, int c0, int bits, uint32_t (&q)[4]) {
    uint32_t w[2];
    fetch_codes4(row, c0, bits, w);
    unpack_codes4(w, bits, q);
}

template <int LPR>
__device__ __forceinline__ float gmax(float v) {
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int LPR>
__device__ __forceinline__ float gmin(float v) {
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 relu4(float4 v) {
    return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float comp(const float4& v, int k) {
    return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
__device__ __forceinline__ void setc(float4& v, int k, float x) {
    if (k == 0) v.x = x; else if (k == 1) v.y = x; else if (k == 2) v.z = x; else v.w = x;
}

__device__ __forceinline__ int find_seg(const int64_t* off, int p, int64_t idx) {
    int s = 0;
    while (s + 1 < p && off[s + 1] <= idx) ++s;
    return s;
}

__device__ __forceinline__ uint4 ld_hdr(const uint8_t* slot) {
    return __ldg(reinterpret_cast<const uint4*>(slot));
}
__device__ __forceinline__ void st_hdr(uint8_t* slot, uint32_t stamp, float lo, float hi) {
    *reinterpret_cast<uint4*>(slot) = make_uint4(stamp, __float_as_uint(lo), __float_as_uint(hi), 0u);
}


// Alg. 2 L3-L9 for one mirror row whose value z sits in the registers of a row group (LPR lanes
// x VPL float4, columns (gl + v·LPR)·4): the snapshot s is loaded, d = z − s tested against
// ε‖s‖∞ (R15), and a sender's codes (or fp32 Δ) and header are stored into its slot, the
// snapshot updated (R11 / Alg. 2 L6) and the send flag recorded.  Reductions use the group's
// lanes only, so other groups of the warp may be elsewhere.  Same arithmetic as
// gather_slot_kernel: identical bits.
template <int LPR, int VPL>
__device__ __forceinline__ void gather_row_fused(const HaloDev& h, const SyncArgs& a, uint8_t* slot, int64_t mrow,
                                                 unsigned gmask, int gl, const float4 (&z)[VPL]) {
    float* sr = a.nocache ? nullptr : a.c.s_mir + mrow * a.ld;
    float4 ss[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
        ss[v] = (sr && c0 < a.ld) ? __ldcs(reinterpret_cast<const float4*>(sr + c0)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float maxs = 0.f, lo = INFINITY, hi = -INFINITY;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        const int c0 = (gl + v * LPR) * 4;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float dk = __fsub_rn(comp(z[v], k), comp(ss[v], k));
            if (c0 + k < a.F) {
                maxs = fmaxf(maxs, fabsf(comp(ss[v], k)));
                lo = fminf(lo, dk);
                hi = fmaxf(hi, dk);
            }
        }
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
        maxs = fmaxf(maxs, __shfl_xor_sync(gmask, maxs, o));
        lo = fminf(lo, __shfl_xor_sync(gmask, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(gmask, hi, o));
    }
    const float maxd = fmaxf(fabsf(lo), fabsf(hi));
    const bool flag = a.nocache || maxd > __fmul_rn(a.eps, maxs);
    if (gl == 0) h.gflag[mrow] = flag ? 1 : 0;
    if (!flag) return;
    const int bits = h.quant;
    if (bits) {
        const QRow qr = qrow(lo, hi, bits);
        const float stp = stepq(lo, hi, bits);
        if (gl == 0) st_hdr(slot, a.gstamp, lo, hi);
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
            const int c0 = (gl + v * LPR) * 4;
            if (c0 >= a.F) continue;
            uint32_t qc[4];
            float dd[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) dd[k] = __fsub_rn(comp(z[v], k), comp(ss[v], k));
            qx4(dd, qr, qc);
            store_codes4(slot + 16, c0, a.F, qc, bits);
            if (sr) {
                float4 snew;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    setc(snew, k, (c0 + k < a.F) ? __fadd_rn(comp(ss[v], k), dqv(qc[k], lo, stp)) : 0.f);
                __stcs(reinterpret_cast<float4*>(sr + c0), snew);
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
            for (int k = 0; k < 4; ++k) setc(dv, k, __fsub_rn(comp(z[v], k), comp(ss[v], k)));
            st4(prow + c0, dv);
            if (sr) st4(sr + c0, z[v]);
        }
    }
}
