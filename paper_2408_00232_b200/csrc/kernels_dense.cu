// Dense kernels: fp32 SIMT GEMM (exact-fp32 mode), ReLU, loss head, reductions,
// optimiser (sm_100a).
//
//   T  = H W                 feature transform (eq. 1; reading R5: Â(HW))
//   dW = Hᵀ S                weight gradient (eq. 5; reading R6), split-K with a
//                            fixed-order reduction (deterministic)
//   δ̈  = (S Wᵀ) ⊙ 𝟙[H > 0]   input gradient (σ' of ReLU, R3)
//   loss: mean CE over masters ∩ train (R7), δ̈^(L) = (softmax − onehot)/N_train
//   optimiser: W ← W − η ΣΔ or Adam (PyTorch update formula)
// The tcgen05 TF32 GEMMs live in gemm_tc.cu; this SIMT GEMM is the exact-fp32 path.
#include <cfloat>

#include "kernels.h"

namespace cdfgnn {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int64_t M, int64_t N, int64_t K,
                                                        const float* __restrict__ A, int64_t lda,
                                                        const float* __restrict__ B, int64_t ldb,
                                                        float* __restrict__ C, int64_t ldc,
                                                        const float* __restrict__ mask, int64_t ldm,
                                                        float* __restrict__ ws, int64_t kchunk,
                                                        int accumulate) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t m0 = (int64_t)blockIdx.y * BM;
    const int64_t n0 = (int64_t)blockIdx.x * BN;
    const int64_t kb = (int64_t)blockIdx.z * kchunk;
    const int64_t ke = min(K, kb + kchunk);
    float acc[4][4] = {};
    for (int64_t k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * 256;
            int mm, kk;
            if (TA) { kk = idx / BM; mm = idx % BM; } else { mm = idx / BK; kk = idx % BK; }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            float va = 0.f;
            if (gm < M && gk < ke) va = TA ? A[gk * lda + gm] : A[gm * lda + gk];
            As[kk][mm] = va;
            int nn, kk2;
            if (TB) { nn = idx / BK; kk2 = idx % BK; } else { kk2 = idx / BN; nn = idx % BN; }
            const int64_t gn = n0 + nn, gk2 = k0 + kk2;
            float vb = 0.f;
            if (gn < N && gk2 < ke) vb = TB ? B[gn * ldb + gk2] : B[gk2 * ldb + gn];
            Bs[kk2][nn] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    if (ws) {   // split-K partial: ws[z][M][N]
        float* wz = ws + (int64_t)blockIdx.z * M * N;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gm = m0 + ty * 4 + i;
            if (gm >= M) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t gn = n0 + tx * 4 + j;
                if (gn < N) wz[gm * N + gn] = acc[i][j];
            }
        }
        return;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t gn = n0 + tx * 4 + j;
            if (gn >= ldc) continue;
            float v = gn < N ? acc[i][j] : 0.f;
            if (mask && gn < N && !(mask[gm * ldm + gn] > 0.f)) v = 0.f;
            if (accumulate && gn < N) v += C[gm * ldc + gn];
            C[gm * ldc + gn] = v;
        }
    }
}

__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const float* __restrict__ ws,
                                     float* __restrict__ C, int64_t ldc, int accumulate) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M * ldc) return;
    const int64_t m = i / ldc, n = i % ldc;
    if (n >= N) { C[i] = 0.f; return; }
    float v = 0.f;
    for (int z = 0; z < splits; ++z) v += ws[(int64_t)z * M * N + m * N + n];   // fixed order
    if (accumulate) v += C[i];
    C[i] = v;
}

__global__ void relu_kernel(const float* __restrict__ Z, float* __restrict__ H, int64_t n4) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n4) return;
    float4 z = reinterpret_cast<const float4*>(Z)[i];
    z.x = fmaxf(z.x, 0.f); z.y = fmaxf(z.y, 0.f); z.z = fmaxf(z.z, 0.f); z.w = fmaxf(z.w, 0.f);
    reinterpret_cast<float4*>(H)[i] = z;
}

constexpr int kMaxClassPerLane = 8;   // C <= 256

// one row of the loss head by a group of LPR lanes (C <= 8·LPR: 8 logits per lane); returns 1
// when the row is a correctly classified train master (R16: argmax ties to the lowest class)
template <int LPR>
__device__ __forceinline__ int loss_row(const float* __restrict__ logits, int64_t ld, int C, int64_t row,
                                        int64_t B, int64_t M, const int32_t* __restrict__ labels,
                                        const uint8_t* __restrict__ train, double inv_ntrain,
                                        float* __restrict__ dlogits, float* __restrict__ rowloss, int* err,
                                        int gl, unsigned gmask) {
    const bool master = row < B || row >= B + M;
    const bool use = master && train[row];
    float* drow = dlogits + row * ld;
    if (!use) {
        for (int c = gl; c < ld; c += LPR) drow[c] = 0.f;
        if (gl == 0) rowloss[row] = 0.f;
        return 0;
    }
    const int y = labels[row];
    if (y < 0 || y >= C) {
        if (gl == 0) atomicExch(err, 3);
        for (int c = gl; c < ld; c += LPR) drow[c] = 0.f;
        if (gl == 0) rowloss[row] = 0.f;
        return 0;
    }
    const float* z = logits + row * ld;
    float v[kMaxClassPerLane];
    float mx = -FLT_MAX;
    int amax = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < kMaxClassPerLane; ++t) {
        const int c = gl + LPR * t;
        v[t] = c < C ? z[c] : -FLT_MAX;
        if (c < C && (v[t] > mx)) { mx = v[t]; amax = c; }
    }
    // group argmax, ties to the lowest class (reading R16)
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(gmask, mx, o);
        const int oa = __shfl_xor_sync(gmask, amax, o);
        if (om > mx || (om == mx && oa < amax)) { mx = om; amax = oa; }
    }
    float s = 0.f;
#pragma unroll
    for (int t = 0; t < kMaxClassPerLane; ++t) {
        const int c = gl + LPR * t;
        if (c < C) s += expf(v[t] - mx);
    }
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
    const float lse = mx + logf(s);
    const float inv = (float)inv_ntrain;
#pragma unroll
    for (int t = 0; t < kMaxClassPerLane; ++t) {
        const int c = gl + LPR * t;
        if (c < C) {
            const float p = expf(v[t] - mx) / s;
            drow[c] = (p - (c == y ? 1.f : 0.f)) * inv;
        } else if (c < ld) {
            drow[c] = 0.f;
        }
    }
    for (int c = gl + LPR * kMaxClassPerLane; c < ld; c += LPR) drow[c] = 0.f;
    if (gl == (y % LPR)) {
        float vy = 0.f;
#pragma unroll
        for (int t = 0; t < kMaxClassPerLane; ++t)
            if (gl + LPR * t == y) vy = v[t];
        rowloss[row] = lse - vy;
    }
    return (gl == 0 && amax == y) ? 1 : 0;
}

// LPR lanes per row (8 when C <= 64: four rows of a warp in flight), grid-stride loop; the correct
// count is reduced per block and added with one atomic per block (a same-address atomic per row
// serialised at L2: ~1.5M per C4 epoch)
template <int LPR>
__global__ void __launch_bounds__(256) loss_kernel(const float* __restrict__ logits, int64_t ld, int C,
                                                   int64_t n, int64_t B, int64_t M,
                                                   const int32_t* __restrict__ labels,
                                                   const uint8_t* __restrict__ train, double inv_ntrain,
                                                   float* __restrict__ dlogits,
                                                   float* __restrict__ rowloss, int* correct, int* err) {
    constexpr int GPW = 32 / LPR;
    const int lane = threadIdx.x & 31;
    const int g = lane / LPR, gl = lane % LPR;
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
    int mine = 0;
    for (int64_t row = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * GPW + g; row < n;
         row += (int64_t)gridDim.x * 8 * GPW)
        mine += loss_row<LPR>(logits, ld, C, row, B, M, labels, train, inv_ntrain, dlogits, rowloss, err, gl, gmask);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    if (lane == 0 && mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(correct, s_cnt);
}

// Σ rowloss in fp64 in a fixed order: block b sums the contiguous chunk b (8 loads in flight per
// thread, tree over the block), then one block adds the kRedBlocks partial sums in block order
constexpr int kRedBlocks = 148;
__global__ void __launch_bounds__(1024) reduce_rows_kernel(const float* __restrict__ x, int64_t n,
                                                           double* __restrict__ part) {
    __shared__ double sh[1024];
    const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
    const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
    constexpr int U = 8;
    double acc[U] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t step = (int64_t)blockDim.x * U;
    for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += step) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t i = i0 + (int64_t)u * blockDim.x;
            if (i < hi) acc[u] += (double)__ldg(x + i);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s += acc[u];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void reduce_parts_kernel(const double* __restrict__ part, int np, double* out) {
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int b = 0; b < np; ++b) s += part[b];
        *out = s;
    }
}

__global__ void count_train_kernel(int64_t n, int64_t B, int64_t M, const uint8_t* train, int* out) {
    const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool use = row < n && (row < B || row >= B + M) && train[row];
    const unsigned b = __ballot_sync(0xffffffffu, use);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, __popc(b));
}

__global__ void optimizer_kernel(int kind, float* __restrict__ W, const float* __restrict__ G,
                                 float* __restrict__ m, float* __restrict__ v, int64_t count,
                                 float lr, float b1, float b2, float eps, float bc1, float bc2,
                                 const int32_t* __restrict__ err) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    if (err && *err) return;      // a halo / data error this epoch (max over ranks): W stays unchanged
    const float g = G[i];
    if (kind == 0) {
        W[i] = W[i] - lr * g;
        return;
    }
    const float mi = b1 * m[i] + (1.f - b1) * g;       // Adam, PyTorch formula
    const float vi = b2 * v[i] + (1.f - b2) * g * g;
    m[i] = mi;
    v[i] = vi;
    const float denom = sqrtf(vi) / sqrtf(bc2) + eps;
    W[i] = W[i] - (lr / bc1) * (mi / denom);
}

__global__ void __launch_bounds__(256) read_probe_kernel(const float4* __restrict__ p, int64_t n4, int reps,
                                                         float* sink) {
    // 8 independent 16-byte L2 reads in flight per thread (ld.global.cg: L1 bypassed), so the
    // probe is bound by L2 -> SM delivery, not by per-thread latency
    constexpr int U = 8;
    float4 acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n4; i0 += stride * U) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t i = i0 + u * stride;
                v[u] = i < n4 ? __ldcg(p + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc[u].x += v[u].x; acc[u].y += v[u].y; acc[u].z += v[u].z; acc[u].w += v[u].w;
            }
        }
    float t = 0.f;
#pragma unroll
    for (int u = 0; u < U; ++u) t += acc[u].x + acc[u].y + acc[u].z + acc[u].w;
    if (t == 1.2345e-30f && sink) sink[0] = t;   // keep the loads alive
}

// out[k] = X[idx[k]]: flattened over (row, float4), grid-stride
__global__ void gather_rows_kernel(const float* __restrict__ X, int64_t ld, const int32_t* __restrict__ idx,
                                   int64_t count, float* __restrict__ out) {
    const int64_t v4 = ld / 4, total = count * v4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / v4, c = i - k * v4;
        reinterpret_cast<float4*>(out)[i] = reinterpret_cast<const float4*>(X + (int64_t)__ldg(idx + k) * ld)[c];
    }
}

}  // namespace

int launch_gather_rows(const float* X, int64_t ld, const int32_t* idx, int64_t count, float* out, cudaStream_t s) {
    if (count <= 0) return 0;
    const int64_t total = count * (ld / 4);
    gather_rows_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(X, ld, idx, count, out);
    return 1;
}

void launch_read_probe(const float4* p, int64_t n4, int reps, float* sink, cudaStream_t s) {
    read_probe_kernel<<<148 * 8, 256, 0, s>>>(p, n4, reps, sink);
}

void launch_gemm_simt(bool TA, bool TB, int64_t M, int64_t N, int64_t K, const float* A,
                      int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                      const float* mask, int64_t ldm, float* splitk_ws, int64_t splitk_cap,
                      bool accumulate, cudaStream_t s) {
    if (M <= 0 || ldc <= 0) return;
    const unsigned gx = (unsigned)((std::max<int64_t>(N, ldc) + BN - 1) / BN);
    const unsigned gy = (unsigned)((M + BM - 1) / BM);
    int splits = 1;
    if (splitk_ws && !mask) {
        // enough CTAs for 148 SMs; the partials must fit the caller's buffer
        const int64_t tiles = (int64_t)gx * gy;
        while (tiles * splits < 4 * 148 && K / (splits * 2) >= 256 &&
               (int64_t)(splits * 2) * M * N <= splitk_cap)
            splits *= 2;
    }
    const int64_t kchunk = splits > 1 ? (((K + splits - 1) / splits + BK - 1) / BK * BK) : K;
    dim3 grid(gx, gy, splits);
    float* ws = splits > 1 ? splitk_ws : nullptr;
    const int acc = accumulate ? 1 : 0;
    if (!TA && !TB) gemm_simt_kernel<false, false><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, mask, ldm, ws, kchunk, acc);
    else if (!TA && TB) gemm_simt_kernel<false, true><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, mask, ldm, ws, kchunk, acc);
    else if (TA && !TB) gemm_simt_kernel<true, false><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, mask, ldm, ws, kchunk, acc);
    else gemm_simt_kernel<true, true><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, mask, ldm, ws, kchunk, acc);
    if (splits > 1) {
        const int64_t tot = M * ldc;
        splitk_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(M, N, splits, ws, C, ldc, acc);
    }
}

void launch_relu(const float* Z, float* H, int64_t count, cudaStream_t s) {
    const int64_t n4 = count / 4;
    if (n4 <= 0) return;
    relu_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, s>>>(Z, H, n4);
}

void launch_loss(const float* logits, int64_t ld, int C, int64_t n, int64_t B, int64_t M,
                 const int32_t* labels, const uint8_t* train, double inv_ntrain, float* dlogits,
                 float* rowloss, int* correct, int* err, cudaStream_t s) {
    if (n <= 0) return;
    if (C <= 8 * kMaxClassPerLane)
        loss_kernel<8><<<(unsigned)std::min<int64_t>((n + 31) / 32, 148 * 8), 256, 0, s>>>(
            logits, ld, C, n, B, M, labels, train, inv_ntrain, dlogits, rowloss, correct, err);
    else
        loss_kernel<32><<<(unsigned)std::min<int64_t>((n + 7) / 8, 148 * 8), 256, 0, s>>>(
            logits, ld, C, n, B, M, labels, train, inv_ntrain, dlogits, rowloss, correct, err);
}

void launch_reduce_rows(const float* rowloss, int64_t n, double* out, double* part, cudaStream_t s) {
    reduce_rows_kernel<<<kRedBlocks, 1024, 0, s>>>(rowloss, n, part);
    reduce_parts_kernel<<<1, 32, 0, s>>>(part, kRedBlocks, out);
}

void launch_count_train(int64_t n, int64_t B, int64_t M, const uint8_t* train, int* out,
                        cudaStream_t s) {
    if (n <= 0) return;
    count_train_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, B, M, train, out);
}

void launch_optimizer(int kind, float* W, const float* G, float* m, float* v, int64_t count,
                      float lr, float b1, float b2, float eps, float bc1, float bc2,
                      const int32_t* err, cudaStream_t s) {
    if (count <= 0) return;
    optimizer_kernel<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(kind, W, G, m, v, count, lr,
                                                                     b1, b2, eps, bc1, bc2, err);
}

}  // namespace cdfgnn
