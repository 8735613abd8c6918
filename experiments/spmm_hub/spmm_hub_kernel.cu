// Community-hub SpMM experiment (round 2), measured and rejected: C3 p=1 256-wide launch
// 30.3 ms (4-lane row groups) / 40.5 ms (warp per row) vs 5.9 ms for the row-per-group kernel
// (profiles/r2/experiments/spmm_hub_C3_p1.txt).  Not built; kept for the record with locality.cpp.
// ---- community-hub SpMM (locality.h) ------------------------------------------------
__global__ void __launch_bounds__(256) permute_rows_kernel(const float* __restrict__ T, const int32_t* __restrict__ order,
                                                           int64_t n, int64_t ld, float* __restrict__ Tp) {
    // one warp per row, 16-byte loads and stores
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const float4* src = reinterpret_cast<const float4*>(T + (int64_t)__ldg(order + i) * ld);
    float4* dst = reinterpret_cast<float4*>(Tp + i * ld);
    for (int64_t q = lane; q < ld / 4; q += 32) dst[q] = __ldcs(src + q);
}

// One CTA per SM, persistent: units (slice k, community t) are taken from a work counter
// slice-major (all communities of slice 0, heaviest first, then slice 1, ...), so the slice of
// T the CTAs gather from at any time is an L2-resident window.  Per unit the CTA stages the
// slice [k·SW, k·SW + SW) of the community's hub rows in shared memory (G = SW/4 lanes x 16
// bytes per row); then one warp per row: its 32/G lane groups take interleaved neighbours
// (R per group in flight), hub neighbours from shared memory, the others from L2, and the
// groups' partial sums are combined by a fixed butterfly — every (row, slice) is summed in a
// fixed order (deterministic).
template <int SW, int R>
__global__ void __launch_bounds__(512, 1) spmm_hub_kernel(HubDev h, const float* __restrict__ Tp,
                                                           float* __restrict__ Y, int64_t ld, int nslices) {
    constexpr int G = SW / 4;           // lanes per row slice
    constexpr int NG = 32 / G;          // lane groups per warp (neighbours in parallel)
    constexpr int B = NG * R;           // neighbours per batch
    extern __shared__ float4 hub_s[];   // [hub count][G]
    __shared__ int s_unit;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane / G, gl = lane % G;
    const int nwarps = blockDim.x >> 5;
    const int total = h.ncomm * nslices;
    for (;;) {
        if (threadIdx.x == 0) s_unit = atomicAdd(h.counter, 1);
        __syncthreads();
        const int u = s_unit;
        if (u >= total) break;
        const int4 cm = __ldg(h.comm + u % h.ncomm);
        const int c0 = (u / h.ncomm) * SW;
        for (int i = threadIdx.x; i < cm.w * G; i += blockDim.x) {
            const int hr = i / G, q = i - hr * G;
            hub_s[i] = (c0 + q * 4 < ld) ? __ldg(reinterpret_cast<const float4*>(Tp + (int64_t)(cm.z + hr) * ld + c0) + q)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        const bool colok = c0 + gl * 4 < ld;
        const float* tcol = Tp + c0 + gl * 4;
        for (int i = cm.x + warp; i < cm.y; i += nwarps) {
            const int rb = __ldg(h.rowptr + i), re = __ldg(h.rowptr + i + 1);
            const int rh = rb + __ldg(h.nhub + i);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            // neighbours inside the community's hub rows: shared memory
            for (int base = rb; base < rh; base += B) {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int e = base + j * NG + g;
                    if (e < rh) {
                        const float w = __ldg(h.val + e);
                        const float4 v = hub_s[(__ldg(h.col + e) - cm.z) * G + gl];
                        acc.x = fmaf(w, v.x, acc.x);
                        acc.y = fmaf(w, v.y, acc.y);
                        acc.z = fmaf(w, v.z, acc.z);
                        acc.w = fmaf(w, v.w, acc.w);
                    }
                }
            }
            // the other neighbours: L2 (the batch's loads are issued before the FMAs)
            for (int base = rh; base < re; base += B) {
                float4 t[R];
                float w[R];
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const int e = base + j * NG + g;
                    const bool live = e < re;
                    w[j] = live ? __ldg(h.val + e) : 0.f;
                    t[j] = (live && colok) ? __ldg(reinterpret_cast<const float4*>(tcol + (int64_t)__ldg(h.col + e) * ld))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    acc.x = fmaf(w[j], t[j].x, acc.x);
                    acc.y = fmaf(w[j], t[j].y, acc.y);
                    acc.z = fmaf(w[j], t[j].z, acc.z);
                    acc.w = fmaf(w[j], t[j].w, acc.w);
                }
            }
            // combine the NG groups' partial sums (fixed butterfly)
#pragma unroll
            for (int o = G; o < 32; o <<= 1) {
                acc.x = __fadd_rn(acc.x, __shfl_xor_sync(0xffffffffu, acc.x, o));
                acc.y = __fadd_rn(acc.y, __shfl_xor_sync(0xffffffffu, acc.y, o));
                acc.z = __fadd_rn(acc.z, __shfl_xor_sync(0xffffffffu, acc.z, o));
                acc.w = __fadd_rn(acc.w, __shfl_xor_sync(0xffffffffu, acc.w, o));
            }
            if (g == 0 && colok)
                *reinterpret_cast<float4*>(Y + (int64_t)__ldg(h.order + i) * ld + c0 + gl * 4) = acc;
        }
        __syncthreads();      // every warp is done with the staged slice
    }
}

constexpr int kHubR = 4;    // neighbours in flight per lane group

void launch_permute_rows(const float* T, const int32_t* order, int64_t n, int64_t ld, float* Tp, cudaStream_t s) {
    if (n <= 0) return;
    permute_rows_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(T, order, n, ld, Tp);
}

int launch_spmm_hub(const HubDev& h, const float* Tp, float* Y, int64_t ld, cudaStream_t s) {
    constexpr int SW = kHubSliceCols;
    const size_t smem = (size_t)h.hub_rows * SW * sizeof(float);
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(spmm_hub_kernel<SW, kHubR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kHubRows * SW * sizeof(float))) != cudaSuccess)
            return 0;
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int nslices = (int)((ld + SW - 1) / SW);
    cudaMemsetAsync(h.counter, 0, sizeof(int32_t), s);
    spmm_hub_kernel<SW, kHubR><<<sms, 512, smem, s>>>(h, Tp, Y, ld, nslices);
    return 1;
}

