// L2 / HBM read-bandwidth probe (debug tool): float4 streaming reads of a buffer of
// the given size, repeated; prints GB/s for each size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ p, long n4, int reps, float* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; ++r)
        for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
            float4 v = __ldcg(p + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x == 1234.5f) out[0] = acc.y + acc.z + acc.w;
}
int main() {
    long sizes[] = {16L << 20, 32L << 20, 64L << 20, 96L << 20, 4L << 30};
    float* buf; cudaMalloc(&buf, 4L << 30); cudaMemset(buf, 0, 4L << 30);
    float* out; cudaMalloc(&out, 16);
    for (long bytes : sizes) {
        long n4 = bytes / 16; int reps = (int)((8L << 30) / bytes); if (reps < 1) reps = 1;
        rd<<<148 * 8, 256>>>((float4*)buf, n4, 1, out);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        rd<<<148 * 8, 256>>>((float4*)buf, n4, reps, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("buffer %6.0f MB: %8.1f GB/s\n", bytes / 1048576.0, (double)bytes * reps / ms / 1e6);
    }
}
