// Which fp32 -> tf32 conversion does kind::tf32 apply to RAW fp32 operands (FLOAT32 tensor map)?  (debug only)
#include "../paper_2408_00232_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <vector>
#include <cmath>
#include <random>
namespace cdfgnn { void set_error(const char* fmt, ...) { va_list ap; va_start(ap, fmt); vprintf(fmt, ap); va_end(ap); printf("\n"); } }
using namespace cdfgnn;
static float h_tf32_rn(float x) { uint32_t u; memcpy(&u, &x, 4); uint32_t r = u + 0xFFFu + ((u >> 13) & 1u); r &= ~0x1FFFu; float y; memcpy(&y, &r, 4); return y; }
static float tf32_rna(float x) { uint32_t u; memcpy(&u, &x, 4); uint32_t r = (u + 0x1000u) & ~0x1FFFu; float y; memcpy(&y, &r, 4); return y; }
static float h_tf32_tr(float x) { uint32_t u; memcpy(&u, &x, 4); u &= ~0x1FFFu; float y; memcpy(&y, &u, 4); return y; }
int main() {
    int M = 256, N = 64, K = 64;
    std::mt19937 g(1); std::normal_distribution<float> nd;
    std::vector<float> A((size_t)M*K), Bt((size_t)N*K), C((size_t)M*N);
    for (auto& x : A) x = nd(g); for (auto& x : Bt) x = nd(g);
    float *dA, *dB, *dC; cudaMalloc(&dA, A.size()*4); cudaMalloc(&dB, Bt.size()*4); cudaMalloc(&dC, C.size()*4);
    cudaMemcpy(dA, A.data(), A.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dB, Bt.data(), Bt.size()*4, cudaMemcpyHostToDevice);
    CUtensorMap ta, tb;
    if (!make_map(&ta, dA, M, K, K, BK, BM, true) || !make_map(&tb, dB, N, K, K, BK, 64, true)) { printf("map fail\n"); return 1; }
    EpiArgs ep{dC, N, nullptr, 0, nullptr, 0, 0, 0};
    CUtensorMap tc;
    int rc = launch_bn<false, false>(64, false, ta, tb, tc, M, N, K, 1, ep, 0); cudaDeviceSynchronize();
    printf("rc %d err %s\n", rc, cudaGetErrorString(cudaGetLastError()));
    cudaMemcpy(C.data(), dC, C.size()*4, cudaMemcpyDeviceToHost);
    double e[4] = {0,0,0,0};
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double r[4] = {0,0,0,0};
        for (int k = 0; k < K; ++k) {
            float a = A[(size_t)m*K+k], b = Bt[(size_t)n*K+k];
            r[0] += (double)a*b; r[1] += (double)h_tf32_rn(a)*h_tf32_rn(b); r[2] += (double)h_tf32_tr(a)*h_tf32_tr(b); r[3] += (double)tf32_rna(a)*tf32_rna(b);
        }
        for (int i = 0; i < 4; ++i) e[i] = fmax(e[i], fabs(r[i] - C[(size_t)m*N+n]));
    }
    printf("max |C - ref|: exact %g  rn-even %g  trunc %g  rn-away %g\n", e[0], e[1], e[2], e[3]);
}
