// MN-major tf32 operand check for gemm_tc.cu (standalone; not part of the library):
// C = A B with A [M x K] K-major and B [K x N] row-major fed MN-major (1xTF32).
#include "../paper_2408_00232_b200/csrc/gemm_tc.cu"
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <vector>
using namespace cdfgnn;
namespace cdfgnn { void set_error(const char* fmt, ...) { va_list ap; va_start(ap, fmt); vprintf(fmt, ap); va_end(ap); printf("\n"); } }

int main(int argc, char** argv) {
    int M = 256, N = 64, K = 64;
    if (argc > 3) { M = atoi(argv[1]); N = atoi(argv[2]); K = atoi(argv[3]); }
    std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N);
    for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) A[(size_t)m * K + k] = (float)((m * 7 + k * 3) % 11 - 5);
    for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) B[(size_t)k * N + n] = (float)((k * 5 + n) % 7 - 3);
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xFF, C.size() * 4);
    const int BN = N >= 256 ? 256 : (N >= 128 ? 128 : 64);
    CUtensorMap ta, tb, tc;
    bool ok = make_map(&ta, dA, M, K, K, BK, BM, false) && make_map(&tb, dB, K, N, N, 32, 32, false, true);
    EpiArgs ep{dC, N, nullptr, 0, nullptr, 0, 0, 0};
    ep.tma = make_store_map(&tc, dC, M, N, N, 1, false) ? 1 : 0;
    int rc = ok ? launch_bn<false, true>(BN, false, ta, tb, tc, M, N, K, 1, ep, 0) : -1;
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0; int bad = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double r = 0; for (int k = 0; k < K; ++k) r += (double)A[(size_t)m*K+k] * B[(size_t)k*N+n];
        double d = fabs(r - C[(size_t)m*N+n]); if (d > maxerr) maxerr = d;
        if (d > 1e-3 && bad < 4) { printf("  C[%d][%d]=%f ref %f\n", m, n, C[(size_t)m*N+n], r); bad++; }
    }
    printf("MN-major B (LBO %d SBO %d) M %d N %d K %d: rc=%d err=%s maxerr %g\n", GEMM_MN_LBO, GEMM_MN_SBO, M, N, K,
           rc, cudaGetErrorString(e), maxerr);
    return 0;
}
