// Debug harness for gemm_tc.cu (standalone; not part of the library).
#include "../paper_2408_00232_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace cdfgnn;
namespace cdfgnn { void set_error(const char* fmt, ...) { va_list ap; va_start(ap, fmt); vprintf(fmt, ap); va_end(ap); printf("\n"); } }

int main(int argc, char** argv) {
    int M = 256, N = 64, K = 64;
    if (argc > 3) { M = atoi(argv[1]); N = atoi(argv[2]); K = atoi(argv[3]); }
    std::vector<float> A((size_t)M * K), B((size_t)K * N), C((size_t)M * N, -7.f);
    for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) A[(size_t)m * K + k] = (float)((m * 7 + k * 3) % 11 - 5);
    for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) B[(size_t)k * N + n] = (float)((k * 5 + n) % 7 - 3);
    float *dA, *dB, *dC, *dBt, *dCt;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
    cudaMalloc(&dBt, B.size() * 4); cudaMalloc(&dCt, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    std::vector<float> Bt((size_t)N * K);
    for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) Bt[(size_t)n * K + k] = B[(size_t)k * N + n];
    cudaMemcpy(dBt, Bt.data(), Bt.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dC, 0xFF, C.size() * 4);
    int rc = gemm_tc_fwd(M, N, K, dA, K, dBt, K, dC, N, SPLIT, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("fwd rc=%d err=%s\n", rc, cudaGetErrorString(e));
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0; int bad = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double r = 0; for (int k = 0; k < K; ++k) r += (double)A[(size_t)m*K+k] * B[(size_t)k*N+n];
        double d = fabs(r - C[(size_t)m*N+n]); if (d > maxerr) maxerr = d; if (d > 1e-3 && bad < 5) { printf("  C[%d][%d]=%f ref %f\n", m, n, C[(size_t)m*N+n], r); bad++; }
    }
    printf("fwd (A K-major, B MN-major) maxerr %g\n", maxerr);
    cudaMemset(dCt, 0xFF, C.size() * 4);
    rc = gemm_tc_bwd_data(M, N, K, dA, K, dBt, K, dCt, N, nullptr, 0, SPLIT, 0);
    e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dCt, C.size() * 4, cudaMemcpyDeviceToHost);
    maxerr = 0; bad = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
        double r = 0; for (int k = 0; k < K; ++k) r += (double)A[(size_t)m*K+k] * B[(size_t)k*N+n];
        double d = fabs(r - C[(size_t)m*N+n]); if (d > maxerr) maxerr = d; if (d > 1e-3 && bad < 5) { printf("  C[%d][%d]=%f ref %f\n", m, n, C[(size_t)m*N+n], r); bad++; }
    }
    printf("bwd_data (A K-major, B K-major) rc=%d err=%s maxerr %g\n", rc, cudaGetErrorString(e), maxerr);
    // wgrad: C[M' x N] = Hᵀ S with H [K' x M'] and S [K' x N]; reuse A as H with K'=M, M'=K
    float* ws; cudaMalloc(&ws, (size_t)64 * K * N * 4);
    std::vector<float> Cw((size_t)K * N);
    float* dCw; cudaMalloc(&dCw, Cw.size() * 4);
    std::vector<float> S((size_t)M * N);
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) S[(size_t)m*N+n] = (float)((m + 2*n) % 5 - 2);
    float* dS; cudaMalloc(&dS, S.size() * 4); cudaMemcpy(dS, S.data(), S.size()*4, cudaMemcpyHostToDevice);
    int launches = 0;
    std::vector<float> At((size_t)K * M), St((size_t)N * M);
    for (int m = 0; m < M; ++m) for (int k = 0; k < K; ++k) At[(size_t)k*M+m] = A[(size_t)m*K+k];
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) St[(size_t)n*M+m] = S[(size_t)m*N+n];
    float *dAt, *dSt; cudaMalloc(&dAt, At.size()*4); cudaMalloc(&dSt, St.size()*4);
    cudaMemcpy(dAt, At.data(), At.size()*4, cudaMemcpyHostToDevice); cudaMemcpy(dSt, St.data(), St.size()*4, cudaMemcpyHostToDevice);
    rc = gemm_tc_wgrad(K, N, M, dAt, M, dSt, M, dCw, N, ws, (size_t)64 * K * N, false, SPLIT, 0, &launches);
    e = cudaDeviceSynchronize();
    cudaMemcpy(Cw.data(), dCw, Cw.size() * 4, cudaMemcpyDeviceToHost);
    maxerr = 0; bad = 0;
    for (int i = 0; i < K; ++i) for (int n = 0; n < N; ++n) {
        double r = 0; for (int m = 0; m < M; ++m) r += (double)A[(size_t)m*K+i] * S[(size_t)m*N+n];
        double d = fabs(r - Cw[(size_t)i*N+n]); if (d > maxerr) maxerr = d; if (d > 1e-3 && bad < 5) { printf("  W[%d][%d]=%f ref %f\n", i, n, Cw[(size_t)i*N+n], r); bad++; }
    }
    printf("wgrad (A MN-major, B MN-major) rc=%d err=%s maxerr %g\n", rc, cudaGetErrorString(e), maxerr);
    return 0;
}
