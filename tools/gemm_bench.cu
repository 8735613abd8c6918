// GEMM timing harness (debug tool): times gemm_tc_fwd / bwd_data / wgrad on GCN shapes.
#include "../paper_2408_00232_b200/csrc/gemm_tc.cu"
#include <cstdio>
#include <functional>
#include <vector>
namespace cdfgnn { void set_error(const char* fmt, ...) { va_list ap; va_start(ap, fmt); vprintf(fmt, ap); va_end(ap); printf("\n"); } }
using namespace cdfgnn;
static float time_it(std::function<void()> f, int reps = 5) {
    f(); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int i = 0; i < reps; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}
int main(int argc, char** argv) {
    struct S { long M, N, K; const char* name; } shapes[] = {
        {232965, 256, 604, "C3 fwd l1"}, {232965, 44, 256, "C3 fwd l2"}, {232965, 256, 44, "C3 bwd_data l2"},
        {1630000, 256, 100, "C4 fwd l1 (p=4)"}, {1630000, 256, 256, "C4 fwd l2 (p=4)"}};
    float *A, *B, *C, *ws;
    cudaMalloc(&A, 2L << 30); cudaMalloc(&B, 64L << 20); cudaMalloc(&C, 2L << 30); cudaMalloc(&ws, 512L << 20);
    cudaMemset(A, 0, 2L << 30); cudaMemset(B, 0, 64L << 20);
    for (int split = 0; split <= 1; ++split) {
        for (auto& sh : shapes) {
            long ldk = (sh.K + 3) / 4 * 4, ldn = (sh.N + 3) / 4 * 4;
            float ms = time_it([&] { gemm_tc_fwd(sh.M, sh.N, sh.K, A, ldk, B, ldk, C, ldn, split, 0); });
            double tf = 2.0 * sh.M * sh.N * sh.K / (ms * 1e-3) / 1e12;
            double gb = (4.0 * sh.M * ldk + 4.0 * sh.M * ldn) / (ms * 1e-3) / 1e9;
            printf("%s %-18s fwd  %8.1f us  %7.1f TF/s(useful)  %7.1f GB/s\n", split ? "3xTF32" : "1xTF32", sh.name, ms * 1e3, tf, gb);
            ms = time_it([&] { gemm_tc_bwd_data(sh.M, sh.N, sh.K, A, ldk, B, ldk, C, ldn, C, ldn, split, 0); });
            printf("%s %-18s data %8.1f us\n", split ? "3xTF32" : "1xTF32", sh.name, ms * 1e3);
        }
        long n = 232965; long npad = (n + 3) / 4 * 4;
        float ms = time_it([&] { int l = 0; gemm_tc_wgrad(604, 256, n, A, npad, A + 604 * npad, npad, C, 256, ws, 128L << 20, false, split, 0, &l); });
        printf("%s %-18s wgrad %8.1f us  %7.1f TF/s(useful)\n", split ? "3xTF32" : "1xTF32", "C3 wgrad l1", ms * 1e3, 2.0 * 604 * 256 * n / (ms * 1e-3) / 1e12);
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
