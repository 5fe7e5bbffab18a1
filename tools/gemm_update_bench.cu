// Developer benchmark (not part of the library): the blocked-GENP trailing
// update C -= A B at the factorisation's shapes through the library's own
// gemm() (this TU includes dgemm.cu / runtime.cu), forced tile configurations,
// and cuBLAS DGEMM (beta = 1, alpha = -1) on the same operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/gemm_update_bench.cu -lcublas -lcuda -o tools/_build/gemm_update_bench
#include <cublas_v2.h>

#include <cstdio>
#include <vector>

#include "../paper_1406_5802_b200/csrc/runtime.cu"
#include "../paper_1406_5802_b200/csrc/dgemm.cu"

using namespace rl;

int main() {
    rl_context* ctx = nullptr;
    if (rl_context_create(0, &ctx) != RL_OK) return 1;
    cublasHandle_t h;
    cublasCreate(&h);
    cublasSetStream(h, ctx->stream);
    const int64_t nmax = 8192;
    double *a, *b, *c;
    cudaMalloc(&a, nmax * nmax * 8);
    cudaMalloc(&b, nmax * nmax * 8);
    cudaMalloc(&c, nmax * nmax * 8);
    std::vector<double> hv(static_cast<size_t>(nmax) * nmax);
    for (size_t i = 0; i < hv.size(); ++i) hv[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
    cudaMemcpy(a, hv.data(), nmax * nmax * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(b, hv.data(), nmax * nmax * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(c, hv.data(), nmax * nmax * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto&& f) {
        f();
        cudaEventRecord(e0, ctx->stream);
        const int reps = 10;
        for (int i = 0; i < reps; ++i) f();
        cudaEventRecord(e1, ctx->stream);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / reps;
    };
    const int64_t ld = nmax;
    for (int64_t m : {8064, 6144, 4096, 2048, 1024}) {
        for (int64_t k : {64, 128, 256, 512}) {
            const double fl = 2.0 * m * m * k;
            const float t_lib = time([&] { gemm(ctx, m, m, k, a, ld, b, ld, c, ld, -1.0, true, nullptr); });
            const float t_small = time([&] {
                run_cfg<SmallCfg, true, false, true>(ctx, m, m, k, a, ld, b, ld, c, ld, -1.0, nullptr, 1, 0, 0);
            });
            const float t_big = time([&] {
                run_cfg<BigCfg, true, false, true>(ctx, m, m, k, a, ld, b, ld, c, ld, -1.0, nullptr, 1, 0, 0);
            });
            const double one = 1.0, mone = -1.0;
            // row-major C (m x m) = C - A B  <=>  column-major C^T = C^T - B^T A^T
            const float t_cub = time([&] {
                cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, k, &mone, b, ld, a, ld, &one, c, ld);
            });
            std::printf("m=n=%5lld k=%4lld  lib %6.3f ms %5.2f TF/s | small %5.2f | big %5.2f | cublas %5.2f TF/s\n",
                        (long long)m, (long long)k, t_lib, fl / t_lib / 1e9, fl / t_small / 1e9, fl / t_big / 1e9,
                        fl / t_cub / 1e9);
        }
    }
    // long K, as the A*G preprocessing product (no accumulate)
    for (int64_t k : {1024, 2048, 8192}) {
        const int64_t m = 8192;
        const double fl = 2.0 * m * m * k;
        const float t_small = time([&] {
            run_cfg<SmallCfg, false, false, true>(ctx, m, m, k, a, ld, b, ld, c, ld, 1.0, nullptr, 1, 0, 0);
        });
        const float t_big = time([&] {
            run_cfg<BigCfg, false, false, true>(ctx, m, m, k, a, ld, b, ld, c, ld, 1.0, nullptr, 1, 0, 0);
        });
        const double one = 1.0, zero = 0.0;
        const float t_cub = time([&] {
            cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, m, k, &one, b, ld, a, ld, &zero, c, ld);
        });
        std::printf("m=n=%5lld k=%4lld (C = A B)  small %5.2f | big %5.2f | cublas %5.2f TF/s\n", (long long)m,
                    (long long)k, fl / t_small / 1e9, fl / t_big / 1e9, fl / t_cub / 1e9);
    }
    return 0;
}
