// Dev check (GPU): the batched kernel's reciprocal (MUFU seed + one cubic step, batched32.cu rcp64)
// against 1.0/x over 4M values: seed error and ulp distance. nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/rcp_check.cu
#include <cstdio>
#include <cmath>
#include <cstdint>
__device__ double rcp64(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    const double t = fma(e, e, e);
    return fma(r, t, r);
}
__global__ void k(const double* x, double* seed_err, long long* ulp, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i]));
    seed_err[i] = fabs(fma(-x[i], r, 1.0));
    const double q = 1.0 / x[i], c = rcp64(x[i]);
    ulp[i] = llabs(__double_as_longlong(q) - __double_as_longlong(c));
}
int main() {
    const int n = 1 << 22;
    double* x; double* se; long long* u;
    cudaMallocManaged(&x, n * 8); cudaMallocManaged(&se, n * 8); cudaMallocManaged(&u, n * 8);
    uint64_t s = 12345;
    for (int i = 0; i < n; ++i) {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        const double m = 1.0 + (double)(s >> 11) / 9007199254740992.0;  // [1,2)
        const int e = (int)((s >> 3) % 80) - 40;
        x[i] = ldexp(m, e) * ((s & 1) ? 1.0 : -1.0);
    }
    k<<<n / 256, 256>>>(x, se, u, n);
    cudaDeviceSynchronize();
    double mse = 0; long long mu = 0; long long cnt1 = 0;
    for (int i = 0; i < n; ++i) { if (se[i] > mse) mse = se[i]; if (u[i] > mu) mu = u[i]; if (u[i]) ++cnt1; }
    printf("max seed rel err %.3e (2^%.1f), max ulp diff vs 1.0/x %lld, nonzero %lld of %d\n", mse, log2(mse), mu, cnt1, n);
    return 0;
}
