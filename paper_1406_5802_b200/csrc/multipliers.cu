// Multiplier specs of the real pipeline (randla::MultiplierSpec,
// multipliers.hpp:20-218) on the device:
//   side_form / sketch_form  how SideMultiplier::make (preprocess.hpp:27-60)
//                            and range_find (lowrank.hpp:62-81) use a spec
//   multiplier_column        first column of a structured (circulant) spec
//   materialize_device       materialize(spec) (multipliers.hpp:174-218)
//   rl_materialize           the same through the C ABI
// Every generator is the reference's, bit for bit (rng_host.cpp,
// rng_device.cu); dense expansions of circulant and skew-circulant columns
// and the circulant x skew-circulant product (gen_circ_skew_product,
// multipliers.hpp:164-172) run on the device.
#include <cstring>
#include <vector>

#include "device_common.cuh"
#include "kernels.cuh"

extern "C" RL_API rl_status rl_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out);
extern "C" RL_API rl_status rl_gen_real_circulant_column(int64_t n, uint64_t seed, double* out);
extern "C" RL_API rl_status rl_gen_finite_set_uniform(int64_t m, int64_t n, uint64_t seed, uint64_t card,
                                                      double* out);

namespace rl {
namespace {

unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__global__ void transpose32_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows, int64_t cols,
                                   double* __restrict__ out, int64_t ldo) {
    __shared__ double t[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) t[i][threadIdx.x] = in[r * ldi + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[c * ldo + r] = t[threadIdx.x][i];
    }
}

// skew_circulant_dense (multipliers.hpp:156-162): (i, j) = c[i - j] for
// i >= j, -c[n + i - j] above the diagonal
__global__ void skew_dense_kernel(const double* __restrict__ c, int64_t n, double* __restrict__ out, int64_t ld) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    const int64_t i = idx / n, j = idx % n;
    out[i * ld + j] = i >= j ? c[i - j] : -c[n + i - j];
}

__global__ void identity_kernel(int64_t n, double* __restrict__ out, int64_t ld) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    const int64_t i = idx / n, j = idx % n;
    out[i * ld + j] = i == j ? 1.0 : 0.0;
}

rl_status complex_family() {
    return set_error(RL_ERR_DIMENSION, "complex multiplier family requested in a real pipeline");
}

bool is_complex(const rl_multiplier* m) {  // multiplier_is_complex (multipliers.hpp:42-52)
    return m->kind == RL_MULT_UNITARY_CIRCULANT || m->kind == RL_MULT_SRFT ||
           (m->kind == RL_MULT_TOEPLITZ_BLOCK && m->variant == RL_TOEPLITZ_UNITARY);
}

bool known(int kind) { return (kind >= RL_MULT_NONE && kind <= RL_MULT_CIRC_SKEW_PRODUCT) || kind == RL_MULT_GAUSSIAN_CIRCULANT; }

rl_status upload(rl_context* ctx, const std::vector<double>& h, double* d) {
    RL_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    RL_CUDA(cudaStreamSynchronize(ctx->stream));  // h is a local of the caller
    return RL_OK;
}

}  // namespace

rl_status StreamBuf::alloc(size_t bytes) {
    RL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes < 16 ? 16 : bytes, s));
    return RL_OK;
}

rl_status transpose_device(rl_context* ctx, const double* in, int64_t ldi, int64_t rows, int64_t cols, double* out,
                           int64_t ldo) {
    transpose32_kernel<<<dim3(nblocks(cols, 32), nblocks(rows, 32)), dim3(32, 8), 0, ctx->stream>>>(in, ldi, rows,
                                                                                                   cols, out, ldo);
    RL_CHECK_LAUNCH("transpose32_kernel");
    return RL_OK;
}

rl_status side_form(const rl_multiplier* m, MForm* out) {
    *out = MForm::NONE;
    if (!m) return RL_OK;
    if (!known(m->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", m->kind);
    if (m->kind == RL_MULT_TOEPLITZ_BLOCK && m->variant != RL_TOEPLITZ_REAL && m->variant != RL_TOEPLITZ_UNITARY)
        return set_error(RL_ERR_INVALID_ARGUMENT, "unknown Toeplitz variant %d", m->variant);
    if (is_complex(m)) return complex_family();
    switch (m->kind) {
        case RL_MULT_NONE: *out = MForm::NONE; break;
        // RealCirculant and the real ToeplitzBlock both keep the full n x n
        // circulant gen_real_circulant(n, seed) structured (preprocess.hpp:36-49)
        case RL_MULT_REAL_CIRCULANT:
        case RL_MULT_TOEPLITZ_BLOCK:
        case RL_MULT_GAUSSIAN_CIRCULANT: *out = MForm::CIRC; break;
        default: *out = MForm::DENSE; break;  // materialize (preprocess.hpp:55-57)
    }
    return RL_OK;
}

rl_status sketch_form(const rl_multiplier* m, int64_t n, int64_t l, MForm* out) {
    *out = MForm::DENSE;
    if (!m) return set_error(RL_ERR_INVALID_ARGUMENT, "range_find: null multiplier spec");
    if (!known(m->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", m->kind);
    if (is_complex(m)) return complex_family();
    switch (m->kind) {
        case RL_MULT_TOEPLITZ_BLOCK:
        case RL_MULT_GAUSSIAN_CIRCULANT: *out = MForm::CIRC; return RL_OK;  // lowrank.hpp:71-73
        case RL_MULT_NONE:
            if (n != l) return set_error(RL_ERR_DIMENSION, "identity multiplier must be square");
            return RL_OK;
        case RL_MULT_REAL_CIRCULANT:
            if (n != l) return set_error(RL_ERR_DIMENSION, "circulant multiplier must be square");
            *out = MForm::CIRC;  // the dense expansion's product equals the circulant's
            return RL_OK;
        case RL_MULT_CIRC_SKEW_PRODUCT:
            if (n != l) return set_error(RL_ERR_DIMENSION, "circulant product multiplier must be square");
            return RL_OK;
        default: return RL_OK;
    }
}

rl_status multiplier_column(const rl_multiplier* m, int64_t n, bool host, std::vector<double>& col) {
    col.assign(static_cast<size_t>(n), 0.0);
    if (m->column) {
        if (host)
            std::memcpy(col.data(), m->column, n * 8);
        else
            RL_CUDA(cudaMemcpy(col.data(), m->column, n * 8, cudaMemcpyDeviceToHost));
        return RL_OK;
    }
    if (m->kind == RL_MULT_GAUSSIAN_CIRCULANT)
        return rl_gen_gaussian(n, 1, m->seed, col.data());  // gen_gaussian_vector (testbed/inputs.hpp:85-90)
    return rl_gen_real_circulant_column(n, m->seed, col.data());  // multipliers.hpp:67-73
}

rl_status materialize_device(rl_context* ctx, const rl_multiplier* m, int64_t rows, int64_t cols, bool host,
                             double* out, int64_t ld) {
    cudaStream_t s = ctx->stream;
    if (!known(m->kind)) return set_error(RL_ERR_INVALID_ARGUMENT, "unknown multiplier kind %d", m->kind);
    if (is_complex(m)) return complex_family();
    if (m->dense) {  // explicit multiplier (rows x cols, row-major)
        RL_CUDA(cudaMemcpy2DAsync(out, ld * 8, m->dense, cols * 8, cols * 8, rows,
                                  host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
        return RL_OK;
    }
    rl_status st;
    switch (m->kind) {
        case RL_MULT_NONE:
            if (rows != cols) return set_error(RL_ERR_DIMENSION, "identity multiplier must be square");
            identity_kernel<<<nblocks(rows * rows, 256), 256, 0, s>>>(rows, out, ld);
            RL_CHECK_LAUNCH("identity_kernel");
            return RL_OK;
        case RL_MULT_GAUSSIAN:  // gen_gaussian(rows, cols, seed), exact, on the device
            return gen_gaussian_device(ctx, rows, cols, m->seed, out, ld, nullptr);
        case RL_MULT_FINITE_SET_UNIFORM: {
            std::vector<double> h(static_cast<size_t>(rows * cols));
            const uint64_t card = m->set_cardinality ? m->set_cardinality : 65536;
            if (card < 2) return set_error(RL_ERR_DIMENSION, "gen_finite_set_uniform: cardinality must be >= 2");
            if ((st = rl_gen_finite_set_uniform(rows, cols, m->seed, card, h.data())) != RL_OK) return st;
            RL_CUDA(cudaMemcpy2DAsync(out, ld * 8, h.data(), cols * 8, cols * 8, rows, cudaMemcpyHostToDevice, s));
            RL_CUDA(cudaStreamSynchronize(s));
            return RL_OK;
        }
        case RL_MULT_REAL_CIRCULANT:
        case RL_MULT_TOEPLITZ_BLOCK:
        case RL_MULT_GAUSSIAN_CIRCULANT: {
            // dense() of the rows x rows circulant (RealCirculant: square) or its
            // leading rows x cols block (gen_real_toeplitz_block(rows, cols, seed))
            if (m->kind == RL_MULT_REAL_CIRCULANT && rows != cols)
                return set_error(RL_ERR_DIMENSION, "circulant multiplier must be square");
            if (cols > rows) return set_error(RL_ERR_DIMENSION, "toeplitz block exceeds parent dimensions");
            std::vector<double> col;
            if ((st = multiplier_column(m, rows, host, col)) != RL_OK) return st;
            StreamBuf dc(s);
            if ((st = dc.alloc(rows * 8)) != RL_OK) return st;
            if ((st = upload(ctx, col, dc.p)) != RL_OK) return st;
            return circulant_dense(ctx, dc.p, rows, rows, cols, out, ld);
        }
        case RL_MULT_CIRC_SKEW_PRODUCT: {
            // gen_circ_skew_product (multipliers.hpp:164-172): the real circulant
            // of derive_seed(seed, 1) times the skew-circulant whose column is
            // next_symmetric draws of derive_seed(seed, 2)
            if (rows != cols) return set_error(RL_ERR_DIMENSION, "circulant product multiplier must be square");
            const int64_t n = rows, ldn = (n + 1) & ~int64_t(1);
            std::vector<double> c1(static_cast<size_t>(n)), c2(static_cast<size_t>(n));
            rl_gen_real_circulant_column(n, rl_derive_seed(m->seed, 1, 0), c1.data());
            rl_gen_real_circulant_column(n, rl_derive_seed(m->seed, 2, 0), c2.data());
            StreamBuf buf(s);
            if ((st = buf.alloc((2 * n + 2 * n * ldn) * 8)) != RL_OK) return st;
            double *d1 = buf.p, *d2 = buf.p + n, *cd = buf.p + 2 * n, *sd = cd + n * ldn;
            RL_CUDA(cudaMemcpyAsync(d1, c1.data(), n * 8, cudaMemcpyHostToDevice, s));
            RL_CUDA(cudaMemcpyAsync(d2, c2.data(), n * 8, cudaMemcpyHostToDevice, s));
            if ((st = circulant_dense(ctx, d1, n, n, n, cd, ldn)) != RL_OK) return st;
            skew_dense_kernel<<<nblocks(n * n, 256), 256, 0, s>>>(d2, n, sd, ldn);
            RL_CHECK_LAUNCH("skew_dense_kernel");
            if ((st = gemm(ctx, n, n, n, cd, ldn, sd, ldn, out, ld, 1.0, false, nullptr)) != RL_OK) return st;
            RL_CUDA(cudaStreamSynchronize(s));  // c1, c2 are locals
            return RL_OK;
        }
        default: return complex_family();
    }
}

}  // namespace rl

using namespace rl;

extern "C" RL_API rl_status rl_materialize(rl_context* ctx, rl_mem mem, const rl_multiplier* spec, int64_t rows,
                                           int64_t cols, double* out) {
    if (!spec || !out) return set_error(RL_ERR_INVALID_ARGUMENT, "materialize: null pointer");
    if (rows <= 0 || cols <= 0) return set_error(RL_ERR_DIMENSION, "materialize: empty shape");
    rl_status st;
    ctx = resolve(ctx, &st);
    if (!ctx) return st;
    const bool host = mem == RL_HOST;
    const int64_t ld = (cols + 1) & ~int64_t(1);
    // the GEMM of the skew product needs even leading dimensions: stage unless
    // device memory already fits
    const bool stage = host || (cols & 1) || (reinterpret_cast<uintptr_t>(out) & 15);
    StreamBuf tmp(ctx->stream);
    double* d = out;
    if (stage) {
        if ((st = tmp.alloc(rows * ld * 8)) != RL_OK) return st;
        d = tmp.p;
    }
    if ((st = materialize_device(ctx, spec, rows, cols, host, d, stage ? ld : cols)) != RL_OK) return st;
    if (stage)
        RL_CUDA(cudaMemcpy2DAsync(out, cols * 8, d, ld * 8, cols * 8, rows,
                                  host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
    if (host) RL_CUDA(cudaStreamSynchronize(ctx->stream));
    return RL_OK;
}
