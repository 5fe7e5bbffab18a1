// TEST INFRASTRUCTURE ONLY — extern "C" entry points over the reference's OWN
// headers (/root/reference/proj/include/randla/*.hpp, compiled read-only from
// where they lie; nothing is copied), built into oracle/_ref/librandla_ref.so
// by oracle/Makefile. Used to validate the plain-C restatement (oracle.c) and
// as bench.py's cpu_baseline / --impl reference arm.
//
// The reference includes <Eigen/Dense>; oracle/ref_shim provides our own
// minimal stand-in whose product routes to the same GEMM hook as oracle.c.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "oracle.h"
#include "randla/block_ge.hpp"
#include "randla/circulant.hpp"
#include "randla/fft.hpp"
#include "randla/lowrank.hpp"
#include "randla/lu.hpp"
#include "randla/multipliers.hpp"
#include "randla/norms.hpp"
#include "randla/parallel.hpp"
#include "randla/preprocess.hpp"
#include "randla/rng.hpp"
#include "randla/stats.hpp"

namespace Eigen::shim {
void gemm_rowmajor(const double* a, const double* b, double* c, Index m, Index k, Index n) {
    or_matmul(m, k, n, a, b, c);
}
void gemm_rowmajor(const std::complex<double>* a, const std::complex<double>* b, std::complex<double>* c,
                   Index m, Index k, Index n) {
    for (Index i = 0; i < m; ++i)
        for (Index j = 0; j < n; ++j) {
            std::complex<double> acc{};
            for (Index t = 0; t < k; ++t) acc += a[i * k + t] * b[t * n + j];
            c[i * n + j] = acc;
        }
}
void singular_values(const double* a, Index m, Index n, double* out) { or_singular_values(m, n, a, out); }
}  // namespace Eigen::shim

using namespace randla;

namespace {
enum { RS_OK = 0, RS_DIM = 1, RS_ZERO_PIVOT = 2, RS_SINGULAR_BLOCK = 3, RS_LOGIC = 5, RS_SINGULAR = 6, RS_OTHER = 9 };

RealMatrix wrap(int64_t m, int64_t n, const double* p) {
    return RealMatrix(static_cast<std::size_t>(m), static_cast<std::size_t>(n), std::vector<double>(p, p + m * n));
}

ComplexMatrix wrapz(int64_t m, int64_t n, const double* p) {
    const Complex* c = reinterpret_cast<const Complex*>(p);
    return ComplexMatrix(static_cast<std::size_t>(m), static_cast<std::size_t>(n), std::vector<Complex>(c, c + m * n));
}

template <typename F>
int guarded(F&& f, int64_t* step = nullptr) {
    try {
        f();
        return RS_OK;
    } catch (const ZeroPivotError& e) {
        if (step) *step = static_cast<int64_t>(e.step);
        return RS_ZERO_PIVOT;
    } catch (const SingularPivotBlockError& e) {
        if (step) *step = static_cast<int64_t>(e.position);
        return RS_SINGULAR_BLOCK;
    } catch (const SingularMatrixError&) {
        return RS_SINGULAR;
    } catch (const DimensionError&) {
        return RS_DIM;
    } catch (const std::logic_error&) {
        return RS_LOGIC;
    } catch (...) {
        return RS_OTHER;
    }
}
}  // namespace

extern "C" {

uint64_t ref_hash_label(const char* s) { return hash_label(s); }
uint64_t ref_derive_seed(uint64_t seed, uint64_t k1, uint64_t k2) { return derive_seed(seed, k1, k2); }

// golden driver (tests/test_testbed.cpp:187-204): trial t draws
// RngStream(derive_seed(seed, hash_label(label), t)).next_double()
// (testbed/experiment.hpp:32-35), then summarize (stats.hpp:19-34)
void ref_golden_draws(const char* label, uint64_t seed, int64_t trials, double* draws, double* stats4) {
    const uint64_t key = hash_label(label);
    std::vector<double> v(static_cast<std::size_t>(trials));
    for (int64_t t = 0; t < trials; ++t) {
        RngStream rng(derive_seed(seed, key, static_cast<uint64_t>(t)));
        v[t] = rng.next_double();
        draws[t] = v[t];
    }
    const StatSummary s = summarize(v);
    stats4[0] = s.mean;
    stats4[1] = s.max;
    stats4[2] = s.min;
    stats4[3] = s.std;
}

void ref_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out) {
    const RealMatrix g = gen_gaussian(static_cast<std::size_t>(m), static_cast<std::size_t>(n), seed);
    std::memcpy(out, g.data(), sizeof(double) * m * n);
}

void ref_gen_finite_set_uniform(int64_t m, int64_t n, uint64_t seed, uint64_t card, double* out) {
    const RealMatrix g = gen_finite_set_uniform(static_cast<std::size_t>(m), static_cast<std::size_t>(n), seed,
                                                static_cast<std::size_t>(card));
    std::memcpy(out, g.data(), sizeof(double) * m * n);
}

// gen_circ_skew_product (multipliers.hpp:164-172), through the shim's GEMM hook
void ref_gen_circ_skew_product(int64_t n, uint64_t seed, double* out) {
    const RealMatrix g = gen_circ_skew_product(static_cast<std::size_t>(n), seed);
    std::memcpy(out, g.data(), sizeof(double) * n * n);
}

void ref_gen_real_circulant_column(int64_t n, uint64_t seed, double* out) {
    const RealCirculant c = gen_real_circulant(static_cast<std::size_t>(n), seed);
    std::memcpy(out, c.first_column().data(), sizeof(double) * n);
}

int ref_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c) {
    return guarded([&] {
        const RealMatrix p = matmul(wrap(m, k, a), wrap(k, n, b));
        std::memcpy(c, p.data(), sizeof(double) * m * n);
    });
}

double ref_spectral_norm_estimate(int64_t m, int64_t n, const double* a) {
    return spectral_norm_estimate(wrap(m, n, a));
}

// genp_factor (lu.hpp:40-58), L and U unpacked into one packed buffer
int ref_genp_factor(int64_t n, const double* a, double* lu, int64_t* zero_step) {
    *zero_step = 0;
    return guarded(
        [&] {
            const LuFactors<double> f = genp_factor(wrap(n, n, a));
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < n; ++j)
                    lu[i * n + j] = (j < i) ? f.lower(static_cast<std::size_t>(i), static_cast<std::size_t>(j))
                                            : f.upper(static_cast<std::size_t>(i), static_cast<std::size_t>(j));
        },
        zero_step);
}

// schur_complement (block_ge.hpp:202-218): E - D B^-1 C for the leading k x k
// block (GEPP on B, so independent of the elimination path)
int ref_schur_complement(int64_t n, const double* a, int64_t k, double* out) {
    return guarded([&] {
        const RealMatrix sc = schur_complement(wrap(n, n, a), static_cast<std::size_t>(k));
        std::memcpy(out, sc.data(), sizeof(double) * (n - k) * (n - k));
    });
}

// lu_solve (lu.hpp:100-123) on packed factors
void ref_lu_solve(int64_t n, const double* lu, const double* b, double* x) {
    LuFactors<double> f{RealMatrix::identity(static_cast<std::size_t>(n)),
                        RealMatrix(static_cast<std::size_t>(n), static_cast<std::size_t>(n)), std::nullopt};
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (j < i)
                f.lower(static_cast<std::size_t>(i), static_cast<std::size_t>(j)) = lu[i * n + j];
            else
                f.upper(static_cast<std::size_t>(i), static_cast<std::size_t>(j)) = lu[i * n + j];
        }
    const std::vector<double> y = lu_solve(f, std::vector<double>(b, b + n));
    std::memcpy(x, y.data(), sizeof(double) * n);
}

int ref_fft(int64_t n, double* z, int inverse) {
    return guarded([&] {
        std::vector<Complex> v(static_cast<std::size_t>(n));
        for (int64_t i = 0; i < n; ++i) v[i] = Complex(z[2 * i], z[2 * i + 1]);
        const std::vector<Complex> w = inverse ? inverse_fft(std::move(v)) : fft(std::move(v));
        for (int64_t i = 0; i < n; ++i) {
            z[2 * i] = w[i].real();
            z[2 * i + 1] = w[i].imag();
        }
    });
}

int ref_circulant_apply(int64_t n, const double* c, const double* x, double* y) {
    return guarded([&] {
        const RealCirculant circ(std::vector<double>(c, c + n));
        const std::vector<double> out = circulant_apply(circ, std::vector<double>(x, x + n));
        std::memcpy(y, out.data(), sizeof(double) * n);
    });
}

int ref_matmul_by_circulant(int64_t m, int64_t n, const double* a, const double* c, double* out) {
    return guarded([&] {
        const RealCirculant circ(std::vector<double>(c, c + n));
        const RealMatrix p = matmul_by_circulant(wrap(m, n, a), circ);
        std::memcpy(out, p.data(), sizeof(double) * m * n);
    });
}

int ref_matmul_by_toeplitz_block(int64_t m, int64_t k, const double* a, int64_t np, const double* c, int64_t l,
                                 double* out) {
    return guarded([&] {
        const ToeplitzBlock<double> t(RealCirculant(std::vector<double>(c, c + np)), static_cast<std::size_t>(k),
                                      static_cast<std::size_t>(l));
        const RealMatrix p = matmul_by_toeplitz_block(wrap(m, k, a), t);
        std::memcpy(out, p.data(), sizeof(double) * m * l);
    });
}

// preprocess_solve(a, b, none, post, refine) (preprocess.hpp:156-180).
// post_kind 0 none, 1 Gaussian with seed, 2 reference RealCirculant (uniform,
// multipliers.hpp:67-73) with seed. history gets refine+1 entries (NaN-padded
// when the loop stopped on divergence).
int ref_preprocess_solve(int64_t n, const double* a, const double* b, int post_kind, uint64_t seed, int64_t refine,
                         double* x, double* history, int* diverged, int64_t* zero_step) {
    *zero_step = 0;
    return guarded(
        [&] {
            MultiplierSpec post;
            post.kind = post_kind == 1   ? MultiplierKind::Gaussian
                        : post_kind == 2 ? MultiplierKind::RealCirculant
                                         : MultiplierKind::None;
            post.seed = seed;
            const SolveOutcome<double> out = preprocess_solve(wrap(n, n, a), std::vector<double>(b, b + n),
                                                              MultiplierSpec{}, post,
                                                              static_cast<std::size_t>(refine));
            std::memcpy(x, out.x.data(), sizeof(double) * n);
            for (int64_t s = 0; s <= refine; ++s)
                history[s] = s < static_cast<int64_t>(out.residual_history.size()) ? out.residual_history[s] : NAN;
            *diverged = out.diverged ? 1 : 0;
        },
        zero_step);
}

// preprocess_solve(a, b, pre, post, refine) with full MultiplierSpecs
// (kinds are the reference's MultiplierKind ordinals, multipliers.hpp:20-29)
int ref_preprocess_solve_spec(int64_t n, const double* a, const double* b, int pre_kind, int pre_variant,
                              uint64_t pre_seed, int post_kind, int post_variant, uint64_t post_seed, uint64_t card,
                              int64_t refine, double* x, double* history, int* diverged, int64_t* zero_step) {
    *zero_step = 0;
    return guarded(
        [&] {
            MultiplierSpec pre, post;
            pre.kind = static_cast<MultiplierKind>(pre_kind);
            pre.variant = static_cast<ToeplitzVariant>(pre_variant);
            pre.seed = pre_seed;
            pre.set_cardinality = static_cast<std::size_t>(card);
            post.kind = static_cast<MultiplierKind>(post_kind);
            post.variant = static_cast<ToeplitzVariant>(post_variant);
            post.seed = post_seed;
            post.set_cardinality = static_cast<std::size_t>(card);
            const SolveOutcome<double> out =
                preprocess_solve(wrap(n, n, a), std::vector<double>(b, b + n), pre, post, static_cast<std::size_t>(refine));
            std::memcpy(x, out.x.data(), sizeof(double) * n);
            for (int64_t s = 0; s <= refine; ++s)
                history[s] = s < static_cast<int64_t>(out.residual_history.size()) ? out.residual_history[s] : NAN;
            *diverged = out.diverged ? 1 : 0;
        },
        zero_step);
}

// the sketch of range_find(a, l, 0, spec, power_steps) (lowrank.hpp:51-81): the
// reference's own multiplier materialization / Toeplitz FFT product and power
// alternation, before its qr (which needs Eigen's Householder QR; the tests
// finish with the restated QR)
int ref_range_sketch(int64_t m, int64_t n, const double* a, int64_t l, int kind, int variant, uint64_t seed,
                     uint64_t card, int64_t power_steps, double* y) {
    return guarded([&] {
        MultiplierSpec spec;
        spec.kind = static_cast<MultiplierKind>(kind);
        spec.variant = static_cast<ToeplitzVariant>(variant);
        spec.seed = seed;
        spec.set_cardinality = static_cast<std::size_t>(card);
        spec.rows = static_cast<std::size_t>(n);
        spec.cols = static_cast<std::size_t>(l);
        const RealMatrix am = wrap(m, n, a);
        RealMatrix sketch(1, 1);
        if (spec.kind == MultiplierKind::ToeplitzBlock) {
            if (spec.variant != ToeplitzVariant::Real) throw DimensionError("complex multiplier family requested in a real pipeline");
            sketch = matmul_by_toeplitz_block(am, gen_real_toeplitz_block(spec.rows, spec.cols, spec.seed));
        } else {
            sketch = matmul(am, materialize<double>(spec));
        }
        for (int64_t s = 0; s < power_steps; ++s) sketch = matmul(am, matmul(am.adjoint(), sketch));
        std::memcpy(y, sketch.data(), sizeof(double) * m * l);
    });
}

// materialize<double>(spec) (multipliers.hpp:174-218)
int ref_materialize(int kind, int variant, uint64_t seed, uint64_t card, int64_t rows, int64_t cols, double* out) {
    return guarded([&] {
        MultiplierSpec spec;
        spec.kind = static_cast<MultiplierKind>(kind);
        spec.variant = static_cast<ToeplitzVariant>(variant);
        spec.seed = seed;
        spec.set_cardinality = static_cast<std::size_t>(card);
        spec.rows = static_cast<std::size_t>(rows);
        spec.cols = static_cast<std::size_t>(cols);
        const RealMatrix g = materialize<double>(spec);
        std::memcpy(out, g.data(), sizeof(double) * rows * cols);
    });
}

// BASELINE config 2 with the reference's own trial pool
// (parallel_for_index, parallel.hpp:14-35): system i uses ts = base + i0 + i
// and the seed mapping of SURVEY §8(d). Returns the number of ZeroPivots.
int64_t ref_batched_config2(int64_t dim, uint64_t base, int64_t i0, int64_t count, double* x_out,
                            double* resid_out) {
    std::vector<int> failed(static_cast<std::size_t>(count), 0);
    const std::size_t d = static_cast<std::size_t>(dim);
    parallel_for_index(static_cast<std::size_t>(count), [&](std::size_t k) {
        const uint64_t ts = base + static_cast<uint64_t>(i0) + k;
        const RealMatrix a = gen_gaussian(d, d, derive_seed(ts, 1));
        RngStream rb(derive_seed(ts, 2));
        std::vector<double> b(d);
        for (double& v : b) v = rb.next_gaussian();
        MultiplierSpec post{MultiplierKind::Gaussian};
        post.seed = derive_seed(ts, 3);
        try {
            const SolveOutcome<double> out = preprocess_solve(a, b, MultiplierSpec{}, post, 0);
            if (x_out) std::memcpy(x_out + k * d, out.x.data(), sizeof(double) * d);
            if (resid_out) resid_out[k] = out.residual_history[0];
        } catch (const ZeroPivotError&) {
            failed[k] = 1;
            if (resid_out) resid_out[k] = NAN;
        }
    });
    int64_t nf = 0;
    for (int f : failed) nf += f;
    return nf;
}

// --impl reference arm: `trials` independent preprocess_solve(A_t, b_t, none,
// {Gaussian, seeds[t]}, 0) calls (the multiplier G_t is generated inside, as
// the reference does) run on the reference's own trial pool
// (parallel_for_index). A_t, b_t are caller-provided so input generation
// stays outside the timed call. Returns the number of ZeroPivots.
int64_t ref_parallel_dense_trials(int64_t n, int64_t trials, const double* a_all, const double* b_all,
                                  const uint64_t* seeds, double* resid_out) {
    std::vector<int> failed(static_cast<std::size_t>(trials), 0);
    const std::size_t nn = static_cast<std::size_t>(n);
    parallel_for_index(static_cast<std::size_t>(trials), [&](std::size_t k) {
        const RealMatrix a = wrap(n, n, a_all + k * nn * nn);
        const std::vector<double> b(b_all + k * nn, b_all + (k + 1) * nn);
        MultiplierSpec post{MultiplierKind::Gaussian};
        post.seed = seeds[k];
        try {
            const SolveOutcome<double> out = preprocess_solve(a, b, MultiplierSpec{}, post, 0);
            if (resid_out) resid_out[k] = out.residual_history[0];
        } catch (const ZeroPivotError&) {
            failed[k] = 1;
            if (resid_out) resid_out[k] = NAN;
        }
    });
    int64_t nf = 0;
    for (int f : failed) nf += f;
    return nf;
}

// gepp_factor (lu.hpp:62-98): packed factors (strict lower of `lower`,
// `upper` on and above the diagonal) and the row permutation
int ref_gepp_factor(int64_t n, const double* a, double* packed, int64_t* perm) {
    return guarded([&] {
        const auto f = gepp_factor(wrap(n, n, a));
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < n; ++j) packed[i * n + j] = j < i ? f.lower(i, j) : f.upper(i, j);
        for (int64_t i = 0; i < n; ++i) perm[i] = static_cast<int64_t>((*f.perm)[i]);
    });
}

// lu_solve / lu_solve_transpose (lu.hpp:100-147) on ref_gepp_factor's output
int ref_gepp_solve(int64_t n, const double* a, const double* b, double* x, int transpose) {
    return guarded([&] {
        const auto f = gepp_factor(wrap(n, n, a));
        const std::vector<double> bv(b, b + n);
        const auto y = transpose ? lu_solve_transpose(f, bv) : lu_solve(f, bv);
        for (int64_t i = 0; i < n; ++i) x[i] = y[i];
    });
}

// block_ge_factor(a, split) (block_ge.hpp:168-181) with pivots(), reassemble(),
// block_solve(b) and the deepest leaf's block_matrix (split.back() squared);
// *position: SingularPivotBlockError's position
int ref_block_ge(int64_t n, const double* a, int64_t nsplit, const int64_t* split, const double* b, double* pivots,
                 double* reassembled, double* x, double* last_leaf, int64_t* position) {
    return guarded(
        [&] {
            std::vector<std::size_t> sp(split, split + nsplit);
            const auto f = block_ge_factor(wrap(n, n, a), sp);
            const auto pv = f.pivots();
            for (int64_t i = 0; i < n; ++i) pivots[i] = pv[i];
            const RealMatrix r = f.reassemble();
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < n; ++j) reassembled[i * n + j] = r(i, j);
            const auto xv = block_solve(f, std::vector<double>(b, b + n));
            for (int64_t i = 0; i < n; ++i) x[i] = xv[i];
            const BlockNode<double>* node = f.root.get();
            while (!node->leaf()) node = node->schur_child.get();
            const int64_t k = static_cast<int64_t>(node->dim);
            for (int64_t i = 0; i < k; ++i)
                for (int64_t j = 0; j < k; ++j) last_leaf[i * k + j] = node->block_matrix(i, j);
        },
        position);
}
// ---- the complex field (Matrix<Complex>): interleaved (re, im) buffers ----

// genp_factor<Complex> (lu.hpp:40-58), packed L\U
int ref_zgenp_factor(int64_t n, const double* a, double* lu, int64_t* zero_step) {
    *zero_step = 0;
    return guarded(
        [&] {
            const LuFactors<Complex> f = genp_factor(wrapz(n, n, a));
            Complex* out = reinterpret_cast<Complex*>(lu);
            for (int64_t i = 0; i < n; ++i)
                for (int64_t j = 0; j < n; ++j)
                    out[i * n + j] = (j < i) ? f.lower(static_cast<std::size_t>(i), static_cast<std::size_t>(j))
                                             : f.upper(static_cast<std::size_t>(i), static_cast<std::size_t>(j));
        },
        zero_step);
}

// preprocess_solve<Complex>(a, b, pre, post, refine) (preprocess.hpp:156-180)
int ref_zpreprocess_solve_spec(int64_t n, const double* a, const double* b, int pre_kind, int pre_variant,
                               uint64_t pre_seed, int post_kind, int post_variant, uint64_t post_seed, uint64_t card,
                               int64_t refine, double* x, double* history, int* diverged, int64_t* zero_step) {
    *zero_step = 0;
    return guarded(
        [&] {
            MultiplierSpec pre, post;
            pre.kind = static_cast<MultiplierKind>(pre_kind);
            pre.variant = static_cast<ToeplitzVariant>(pre_variant);
            pre.seed = pre_seed;
            pre.set_cardinality = static_cast<std::size_t>(card);
            post.kind = static_cast<MultiplierKind>(post_kind);
            post.variant = static_cast<ToeplitzVariant>(post_variant);
            post.seed = post_seed;
            post.set_cardinality = static_cast<std::size_t>(card);
            const Complex* bz = reinterpret_cast<const Complex*>(b);
            const SolveOutcome<Complex> out = preprocess_solve(wrapz(n, n, a), std::vector<Complex>(bz, bz + n), pre,
                                                               post, static_cast<std::size_t>(refine));
            std::memcpy(x, out.x.data(), sizeof(Complex) * n);
            for (int64_t s = 0; s <= refine; ++s)
                history[s] = s < static_cast<int64_t>(out.residual_history.size()) ? out.residual_history[s] : NAN;
            *diverged = out.diverged ? 1 : 0;
        },
        zero_step);
}

// materialize<Complex>(spec) (multipliers.hpp:174-218)
int ref_zmaterialize(int kind, int variant, uint64_t seed, uint64_t card, int64_t rows, int64_t cols, double* out) {
    return guarded([&] {
        MultiplierSpec spec;
        spec.kind = static_cast<MultiplierKind>(kind);
        spec.variant = static_cast<ToeplitzVariant>(variant);
        spec.seed = seed;
        spec.set_cardinality = static_cast<std::size_t>(card);
        spec.rows = static_cast<std::size_t>(rows);
        spec.cols = static_cast<std::size_t>(cols);
        const ComplexMatrix g = materialize<Complex>(spec);
        std::memcpy(out, g.data(), sizeof(Complex) * rows * cols);
    });
}

// the sketch of range_find<Complex> (lowrank.hpp:51-81) before its qr
int ref_zrange_sketch(int64_t m, int64_t n, const double* a, int64_t l, int kind, int variant, uint64_t seed,
                      uint64_t card, int64_t power_steps, double* y) {
    return guarded([&] {
        MultiplierSpec spec;
        spec.kind = static_cast<MultiplierKind>(kind);
        spec.variant = static_cast<ToeplitzVariant>(variant);
        spec.seed = seed;
        spec.set_cardinality = static_cast<std::size_t>(card);
        spec.rows = static_cast<std::size_t>(n);
        spec.cols = static_cast<std::size_t>(l);
        const ComplexMatrix am = wrapz(m, n, a);
        ComplexMatrix sketch(1, 1);
        if (spec.kind == MultiplierKind::ToeplitzBlock) {
            if (spec.variant == ToeplitzVariant::Real)
                sketch = matmul_by_toeplitz_block(am, gen_real_toeplitz_block(spec.rows, spec.cols, spec.seed));
            else
                sketch = matmul_by_toeplitz_block(am, gen_unitary_toeplitz_block(spec.rows, spec.cols, spec.seed));
        } else {
            sketch = matmul(am, materialize<Complex>(spec));
        }
        for (int64_t s = 0; s < power_steps; ++s) sketch = matmul(am, matmul(am.adjoint(), sketch));
        std::memcpy(y, sketch.data(), sizeof(Complex) * m * l);
    });
}

// first column of gen_unitary_circulant (multipliers.hpp:75-82)
void ref_gen_unitary_circulant(int64_t n, uint64_t seed, double* out) {
    const ComplexCirculant c = gen_unitary_circulant(static_cast<std::size_t>(n), seed);
    std::memcpy(out, c.first_column().data(), sizeof(Complex) * n);
}

// srft_columns (multipliers.hpp:132-138)
void ref_srft_columns(int64_t n, int64_t l, uint64_t seed, int64_t* out) {
    const auto cols = srft_columns(static_cast<std::size_t>(n), static_cast<std::size_t>(l), seed);
    for (int64_t j = 0; j < l; ++j) out[j] = static_cast<int64_t>(cols[j]);
}

// the sketching matrix of srft_sketch_check (lowrank.hpp:235-246) for a given
// width l: gen_srft, or the same columns of the unitary circulant drawn from
// the same phases (restated from those lines with the reference's functions)
int ref_srft_matrix(int64_t n, int64_t l, uint64_t seed, int variant, double* out) {
    return guarded([&] {
        const std::size_t nn = static_cast<std::size_t>(n), ll = static_cast<std::size_t>(l);
        ComplexMatrix s(1, 1);
        if (variant == 0) {
            s = gen_srft(nn, ll, seed);
        } else {
            const ComplexCirculant circ = gen_unitary_circulant(nn, seed);
            const auto cols = srft_columns(nn, ll, seed);
            s = ComplexMatrix(nn, ll);
            for (std::size_t i = 0; i < nn; ++i)
                for (std::size_t j = 0; j < ll; ++j) s(i, j) = circ.entry(i, cols[j]);
        }
        std::memcpy(out, s.data(), sizeof(Complex) * n * l);
    });
}

// RngStream(seed).derived(key).next_gaussian() x count (rng.hpp:20-24, :56-71)
void ref_gaussian_derived(uint64_t seed, uint64_t key, int64_t count, double* out) {
    RngStream s = RngStream(seed).derived(key);
    for (int64_t i = 0; i < count; ++i) out[i] = s.next_gaussian();
}

double ref_zspectral_norm_estimate(int64_t m, int64_t n, const double* a) {
    return spectral_norm_estimate(wrapz(m, n, a));
}

// gen_dft_input (testbed/inputs.hpp:52-55) = dft_dense(n) (fft.hpp:21-30)
int ref_dft_dense(int64_t n, double* out) {
    return guarded([&] {
        const ComplexMatrix d = dft_dense(static_cast<std::size_t>(n));
        std::memcpy(out, d.data(), sizeof(Complex) * n * n);
    });
}

}  // extern "C"
