// randla_b200/randla.hpp — C++ drop-in for the hot path of the reference
// `randla` header library (namespace randla, /root/reference/proj/include/
// randla/*.hpp, double instantiation), implemented over the C ABI in
// randla_capi.h. A reference user swaps the reference's includes
//     #include "randla/preprocess.hpp"   ->   #include "randla_b200/randla.hpp"
// (or puts include/randla_dropin first on the include path, whose
// randla/*.hpp files forward here) and links librandla_b200.so; the names,
// argument meaning and exception types below are the reference's. Every
// computation on the path runs on the GPU; there is no CPU fallback (a host
// without a CUDA device gets DeviceError). Requires C++20, as the reference.
//
// Covered (reference file:line):
//   Complex, field, tol_*, exception types   types.hpp:9-78
//   RngStream, hash_label                    rng.hpp:16-95 (host, bit-identical)
//   Matrix<T> (double and Complex), matmul,
//   +, -, scalar *, matvec, frobenius_norm,
//   max_abs, norm2, to_complex               matrix.hpp:15-203 (matmul<double> on the GPU)
//   svd_values, spectral_norm, TruncatedSVD  svd.hpp:32-88, norms.hpp:11-14 (device Jacobi)
//   spectral_norm_estimate                   norms.hpp:35-78
//   fft, inverse_fft, dft_dense              fft.hpp:21-98 (GPU transforms)
//   CirculantMatrix/RealCirculant,
//   circulant_apply, circulant_solve,
//   spectrum_range, circulant_is_singular,
//   ToeplitzBlock, matmul_by_circulant,
//   matmul_by_toeplitz_block                 circulant.hpp:17-203
//   MultiplierKind, ToeplitzVariant,
//   MultiplierSpec, multiplier_is_complex,
//   derive_seed, gen_gaussian,
//   gen_real_circulant, gen_real_toeplitz_block,
//   gen_finite_set_uniform, gen_circ_skew_product,
//   materialize                              multipliers.hpp:20-218
//   LuFactors, genp_factor, lu_solve         lu.hpp:17-28, :40-58, :100-123
//   gepp_factor, lu_solve_transpose          lu.hpp:62-98, :127-147 (bit-identical)
//   BlockNode, BlockFactorization,
//   block_ge_factor, block_solve,
//   balanced_split, schur_complement         block_ge.hpp:18-218 (bit-identical)
//   relative_residual                        lu.hpp:155-161
//   SolveOutcome, SideMultiplier,
//   iterative_refine, preprocess_solve,
//   preprocess_solve_with_retry              preprocess.hpp:9-196
//   QrResult, qr, orthonormal_basis          qr.hpp:17-54 (CholeskyQR2 on the GPU)
//   LowRankResult, range_find_with,
//   range_find, approximation_residual,
//   basis_residual, subspace_residual        lowrank.hpp:21-113
//   testbed::gen_lownumrank, gen_hard_block,
//   gen_gaussian_vector, LowRankInstance     testbed/inputs.hpp:18-90
//   batched_preprocess_solve_32              BASELINE config 2 (no reference counterpart:
//                                            the reference loops preprocess_solve per trial)
//   the complex field: ComplexCirculant, gen_unitary_circulant,
//   gen_unitary_toeplitz_block, gen_srft, srft_from_parts, srft_columns,
//   materialize<Complex>, genp_factor / lu_solve / preprocess_solve /
//   range_find / qr over Complex, srft_sketch_check  multipliers.hpp:75-138,
//                                            lowrank.hpp:199-261 (complex.cu on the GPU)
//   parse/format_multiplier_token            multipliers.hpp:222-275
//   StatSummary, summarize, parallel_for_index,
//   RandomNormStats, probe_norm_stats        stats.hpp, parallel.hpp, norm_stats.hpp
// Elementwise Matrix<T> arithmetic (+, -, scalar *, matvec) is host code, as in
// the reference; every product, factorization, transform and sketch runs on
// the GPU.
#pragma once

#include <algorithm>
#include <cmath>
#include <complex>
#include <concepts>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <numbers>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "randla_capi.h"

namespace randla {

// ---- scalar fields, tolerances, error contract (types.hpp:9-78) -------------
using Complex = std::complex<double>;

template <typename T>
struct field {
    static constexpr bool is_complex = false;
    using real_type = T;
    static T conj(T x) { return x; }
    static double abs2(T x) { return x * x; }
    static double real(T x) { return x; }
    static double imag(T) { return 0.0; }
};
template <>
struct field<Complex> {
    static constexpr bool is_complex = true;
    using real_type = double;
    static Complex conj(Complex x) { return std::conj(x); }
    static double abs2(Complex x) { return std::norm(x); }
    static double real(Complex x) { return x.real(); }
    static double imag(Complex x) { return x.imag(); }
};
template <typename T>
concept ScalarField = std::is_same_v<T, double> || std::is_same_v<T, Complex>;

inline double tol_orth(std::size_t m, std::size_t n) { return 1e-10 * static_cast<double>(std::max(m, n)); }
inline double tol_recon(std::size_t m, std::size_t n) { return 1e-10 * static_cast<double>(std::max(m, n)); }
inline double tol_rank(std::size_t m, std::size_t n) { return 1e-13 * static_cast<double>(std::max(m, n)); }
inline double tol_pivot(std::size_t n) { return 1e-13 * static_cast<double>(n); }

struct DimensionError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct SingularMatrixError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RankDeficiencyError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ZeroPivotError : std::runtime_error {
    std::size_t step;
    explicit ZeroPivotError(std::size_t s)
        : std::runtime_error("zero pivot at elimination step " + std::to_string(s)), step(s) {}
};
struct SingularPivotBlockError : std::runtime_error {
    std::size_t position;
    explicit SingularPivotBlockError(std::size_t p)
        : std::runtime_error("numerically singular pivot block at position " + std::to_string(p)), position(p) {}
};
struct ConvergenceError : std::runtime_error {
    std::size_t iterations;
    ConvergenceError(const std::string& what, std::size_t it)
        : std::runtime_error(what + " (after " + std::to_string(it) + " iterations)"), iterations(it) {}
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
// the device failed (no GPU, CUDA error, out of memory): no reference counterpart
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(rl_status st, int64_t where = 0) {
    switch (st) {
        case RL_OK: return;
        case RL_ERR_DIMENSION: throw DimensionError(rl_last_error());
        case RL_ERR_ZERO_PIVOT: throw ZeroPivotError(static_cast<std::size_t>(where));
        case RL_ERR_SINGULAR_PIVOT_BLOCK: throw SingularPivotBlockError(static_cast<std::size_t>(where));
        case RL_ERR_RANK_DEFICIENCY: throw RankDeficiencyError(rl_last_error());
        case RL_ERR_SINGULAR_MATRIX: throw SingularMatrixError(rl_last_error());
        case RL_ERR_LOGIC: throw std::logic_error(rl_last_error());
        default: throw DeviceError(std::string("librandla_b200: ") + rl_last_error());
    }
}
inline int64_t i64(std::size_t v) { return static_cast<int64_t>(v); }
}  // namespace detail

// ---- seeded streams (rng.hpp:16-95), host, the reference's arithmetic -----------
// splitmix64 counter stream: every draw is finalize(state + k * golden); the
// Gaussian is Marsaglia's polar method with the spare kept.
class RngStream {
  public:
    explicit RngStream(std::uint64_t seed) : state_(mix_key(kGolden, seed)) {}
    RngStream derived(std::uint64_t key) const {
        RngStream s(*this);
        s.state_ = mix_key(s.state_, key);
        s.has_spare_ = false;
        return s;
    }
    RngStream derived(std::uint64_t key1, std::uint64_t key2) const { return derived(key1).derived(key2); }
    std::uint64_t next_u64() {
        state_ += kGolden;
        return finalize(state_);
    }
    double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_symmetric() { return 2.0 * next_double() - 1.0; }
    std::uint64_t next_below(std::uint64_t bound) {
        const std::uint64_t limit = bound * (~std::uint64_t{0} / bound);
        for (;;) {
            const std::uint64_t v = next_u64();
            if (v < limit) return v % bound;
        }
    }
    double next_gaussian() {
        if (has_spare_) {
            has_spare_ = false;
            return spare_;
        }
        for (;;) {
            const double u = next_symmetric();
            const double v = next_symmetric();
            const double s = u * u + v * v;
            if (s >= 1.0 || s == 0.0) continue;
            const double f = std::sqrt(-2.0 * std::log(s) / s);
            spare_ = v * f;
            has_spare_ = true;
            return u * f;
        }
    }

  private:
    static constexpr std::uint64_t kGolden = 0x9E3779B97F4A7C15ull;
    static std::uint64_t finalize(std::uint64_t z) {
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    static std::uint64_t mix_key(std::uint64_t state, std::uint64_t key) {
        state ^= key + kGolden + (state << 6) + (state >> 2);
        return finalize(state + kGolden);
    }
    std::uint64_t state_;
    bool has_spare_ = false;
    double spare_ = 0.0;
};

inline std::uint64_t hash_label(const char* s) { return rl_hash_label(s); }

// ---- dense row-major matrix (matrix.hpp:15-110) ----------------------------------
template <ScalarField T>
class Matrix {
  public:
    using value_type = T;
    Matrix() = default;
    Matrix(std::size_t rows, std::size_t cols, T fill = T{}) : r_(rows), c_(cols), e_(rows * cols, fill) {
        if (rows == 0 || cols == 0) throw DimensionError("matrix dimensions must be positive");
    }
    Matrix(std::size_t rows, std::size_t cols, std::vector<T> entries) : r_(rows), c_(cols), e_(std::move(entries)) {
        if (rows == 0 || cols == 0) throw DimensionError("matrix dimensions must be positive");
        if (e_.size() != rows * cols) throw DimensionError("entry count does not match rows*cols");
    }
    static Matrix identity(std::size_t n) {
        Matrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = T{1};
        return m;
    }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    T& operator()(std::size_t i, std::size_t j) { return e_[i * c_ + j]; }
    const T& operator()(std::size_t i, std::size_t j) const { return e_[i * c_ + j]; }
    const std::vector<T>& entries() const { return e_; }
    T* data() { return e_.data(); }
    const T* data() const { return e_.data(); }

    Matrix leading_block(std::size_t k, std::size_t l) const {
        if (k == 0 || l == 0 || k > r_ || l > c_) throw DimensionError("leading block exceeds matrix dimensions");
        return block(0, 0, k, l);
    }
    Matrix block(std::size_t row0, std::size_t col0, std::size_t k, std::size_t l) const {
        if (row0 + k > r_ || col0 + l > c_) throw DimensionError("block exceeds matrix dimensions");
        Matrix out(k, l);
        for (std::size_t i = 0; i < k; ++i)
            std::copy_n(e_.begin() + static_cast<std::ptrdiff_t>((row0 + i) * c_ + col0), l,
                        out.e_.begin() + static_cast<std::ptrdiff_t>(i * l));
        return out;
    }
    void set_block(std::size_t row0, std::size_t col0, const Matrix& b) {
        if (row0 + b.rows() > r_ || col0 + b.cols() > c_) throw DimensionError("block exceeds matrix dimensions");
        for (std::size_t i = 0; i < b.rows(); ++i)
            std::copy_n(b.e_.begin() + static_cast<std::ptrdiff_t>(i * b.c_), b.c_,
                        e_.begin() + static_cast<std::ptrdiff_t>((row0 + i) * c_ + col0));
    }
    Matrix transpose() const {
        Matrix out(c_, r_);
        for (std::size_t i = 0; i < r_; ++i)
            for (std::size_t j = 0; j < c_; ++j) out(j, i) = (*this)(i, j);
        return out;
    }
    Matrix adjoint() const {  // conjugate transpose; plain transpose over the reals
        Matrix out(c_, r_);
        for (std::size_t i = 0; i < r_; ++i)
            for (std::size_t j = 0; j < c_; ++j) out(j, i) = field<T>::conj((*this)(i, j));
        return out;
    }
    std::vector<T> col(std::size_t j) const {
        std::vector<T> v(r_);
        for (std::size_t i = 0; i < r_; ++i) v[i] = (*this)(i, j);
        return v;
    }
    std::vector<T> row(std::size_t i) const {
        return std::vector<T>(e_.begin() + static_cast<std::ptrdiff_t>(i * c_),
                              e_.begin() + static_cast<std::ptrdiff_t>((i + 1) * c_));
    }
    bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && e_ == o.e_; }

  private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<T> e_;
};
using RealMatrix = Matrix<double>;
using ComplexMatrix = Matrix<Complex>;

// C = A B (matrix.hpp:115-121): the FP64 DMMA GEMM; a complex product runs
// as one real GEMM on [Ar | Ai] x [[Br, Bi], [-Bi, Br]]
template <ScalarField T>
Matrix<T> matmul(const Matrix<T>& a, const Matrix<T>& b) {
    if (a.cols() != b.rows()) throw DimensionError("matmul: inner dimensions differ");
    Matrix<T> out(a.rows(), b.cols());
    const std::size_t m = a.rows(), k = a.cols(), n = b.cols();
    if constexpr (std::is_same_v<T, double>) {
        detail::check(rl_dgemm(nullptr, RL_HOST, detail::i64(m), detail::i64(n), detail::i64(k), a.data(),
                               detail::i64(k), b.data(), detail::i64(n), out.data(), detail::i64(n)));
    } else {
        detail::check(rl_zgemm(nullptr, RL_HOST, detail::i64(m), detail::i64(n), detail::i64(k),
                               reinterpret_cast<const double*>(a.data()), reinterpret_cast<const double*>(b.data()),
                               reinterpret_cast<double*>(out.data())));
    }
    return out;
}

template <ScalarField T>
Matrix<T> operator+(const Matrix<T>& a, const Matrix<T>& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw DimensionError("add: shape mismatch");
    Matrix<T> out(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) out(i, j) = a(i, j) + b(i, j);
    return out;
}
template <ScalarField T>
Matrix<T> operator-(const Matrix<T>& a, const Matrix<T>& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw DimensionError("sub: shape mismatch");
    Matrix<T> out(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) out(i, j) = a(i, j) - b(i, j);
    return out;
}
template <ScalarField T, typename S>
Matrix<T> operator*(S scalar, const Matrix<T>& a) {
    Matrix<T> out(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) out(i, j) = T(scalar) * a(i, j);
    return out;
}

template <ScalarField T>
std::vector<T> matvec(const Matrix<T>& a, const std::vector<T>& x) {  // matrix.hpp:146-156
    if (a.cols() != x.size()) throw DimensionError("matvec: shape mismatch");
    std::vector<T> y(a.rows(), T{});
    for (std::size_t i = 0; i < a.rows(); ++i) {
        T acc{};
        for (std::size_t j = 0; j < a.cols(); ++j) acc += a(i, j) * x[j];
        y[i] = acc;
    }
    return y;
}
template <ScalarField T>
double frobenius_norm(const Matrix<T>& a) {
    double s = 0.0;
    for (const T& v : a.entries()) s += field<T>::abs2(v);
    return std::sqrt(s);
}
template <ScalarField T>
double max_abs(const Matrix<T>& a) {
    double m = 0.0;
    for (const T& v : a.entries()) m = std::max(m, std::sqrt(field<T>::abs2(v)));
    return m;
}
template <ScalarField T>
double norm2(const std::vector<T>& v) {
    double s = 0.0;
    for (const T& x : v) s += field<T>::abs2(x);
    return std::sqrt(s);
}
inline ComplexMatrix to_complex(const RealMatrix& a) {
    ComplexMatrix out(a.rows(), a.cols());
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) out(i, j) = Complex(a(i, j), 0.0);
    return out;
}
inline const ComplexMatrix& to_complex(const ComplexMatrix& a) { return a; }
namespace detail {
inline std::vector<Complex> to_complex_vec(const std::vector<double>& v) {
    std::vector<Complex> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = Complex(v[i], 0.0);
    return out;
}
inline const std::vector<Complex>& to_complex_vec(const std::vector<Complex>& v) { return v; }
}  // namespace detail
inline std::vector<Complex> to_complex(const std::vector<double>& v) {
    std::vector<Complex> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = Complex(v[i], 0.0);
    return out;
}

// ---- singular values (svd.hpp:32-88, norms.hpp:11-33) ------------------------------
// svd_values by the device's one-sided Jacobi; a complex A = X + iY through its
// real embedding [[X, -Y], [Y, X]], whose singular values are A's, each twice
template <ScalarField T>
std::vector<double> svd_values(const Matrix<T>& a) {
    if constexpr (std::is_same_v<T, double>) {
        std::vector<double> sv(std::min(a.rows(), a.cols()));
        detail::check(rl_singular_values(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                         sv.data()));
        return sv;
    } else {
        const std::size_t m = a.rows(), n = a.cols();
        RealMatrix e(2 * m, 2 * n);
        for (std::size_t i = 0; i < m; ++i)
            for (std::size_t j = 0; j < n; ++j) {
                e(i, j) = e(m + i, n + j) = a(i, j).real();
                e(m + i, j) = a(i, j).imag();
                e(i, n + j) = -a(i, j).imag();
            }
        const std::vector<double> twice = svd_values(e);
        std::vector<double> sv(std::min(m, n));
        for (std::size_t i = 0; i < sv.size(); ++i) sv[i] = twice[2 * i];
        return sv;
    }
}
template <ScalarField T>
double spectral_norm(const Matrix<T>& a) {
    return svd_values(a).front();
}
template <ScalarField T>
double pseudo_inverse_norm(const Matrix<T>& a) {
    const double smin = svd_values(a).back();
    if (smin == 0.0) throw SingularMatrixError("pseudo-inverse norm of an exactly singular matrix");
    return 1.0 / smin;
}
template <ScalarField T>
double condition_number(const Matrix<T>& a) {
    const auto sv = svd_values(a);
    if (sv.back() == 0.0) throw SingularMatrixError("condition number of an exactly singular matrix");
    return sv.front() / sv.back();
}

template <ScalarField T>
struct TruncatedSVD {
    Matrix<T> left;                 // m-by-r
    std::vector<double> singulars;  // r leading values
    Matrix<T> right;                // n-by-r
    Matrix<T> reconstruct() const {
        Matrix<T> scaled = left;
        for (std::size_t j = 0; j < singulars.size(); ++j)
            for (std::size_t i = 0; i < scaled.rows(); ++i) scaled(i, j) *= T(singulars[j]);
        return matmul(scaled, right.adjoint());
    }
};

// spectral_norm_estimate (norms.hpp:35-78): the reference's power iteration, in
// its summation order, on the GPU
inline double spectral_norm_estimate(const RealMatrix& a) {
    double out = 0.0;
    detail::check(rl_spectral_norm_estimate(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                            &out));
    return out;
}
// complex A: the same power iteration on the real embedding [[X, -Y], [Y, X]]
// (the same singular values and row / column norms; the start vector differs,
// so the estimate agrees to the iteration's 1e-9 stopping tolerance)
inline double spectral_norm_estimate(const ComplexMatrix& a) {
    const std::size_t m = a.rows(), n = a.cols();
    RealMatrix e(2 * m, 2 * n);
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            e(i, j) = e(m + i, n + j) = a(i, j).real();
            e(m + i, j) = a(i, j).imag();
            e(i, n + j) = -a(i, j).imag();
        }
    return spectral_norm_estimate(e);
}

// ---- transforms (fft.hpp) ----------------------------------------------------------
inline bool is_power_of_two(std::size_t n) { return n != 0 && (n & (n - 1)) == 0; }

// n-by-n matrix with entry (i, j) = omega^{ij}, omega = exp(+2 pi i / n)
inline ComplexMatrix dft_dense(std::size_t n) {
    if (n < 1) throw DimensionError("dft_dense: n must be positive");
    std::vector<Complex> root(n);
    for (std::size_t k = 0; k < n; ++k)
        root[k] = std::polar(1.0, 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n));
    ComplexMatrix out(n, n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) out(i, j) = root[(i * j) % n];
    return out;
}

namespace detail {
inline std::vector<Complex> transform(std::vector<Complex> v, bool inverse) {
    if (v.empty()) throw DimensionError(inverse ? "inverse_fft: empty input" : "fft: empty input");
    check(rl_fft(nullptr, RL_HOST, 1, i64(v.size()), reinterpret_cast<double*>(v.data()), inverse ? 1 : 0));
    return v;
}
}  // namespace detail

inline std::vector<Complex> fft(std::vector<Complex> v) { return detail::transform(std::move(v), false); }
inline std::vector<Complex> fft(const std::vector<double>& v) { return fft(to_complex(v)); }
inline std::vector<Complex> inverse_fft(std::vector<Complex> v) { return detail::transform(std::move(v), true); }

// ---- circulants (circulant.hpp:17-203), real field -------------------------------
template <ScalarField T>
class CirculantMatrix {
  public:
    explicit CirculantMatrix(std::vector<T> first_column) : c_(std::move(first_column)) {
        if (c_.empty()) throw DimensionError("circulant: empty first column");
        spectrum_ = fft(c_);  // eager, as the reference (circulant.hpp:19-22)
    }
    std::size_t size() const { return c_.size(); }
    const std::vector<T>& first_column() const { return c_; }
    const std::vector<Complex>& spectrum() const { return spectrum_; }
    T entry(std::size_t i, std::size_t j) const { return c_[(i + c_.size() - j) % c_.size()]; }
    Matrix<T> dense() const {
        const std::size_t n = c_.size();
        Matrix<T> out(n, n);
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = 0; j < n; ++j) out(i, j) = entry(i, j);
        return out;
    }
    CirculantMatrix transposed() const {  // first column c[(n - i) mod n]
        const std::size_t n = c_.size();
        std::vector<T> rev(n);
        for (std::size_t i = 0; i < n; ++i) rev[i] = c_[(n - i) % n];
        return CirculantMatrix(std::move(rev));
    }

  private:
    std::vector<T> c_;
    std::vector<Complex> spectrum_;
};
using RealCirculant = CirculantMatrix<double>;

// C x through the FFT kernel (circulant.hpp:91-96)
inline std::vector<double> circulant_apply(const RealCirculant& c, const std::vector<double>& x) {
    if (x.size() != c.size()) throw DimensionError("circulant_apply: length mismatch");
    std::vector<double> y(x.size());
    detail::check(rl_circulant_apply(nullptr, RL_HOST, detail::i64(c.size()), c.first_column().data(), x.data(), y.data()));
    return y;
}
// real circulant times complex input (circulant.hpp:98-101): the real and
// imaginary parts separately (C is real, so this is C x exactly)
inline std::vector<Complex> circulant_apply(const RealCirculant& c, const std::vector<Complex>& x) {
    if (x.size() != c.size()) throw DimensionError("circulant_apply: length mismatch");
    std::vector<double> re(x.size()), im(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) {
        re[i] = x[i].real();
        im[i] = x[i].imag();
    }
    const std::vector<double> yr = circulant_apply(c, re), yi = circulant_apply(c, im);
    std::vector<Complex> y(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) y[i] = Complex(yr[i], yi[i]);
    return y;
}

using ComplexCirculant = CirculantMatrix<Complex>;
// C x for a complex circulant (circulant.hpp:81-89), on the GPU
inline std::vector<Complex> circulant_apply(const ComplexCirculant& c, const std::vector<Complex>& x) {
    if (x.size() != c.size()) throw DimensionError("circulant_apply: length mismatch");
    std::vector<Complex> y(x.size());
    detail::check(rl_zcirculant_apply(nullptr, RL_HOST, detail::i64(c.size()),
                                      reinterpret_cast<const double*>(c.first_column().data()),
                                      reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())));
    return y;
}

template <ScalarField T>
std::pair<double, double> spectrum_range(const CirculantMatrix<T>& c) {
    double lo = std::abs(c.spectrum().front()), hi = lo;
    for (const Complex& u : c.spectrum()) {
        lo = std::min(lo, std::abs(u));
        hi = std::max(hi, std::abs(u));
    }
    return {lo, hi};
}
template <ScalarField T>
bool circulant_is_singular(const CirculantMatrix<T>& c) {
    const auto [lo, hi] = spectrum_range(c);
    return lo <= tol_rank(c.size(), c.size()) * hi;
}

// C^-1 b by spectral division (circulant.hpp:111-139); the transforms on the GPU
inline std::vector<double> circulant_solve(const RealCirculant& c, const std::vector<double>& b) {
    if (b.size() != c.size()) throw DimensionError("circulant_solve: length mismatch");
    if (circulant_is_singular(c)) throw SingularMatrixError("circulant is numerically singular");
    std::vector<Complex> y = fft(b);
    for (std::size_t i = 0; i < y.size(); ++i) y[i] /= c.spectrum()[i];
    y = inverse_fft(std::move(y));
    const auto [lo, hi] = spectrum_range(c);
    (void)hi;
    const double scale = lo > 0.0 ? norm2(b) / lo : norm2(b);
    double imag2 = 0.0, full2 = 0.0;
    for (const Complex& v : y) {
        imag2 += v.imag() * v.imag();
        full2 += std::norm(v);
    }
    if (std::sqrt(imag2) > 1e-11 * (std::sqrt(full2) + scale))
        throw std::logic_error("real circulant product produced non-negligible imaginary part");
    std::vector<double> out(y.size());
    for (std::size_t i = 0; i < y.size(); ++i) out[i] = y[i].real();
    return out;
}

// C^-1 b for a complex circulant (circulant.hpp:111-135), transforms on the GPU
inline std::vector<Complex> circulant_solve(const ComplexCirculant& c, const std::vector<Complex>& b) {
    if (b.size() != c.size()) throw DimensionError("circulant_solve: length mismatch");
    if (circulant_is_singular(c)) throw SingularMatrixError("circulant is numerically singular");
    std::vector<Complex> y = fft(b);
    for (std::size_t i = 0; i < y.size(); ++i) y[i] /= c.spectrum()[i];
    return inverse_fft(std::move(y));
}

template <ScalarField T>
class ToeplitzBlock {  // leading rows x cols block of a circulant (circulant.hpp:143-169)
  public:
    ToeplitzBlock(CirculantMatrix<T> parent, std::size_t rows, std::size_t cols)
        : parent_(std::move(parent)), rows_(rows), cols_(cols) {
        if (rows == 0 || cols == 0 || rows > parent_.size() || cols > parent_.size())
            throw DimensionError("toeplitz block exceeds parent dimensions");
    }
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    const CirculantMatrix<T>& parent() const { return parent_; }
    T entry(std::size_t i, std::size_t j) const { return parent_.entry(i, j); }
    Matrix<T> dense() const {
        Matrix<T> out(rows_, cols_);
        for (std::size_t i = 0; i < rows_; ++i)
            for (std::size_t j = 0; j < cols_; ++j) out(i, j) = entry(i, j);
        return out;
    }

  private:
    CirculantMatrix<T> parent_;
    std::size_t rows_, cols_;
};

// A C, every row through the FFT kernel (circulant.hpp:171-185)
inline RealMatrix matmul_by_circulant(const RealMatrix& a, const RealCirculant& c) {
    if (a.cols() != c.size()) throw DimensionError("matmul_by_circulant: shape mismatch");
    RealMatrix out(a.rows(), a.cols());
    detail::check(rl_circulant_right_multiply(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                              c.first_column().data(), out.data()));
    return out;
}
// A T for a leading Toeplitz block (circulant.hpp:187-203)
inline RealMatrix matmul_by_toeplitz_block(const RealMatrix& a, const ToeplitzBlock<double>& t) {
    if (a.cols() != t.rows()) throw DimensionError("matmul_by_toeplitz_block: shape mismatch");
    RealMatrix out(a.rows(), t.cols());
    const auto& c = t.parent().first_column();
    detail::check(rl_toeplitz_right_multiply(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                             detail::i64(c.size()), c.data(), detail::i64(t.cols()), out.data()));
    return out;
}
// the complex field (circulant.hpp:171-203 with a complex operand): every row
// through the complex FFT on the GPU
namespace detail {
template <ScalarField TA, ScalarField TC>
ComplexMatrix zcirc_rows(const Matrix<TA>& a, const std::vector<TC>& parent, std::size_t cols) {
    const ComplexMatrix ac = to_complex(a);
    const std::vector<Complex> c = to_complex_vec(parent);
    ComplexMatrix out(a.rows(), cols);
    check(rl_zcirculant_right_multiply(nullptr, RL_HOST, i64(a.rows()), i64(a.cols()),
                                       reinterpret_cast<const double*>(ac.data()), i64(c.size()),
                                       reinterpret_cast<const double*>(c.data()), i64(cols),
                                       reinterpret_cast<double*>(out.data())));
    return out;
}
}  // namespace detail
template <ScalarField TA, ScalarField TC>
    requires(field<TA>::is_complex || field<TC>::is_complex)
ComplexMatrix matmul_by_circulant(const Matrix<TA>& a, const CirculantMatrix<TC>& c) {
    if (a.cols() != c.size()) throw DimensionError("matmul_by_circulant: shape mismatch");
    return detail::zcirc_rows(a, c.first_column(), c.size());
}
template <ScalarField TA, ScalarField TC>
    requires(field<TA>::is_complex || field<TC>::is_complex)
ComplexMatrix matmul_by_toeplitz_block(const Matrix<TA>& a, const ToeplitzBlock<TC>& t) {
    if (a.cols() != t.rows()) throw DimensionError("matmul_by_toeplitz_block: shape mismatch");
    return detail::zcirc_rows(a, t.parent().first_column(), t.cols());
}

// first-column forms (no spectrum on the host)
inline RealMatrix matmul_by_circulant(const RealMatrix& a, const std::vector<double>& first_column) {
    if (a.cols() != first_column.size()) throw DimensionError("matmul_by_circulant: shape mismatch");
    RealMatrix out(a.rows(), a.cols());
    detail::check(rl_circulant_right_multiply(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                              first_column.data(), out.data()));
    return out;
}
inline RealMatrix matmul_by_toeplitz_block(const RealMatrix& a, const std::vector<double>& parent_column,
                                           std::size_t cols) {
    RealMatrix out(a.rows(), cols);
    detail::check(rl_toeplitz_right_multiply(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                             detail::i64(parent_column.size()), parent_column.data(),
                                             detail::i64(cols), out.data()));
    return out;
}

// ---- multiplier families (multipliers.hpp:20-218) -----------------------------------
// The reference's ordinals; GaussianCirculant is the B200 extension outside
// them: RealCirculant(gen_gaussian_vector(n, seed)) (BASELINE configs 3, 5).
enum class MultiplierKind {
    None = RL_MULT_NONE,
    Gaussian = RL_MULT_GAUSSIAN,
    RealCirculant = RL_MULT_REAL_CIRCULANT,
    UnitaryCirculant = RL_MULT_UNITARY_CIRCULANT,
    ToeplitzBlock = RL_MULT_TOEPLITZ_BLOCK,
    Srft = RL_MULT_SRFT,
    FiniteSetUniform = RL_MULT_FINITE_SET_UNIFORM,
    CircSkewProduct = RL_MULT_CIRC_SKEW_PRODUCT,
    GaussianCirculant = RL_MULT_GAUSSIAN_CIRCULANT,
};
enum class ToeplitzVariant { Real = RL_TOEPLITZ_REAL, Unitary = RL_TOEPLITZ_UNITARY };

struct MultiplierSpec {
    MultiplierKind kind = MultiplierKind::None;
    std::size_t rows = 0;
    std::size_t cols = 0;  // cols <= rows for sketching uses
    std::uint64_t seed = 0;
    std::size_t set_cardinality = 65536;              // FiniteSetUniform only
    ToeplitzVariant variant = ToeplitzVariant::Real;  // ToeplitzBlock only
};

inline bool multiplier_is_complex(const MultiplierSpec& spec) {
    return spec.kind == MultiplierKind::UnitaryCirculant || spec.kind == MultiplierKind::Srft ||
           (spec.kind == MultiplierKind::ToeplitzBlock && spec.variant == ToeplitzVariant::Unitary);
}

namespace detail {
inline rl_multiplier to_abi(const MultiplierSpec& s) {
    rl_multiplier m{};
    m.kind = static_cast<int32_t>(s.kind);
    m.variant = static_cast<int32_t>(s.variant);
    m.seed = s.seed;
    m.set_cardinality = s.set_cardinality;
    return m;
}
}  // namespace detail

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t k1, std::uint64_t k2 = 0) {
    return rl_derive_seed(seed, k1, k2);
}

inline RealMatrix gen_gaussian(std::size_t m, std::size_t n, std::uint64_t seed) {
    RealMatrix out(m, n);
    detail::check(rl_gen_gaussian(detail::i64(m), detail::i64(n), seed, out.data()));
    return out;
}
inline std::vector<double> gen_gaussian_vector(std::size_t n, std::uint64_t seed) {
    std::vector<double> v(n);
    detail::check(rl_gen_gaussian(detail::i64(n), 1, seed, v.data()));
    return v;
}
inline RealCirculant gen_real_circulant(std::size_t n, std::uint64_t seed) {
    std::vector<double> c(n);
    detail::check(rl_gen_real_circulant_column(detail::i64(n), seed, c.data()));
    return RealCirculant(std::move(c));
}
inline ToeplitzBlock<double> gen_real_toeplitz_block(std::size_t n, std::size_t l, std::uint64_t seed) {
    return ToeplitzBlock<double>(gen_real_circulant(n, seed), n, l);
}
inline RealMatrix gen_finite_set_uniform(std::size_t m, std::size_t n, std::uint64_t seed, std::size_t cardinality) {
    if (cardinality < 2) throw DimensionError("gen_finite_set_uniform: cardinality must be >= 2");
    RealMatrix out(m, n);
    detail::check(rl_gen_finite_set_uniform(detail::i64(m), detail::i64(n), seed, cardinality, out.data()));
    return out;
}

// ---- the complex families (multipliers.hpp:75-138) -----------------------------------
// spectrum u_j = polar(1, 2 pi phi_j) from the reference's stream (host, the
// same libm), first column inverse_fft(u) on the GPU
inline ComplexCirculant gen_unitary_circulant(std::size_t n, std::uint64_t seed) {
    if (n == 0) throw DimensionError("circulant: empty first column");
    std::vector<Complex> c(n);
    detail::check(rl_gen_unitary_circulant(nullptr, RL_HOST, detail::i64(n), seed, reinterpret_cast<double*>(c.data())));
    return ComplexCirculant(std::move(c));
}
inline ToeplitzBlock<Complex> gen_unitary_toeplitz_block(std::size_t n, std::size_t l, std::uint64_t seed) {
    return ToeplitzBlock<Complex>(gen_unitary_circulant(n, seed), n, l);
}
// sqrt(n/l) D Omega R from explicit parts (multipliers.hpp:92-110)
inline ComplexMatrix srft_from_parts(std::size_t n, const std::vector<double>& phases,
                                     const std::vector<std::size_t>& columns) {
    const std::size_t l = columns.size();
    if (phases.size() != n || l == 0 || l > n) throw DimensionError("srft_from_parts: bad shapes");
    std::vector<Complex> root(n);
    for (std::size_t k = 0; k < n; ++k)
        root[k] = std::polar(1.0, 2.0 * std::numbers::pi * static_cast<double>(k) / static_cast<double>(n));
    const double scale = std::sqrt(static_cast<double>(n) / static_cast<double>(l));
    ComplexMatrix out(n, l);
    for (std::size_t i = 0; i < n; ++i) {
        const Complex d = scale * std::polar(1.0, 2.0 * std::numbers::pi * phases[i]);
        for (std::size_t j = 0; j < l; ++j) out(i, j) = d * root[(i * columns[j]) % n];
    }
    return out;
}
// l sorted indices out of n without replacement (multipliers.hpp:112-121)
inline std::vector<std::size_t> sample_without_replacement(std::size_t n, std::size_t l, RngStream& rng) {
    std::vector<std::size_t> pool(n);
    for (std::size_t i = 0; i < n; ++i) pool[i] = i;
    for (std::size_t i = 0; i < l; ++i) std::swap(pool[i], pool[i + static_cast<std::size_t>(rng.next_below(n - i))]);
    std::vector<std::size_t> out(pool.begin(), pool.begin() + static_cast<std::ptrdiff_t>(l));
    std::sort(out.begin(), out.end());
    return out;
}
inline std::vector<std::size_t> srft_columns(std::size_t n, std::size_t l, std::uint64_t seed) {
    std::vector<int64_t> c(l);
    detail::check(rl_srft_columns(detail::i64(n), detail::i64(l), seed, c.data()));
    return std::vector<std::size_t>(c.begin(), c.end());
}

// materialize<T>(spec) (multipliers.hpp:174-218): the dense sample of the
// named family in the requested field, from the reference's generators (the
// expansions, the skew product and the complex families on the GPU)
template <ScalarField T>
Matrix<T> materialize(const MultiplierSpec& spec) {
    if constexpr (!field<T>::is_complex) {
        if (multiplier_is_complex(spec)) throw DimensionError("complex multiplier family requested in a real pipeline");
        RealMatrix out(spec.rows, spec.cols);
        const rl_multiplier m = detail::to_abi(spec);
        detail::check(rl_materialize(nullptr, RL_HOST, &m, detail::i64(spec.rows), detail::i64(spec.cols), out.data()));
        return out;
    } else {
        ComplexMatrix out(spec.rows, spec.cols);
        const rl_multiplier m = detail::to_abi(spec);
        detail::check(rl_zmaterialize(nullptr, RL_HOST, &m, detail::i64(spec.rows), detail::i64(spec.cols),
                                      reinterpret_cast<double*>(out.data())));
        return out;
    }
}
inline RealMatrix gen_circ_skew_product(std::size_t n, std::uint64_t seed) {
    MultiplierSpec s{MultiplierKind::CircSkewProduct, n, n, seed};
    return materialize<double>(s);
}
inline ComplexMatrix gen_srft(std::size_t n, std::size_t l, std::uint64_t seed) {
    if (l < 1 || l > n) throw DimensionError("gen_srft: need 1 <= l <= n");
    MultiplierSpec s{MultiplierKind::Srft, n, l, seed};
    return materialize<Complex>(s);
}

// CLI token forms (multipliers.hpp:222-275)
inline std::string format_multiplier_token(const MultiplierSpec& spec) {
    switch (spec.kind) {
        case MultiplierKind::None: return "none";
        case MultiplierKind::Gaussian: return "gaussian";
        case MultiplierKind::RealCirculant: return "circulant";
        case MultiplierKind::UnitaryCirculant: return "unitary-circulant";
        case MultiplierKind::ToeplitzBlock:
            return spec.variant == ToeplitzVariant::Real ? "toeplitz:variant=real" : "toeplitz:variant=unitary";
        case MultiplierKind::Srft: return "srft";
        case MultiplierKind::FiniteSetUniform: return "finite:card=" + std::to_string(spec.set_cardinality);
        case MultiplierKind::CircSkewProduct: return "circskew";
        case MultiplierKind::GaussianCirculant: return "gaussian-circulant";
    }
    return "none";
}
inline MultiplierSpec parse_multiplier_token(const std::string& token) {
    MultiplierSpec spec;
    const std::size_t colon = token.find(':');
    const std::string head = token.substr(0, colon);
    const std::string opts = colon == std::string::npos ? "" : token.substr(colon + 1);
    static const std::pair<const char*, MultiplierKind> kinds[] = {
        {"none", MultiplierKind::None},       {"gaussian", MultiplierKind::Gaussian},
        {"circulant", MultiplierKind::RealCirculant}, {"unitary-circulant", MultiplierKind::UnitaryCirculant},
        {"toeplitz", MultiplierKind::ToeplitzBlock},  {"srft", MultiplierKind::Srft},
        {"finite", MultiplierKind::FiniteSetUniform}, {"circskew", MultiplierKind::CircSkewProduct},
        {"gaussian-circulant", MultiplierKind::GaussianCirculant}};
    bool found = false;
    for (const auto& [name, kind] : kinds)
        if (head == name) {
            spec.kind = kind;
            found = true;
        }
    if (!found) throw IoError("unknown multiplier token: " + token);
    for (std::size_t pos = 0; pos < opts.size();) {
        const std::size_t comma = opts.find(',', pos);
        const std::size_t end = comma == std::string::npos ? opts.size() : comma;
        const std::string kv = opts.substr(pos, end - pos);
        const std::size_t eq = kv.find('=');
        if (eq == std::string::npos) throw IoError("bad multiplier option: " + kv);
        const std::string key = kv.substr(0, eq), value = kv.substr(eq + 1);
        if (key == "variant" && spec.kind == MultiplierKind::ToeplitzBlock) {
            if (value == "real")
                spec.variant = ToeplitzVariant::Real;
            else if (value == "unitary")
                spec.variant = ToeplitzVariant::Unitary;
            else
                throw IoError("bad toeplitz variant: " + value);
        } else if (key == "card" && spec.kind == MultiplierKind::FiniteSetUniform) {
            spec.set_cardinality = std::stoull(value);
        } else {
            throw IoError("bad multiplier option: " + kv);
        }
        pos = end + 1;
    }
    return spec;
}

// ---- GENP (lu.hpp) --------------------------------------------------------------------
template <ScalarField T = double>
struct LuFactors {
    Matrix<T> lower;
    Matrix<T> upper;
    std::optional<std::vector<std::size_t>> perm;  // empty for GENP; GEPP: original row at position i
    std::vector<T> pivots() const {
        std::vector<T> p(upper.rows());
        for (std::size_t j = 0; j < upper.rows(); ++j) p[j] = upper(j, j);
        return p;
    }
};

namespace detail {
template <ScalarField T>
LuFactors<T> unpack(const Matrix<T>& packed) {
    const std::size_t n = packed.rows();
    LuFactors<T> f{Matrix<T>::identity(n), Matrix<T>(n, n), std::nullopt};
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) (j < i ? f.lower(i, j) : f.upper(i, j)) = packed(i, j);
    return f;
}
template <ScalarField T>
Matrix<T> pack(const LuFactors<T>& f) {
    const std::size_t n = f.upper.rows();
    Matrix<T> p(n, n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) p(i, j) = j < i ? f.lower(i, j) : f.upper(i, j);
    return p;
}
}  // namespace detail

inline LuFactors<double> genp_factor(const RealMatrix& a) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("genp_factor: square input required");
    RealMatrix packed(n, n);
    rl_solve_info info{};
    const rl_status st = rl_genp_factor(nullptr, RL_HOST, detail::i64(n), a.data(), packed.data(), &info);
    detail::check(st, info.zero_pivot_step);
    return detail::unpack(packed);
}
// over the complex field: the panel-planar blocked GENP of complex.cu
inline LuFactors<Complex> genp_factor(const ComplexMatrix& a) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("genp_factor: square input required");
    ComplexMatrix packed(n, n);
    rl_solve_info info{};
    const rl_status st = rl_zgenp_factor(nullptr, RL_HOST, detail::i64(n), reinterpret_cast<const double*>(a.data()),
                                         reinterpret_cast<double*>(packed.data()), &info);
    detail::check(st, info.zero_pivot_step);
    return detail::unpack(packed);
}

namespace detail {
inline std::vector<double> gepp_solve(const LuFactors<double>& f, const std::vector<double>& b, bool transpose);
}
inline std::vector<double> lu_solve(const LuFactors<double>& f, const std::vector<double>& b) {
    if (f.perm) return detail::gepp_solve(f, b, false);
    const std::size_t n = f.upper.rows();
    if (b.size() != n) throw DimensionError("lu_solve: length mismatch");
    const RealMatrix packed = detail::pack(f);
    std::vector<double> x(n);
    detail::check(rl_lu_solve(nullptr, RL_HOST, detail::i64(n), packed.data(), b.data(), x.data()));
    return x;
}
inline std::vector<Complex> lu_solve(const LuFactors<Complex>& f, const std::vector<Complex>& b) {
    if (f.perm) throw DimensionError("lu_solve: complex pivoted factors are off the B200 path");
    const std::size_t n = f.upper.rows();
    if (b.size() != n) throw DimensionError("lu_solve: length mismatch");
    const ComplexMatrix packed = detail::pack(f);
    std::vector<Complex> x(n);
    detail::check(rl_zlu_solve(nullptr, RL_HOST, detail::i64(n), reinterpret_cast<const double*>(packed.data()),
                               reinterpret_cast<const double*>(b.data()), reinterpret_cast<double*>(x.data())));
    return x;
}

// ---- GEPP and block elimination (lu.hpp:62-147, block_ge.hpp) ----------------
// The device keeps the reference's arithmetic order: factors, permutations,
// pivots, Schur complements and block_solve results are bit-identical.
namespace detail {
inline RealMatrix pack_lu(const LuFactors<double>& f) { return pack(f); }
inline std::vector<int64_t> perm_of(const LuFactors<double>& f) {
    const std::size_t n = f.upper.rows();
    std::vector<int64_t> p(n);
    for (std::size_t i = 0; i < n; ++i) p[i] = f.perm ? static_cast<int64_t>((*f.perm)[i]) : static_cast<int64_t>(i);
    return p;
}
inline std::vector<double> gepp_solve(const LuFactors<double>& f, const std::vector<double>& b, bool transpose) {
    const std::size_t n = f.upper.rows();
    if (b.size() != n) throw DimensionError(transpose ? "lu_solve_transpose: length mismatch" : "lu_solve: length mismatch");
    const RealMatrix packed = pack(f);
    const std::vector<int64_t> p = perm_of(f);
    std::vector<double> x(n);
    check(rl_gepp_solve(nullptr, RL_HOST, static_cast<int64_t>(n), 1, packed.data(), p.data(), b.data(), x.data(),
                        transpose ? 1 : 0));
    return x;
}
}  // namespace detail

inline LuFactors<double> gepp_factor(const RealMatrix& a) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("gepp_factor: square input required");
    RealMatrix packed(n, n);
    std::vector<int64_t> p(n);
    int64_t step = 0;
    detail::check(rl_gepp_factor(nullptr, RL_HOST, static_cast<int64_t>(n), a.data(), packed.data(), p.data(), &step));
    LuFactors<double> f = detail::unpack(packed);
    f.perm = std::vector<std::size_t>(p.begin(), p.end());
    return f;
}

inline std::vector<double> lu_solve_transpose(const LuFactors<double>& f, const std::vector<double>& c) {
    return detail::gepp_solve(f, c, true);
}

struct BlockNode {  // block_ge.hpp:18-35
    std::size_t dim = 0, offset = 0, pivot_size = 0;
    RealMatrix block_matrix;
    std::optional<LuFactors<double>> block_lu;
    RealMatrix db_inv, b_inv_c;
    std::unique_ptr<BlockNode> pivot_child, schur_child;
    bool leaf() const { return pivot_size == 0; }
};

struct BlockFactorization {  // block_ge.hpp:37-83
    std::unique_ptr<BlockNode> root;
    std::vector<std::size_t> split;
    RealMatrix factors;           // flat device layout (rl_block_ge_factor)
    std::vector<int64_t> perm;
    std::vector<double> pivots() const {
        std::vector<double> p(factors.rows());
        for (std::size_t j = 0; j < p.size(); ++j) p[j] = factors(j, j);
        return p;
    }
    RealMatrix reassemble() const { return reassemble_node(*root); }

  private:
    static RealMatrix reassemble_node(const BlockNode& node) {
        const std::size_t d = node.dim;
        if (node.leaf()) {
            const RealMatrix lu = matmul(node.block_lu->lower, node.block_lu->upper);
            RealMatrix out(d, d);
            for (std::size_t i = 0; i < d; ++i)
                for (std::size_t j = 0; j < d; ++j) out((*node.block_lu->perm)[i], j) = lu(i, j);
            return out;
        }
        const RealMatrix b = reassemble_node(*node.pivot_child), s = reassemble_node(*node.schur_child);
        const std::size_t k = node.pivot_size;
        const RealMatrix c = matmul(b, node.b_inv_c), dd = matmul(node.db_inv, b), t = matmul(node.db_inv, c);
        RealMatrix out(d, d);
        for (std::size_t i = 0; i < d; ++i)
            for (std::size_t j = 0; j < d; ++j)
                out(i, j) = i < k ? (j < k ? b(i, j) : c(i, j - k)) : (j < k ? dd(i - k, j) : s(i - k, j - k) + t(i - k, j - k));
        return out;
    }
};

inline std::vector<std::size_t> balanced_split(std::size_t n) {  // block_ge.hpp:184-194
    std::vector<std::size_t> out;
    std::size_t remaining = n;
    while (remaining > 1) {
        const std::size_t half = remaining / 2;
        out.push_back(half);
        remaining -= half;
    }
    out.push_back(remaining);
    return out;
}

inline BlockFactorization block_ge_factor(const RealMatrix& a, const std::vector<std::size_t>& split) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("block_ge_factor: square input required");
    std::vector<int64_t> sp(split.begin(), split.end());
    BlockFactorization f;
    f.split = split;
    f.factors = RealMatrix(n, n);
    f.perm.assign(n, 0);
    RealMatrix leaves(n, n);
    int64_t position = 0;
    const rl_status st = rl_block_ge_factor(nullptr, RL_HOST, static_cast<int64_t>(n), a.data(),
                                            static_cast<int64_t>(sp.size()), sp.empty() ? nullptr : sp.data(),
                                            f.factors.data(), f.perm.data(), leaves.data(), &position);
    detail::check(st, position);
    auto sub = [&](const RealMatrix& m, std::size_t r0, std::size_t c0, std::size_t r, std::size_t c) {
        RealMatrix out(r, c);
        for (std::size_t i = 0; i < r; ++i)
            for (std::size_t j = 0; j < c; ++j) out(i, j) = m(r0 + i, c0 + j);
        return out;
    };
    auto leaf = [&](std::size_t o, std::size_t k) {
        auto node = std::make_unique<BlockNode>();
        node->dim = k;
        node->offset = o;
        node->block_matrix = sub(leaves, o, o, k, k);
        LuFactors<double> lu = detail::unpack(sub(f.factors, o, o, k, k));
        lu.perm = std::vector<std::size_t>(f.perm.begin() + static_cast<std::ptrdiff_t>(o),
                                           f.perm.begin() + static_cast<std::ptrdiff_t>(o + k));
        node->block_lu = std::move(lu);
        return node;
    };
    std::vector<std::pair<std::size_t, std::size_t>> levels;
    std::size_t o = 0;
    for (std::size_t i = 0; i < split.size(); ++i) {
        const std::size_t k = i + 1 == split.size() ? n - o : split[i];
        levels.emplace_back(o, k);
        o += k;
    }
    std::unique_ptr<BlockNode> node;
    for (auto it = levels.rbegin(); it != levels.rend(); ++it) {
        const auto [oo, k] = *it;
        if (!node) {
            node = leaf(oo, k);
            continue;
        }
        auto in = std::make_unique<BlockNode>();
        in->dim = n - oo;
        in->offset = oo;
        in->pivot_size = k;
        in->db_inv = sub(f.factors, oo + k, oo, n - oo - k, k);
        in->b_inv_c = sub(f.factors, oo, oo + k, k, n - oo - k);
        in->pivot_child = leaf(oo, k);
        in->schur_child = std::move(node);
        node = std::move(in);
    }
    f.root = std::move(node);
    return f;
}

inline std::vector<double> block_solve(const BlockFactorization& f, const std::vector<double>& b) {
    const std::size_t n = f.factors.rows();
    if (b.size() != n) throw DimensionError("block_solve: length mismatch");
    std::vector<int64_t> sp(f.split.begin(), f.split.end());
    std::vector<double> x(n);
    detail::check(rl_block_solve(nullptr, RL_HOST, static_cast<int64_t>(n), static_cast<int64_t>(sp.size()), sp.data(),
                                 f.factors.data(), f.perm.data(), b.data(), x.data()));
    return x;
}

inline RealMatrix schur_complement(const RealMatrix& a, std::size_t k) {  // block_ge.hpp:202-218
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("schur_complement: square input required");
    if (k == 0 || k >= n) throw DimensionError("schur_complement: need 0 < k < n");
    RealMatrix b(k, k), c(k, n - k), d(n - k, k);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) {
            if (i < k && j < k) b(i, j) = a(i, j);
            else if (i < k) c(i, j - k) = a(i, j);
            else if (j < k) d(i - k, j) = a(i, j);
        }
    const LuFactors<double> b_lu = gepp_factor(b);
    const RealMatrix packed = detail::pack(b_lu);
    const std::vector<int64_t> p = detail::perm_of(b_lu);
    RealMatrix x(k, n - k);
    detail::check(rl_gepp_solve(nullptr, RL_HOST, static_cast<int64_t>(k), static_cast<int64_t>(n - k), packed.data(),
                                p.data(), c.data(), x.data(), 0));
    const RealMatrix dx = matmul(d, x);
    RealMatrix out(n - k, n - k);
    for (std::size_t i = 0; i < n - k; ++i)
        for (std::size_t j = 0; j < n - k; ++j) out(i, j) = a(k + i, k + j) - dx(i, j);
    return out;
}

template <ScalarField T>
double relative_residual(const Matrix<T>& a, const std::vector<T>& x, const std::vector<T>& b) {
    const std::vector<T> ax = matvec(a, x);
    double num = 0.0;
    for (std::size_t i = 0; i < b.size(); ++i) num += field<T>::abs2(ax[i] - b[i]);
    return std::sqrt(num) / norm2(b);
}

// ---- preprocessing (preprocess.hpp) ------------------------------------------------
template <ScalarField T = double>
struct SolveOutcome {
    std::vector<T> x;
    std::vector<double> residual_history;  // ||Ax - b|| / ||b|| after the solve and each refinement
    bool diverged = false;
    rl_solve_info info{};                  // device diagnostics (growth, pivots, stage times)
};

// One side of A -> F A H (preprocess.hpp:20-110): identity, a dense sample, or
// a circulant kept structured; products on the GPU.
template <ScalarField T = double>
class SideMultiplier {
  public:
    static SideMultiplier identity() { return SideMultiplier(); }
    static SideMultiplier make(MultiplierSpec spec, std::size_t n) {
        if (spec.rows == 0) spec.rows = n;
        if (spec.cols == 0) spec.cols = n;
        if (spec.rows != n || spec.cols != n)
            throw DimensionError("solve preprocessing takes square n-by-n multipliers");
        SideMultiplier out;
        switch (spec.kind) {
            case MultiplierKind::None: return out;
            case MultiplierKind::RealCirculant:
                out.real_circ_.emplace(gen_real_circulant(n, spec.seed));
                return out;
            case MultiplierKind::GaussianCirculant:
                out.real_circ_.emplace(gen_gaussian_vector(n, spec.seed));
                return out;
            case MultiplierKind::UnitaryCirculant:
                if constexpr (field<T>::is_complex) {
                    out.complex_circ_.emplace(gen_unitary_circulant(n, spec.seed));
                    return out;
                }
                break;
            case MultiplierKind::ToeplitzBlock:
                if (spec.variant == ToeplitzVariant::Real) {
                    out.real_circ_.emplace(gen_real_circulant(n, spec.seed));
                    return out;
                }
                if constexpr (field<T>::is_complex) {
                    out.complex_circ_.emplace(gen_unitary_circulant(n, spec.seed));
                    return out;
                }
                break;
            default: out.dense_.emplace(materialize<T>(spec)); return out;
        }
        throw DimensionError("complex multiplier family requested in a real pipeline");
    }
    bool is_identity() const { return !dense_ && !real_circ_ && !complex_circ_; }
    Matrix<T> right_multiply(const Matrix<T>& a) const {  // A H
        if (is_identity()) return a;
        if (dense_) return matmul(a, *dense_);
        if (real_circ_) return coerce(matmul_by_circulant(a, *real_circ_));
        return coerce(matmul_by_circulant(a, *complex_circ_));
    }
    Matrix<T> left_multiply(const Matrix<T>& a) const {  // F A, column by column for the structured forms
        if (is_identity()) return a;
        if (dense_) return matmul(*dense_, a);
        // F A = (A^T F^T)^T: every column through the circulant at once
        if (real_circ_) return coerce(matmul_by_circulant(a.transpose(), real_circ_->transposed())).transpose();
        return coerce(matmul_by_circulant(a.transpose(), complex_circ_->transposed())).transpose();
    }
    std::vector<T> apply_vec(const std::vector<T>& v) const {  // H v
        if (is_identity()) return v;
        if (dense_) return matvec(*dense_, v);
        if (real_circ_) return circulant_apply(*real_circ_, v);
        if constexpr (field<T>::is_complex) return circulant_apply(*complex_circ_, v);
        throw std::logic_error("unreachable multiplier state");
    }

  private:
    SideMultiplier() = default;
    template <typename M>
    static Matrix<T> coerce(M&& m) {
        if constexpr (std::is_same_v<std::decay_t<M>, Matrix<T>>)
            return std::forward<M>(m);
        else
            throw std::logic_error("unreachable multiplier field mix");
    }
    std::optional<Matrix<T>> dense_;
    std::optional<RealCirculant> real_circ_;
    std::optional<ComplexCirculant> complex_circ_;
};

// residual-correction loop reusing one factorization through `solver`
// (preprocess.hpp:115-143): two consecutive increases set `diverged`
template <ScalarField T>
SolveOutcome<T> iterative_refine(const Matrix<T>& a, const std::function<std::vector<T>(const std::vector<T>&)>& solver,
                                 const std::vector<T>& b, std::vector<T> x0, std::size_t steps) {
    SolveOutcome<T> out;
    out.x = std::move(x0);
    const double bnorm = norm2(b);
    auto residual = [&](const std::vector<T>& x) {
        std::vector<T> r = matvec(a, x);
        for (std::size_t i = 0; i < r.size(); ++i) r[i] = b[i] - r[i];
        return r;
    };
    std::vector<T> r = residual(out.x);
    out.residual_history.push_back(norm2(r) / bnorm);
    std::size_t streak = 0;
    for (std::size_t s = 0; s < steps; ++s) {
        const std::vector<T> d = solver(r);
        for (std::size_t i = 0; i < out.x.size(); ++i) out.x[i] += d[i];
        r = residual(out.x);
        const double rel = norm2(r) / bnorm;
        streak = rel > out.residual_history.back() ? streak + 1 : 0;
        out.residual_history.push_back(rel);
        if (streak >= 2) {
            out.diverged = true;
            break;
        }
    }
    return out;
}
template <ScalarField T>
SolveOutcome<T> iterative_refine(const Matrix<T>& a, const LuFactors<T>& factors, const std::vector<T>& b,
                                 std::vector<T> x0, std::size_t steps) {
    return iterative_refine<T>(
        a, [&](const std::vector<T>& r) { return lu_solve(factors, r); }, b, std::move(x0), steps);
}

// preprocess_solve(a, b, pre, post, refine) (preprocess.hpp:156-180): one
// device call: F (A H), blocked GENP with the reference's pivot verdict, chain
// solve H (LU)^-1 (F r) and the refinement loop; over either field
template <ScalarField T>
SolveOutcome<T> preprocess_solve(const Matrix<T>& a, const std::vector<T>& b, const MultiplierSpec& pre_spec,
                                 const MultiplierSpec& post_spec, std::size_t refine_steps) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("preprocess_solve: square input required");
    if (b.size() != n) throw DimensionError("preprocess_solve: length mismatch");
    for (const MultiplierSpec* s : {&pre_spec, &post_spec})
        if ((s->rows != 0 && s->rows != n) || (s->cols != 0 && s->cols != n))
            throw DimensionError("solve preprocessing takes square n-by-n multipliers");
    if constexpr (!field<T>::is_complex)
        for (const MultiplierSpec* s : {&pre_spec, &post_spec})
            if (multiplier_is_complex(*s)) throw DimensionError("complex multiplier family requested in a real pipeline");
    const rl_multiplier pre = detail::to_abi(pre_spec), post = detail::to_abi(post_spec);
    SolveOutcome<T> out;
    out.x.resize(n);
    out.residual_history.assign(refine_steps + 1, 0.0);
    out.info.history = out.residual_history.data();
    out.info.history_capacity = detail::i64(refine_steps + 1);
    rl_status st;
    if constexpr (field<T>::is_complex)
        st = rl_zpreprocessed_genp_solve(nullptr, RL_HOST, detail::i64(n), reinterpret_cast<const double*>(a.data()),
                                         reinterpret_cast<const double*>(b.data()), &pre, &post,
                                         detail::i64(refine_steps), reinterpret_cast<double*>(out.x.data()), nullptr,
                                         &out.info);
    else
        st = rl_preprocessed_genp_solve(nullptr, RL_HOST, detail::i64(n), a.data(), b.data(), &pre, &post,
                                        detail::i64(refine_steps), out.x.data(), nullptr, 0, &out.info);
    detail::check(st, out.info.zero_pivot_step);
    out.residual_history.resize(static_cast<std::size_t>(out.info.history_len));
    out.info.history = nullptr;
    out.diverged = out.info.diverged != 0;
    return out;
}

template <ScalarField T>
SolveOutcome<T> preprocess_solve_with_retry(const Matrix<T>& a, const std::vector<T>& b, MultiplierSpec pre_spec,
                                            MultiplierSpec post_spec, std::size_t refine_steps,
                                            std::size_t max_retries = 3) {
    for (std::size_t attempt = 0;; ++attempt) {
        try {
            return preprocess_solve(a, b, pre_spec, post_spec, refine_steps);
        } catch (const ZeroPivotError&) {
            if (attempt >= max_retries) throw;
            pre_spec.seed = derive_seed(pre_spec.seed, 0x52455452ull, attempt + 1);
            post_spec.seed = derive_seed(post_spec.seed, 0x52455452ull, attempt + 1);
        }
    }
}

// ---- QR (qr.hpp:17-76): CholeskyQR2 on the GPU, positive (real) diagonal R ----------
template <ScalarField T = double>
struct QrResult {
    Matrix<T> q;  // m-by-n
    Matrix<T> r;  // n-by-n
};
inline QrResult<double> qr(const RealMatrix& y) {
    if (y.rows() < y.cols()) throw DimensionError("qr: expected rows >= cols");
    QrResult<double> out{RealMatrix(y.rows(), y.cols()), RealMatrix(y.cols(), y.cols())};
    int64_t bad = 0;
    const rl_status st = rl_cholqr2(nullptr, RL_HOST, detail::i64(y.rows()), detail::i64(y.cols()), y.data(),
                                    out.q.data(), out.r.data(), &bad);
    if (st == RL_ERR_RANK_DEFICIENCY)
        throw RankDeficiencyError("qr: numerically rank-deficient at column " + std::to_string(bad));
    detail::check(st);
    return out;
}
namespace detail {
inline ComplexMatrix zbasis(const ComplexMatrix& y, bool unchecked) {
    if (y.rows() < y.cols()) throw DimensionError("qr: expected rows >= cols");
    ComplexMatrix q(y.rows(), y.cols());
    int64_t bad = 0;
    const rl_status st = rl_zorthonormal_basis(nullptr, RL_HOST, i64(y.rows()), i64(y.cols()),
                                               reinterpret_cast<const double*>(y.data()),
                                               reinterpret_cast<double*>(q.data()), unchecked ? 1 : 0, &bad);
    if (st == RL_ERR_RANK_DEFICIENCY)
        throw RankDeficiencyError("qr: numerically rank-deficient at column " + std::to_string(bad));
    check(st);
    return q;
}
}  // namespace detail
// complex: the basis through the real embedding (complex.cu), R = Q^H Y
inline QrResult<Complex> qr(const ComplexMatrix& y) {
    ComplexMatrix q = detail::zbasis(y, false);
    ComplexMatrix r = matmul(q.adjoint(), y);
    for (std::size_t i = 0; i < r.rows(); ++i) {
        for (std::size_t j = 0; j < i; ++j) r(i, j) = Complex{};
        r(i, i) = Complex(r(i, i).real(), 0.0);  // real positive by construction
    }
    return {std::move(q), std::move(r)};
}
inline RealMatrix orthonormal_basis(const RealMatrix& y) { return qr(y).q; }
inline ComplexMatrix orthonormal_basis(const ComplexMatrix& y) { return detail::zbasis(y, false); }
// without the rank check (qr.hpp:58-76)
inline RealMatrix orthonormal_basis_unchecked(const RealMatrix& y) {
    if (y.rows() < y.cols()) throw DimensionError("qr: expected rows >= cols");
    RealMatrix q(y.rows(), y.cols());
    detail::check(rl_orthonormal_basis_unchecked(nullptr, RL_HOST, detail::i64(y.rows()), detail::i64(y.cols()),
                                                 y.data(), q.data()));
    return q;
}
inline ComplexMatrix orthonormal_basis_unchecked(const ComplexMatrix& y) { return detail::zbasis(y, true); }

// ---- range finder (lowrank.hpp:21-113) ------------------------------------------------
template <ScalarField T = double>
struct LowRankResult {
    Matrix<T> q;  // m-by-l, orthonormal columns
    std::size_t rank = 0;
    std::size_t oversample = 0;
    std::size_t power_steps = 0;

    std::size_t sketch_width() const { return q.cols(); }
    std::vector<T> apply_projection(const std::vector<T>& v) const { return matvec(q, matvec(q.adjoint(), v)); }
    Matrix<T> apply_approximation(const Matrix<T>& a) const { return matmul(q, matmul(q.adjoint(), a)); }
    Matrix<T> projector_dense() const {
        if (q.rows() > 2048) throw DimensionError("projector materialization capped at 2048");
        return matmul(q, q.adjoint());
    }
};

// range finder on a supplied sketch: power steps (A A^H)^s, then the basis
template <ScalarField T>
LowRankResult<T> range_find_with(const Matrix<T>& a, Matrix<T> sketch, std::size_t r, std::size_t p,
                                 std::size_t power_steps) {
    if (r < 1 || r + p > std::min(a.rows(), a.cols()))
        throw DimensionError("range_find: rank plus oversampling exceeds matrix size");
    for (std::size_t s = 0; s < power_steps; ++s) sketch = matmul(a, matmul(a.adjoint(), sketch));
    return LowRankResult<T>{orthonormal_basis(sketch), r, p, power_steps};
}

// range_find (lowrank.hpp:62-83): one device call (sketch by the spec's family,
// power steps, CholeskyQR2), over either field
template <ScalarField T>
LowRankResult<T> range_find(const Matrix<T>& a, std::size_t r, std::size_t p, MultiplierSpec spec,
                            std::size_t power_steps) {
    const std::size_t n = a.cols(), l = r + p;
    if (r < 1 || l > std::min(a.rows(), a.cols()))
        throw DimensionError("range_find: rank plus oversampling exceeds matrix size");
    spec.rows = n;
    spec.cols = l;
    const rl_multiplier m = detail::to_abi(spec);
    LowRankResult<T> out{Matrix<T>(a.rows(), l), r, p, power_steps};
    rl_lowrank_info info{};
    rl_status st;
    if constexpr (field<T>::is_complex)
        st = rl_zrange_find_residual(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(n),
                                     reinterpret_cast<const double*>(a.data()), detail::i64(l), &m,
                                     detail::i64(power_steps), reinterpret_cast<double*>(out.q.data()), &info);
    else
        st = rl_range_find(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(n), a.data(), detail::i64(l), &m,
                           detail::i64(power_steps), out.q.data(), &info);
    if (st == RL_ERR_RANK_DEFICIENCY)
        throw RankDeficiencyError("qr: numerically rank-deficient at column " +
                                  std::to_string(info.rank_deficient_column));
    detail::check(st);
    return out;
}

// ||A - Q (Q^H A)||_2 for this A (lowrank.hpp:99-102), on the GPU: B = Q^H A,
// the residual never stored, its 2-norm by the restated power iteration
template <ScalarField T>
double approximation_residual(const Matrix<T>& a, const LowRankResult<T>& result) {
    if (a.rows() != result.q.rows()) throw DimensionError("approximation_residual: shape mismatch");
    rl_lowrank_info info{};
    if constexpr (field<T>::is_complex)
        detail::check(rl_zapproximation_residual(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()),
                                                 reinterpret_cast<const double*>(a.data()), detail::i64(result.q.cols()),
                                                 reinterpret_cast<const double*>(result.q.data()), &info));
    else
        detail::check(rl_approximation_residual(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()),
                                                a.data(), detail::i64(result.q.cols()), result.q.data(), &info));
    return info.residual_spectral;
}

struct SubspaceResiduals {
    double rn1 = 0.0;  // projection residual of the leading left singular basis
    double rn2 = 0.0;  // ||A - Q Q^H A||
};
template <ScalarField T>
double basis_residual(const LowRankResult<T>& result, const TruncatedSVD<T>& truth) {
    const Matrix<T> y = matmul(result.q.adjoint(), truth.left);
    return spectral_norm(matmul(result.q, y) - truth.left);
}
template <ScalarField T>
SubspaceResiduals subspace_residual(const Matrix<T>& a, const LowRankResult<T>& result, const TruncatedSVD<T>& truth) {
    return {basis_residual(result, truth), approximation_residual(a, result)};
}
inline TruncatedSVD<Complex> to_complex(const TruncatedSVD<double>& t) {
    return {to_complex(t.left), t.singulars, to_complex(t.right)};
}

// ---- error bounds and the a-posteriori estimate (lowrank.hpp:114-196) --------------------
struct ReferenceBounds {  // expected-error reference values, oversampling p >= 2
    double frobenius = 0.0;
    double spectral = 0.0;
    double spectral_simplified = 0.0;
};
struct BoundReport {
    double delta_plus = 0.0;
    double delta_plus_prime = 0.0;
    double sigma_r = 0.0;
    double sigma_r1 = 0.0;
    double h_frobenius = 0.0;
    double t_h_inv_norm = 0.0;
    std::optional<ReferenceBounds> reference;
};
// delta_plus = sqrt(2) ||H||_F ||(T_r^H H)^+|| sigma_{r+1} / sigma_r and
// delta_plus_prime = sigma_{r+1} + 2 delta_plus ||A||; T_r^H H and its
// singular values on the GPU
template <ScalarField T>
BoundReport error_bounds_from_parts(const Matrix<T>& t_r, const std::vector<double>& singulars, const Matrix<T>& h,
                                    std::size_t r) {
    if (r < 1 || r > singulars.size()) throw DimensionError("error_bounds: rank out of range");
    if (t_r.cols() != r || t_r.rows() != h.rows()) throw DimensionError("error_bounds: shape mismatch");
    if (h.cols() < r) throw DimensionError("error_bounds: sketch narrower than rank");
    BoundReport rep;
    rep.sigma_r = singulars[r - 1];
    rep.sigma_r1 = r < singulars.size() ? singulars[r] : 0.0;
    rep.h_frobenius = frobenius_norm(h);
    const auto gsv = svd_values(matmul(t_r.adjoint(), h));
    if (gsv.back() <= 0.0) throw SingularMatrixError("unlucky multiplier: T_r^H H is singular, the bound is undefined");
    rep.t_h_inv_norm = 1.0 / gsv.back();
    rep.delta_plus = std::numbers::sqrt2 * rep.h_frobenius * rep.t_h_inv_norm * rep.sigma_r1 / rep.sigma_r;
    rep.delta_plus_prime = rep.sigma_r1 + 2.0 * rep.delta_plus * singulars.front();
    const std::size_t p = h.cols() - r;
    if (p >= 2) {
        double tail = 0.0;
        for (std::size_t j = r; j < singulars.size(); ++j) tail += singulars[j] * singulars[j];
        const double rd = static_cast<double>(r), pd = static_cast<double>(p);
        ReferenceBounds ref;
        ref.frobenius = std::sqrt(1.0 + rd / (pd - 1.0)) * std::sqrt(tail);
        ref.spectral = (1.0 + std::sqrt(rd / (pd - 1.0))) * rep.sigma_r1 +
                       (std::numbers::e * std::sqrt(rd + pd) / pd) * std::sqrt(tail);
        ref.spectral_simplified =
            (1.0 + 4.0 * std::sqrt(rd + pd) / (pd - 1.0) * std::sqrt(static_cast<double>(singulars.size()))) *
            rep.sigma_r1;
        rep.reference = ref;
    }
    return rep;
}
// 10 sqrt(2/pi) max_j ||(A - Q Q^H A) g_j|| over r_probes Gaussian probes
// g_j from RngStream(seed).derived(j + 1)
template <ScalarField T>
double posterior_estimate(const Matrix<T>& a, const LowRankResult<T>& result, std::size_t r_probes,
                          std::uint64_t seed) {
    if (r_probes < 1) throw DimensionError("posterior_estimate: need at least one probe");
    Matrix<T> g(a.cols(), r_probes);
    for (std::size_t j = 0; j < r_probes; ++j) {
        RngStream stream = RngStream(seed).derived(j + 1);
        for (std::size_t i = 0; i < a.cols(); ++i) g(i, j) = T(stream.next_gaussian());
    }
    const Matrix<T> ag = matmul(a, g);  // all probes at once on the GPU
    const Matrix<T> proj = result.apply_approximation(ag);
    double worst = 0.0;
    for (std::size_t j = 0; j < r_probes; ++j) {
        double norm_sq = 0.0;
        for (std::size_t i = 0; i < ag.rows(); ++i) norm_sq += field<T>::abs2(ag(i, j) - proj(i, j));
        worst = std::max(worst, std::sqrt(norm_sq));
    }
    return 10.0 * std::sqrt(2.0 / std::numbers::pi) * worst;
}
// gauge fix for comparing orthonormal factors (lowrank.hpp:263-282): each
// column rotated so its largest-magnitude entry is real and positive
template <ScalarField T>
void canonicalize_columns(Matrix<T>& q) {
    for (std::size_t j = 0; j < q.cols(); ++j) {
        std::size_t imax = 0;
        double best = -1.0;
        for (std::size_t i = 0; i < q.rows(); ++i) {
            const double mag = field<T>::abs2(q(i, j));
            if (mag > best) {
                best = mag;
                imax = i;
            }
        }
        const double mag = std::sqrt(best);
        if (mag == 0.0) continue;
        const T phase = field<T>::conj(q(imax, j)) * T(1.0 / mag);
        for (std::size_t i = 0; i < q.rows(); ++i) q(i, j) *= phase;
    }
}

// ---- the sampled-transform sketch check (lowrank.hpp:199-261) ---------------------------
enum class SketchVariant { Srft, CirculantPermutation };
struct SrftCheckResult {
    double residual = 0.0;  // ||(I - P_Y) A||
    double bound = 0.0;     // sqrt(1 + 7 n / l) sigma_{r+1}
    std::size_t sketch_width = 0;
    bool clamped = false;   // the prescribed width reached n and was cut back
};
// one device call: the sketch at its prescribed width (clamped to n), the
// unchecked basis, the residual norm and the bound
template <ScalarField T>
SrftCheckResult srft_sketch_check(const Matrix<T>& a, std::size_t r, std::uint64_t seed,
                                  SketchVariant variant = SketchVariant::Srft,
                                  std::optional<double> known_sigma_r1 = std::nullopt) {
    static_assert(std::is_same_v<T, double>, "srft_sketch_check takes the real input it lifts");
    rl_srft_check out{};
    detail::check(rl_srft_sketch_check(nullptr, RL_HOST, detail::i64(a.rows()), detail::i64(a.cols()), a.data(),
                                       detail::i64(r), seed, variant == SketchVariant::Srft ? 0 : 1,
                                       known_sigma_r1 ? *known_sigma_r1 : -1.0, &out));
    return {out.residual, out.bound, static_cast<std::size_t>(out.sketch_width), out.clamped != 0};
}

// ---- testbed inputs (testbed/inputs.hpp) ------------------------------------------------
namespace testbed {

// hard-block GENP input (inputs.hpp:18-49): leading n/2 block with four zero
// singular values, Gaussian Toeplitz borders scaled to unit estimate
inline RealMatrix gen_hard_block(std::size_t n, std::uint64_t seed) {
    if (n < 8 || n % 2 != 0) throw DimensionError("gen_hard_block: need even n >= 8");
    const std::size_t k = n / 2;
    const RealMatrix u = orthonormal_basis(gen_gaussian(k, k, derive_seed(seed, 1)));
    const RealMatrix v = orthonormal_basis(gen_gaussian(k, k, derive_seed(seed, 2)));
    RealMatrix scaled = u;
    for (std::size_t j = k - 4; j < k; ++j)
        for (std::size_t i = 0; i < k; ++i) scaled(i, j) = 0.0;
    const RealMatrix a_k = matmul(scaled, v.transpose());
    auto toeplitz = [&](std::uint64_t s) {
        RngStream rng(s);
        std::vector<double> diag(2 * k - 1);  // index (i - j) + (k - 1)
        for (double& t : diag) t = rng.next_gaussian();
        RealMatrix t(k, k);
        for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = 0; j < k; ++j) t(i, j) = diag[i + (k - 1) - j];
        const double norm = spectral_norm_estimate(t);
        for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = 0; j < k; ++j) t(i, j) /= norm;
        return t;
    };
    RealMatrix out(n, n);
    out.set_block(0, 0, a_k);
    out.set_block(0, k, toeplitz(derive_seed(seed, 3)));
    out.set_block(k, 0, toeplitz(derive_seed(seed, 4)));
    out.set_block(k, k, toeplitz(derive_seed(seed, 5)));
    return out;
}

struct LowRankInstance {
    RealMatrix a;
    TruncatedSVD<double> truth;
    std::vector<double> singulars;
};

// known numerical rank r (inputs.hpp:67-83): sigma_j = 1/(j+1) up to r, 1e-10 beyond
inline LowRankInstance gen_lownumrank(std::size_t n, std::size_t r, std::uint64_t seed) {
    if (r < 1 || r >= n) throw DimensionError("gen_lownumrank: need 1 <= r < n");
    const RealMatrix s = orthonormal_basis(gen_gaussian(n, n, derive_seed(seed, 1)));
    const RealMatrix t = orthonormal_basis(gen_gaussian(n, n, derive_seed(seed, 2)));
    std::vector<double> sigma(n);
    for (std::size_t j = 0; j < n; ++j) sigma[j] = (j < r) ? 1.0 / static_cast<double>(j + 1) : 1e-10;
    RealMatrix scaled = s;
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t i = 0; i < n; ++i) scaled(i, j) *= sigma[j];
    return LowRankInstance{matmul(scaled, t.transpose()),
                           TruncatedSVD<double>{s.leading_block(n, r),
                                                std::vector<double>(sigma.begin(), sigma.begin() + static_cast<std::ptrdiff_t>(r)),
                                                t.leading_block(n, r)},
                           std::move(sigma)};
}

inline std::vector<double> gen_gaussian_vector(std::size_t n, std::uint64_t seed) {
    return randla::gen_gaussian_vector(n, seed);
}

// the transform matrix itself (inputs.hpp:49-55)
inline ComplexMatrix gen_dft_input(std::size_t n) {
    if (!is_power_of_two(n) || n < 64) throw DimensionError("gen_dft_input: need a power of two >= 64");
    return dft_dense(n);
}

}  // namespace testbed

// ---- testbed statistics helpers (stats.hpp, parallel.hpp, norm_stats.hpp) --------------
struct StatSummary {  // stats.hpp: population statistics in a two-pass sweep
    double mean = 0.0;
    double max = 0.0;
    double min = 0.0;
    double std = 0.0;
};
inline StatSummary summarize(const std::vector<double>& values) {
    if (values.empty()) throw std::invalid_argument("summarize: no values");
    StatSummary s;
    s.min = s.max = values.front();
    double sum = 0.0;
    for (double v : values) {
        sum += v;
        s.min = std::min(s.min, v);
        s.max = std::max(s.max, v);
    }
    s.mean = sum / static_cast<double>(values.size());
    double var = 0.0;
    for (double v : values) var += (v - s.mean) * (v - s.mean);
    s.std = std::sqrt(var / static_cast<double>(values.size()));
    return s;
}
// fn(i) for i in [0, count) over the host's threads, every index its own
// result slot; the first exception is rethrown (parallel.hpp). Each worker
// thread gets its own device context and stream in the library.
inline void parallel_for_index(std::size_t count, const std::function<void(std::size_t)>& fn) {
    const std::size_t hw = std::max<std::size_t>(1, std::thread::hardware_concurrency());
    const std::size_t workers = std::min(hw, count);
    if (workers <= 1) {
        for (std::size_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errors(workers);
    for (std::size_t w = 0; w < workers; ++w)
        pool.emplace_back([&, w]() {
            try {
                for (std::size_t i = w; i < count; i += workers) fn(i);
            } catch (...) {
                errors[w] = std::current_exception();
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errors)
        if (e) std::rethrow_exception(e);
}
// Monte-Carlo condition statistics of a multiplier family (norm_stats.hpp)
struct RandomNormStats {
    MultiplierSpec family;
    std::size_t samples = 0;
    StatSummary norm;       // sigma_1
    StatSummary pinv_norm;  // 1 / sigma_min
    StatSummary cond;       // sigma_1 / sigma_min
};
inline RandomNormStats probe_norm_stats(const MultiplierSpec& spec, std::size_t trials) {
    if (trials < 1) throw DimensionError("probe_norm_stats: trials must be >= 1");
    std::vector<double> norms(trials), pinvs(trials), conds(trials);
    parallel_for_index(trials, [&](std::size_t t) {
        MultiplierSpec draw = spec;
        draw.seed = derive_seed(spec.seed, t);
        const std::vector<double> sv = multiplier_is_complex(draw) ? svd_values(materialize<Complex>(draw))
                                                                   : svd_values(materialize<double>(draw));
        norms[t] = sv.front();
        pinvs[t] = 1.0 / sv.back();
        conds[t] = sv.front() / sv.back();
    });
    return RandomNormStats{spec, trials, summarize(norms), summarize(pinvs), summarize(conds)};
}

// ---- BASELINE config 2: many independent 32x32 preprocessed solves ---------------
struct BatchedSolve {
    std::vector<double> x, residual, growth, lu;
    std::vector<int32_t> status;
    rl_batch_summary summary{};
};

inline BatchedSolve batched_preprocess_solve_32(const std::vector<double>& a, const std::vector<double>& g,
                                                const std::vector<double>& b) {
    const std::size_t batch = b.size() / 32;
    if (a.size() != batch * 1024 || g.size() != batch * 1024 || b.size() != batch * 32)
        throw DimensionError("batched_preprocess_solve_32: shapes must be (B,32,32), (B,32,32), (B,32)");
    BatchedSolve out;
    out.x.resize(batch * 32);
    out.residual.resize(batch);
    out.growth.resize(batch);
    out.lu.resize(batch * 1024);
    out.status.resize(batch);
    detail::check(rl_batched_genp_solve_32(nullptr, RL_HOST, static_cast<int64_t>(batch), a.data(), g.data(),
                                           b.data(), out.lu.data(), out.x.data(), out.residual.data(),
                                           out.growth.data(), out.status.data(), &out.summary));
    return out;
}

}  // namespace randla
