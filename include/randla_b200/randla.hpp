// randla_b200/randla.hpp — C++ drop-in for the hot path of the reference
// `randla` header library (namespace randla, /root/reference/proj/include/
// randla/*.hpp, double instantiation), implemented over the C ABI in
// randla_capi.h. A reference user swaps
//     #include "randla/preprocess.hpp"   ->   #include "randla_b200/randla.hpp"
// and links librandla_b200.so; the names, argument meaning and exception
// types below are the reference's. Every computation runs on the GPU; there
// is no CPU fallback (a host without a CUDA device gets DeviceError).
//
// Covered (reference file:line):
//   Matrix<double>/RealMatrix           matrix.hpp:15-110  (value type, row-major)
//   matmul                               matrix.hpp:115-121
//   derive_seed, hash_label              multipliers.hpp:54-56, rng.hpp:87-95
//   gen_gaussian, gen_gaussian_vector    multipliers.hpp:58-65, testbed/inputs.hpp:85-90
//   MultiplierKind/MultiplierSpec        multipliers.hpp:20-40
//   spectral_norm_estimate               norms.hpp:35-78
//   LuFactors, genp_factor, lu_solve     lu.hpp:17-28, :40-58, :100-123
//   gepp_factor, lu_solve_transpose      lu.hpp:62-98, :127-147 (bit-identical)
//   BlockNode, BlockFactorization,
//   block_ge_factor, block_solve,
//   balanced_split, schur_complement     block_ge.hpp:18-218 (bit-identical pivots,
//                                        Schur leaves and block_solve results)
//   relative_residual                    lu.hpp:155-161 (host arithmetic, as in the reference)
//   SolveOutcome, preprocess_solve,
//   preprocess_solve_with_retry          preprocess.hpp:9-14, :156-196
//   matmul_by_circulant,
//   matmul_by_toeplitz_block             circulant.hpp:171-203 (first-column forms)
//   orthonormal_basis, range_find,
//   approximation_residual               qr.hpp:51-54, lowrank.hpp:62-83, :99-102
//   batched_preprocess_solve_32          BASELINE config 2 (no reference counterpart:
//                                        the reference loops preprocess_solve per trial)
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "randla_capi.h"

namespace randla {

// ---- error contract (types.hpp:44-78) -------------------------------------
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
}  // namespace detail

// ---- dense row-major matrix (matrix.hpp:15-110) ------------------------------
class RealMatrix {
  public:
    RealMatrix() = default;
    RealMatrix(std::size_t rows, std::size_t cols, double fill = 0.0) : r_(rows), c_(cols), e_(rows * cols, fill) {
        if (rows == 0 || cols == 0) throw DimensionError("matrix dimensions must be positive");
    }
    RealMatrix(std::size_t rows, std::size_t cols, std::vector<double> entries)
        : r_(rows), c_(cols), e_(std::move(entries)) {
        if (rows == 0 || cols == 0) throw DimensionError("matrix dimensions must be positive");
        if (e_.size() != rows * cols) throw DimensionError("entry count does not match rows*cols");
    }
    static RealMatrix identity(std::size_t n) {
        RealMatrix m(n, n);
        for (std::size_t i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    std::size_t rows() const { return r_; }
    std::size_t cols() const { return c_; }
    double& operator()(std::size_t i, std::size_t j) { return e_[i * c_ + j]; }
    const double& operator()(std::size_t i, std::size_t j) const { return e_[i * c_ + j]; }
    const std::vector<double>& entries() const { return e_; }
    double* data() { return e_.data(); }
    const double* data() const { return e_.data(); }
    bool operator==(const RealMatrix& o) const { return r_ == o.r_ && c_ == o.c_ && e_ == o.e_; }

  private:
    std::size_t r_ = 0, c_ = 0;
    std::vector<double> e_;
};
template <typename T>
using Matrix = RealMatrix;  // the double instantiation is the one on the path

inline RealMatrix matmul(const RealMatrix& a, const RealMatrix& b) {
    if (a.cols() != b.rows()) throw DimensionError("matmul: inner dimensions differ");
    RealMatrix out(a.rows(), b.cols());
    const int64_t m = static_cast<int64_t>(a.rows()), k = static_cast<int64_t>(a.cols()),
                  n = static_cast<int64_t>(b.cols());
    detail::check(rl_dgemm(nullptr, RL_HOST, m, n, k, a.data(), k, b.data(), n, out.data(), n));
    return out;
}

inline std::vector<double> matvec(const RealMatrix& a, const std::vector<double>& x) {
    if (a.cols() != x.size()) throw DimensionError("matvec: shape mismatch");
    std::vector<double> y(a.rows(), 0.0);
    for (std::size_t i = 0; i < a.rows(); ++i) {
        double acc = 0.0;
        for (std::size_t j = 0; j < a.cols(); ++j) acc += a(i, j) * x[j];
        y[i] = acc;
    }
    return y;
}

inline double norm2(const std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
}

// ---- multipliers (multipliers.hpp) ---------------------------------------------
enum class MultiplierKind { None, Gaussian, RealCirculant, GaussianCirculant };

struct MultiplierSpec {
    MultiplierKind kind = MultiplierKind::None;
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::uint64_t seed = 0;
};

inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t k1, std::uint64_t k2 = 0) {
    return rl_derive_seed(seed, k1, k2);
}
inline std::uint64_t hash_label(const char* s) { return rl_hash_label(s); }

inline RealMatrix gen_gaussian(std::size_t m, std::size_t n, std::uint64_t seed) {
    RealMatrix out(m, n);
    detail::check(rl_gen_gaussian(static_cast<int64_t>(m), static_cast<int64_t>(n), seed, out.data()));
    return out;
}
inline std::vector<double> gen_gaussian_vector(std::size_t n, std::uint64_t seed) {
    std::vector<double> v(n);
    detail::check(rl_gen_gaussian(static_cast<int64_t>(n), 1, seed, v.data()));
    return v;
}

// ---- norms / GENP (norms.hpp, lu.hpp) ---------------------------------------------
inline double spectral_norm_estimate(const RealMatrix& a) {
    double out = 0.0;
    detail::check(rl_spectral_norm_estimate(nullptr, RL_HOST, static_cast<int64_t>(a.rows()),
                                            static_cast<int64_t>(a.cols()), a.data(), &out));
    return out;
}

struct LuFactors {
    RealMatrix lower;
    RealMatrix upper;
    std::optional<std::vector<std::size_t>> perm;  // empty for GENP; GEPP: original row at position i
    std::vector<double> pivots() const {
        std::vector<double> p(upper.rows());
        for (std::size_t j = 0; j < upper.rows(); ++j) p[j] = upper(j, j);
        return p;
    }
};

namespace detail {
inline LuFactors unpack(const RealMatrix& packed) {
    const std::size_t n = packed.rows();
    LuFactors f{RealMatrix::identity(n), RealMatrix(n, n), std::nullopt};
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) (j < i ? f.lower(i, j) : f.upper(i, j)) = packed(i, j);
    return f;
}
inline RealMatrix pack(const LuFactors& f) {
    const std::size_t n = f.upper.rows();
    RealMatrix p(n, n);
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t j = 0; j < n; ++j) p(i, j) = j < i ? f.lower(i, j) : f.upper(i, j);
    return p;
}
}  // namespace detail

inline LuFactors genp_factor(const RealMatrix& a) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("genp_factor: square input required");
    RealMatrix packed(n, n);
    rl_solve_info info{};
    const rl_status st = rl_genp_factor(nullptr, RL_HOST, static_cast<int64_t>(n), a.data(), packed.data(), &info);
    detail::check(st, info.zero_pivot_step);  // step read after the call
    return detail::unpack(packed);
}

namespace detail {
inline std::vector<double> gepp_solve(const LuFactors& f, const std::vector<double>& b, bool transpose);
}
inline std::vector<double> lu_solve(const LuFactors& f, const std::vector<double>& b) {
    if (f.perm) return detail::gepp_solve(f, b, false);
    const std::size_t n = f.upper.rows();
    if (b.size() != n) throw DimensionError("lu_solve: length mismatch");
    const RealMatrix packed = detail::pack(f);
    std::vector<double> x(n);
    detail::check(rl_lu_solve(nullptr, RL_HOST, static_cast<int64_t>(n), packed.data(), b.data(), x.data()));
    return x;
}

// ---- GEPP and block elimination (lu.hpp:62-147, block_ge.hpp) ----------------
// The device keeps the reference's arithmetic order: factors, permutations,
// pivots, Schur complements and block_solve results are bit-identical.
namespace detail {
inline RealMatrix pack_lu(const LuFactors& f) { return pack(f); }
inline std::vector<int64_t> perm_of(const LuFactors& f) {
    const std::size_t n = f.upper.rows();
    std::vector<int64_t> p(n);
    for (std::size_t i = 0; i < n; ++i) p[i] = f.perm ? static_cast<int64_t>((*f.perm)[i]) : static_cast<int64_t>(i);
    return p;
}
inline std::vector<double> gepp_solve(const LuFactors& f, const std::vector<double>& b, bool transpose) {
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

inline LuFactors gepp_factor(const RealMatrix& a) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("gepp_factor: square input required");
    RealMatrix packed(n, n);
    std::vector<int64_t> p(n);
    int64_t step = 0;
    detail::check(rl_gepp_factor(nullptr, RL_HOST, static_cast<int64_t>(n), a.data(), packed.data(), p.data(), &step));
    LuFactors f = detail::unpack(packed);
    f.perm = std::vector<std::size_t>(p.begin(), p.end());
    return f;
}

inline std::vector<double> lu_solve_transpose(const LuFactors& f, const std::vector<double>& c) {
    return detail::gepp_solve(f, c, true);
}

struct BlockNode {  // block_ge.hpp:18-35
    std::size_t dim = 0, offset = 0, pivot_size = 0;
    RealMatrix block_matrix;
    std::optional<LuFactors> block_lu;
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
        LuFactors lu = detail::unpack(sub(f.factors, o, o, k, k));
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
    const LuFactors b_lu = gepp_factor(b);
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

inline double relative_residual(const RealMatrix& a, const std::vector<double>& x, const std::vector<double>& b) {
    const std::vector<double> ax = matvec(a, x);
    double num = 0.0;
    for (std::size_t i = 0; i < b.size(); ++i) num += (ax[i] - b[i]) * (ax[i] - b[i]);
    return std::sqrt(num) / norm2(b);
}

// ---- preprocessed solve (preprocess.hpp) -----------------------------------------
struct SolveOutcome {
    std::vector<double> x;
    std::vector<double> residual_history;
    bool diverged = false;
    rl_solve_info info{};
};

inline SolveOutcome preprocess_solve(const RealMatrix& a, const std::vector<double>& b, const MultiplierSpec& pre_spec,
                                     const MultiplierSpec& post_spec, std::size_t refine_steps) {
    const std::size_t n = a.rows();
    if (a.cols() != n) throw DimensionError("preprocess_solve: square input required");
    if (b.size() != n) throw DimensionError("preprocess_solve: length mismatch");
    if (pre_spec.kind != MultiplierKind::None)
        throw DimensionError("preprocess_solve: left multipliers are not on the B200 path");
    rl_multiplier m{};
    switch (post_spec.kind) {
        case MultiplierKind::None: m.kind = RL_MULT_NONE; break;
        case MultiplierKind::Gaussian: m.kind = RL_MULT_GAUSSIAN; break;
        case MultiplierKind::RealCirculant: m.kind = RL_MULT_REAL_CIRCULANT; break;
        case MultiplierKind::GaussianCirculant: m.kind = RL_MULT_GAUSSIAN_CIRCULANT; break;
    }
    m.seed = post_spec.seed;
    SolveOutcome out;
    out.x.resize(n);
    const rl_status st = rl_preprocessed_genp_solve(nullptr, RL_HOST, static_cast<int64_t>(n), a.data(), b.data(), &m,
                                                    static_cast<int64_t>(refine_steps), out.x.data(), nullptr, 0,
                                                    &out.info);
    detail::check(st, out.info.zero_pivot_step);
    out.residual_history.assign(out.info.residual_history, out.info.residual_history + out.info.history_len);
    out.diverged = out.info.diverged != 0;
    return out;
}

inline SolveOutcome preprocess_solve_with_retry(const RealMatrix& a, const std::vector<double>& b,
                                                MultiplierSpec pre_spec, MultiplierSpec post_spec,
                                                std::size_t refine_steps, std::size_t max_retries = 3) {
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

// ---- structured multipliers (circulant.hpp), first-column forms ------------------
inline RealMatrix matmul_by_circulant(const RealMatrix& a, const std::vector<double>& first_column) {
    if (a.cols() != first_column.size()) throw DimensionError("matmul_by_circulant: shape mismatch");
    RealMatrix out(a.rows(), a.cols());
    detail::check(rl_circulant_right_multiply(nullptr, RL_HOST, static_cast<int64_t>(a.rows()),
                                              static_cast<int64_t>(a.cols()), a.data(), first_column.data(),
                                              out.data()));
    return out;
}

inline RealMatrix matmul_by_toeplitz_block(const RealMatrix& a, const std::vector<double>& parent_column,
                                           std::size_t cols) {
    RealMatrix out(a.rows(), cols);
    detail::check(rl_toeplitz_right_multiply(nullptr, RL_HOST, static_cast<int64_t>(a.rows()),
                                             static_cast<int64_t>(a.cols()), a.data(),
                                             static_cast<int64_t>(parent_column.size()), parent_column.data(),
                                             static_cast<int64_t>(cols), out.data()));
    return out;
}

// ---- low-rank (qr.hpp, lowrank.hpp) ------------------------------------------------
inline RealMatrix orthonormal_basis(const RealMatrix& y) {
    RealMatrix q(y.rows(), y.cols());
    int64_t bad = 0;
    const rl_status st = rl_cholqr2(nullptr, RL_HOST, static_cast<int64_t>(y.rows()), static_cast<int64_t>(y.cols()),
                                    y.data(), q.data(), nullptr, &bad);
    if (st == RL_ERR_RANK_DEFICIENCY)
        throw RankDeficiencyError("qr: numerically rank-deficient at column " + std::to_string(bad));
    detail::check(st);
    return q;
}

struct LowRankResult {
    RealMatrix q;
    std::size_t rank = 0, oversample = 0, power_steps = 0;
    rl_lowrank_info info{};
};

inline LowRankResult range_find(const RealMatrix& a, std::size_t r, std::size_t p, MultiplierSpec spec,
                                std::size_t power_steps = 0) {
    if (power_steps != 0) throw DimensionError("range_find: power steps are not on the B200 path");
    const std::size_t l = r + p;
    LowRankResult out{RealMatrix(a.rows(), l), r, p, power_steps, {}};
    rl_multiplier m{};
    m.kind = spec.kind == MultiplierKind::Gaussian ? RL_MULT_GAUSSIAN : RL_MULT_GAUSSIAN_CIRCULANT;
    m.seed = spec.seed;
    const rl_status st = rl_range_find_residual(nullptr, RL_HOST, static_cast<int64_t>(a.rows()),
                                                static_cast<int64_t>(a.cols()), a.data(), static_cast<int64_t>(l), &m,
                                                out.q.data(), &out.info);
    if (st == RL_ERR_RANK_DEFICIENCY)
        throw RankDeficiencyError("qr: numerically rank-deficient at column " +
                                  std::to_string(out.info.rank_deficient_column));
    detail::check(st);
    return out;
}

// ||A - Q Q^T A||_2 of the range_find result, evaluated with A (lowrank.hpp:99-102)
inline double approximation_residual(const RealMatrix&, const LowRankResult& result) {
    return result.info.residual_spectral;
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
