/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain-C restatement of the
 * reference's hot path). See oracle.h for scope and pinning. Built with
 * -ffp-contract=off and no -march flags so every expression rounds exactly as
 * the reference's x86-64 build does (no FMA contraction).
 */
#include "oracle.h"

#include <dlfcn.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- RNG --- */
/* rng.hpp:74-80 mix_key */
static uint64_t mix_key(uint64_t state, uint64_t key) {
    state ^= key + 0x9E3779B97F4A7C15ull + (state << 6) + (state >> 2);
    uint64_t z = state + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* rng.hpp:18 */
void or_rng_init(or_rng* r, uint64_t seed) {
    r->state = mix_key(0x9E3779B97F4A7C15ull, seed);
    r->has_spare = 0;
    r->spare = 0.0;
}

/* rng.hpp:20-25 */
void or_rng_derived(const or_rng* r, uint64_t key, or_rng* out) {
    *out = *r;
    out->state = mix_key(out->state, key);
    out->has_spare = 0;
}

/* rng.hpp:31-37 */
uint64_t or_rng_next_u64(or_rng* r) {
    r->state += 0x9E3779B97F4A7C15ull;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* rng.hpp:40 */
double or_rng_next_double(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:43 */
double or_rng_next_symmetric(or_rng* r) { return 2.0 * or_rng_next_double(r) - 1.0; }

/* rng.hpp:56-71 Marsaglia polar */
double or_rng_next_gaussian(or_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u, v, s;
    do {
        u = or_rng_next_symmetric(r);
        v = or_rng_next_symmetric(r);
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double f = sqrt(-2.0 * log(s) / s);
    r->spare = v * f;
    r->has_spare = 1;
    return u * f;
}

/* rng.hpp:87-95 FNV-1a */
uint64_t or_hash_label(const char* s) {
    uint64_t h = 1469598103934665603ull;
    for (; *s; ++s) {
        h ^= (uint64_t)(unsigned char)*s;
        h *= 1099511628211ull;
    }
    return h;
}

/* multipliers.hpp:54-56 */
uint64_t or_derive_seed(uint64_t seed, uint64_t k1, uint64_t k2) {
    or_rng a, b, c;
    or_rng_init(&a, seed);
    or_rng_derived(&a, k1, &b);
    or_rng_derived(&b, k2, &c);
    return or_rng_next_u64(&c);
}

/* multipliers.hpp:58-65: entry (i, j) is draw i*n + j of one stream */
void or_gen_gaussian(int64_t m, int64_t n, uint64_t seed, double* out) {
    or_rng r;
    or_rng_init(&r, seed);
    for (int64_t i = 0; i < m * n; ++i) out[i] = or_rng_next_gaussian(&r);
}

/* testbed/inputs.hpp:85-90 */
void or_gen_gaussian_vector(int64_t n, uint64_t seed, double* out) { or_gen_gaussian(n, 1, seed, out); }

/* multipliers.hpp:67-73 (uniform [-1, 1] first column, Example 6.1) */
void or_gen_real_circulant_column(int64_t n, uint64_t seed, double* out) {
    or_rng r;
    or_rng_init(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = or_rng_next_symmetric(&r);
}

/* ------------------------------------------------------ dense products --- */
/* matrix.hpp:115-121 delegates to Eigen's GEMM; here OpenBLAS (numpy's
 * bundled scipy-openblas, ILP64) single-threaded when it can be found, else
 * an i-k-j loop. Both differ from Eigen only in summation order. */
typedef void (*dgemm_fn)(const char*, const char*, const int64_t*, const int64_t*, const int64_t*,
                         const double*, const double*, const int64_t*, const double*, const int64_t*,
                         const double*, double*, const int64_t*, size_t, size_t);
static dgemm_fn g_dgemm = 0;
static int g_dgemm_probed = 0;
static pthread_mutex_t g_probe_mu = PTHREAD_MUTEX_INITIALIZER;

static void probe_blas(void) {
    pthread_mutex_lock(&g_probe_mu);
    if (!g_dgemm_probed) {
        const char* path = getenv("RANDLA_ORACLE_OPENBLAS");
        if (path && *path) {
            void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
            if (h) {
                g_dgemm = (dgemm_fn)dlsym(h, "scipy_dgemm_64_");
                void (*set_threads)(int) = (void (*)(int))dlsym(h, "scipy_openblas_set_num_threads64_");
                if (set_threads) set_threads(1);
            }
        }
        g_dgemm_probed = 1;
    }
    pthread_mutex_unlock(&g_probe_mu);
}

int or_matmul_uses_blas(void) {
    probe_blas();
    return g_dgemm != 0;
}

void or_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c) {
    probe_blas();
    if (g_dgemm) {
        /* row-major C = A B  <=>  column-major C^T = B^T A^T */
        const double one = 1.0, zero = 0.0;
        g_dgemm("N", "N", &n, &m, &k, &one, b, &n, a, &k, &zero, c, &n, 1, 1);
        return;
    }
    for (int64_t i = 0; i < m; ++i) {
        double* ci = c + i * n;
        for (int64_t j = 0; j < n; ++j) ci[j] = 0.0;
        for (int64_t t = 0; t < k; ++t) {
            const double ait = a[i * k + t];
            const double* bt = b + t * n;
            for (int64_t j = 0; j < n; ++j) ci[j] += ait * bt[j];
        }
    }
}

/* matrix.hpp:146-156 */
void or_matvec(int64_t m, int64_t n, const double* a, const double* x, double* y) {
    for (int64_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int64_t j = 0; j < n; ++j) acc += a[i * n + j] * x[j];
        y[i] = acc;
    }
}

/* matrix.hpp:172-177 */
double or_norm2(int64_t n, const double* v) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* matrix.hpp:158-163 */
double or_frobenius_norm(int64_t m, int64_t n, const double* a) { return or_norm2(m * n, a); }

/* matrix.hpp:165-170 */
double or_max_abs(int64_t m, int64_t n, const double* a) {
    double r = 0.0;
    for (int64_t i = 0; i < m * n; ++i) {
        const double v = sqrt(a[i] * a[i]);
        r = r > v ? r : v;
    }
    return r;
}

/* norms.hpp:35-78: floor = largest column/row norm; power iteration on
 * A^T A from x_j = 1 + j/(n+1), at most 200 steps, stop when
 * |‖Ax‖ - est| <= 1e-9 ‖Ax‖. */
double or_spectral_norm_estimate(int64_t m, int64_t n, const double* a) {
    double floor_norm = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s += a[i * n + j] * a[i * n + j];
        floor_norm = floor_norm > s ? floor_norm : s;
    }
    for (int64_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += a[i * n + j] * a[i * n + j];
        floor_norm = floor_norm > s ? floor_norm : s;
    }
    floor_norm = sqrt(floor_norm);
    if (floor_norm == 0.0) return 0.0;

    double* x = (double*)malloc(sizeof(double) * n);
    double* y = (double*)malloc(sizeof(double) * n);
    double* ax = (double*)malloc(sizeof(double) * m);
    for (int64_t j = 0; j < n; ++j) x[j] = 1.0 + (double)j / ((double)n + 1.0);
    const double nx = or_norm2(n, x);
    for (int64_t j = 0; j < n; ++j) x[j] = (1.0 / nx) * x[j];
    double est = 0.0;
    for (int it = 0; it < 200; ++it) {
        or_matvec(m, n, a, x, ax);
        const double nax = or_norm2(m, ax);
        if (nax == 0.0) break;
        for (int64_t j = 0; j < n; ++j) y[j] = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            const double axi = ax[i];
            for (int64_t j = 0; j < n; ++j) y[j] += a[i * n + j] * axi;
        }
        const double ny = or_norm2(n, y);
        if (ny == 0.0) break;
        for (int64_t j = 0; j < n; ++j) x[j] = (1.0 / ny) * y[j];
        if (fabs(nax - est) <= 1e-9 * nax) {
            est = nax;
            break;
        }
        est = nax;
    }
    free(x);
    free(y);
    free(ax);
    return est > floor_norm ? est : floor_norm;
}

/* ------------------------------------------------------------- GENP --- */
/* lu.hpp:40-58 (tolerance types.hpp:42): natural-order elimination, no row
 * exchanges, verdict ZeroPivot(j+1) when |u_jj| <= 1e-13 n ‖a‖_est. */
int or_genp_factor(int64_t n, const double* a, double* lu, int64_t* zero_step, double* tol_out) {
    const double tol = (1e-13 * (double)n) * or_spectral_norm_estimate(n, n, a);
    if (tol_out) *tol_out = tol;
    if (lu != a) memcpy(lu, a, sizeof(double) * n * n);
    if (zero_step) *zero_step = 0;
    for (int64_t j = 0; j < n; ++j) {
        const double piv = lu[j * n + j];
        if (sqrt(piv * piv) <= tol) {
            if (zero_step) *zero_step = j + 1;
            return OR_ZERO_PIVOT;
        }
        for (int64_t i = j + 1; i < n; ++i) {
            const double l = lu[i * n + j] / piv;
            lu[i * n + j] = l; /* lower(i, j) */
            for (int64_t k = j + 1; k < n; ++k) lu[i * n + k] = lu[i * n + k] - l * lu[j * n + k];
        }
    }
    return OR_OK;
}

/* elimination steps j0..j1-1 of genp_factor's loop (lu.hpp:47-56), in place on
 * the n x n matrix `lu` (no verdict): the bounded sample of the full-size GENP
 * workload that bench.py's cpu_baseline times (the same arithmetic and memory
 * traffic per step as or_genp_factor) */
void or_genp_steps(int64_t n, double* lu, int64_t j0, int64_t j1) {
    for (int64_t j = j0; j < j1 && j < n; ++j) {
        const double piv = lu[j * n + j];
        for (int64_t i = j + 1; i < n; ++i) {
            const double l = lu[i * n + j] / piv;
            lu[i * n + j] = l;
            for (int64_t k = j + 1; k < n; ++k) lu[i * n + k] = lu[i * n + k] - l * lu[j * n + k];
        }
    }
}

/* lu.hpp:100-123 (no permutation) */
void or_lu_solve(int64_t n, const double* lu, const double* b, double* x) {
    if (x != b) memcpy(x, b, sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) {
        double acc = x[i];
        for (int64_t k = 0; k < i; ++k) acc -= lu[i * n + k] * x[k];
        x[i] = acc;
    }
    for (int64_t ii = n; ii-- > 0;) {
        double acc = x[ii];
        for (int64_t k = ii + 1; k < n; ++k) acc -= lu[ii * n + k] * x[k];
        x[ii] = acc / lu[ii * n + ii];
    }
}

/* lu.hpp:155-161 */
double or_relative_residual(int64_t n, const double* a, const double* x, const double* b) {
    double* ax = (double*)malloc(sizeof(double) * n);
    or_matvec(n, n, a, x, ax);
    double num = 0.0;
    for (int64_t i = 0; i < n; ++i) num += (ax[i] - b[i]) * (ax[i] - b[i]);
    free(ax);
    return sqrt(num) / or_norm2(n, b);
}

/* -------------------------------------------------------------- FFT --- */
static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

/* complex product exactly as GCC evaluates std::complex<double> * for finite
 * values on x86-64 (no contraction): (ac - bd, ad + bc) */
static inline void cmul(double a, double b, double c, double d, double* re, double* im) {
    *re = a * c - b * d;
    *im = a * d + b * c;
}

/* fft.hpp:35-57 iterative radix-2, bit reversal first, twiddle recurrence */
static void fft_pow2(int64_t n, double* z, double sign) {
    for (int64_t i = 1, j = 0; i < n; ++i) {
        int64_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) {
            double t0 = z[2 * i], t1 = z[2 * i + 1];
            z[2 * i] = z[2 * j];
            z[2 * i + 1] = z[2 * j + 1];
            z[2 * j] = t0;
            z[2 * j + 1] = t1;
        }
    }
    for (int64_t len = 2; len <= n; len <<= 1) {
        const double ang = sign * 2.0 * M_PI / (double)len;
        const double wr0 = cos(ang), wi0 = sin(ang);
        for (int64_t i = 0; i < n; i += len) {
            double wr = 1.0, wi = 0.0;
            for (int64_t j = 0; j < len / 2; ++j) {
                const double ur = z[2 * (i + j)], ui = z[2 * (i + j) + 1];
                double vr, vi;
                cmul(z[2 * (i + j + len / 2)], z[2 * (i + j + len / 2) + 1], wr, wi, &vr, &vi);
                z[2 * (i + j)] = ur + vr;
                z[2 * (i + j) + 1] = ui + vi;
                z[2 * (i + j + len / 2)] = ur - vr;
                z[2 * (i + j + len / 2) + 1] = ui - vi;
                double nr, ni;
                cmul(wr, wi, wr0, wi0, &nr, &ni);
                wr = nr;
                wi = ni;
            }
        }
    }
}

/* fft.hpp:21-30 dense fallback for non-power-of-two lengths */
static void dft_dense_apply(int64_t n, double* z, double sign) {
    double* root = (double*)malloc(sizeof(double) * 2 * n);
    double* out = (double*)calloc(2 * n, sizeof(double));
    for (int64_t k = 0; k < n; ++k) {
        const double ang = sign * 2.0 * M_PI * (double)k / (double)n;
        root[2 * k] = cos(ang);
        root[2 * k + 1] = sin(ang);
    }
    for (int64_t i = 0; i < n; ++i) {
        double ar = 0.0, ai = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const int64_t k = (i * j) % n;
            double pr, pi;
            cmul(root[2 * k], root[2 * k + 1], z[2 * j], z[2 * j + 1], &pr, &pi);
            ar += pr;
            ai += pi;
        }
        out[2 * i] = ar;
        out[2 * i + 1] = ai;
    }
    memcpy(z, out, sizeof(double) * 2 * n);
    free(root);
    free(out);
}

/* fft.hpp:76-83 */
int or_fft(int64_t n, double* z) {
    if (n < 1) return OR_DIMENSION_ERROR;
    if (is_pow2(n))
        fft_pow2(n, z, +1.0);
    else
        dft_dense_apply(n, z, +1.0);
    return OR_OK;
}

/* fft.hpp:88-98 */
int or_inverse_fft(int64_t n, double* z) {
    if (n < 1) return OR_DIMENSION_ERROR;
    const double inv_n = 1.0 / (double)n;
    if (is_pow2(n))
        fft_pow2(n, z, -1.0);
    else
        dft_dense_apply(n, z, -1.0);
    for (int64_t i = 0; i < 2 * n; ++i) z[i] *= inv_n;
    return OR_OK;
}

/* circulant.hpp:57-68 strip_imag + :70-76 spectral_apply + :85-91
 * circulant_apply (real). spectrum = fft(c) (circulant.hpp:19-22). */
static int circulant_apply_spec(int64_t n, const double* spectrum, double cmax, const double* x, double* y,
                                double* work) {
    for (int64_t i = 0; i < n; ++i) {
        work[2 * i] = x[i];
        work[2 * i + 1] = 0.0;
    }
    or_fft(n, work);
    for (int64_t i = 0; i < n; ++i) {
        double re, im;
        cmul(work[2 * i], work[2 * i + 1], spectrum[2 * i], spectrum[2 * i + 1], &re, &im);
        work[2 * i] = re;
        work[2 * i + 1] = im;
    }
    or_inverse_fft(n, work);
    const double scale = cmax * or_norm2(n, x);
    double imag2 = 0.0, full2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        imag2 += work[2 * i + 1] * work[2 * i + 1];
        full2 += work[2 * i] * work[2 * i] + work[2 * i + 1] * work[2 * i + 1];
    }
    if (sqrt(imag2) > 1e-11 * (sqrt(full2) + scale)) return OR_LOGIC_ERROR;
    for (int64_t i = 0; i < n; ++i) y[i] = work[2 * i];
    return OR_OK;
}

static double* spectrum_of(int64_t n, const double* c) {
    double* s = (double*)malloc(sizeof(double) * 2 * n);
    for (int64_t i = 0; i < n; ++i) {
        s[2 * i] = c[i];
        s[2 * i + 1] = 0.0;
    }
    or_fft(n, s);
    return s;
}

static double max_abs_vec(int64_t n, const double* c) {
    double m = 0.0;
    for (int64_t i = 0; i < n; ++i) m = m > fabs(c[i]) ? m : fabs(c[i]);
    return m;
}

int or_circulant_apply(int64_t n, const double* c, const double* x, double* y) {
    double* spec = spectrum_of(n, c);
    double* work = (double*)malloc(sizeof(double) * 2 * n);
    const int st = circulant_apply_spec(n, spec, max_abs_vec(n, c), x, y, work);
    free(spec);
    free(work);
    return st;
}

/* circulant.hpp:40-45: transposed circulant has first column c[(n-i) mod n] */
static void transposed_column(int64_t n, const double* c, double* ct) {
    for (int64_t i = 0; i < n; ++i) ct[i] = c[(n - i) % n];
}

/* circulant.hpp:171-185: row i of A C = C^T a_i */
int or_matmul_by_circulant(int64_t m, int64_t n, const double* a, const double* c, double* out) {
    double* ct = (double*)malloc(sizeof(double) * n);
    transposed_column(n, c, ct);
    double* spec = spectrum_of(n, ct);
    const double cmax = max_abs_vec(n, ct);
    double* work = (double*)malloc(sizeof(double) * 2 * n);
    int st = OR_OK;
    for (int64_t i = 0; i < m && st == OR_OK; ++i) st = circulant_apply_spec(n, spec, cmax, a + i * n, out + i * n, work);
    free(ct);
    free(spec);
    free(work);
    return st;
}

/* circulant.hpp:187-203: pad each row of A to the parent size, apply the
 * transposed parent, keep the first l entries */
int or_matmul_by_toeplitz_block(int64_t m, int64_t k, const double* a, int64_t np, const double* c, int64_t l,
                                double* out) {
    if (k > np || l > np || k < 1 || l < 1) return OR_DIMENSION_ERROR;
    double* ct = (double*)malloc(sizeof(double) * np);
    transposed_column(np, c, ct);
    double* spec = spectrum_of(np, ct);
    const double cmax = max_abs_vec(np, ct);
    double* work = (double*)malloc(sizeof(double) * 2 * np);
    double* row = (double*)calloc(np, sizeof(double));
    double* prod = (double*)malloc(sizeof(double) * np);
    int st = OR_OK;
    for (int64_t i = 0; i < m && st == OR_OK; ++i) {
        memcpy(row, a + i * k, sizeof(double) * k);
        st = circulant_apply_spec(np, spec, cmax, row, prod, work);
        memcpy(out + i * l, prod, sizeof(double) * l);
    }
    free(ct);
    free(spec);
    free(work);
    free(row);
    free(prod);
    return st;
}

/* ------------------------------------------------ preprocessed solve --- */
/* preprocess.hpp:156-180 with pre = none; iterative_refine :115-143 with
 * x0 = 0 and refine+1 steps, first history entry dropped. */
int or_preprocess_solve(int64_t n, const double* a, const double* b, int post_kind, const double* post,
                        int64_t refine, double* x, double* history, int* diverged, int64_t* zero_step,
                        double* lu_out, double* product_out) {
    double* product = (double*)malloc(sizeof(double) * n * n);
    int st = OR_OK;
    if (post_kind == OR_POST_DENSE)
        or_matmul(n, n, n, a, post, product);
    else if (post_kind == OR_POST_CIRCULANT)
        st = or_matmul_by_circulant(n, n, a, post, product);
    else
        memcpy(product, a, sizeof(double) * n * n);
    if (product_out && st == OR_OK) memcpy(product_out, product, sizeof(double) * n * n);
    if (st != OR_OK) {
        free(product);
        return st;
    }
    double* lu = lu_out ? lu_out : (double*)malloc(sizeof(double) * n * n);
    int64_t zs = 0;
    st = or_genp_factor(n, product, lu, &zs, 0);
    if (zero_step) *zero_step = zs;
    free(product);
    if (st != OR_OK) {
        if (!lu_out) free(lu);
        return st;
    }
    double* r = (double*)malloc(sizeof(double) * n);
    double* y = (double*)malloc(sizeof(double) * n);
    double* d = (double*)malloc(sizeof(double) * n);
    const double bnorm = or_norm2(n, b);
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    /* residual(x0 = 0) */
    or_matvec(n, n, a, x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double last = or_norm2(n, r) / bnorm;
    int streak = 0, div = 0;
    const int64_t steps = refine + 1;
    int64_t h = 0;
    for (int64_t s = 0; s < steps; ++s) {
        or_lu_solve(n, lu, r, y);
        if (post_kind == OR_POST_DENSE)
            or_matvec(n, n, post, y, d);
        else if (post_kind == OR_POST_CIRCULANT)
            st = or_circulant_apply(n, post, y, d);
        else
            memcpy(d, y, sizeof(double) * n);
        if (st != OR_OK) break;
        for (int64_t i = 0; i < n; ++i) x[i] += d[i];
        or_matvec(n, n, a, x, r);
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
        const double rel = or_norm2(n, r) / bnorm;
        streak = (rel > last) ? streak + 1 : 0;
        if (history) history[h] = rel;
        ++h;
        last = rel;
        if (streak >= 2) {
            div = 1;
            break;
        }
    }
    if (history)
        for (; h < steps; ++h) history[h] = NAN; /* loop stopped early */
    if (diverged) *diverged = div;
    free(r);
    free(y);
    free(d);
    if (!lu_out) free(lu);
    return st;
}

/* ------------------------------------------------------ config-2 driver --- */
typedef struct {
    int64_t dim;
    uint64_t base;
    int64_t i0, count;
    int workers, w;
    double *a_out, *g_out, *b_out, *x_out, *resid_out, *growth_out, *lu_out;
    int64_t* status_out;
} batch_job;

static void* batch_worker(void* p) {
    batch_job* j = (batch_job*)p;
    const int64_t d = j->dim, dd = d * d;
    double* a = (double*)malloc(sizeof(double) * dd);
    double* g = (double*)malloc(sizeof(double) * dd);
    double* b = (double*)malloc(sizeof(double) * d);
    double* x = (double*)malloc(sizeof(double) * d);
    double* lu = (double*)malloc(sizeof(double) * dd);
    double* prod = (double*)malloc(sizeof(double) * dd);
    double hist[1];
    for (int64_t k = j->w; k < j->count; k += j->workers) {
        const uint64_t ts = j->base + (uint64_t)(j->i0 + k);
        or_gen_gaussian(d, d, or_derive_seed(ts, 1, 0), a);
        or_gen_gaussian_vector(d, or_derive_seed(ts, 2, 0), b);
        or_gen_gaussian(d, d, or_derive_seed(ts, 3, 0), g);
        int div = 0;
        int64_t zs = 0;
        const int st = or_preprocess_solve(d, a, b, OR_POST_DENSE, g, 0, x, hist, &div, &zs, lu, prod);
        if (j->a_out) memcpy(j->a_out + k * dd, a, sizeof(double) * dd);
        if (j->g_out) memcpy(j->g_out + k * dd, g, sizeof(double) * dd);
        if (j->b_out) memcpy(j->b_out + k * d, b, sizeof(double) * d);
        if (j->x_out) memcpy(j->x_out + k * d, x, sizeof(double) * d);
        if (j->lu_out) memcpy(j->lu_out + k * dd, lu, sizeof(double) * dd);
        if (j->resid_out) j->resid_out[k] = st == OR_OK ? hist[0] : NAN;
        if (j->status_out) j->status_out[k] = st == OR_OK ? 0 : (st == OR_ZERO_PIVOT ? zs : -st);
        if (j->growth_out) {
            /* growth = max|U| / max|AG| (SURVEY App. A decision) */
            double mu = 0.0;
            for (int64_t r = 0; r < d; ++r)
                for (int64_t c = r; c < d; ++c) mu = mu > fabs(lu[r * d + c]) ? mu : fabs(lu[r * d + c]);
            j->growth_out[k] = st == OR_OK ? mu / or_max_abs(d, d, prod) : NAN;
        }
    }
    free(a);
    free(g);
    free(b);
    free(x);
    free(lu);
    free(prod);
    return 0;
}

void or_batched_config2(int64_t dim, uint64_t base, int64_t i0, int64_t count, int threads, double* a_out,
                        double* g_out, double* b_out, double* x_out, double* resid_out, int64_t* status_out,
                        double* growth_out, double* lu_out) {
    if (threads < 1) threads = 1;
    if (threads > count) threads = (int)count;
    if (threads < 1) return;
    batch_job* jobs = (batch_job*)calloc(threads, sizeof(batch_job));
    pthread_t* tids = (pthread_t*)calloc(threads, sizeof(pthread_t));
    for (int w = 0; w < threads; ++w) {
        batch_job* j = &jobs[w];
        j->dim = dim;
        j->base = base;
        j->i0 = i0;
        j->count = count;
        j->workers = threads;
        j->w = w;
        j->a_out = a_out;
        j->g_out = g_out;
        j->b_out = b_out;
        j->x_out = x_out;
        j->resid_out = resid_out;
        j->status_out = status_out;
        j->growth_out = growth_out;
        j->lu_out = lu_out;
        if (threads == 1)
            batch_worker(j);
        else
            pthread_create(&tids[w], 0, batch_worker, j);
    }
    if (threads > 1)
        for (int w = 0; w < threads; ++w) pthread_join(tids[w], 0);
    free(jobs);
    free(tids);
}

/* ---------------------------------------------------------------- QR --- */
/* qr.hpp:21-47: Householder thin QR (reflector convention beta =
 * -sign(x0)‖x‖ as in the standard LAPACK/Eigen makeHouseholder), then the
 * phase normalisation making diag(R) > 0 and the rank check
 * |r_jj| <= tol_rank(m, n) * spectral_norm_estimate(a). */
int or_qr(int64_t m, int64_t l, const double* a, double* q, double* r, int64_t* bad_col) {
    if (m < l) return OR_DIMENSION_ERROR;
    double* w = (double*)malloc(sizeof(double) * m * l); /* column-major working copy */
    double* tau = (double*)malloc(sizeof(double) * l);
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < l; ++j) w[j * m + i] = a[i * l + j];
    for (int64_t k = 0; k < l; ++k) {
        double* col = w + k * m;
        const double c0 = col[k];
        double tail = 0.0;
        for (int64_t i = k + 1; i < m; ++i) tail += col[i] * col[i];
        double beta;
        if (tail == 0.0) {
            tau[k] = 0.0;
            beta = c0;
            for (int64_t i = k + 1; i < m; ++i) col[i] = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int64_t i = k + 1; i < m; ++i) col[i] /= (c0 - beta);
            tau[k] = (beta - c0) / beta;
        }
        col[k] = beta;
        /* apply H = I - tau v v^T (v = [1; col[k+1:]]) to the trailing columns */
        for (int64_t j = k + 1; j < l; ++j) {
            double* cj = w + j * m;
            double dot = cj[k];
            for (int64_t i = k + 1; i < m; ++i) dot += col[i] * cj[i];
            dot *= tau[k];
            cj[k] -= dot;
            for (int64_t i = k + 1; i < m; ++i) cj[i] -= dot * col[i];
        }
    }
    /* R */
    for (int64_t i = 0; i < l; ++i)
        for (int64_t j = 0; j < l; ++j) r[i * l + j] = (j >= i) ? w[j * m + i] : 0.0;
    /* thin Q = H_0 ... H_{l-1} [I; 0], built backwards, column-major in qc */
    double* qc = (double*)calloc(m * l, sizeof(double));
    for (int64_t j = 0; j < l; ++j) qc[j * m + j] = 1.0;
    for (int64_t k = l - 1; k >= 0; --k) {
        const double* v = w + k * m;
        for (int64_t j = 0; j < l; ++j) {
            double* cj = qc + j * m;
            double dot = cj[k];
            for (int64_t i = k + 1; i < m; ++i) dot += v[i] * cj[i];
            dot *= tau[k];
            cj[k] -= dot;
            for (int64_t i = k + 1; i < m; ++i) cj[i] -= dot * v[i];
        }
    }
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < l; ++j) q[i * l + j] = qc[j * m + i];
    free(qc);
    free(w);
    free(tau);
    const double scale = or_spectral_norm_estimate(m, l, a);
    const double tol = 1e-13 * (double)(m > l ? m : l);
    if (bad_col) *bad_col = 0;
    for (int64_t j = 0; j < l; ++j) {
        const double d = r[j * l + j];
        const double mag = sqrt(d * d);
        if (mag <= tol * scale) {
            if (bad_col) *bad_col = j + 1;
            return OR_RANK_DEFICIENCY;
        }
        const double phase = d * (1.0 / mag);
        for (int64_t i = 0; i < m; ++i) q[i * l + j] *= phase;
        for (int64_t k = j; k < l; ++k) r[j * l + k] *= phase;
        r[j * l + j] = mag;
    }
    return OR_OK;
}

/* ------------------------------------------------------ singular values --- */
/* One-sided Jacobi on the columns of A (or of A^T when m < n), cyclic pair
 * order, until no pair has |a_p . a_q| > 1e-15 sqrt(|a_p|^2 |a_q|^2); the
 * singular values are the column norms, sorted non-increasing. */
static int cmp_desc(const void* x, const void* y) {
    const double a = *(const double*)x, b = *(const double*)y;
    return a < b ? 1 : (a > b ? -1 : 0);
}

void or_singular_values(int64_t m, int64_t n, const double* a, double* out) {
    const int tr = m < n;
    const int64_t rows = tr ? n : m, cols = tr ? m : n;
    double* w = (double*)malloc(sizeof(double) * rows * cols); /* column p at w + p * rows */
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            if (tr) w[i * rows + j] = a[i * n + j];
            else w[j * rows + i] = a[i * n + j];
        }
    for (int sweep = 0; sweep < 60; ++sweep) {
        int rotated = 0;
        for (int64_t p = 0; p + 1 < cols; ++p)
            for (int64_t q = p + 1; q < cols; ++q) {
                double* wp = w + p * rows;
                double* wq = w + q * rows;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int64_t i = 0; i < rows; ++i) {
                    al += wp[i] * wp[i];
                    be += wq[i] * wq[i];
                    ga += wp[i] * wq[i];
                }
                if (ga == 0.0 || fabs(ga) <= 1e-15 * sqrt(al * be)) continue;
                rotated = 1;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
                for (int64_t i = 0; i < rows; ++i) {
                    const double xp = wp[i], xq = wq[i];
                    wp[i] = c * xp - s * xq;
                    wq[i] = s * xp + c * xq;
                }
            }
        if (!rotated) break;
    }
    for (int64_t p = 0; p < cols; ++p) {
        double s2 = 0.0;
        for (int64_t i = 0; i < rows; ++i) s2 += w[p * rows + i] * w[p * rows + i];
        out[p] = sqrt(s2);
    }
    qsort(out, (size_t)cols, sizeof(double), cmp_desc);
    free(w);
}
