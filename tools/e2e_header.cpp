// End-to-end timing of the C++ drop-in exactly as a reference user calls it:
// preprocess_solve(A, b, none, {Gaussian, seed 2}, 0) on RealMatrix /
// std::vector (pageable host memory) through include/randla_b200/randla.hpp
// (preprocess.hpp:156-180 signature). Every step uploads A and b, draws G on
// the device, factors, solves and brings x back. Prints one JSON line.
// Usage: e2e_header [n] [steps] [warmup]
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "randla_b200/randla.hpp"

int main(int argc, char** argv) {
    using namespace randla;
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 8192;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 10;
    const int warmup = argc > 3 ? std::atoi(argv[3]) : 2;
    const RealMatrix a = gen_gaussian(n, n, 1);
    const std::vector<double> b = gen_gaussian_vector(n, 3);
    MultiplierSpec post{MultiplierKind::Gaussian};
    post.seed = 2;
    SolveOutcome<double> out;
    for (int i = 0; i < warmup; ++i) out = preprocess_solve(a, b, MultiplierSpec{}, post, 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < steps; ++i) out = preprocess_solve(a, b, MultiplierSpec{}, post, 0);
    const auto t1 = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / steps;
    std::printf("{\"n\": %zu, \"steps\": %d, \"warmup\": %d, \"ms_per_step\": %.4f, \"residual\": %.6e, \"x0\": %.17g}\n",
                n, steps, warmup, ms, out.residual_history[0], out.x[0]);
    return 0;
}
