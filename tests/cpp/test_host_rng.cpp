// Host-only checks of the drop-in header (no GPU needed): the header's
// RngStream (rng.hpp:16-85 restated) against the library's exact generators
// (rl_gen_gaussian, rl_gen_real_circulant_column, rl_gen_finite_set_uniform,
// rl_derive_seed), i.e. against the same reference streams the device
// multipliers are pinned to. Exit code 0 = all passed.
#include <cstdio>

#include "randla_b200/randla.hpp"

using namespace randla;

static int failures = 0;
#define CHECK(c)                                                     \
    do {                                                             \
        if (!(c)) {                                                  \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            ++failures;                                              \
        }                                                            \
    } while (0)

int main() {
    for (std::uint64_t seed : {0ull, 1ull, 2ull, 12345ull, 0xFFFFFFFFFFFFFFFFull}) {
        const RealMatrix g = gen_gaussian(33, 17, seed);
        RngStream rng(seed);
        bool same = true;
        for (std::size_t i = 0; i < 33; ++i)
            for (std::size_t j = 0; j < 17; ++j) same = same && rng.next_gaussian() == g(i, j);
        CHECK(same);
        std::vector<double> col(64);
        rl_gen_real_circulant_column(64, seed, col.data());
        RngStream r2(seed);
        bool same_col = true;
        for (double v : col) same_col = same_col && r2.next_symmetric() == v;
        CHECK(same_col);
        for (std::size_t card : {2ull, 3ull, 1000ull, 65536ull, (1ull << 63) + 5ull}) {
            const RealMatrix f = gen_finite_set_uniform(9, 11, seed, card);
            RngStream r3(seed);
            const auto off = static_cast<std::int64_t>(card / 2);
            bool same_f = true;
            for (std::size_t i = 0; i < 9; ++i)
                for (std::size_t j = 0; j < 11; ++j)
                    same_f = same_f && f(i, j) == static_cast<double>(static_cast<std::int64_t>(r3.next_below(card)) - off);
            CHECK(same_f);
        }
        CHECK(derive_seed(seed, 3, 9) == RngStream(seed).derived(3, 9).next_u64());
    }
    std::printf(failures ? "%d failed\n" : "all passed\n", failures);
    return failures ? 1 : 0;
}
