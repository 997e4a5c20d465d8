// The overlay's shuffle-based cube move (include/bida_fast_apply.hpp) against
// the reference's RubiksCube::apply (rubiks.hpp:81-95) for all 18 moves on
// random valid states, random byte soup (fallback path) and random walks.
// Exit 0 = identical everywhere.
#include <cstdio>
#include <cstring>
#include <random>

#include "bida/rubiks.hpp"
#include "bida_fast_apply.hpp"

using bida::RubiksCube;

int main() {
    std::mt19937_64 rng(9);
    long bad = 0, n = 0, fast = 0;
    RubiksCube::State w = RubiksCube::solved();
    for (int t = 0; t < 400000; ++t) {
        RubiksCube::State s;
        const int kind = t % 3;
        if (kind == 0) {  // walk state (valid)
            w = RubiksCube::apply(w, static_cast<std::uint8_t>(rng() % 18));
            s = w;
        } else if (kind == 1) {  // in-range bytes, not necessarily a valid cube
            for (auto &v : s.cp) v = static_cast<std::uint8_t>(rng() % 8);
            for (auto &v : s.co) v = static_cast<std::uint8_t>(rng() % 3);
            for (auto &v : s.ep) v = static_cast<std::uint8_t>(rng() % 12);
            for (auto &v : s.eo) v = static_cast<std::uint8_t>(rng() % 2);
        } else {  // byte soup: orientation out of range -> reference path
            for (auto &v : s.cp) v = static_cast<std::uint8_t>(rng());
            for (auto &v : s.co) v = static_cast<std::uint8_t>(rng());
            for (auto &v : s.ep) v = static_cast<std::uint8_t>(rng());
            for (auto &v : s.eo) v = static_cast<std::uint8_t>(rng());
        }
        for (std::uint8_t a = 0; a < 18; ++a) {
            const RubiksCube::State r = RubiksCube::apply(s, a);
            const RubiksCube::State f = bida_fast::apply<RubiksCube>(s, a);
            bad += std::memcmp(&r, &f, sizeof(r)) != 0;
            ++n;
#if defined(__x86_64__)
            RubiksCube::State tmp;
            fast += bida_fast::has_ssse3() && bida_fast::rc_apply_simd(s, a, tmp);
#endif
        }
    }
    std::printf("apply_check: %ld of %ld moves differ from RubiksCube::apply (%ld via shuffles)\n", bad, n, fast);
    return bad ? 1 : 0;
}
