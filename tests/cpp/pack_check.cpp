// The agent's fast state packing (include/bida_gpu_backend.hpp DomainOf<D>::pack,
// PEXT when BMI2 is present) against the reference's own D::pack
// (rubiks.hpp:126-137, stp.hpp:121-126) on random in-range and out-of-range
// states.  Exit 0 = identical everywhere.
#include <cstdio>
#include <cstring>
#include <random>

#include "bida/rubiks.hpp"
#include "bida/stp.hpp"
#include "bida_gpu_backend.hpp"

int main() {
    std::mt19937_64 rng(5);
    long bad = 0, n = 0;
    for (int t = 0; t < 2000000; ++t) {
        bida::RubiksCube::State s;
        const bool wild = t % 7 == 0;  // bytes outside the field ranges
        for (auto &v : s.cp) v = static_cast<std::uint8_t>(wild ? rng() & 0xFF : rng() % 8);
        for (auto &v : s.co) v = static_cast<std::uint8_t>(wild ? rng() & 0xFF : rng() % 3);
        for (auto &v : s.ep) v = static_cast<std::uint8_t>(wild ? rng() & 0xFF : rng() % 12);
        for (auto &v : s.eo) v = static_cast<std::uint8_t>(wild ? rng() & 0xFF : rng() % 2);
        unsigned char a[16];
        bida_gpu::DomainOf<bida::RubiksCube>::pack(s, a);
        const auto r = bida::RubiksCube::pack(s);
        bad += std::memcmp(a, &r.lo, 8) != 0 || std::memcmp(a + 8, &r.hi, 8) != 0;
        ++n;
        bida::TilePuzzle<4>::State q;
        for (auto &v : q.tiles) v = static_cast<std::uint8_t>(wild ? rng() & 0xFF : rng() % 16);
        unsigned char b[8];
        bida_gpu::DomainOf<bida::TilePuzzle<4>>::pack(q, b);
        const std::uint64_t w = bida::TilePuzzle<4>::pack(q);
        bad += std::memcmp(b, &w, 8) != 0;
        ++n;
    }
    std::printf("pack_check: %ld of %ld packed states differ from D::pack (bmi2 %s)\n", bad, n,
                bida_gpu::pack_detail::has_bmi2() ? "on" : "off");
    return bad ? 1 : 0;
}
