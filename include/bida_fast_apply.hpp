// bida_fast_apply.hpp — RubiksCube::apply (rubiks.hpp:81-95) as byte shuffles,
// for the CB-DFS overlay's per-child move (include/bida_fast_cbdfs.hpp).
//
// The reference applies a twist element by element: the cubie at position
// cf[i] moves to position i and gains twist co[i] (mod 3), edges likewise
// (ef, eo mod 2), over the 40-byte State {cp[8], co[8], ep[12], eo[12]}.  Here
// cp|co is one 16-byte vector gathered by one PSHUFB, ep|eo two overlapping
// 16-byte vectors gathered by four; the twists are a byte add and a modulo by
// conditional subtract.  Exactly the reference's result for every state whose
// orientation bytes are in range (co <= 2, eo <= 1: every state the search
// generates from a valid start); any other state takes RubiksCube::apply.
// The move tables are the reference's quarter turns (rubiks.hpp:340-364)
// composed as it composes them.  tests/cpp/apply_check.cpp compares against
// RubiksCube::apply on random states for all 18 moves.
#pragma once

#include <array>
#include <cstdint>
#include <cstring>

#include "bida/rubiks.hpp"

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace bida_fast {

struct RcShuffles {
    alignas(16) std::uint8_t corner[18][16];      // gather cp|co
    alignas(16) std::uint8_t corner_add[18][16];  // + co twist (co half)
    alignas(16) std::uint8_t e0_from0[18][16];    // bytes 16..31: ep0..11 from E0
    alignas(16) std::uint8_t e0_from1[18][16];    //               eo0..3  from E1
    alignas(16) std::uint8_t e0_add[18][16];
    alignas(16) std::uint8_t e1_from0[18][16];    // bytes 24..39: ep8..11 from E0
    alignas(16) std::uint8_t e1_from1[18][16];    //               eo0..11 from E1
    alignas(16) std::uint8_t e1_add[18][16];
};

inline const RcShuffles &rc_shuffles() {
    static const RcShuffles t = [] {
        struct Q {
            std::uint8_t cf[8], co[8], ef[12], eo[12];
        };
        const Q q[6] = {
            {{3, 0, 1, 2, 4, 5, 6, 7}, {0, 0, 0, 0, 0, 0, 0, 0}, {3, 0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11}, {0}},
            {{0, 1, 2, 3, 5, 6, 7, 4}, {0, 0, 0, 0, 0, 0, 0, 0}, {0, 1, 2, 3, 5, 6, 7, 4, 8, 9, 10, 11}, {0}},
            {{0, 2, 6, 3, 4, 1, 5, 7}, {0, 1, 2, 0, 0, 2, 1, 0}, {0, 1, 10, 3, 4, 5, 9, 7, 8, 2, 6, 11}, {0}},
            {{4, 1, 2, 0, 7, 5, 6, 3}, {2, 0, 0, 1, 1, 0, 0, 2}, {8, 1, 2, 3, 11, 5, 6, 7, 4, 9, 10, 0}, {0}},
            {{1, 5, 2, 3, 0, 4, 6, 7}, {1, 2, 0, 0, 2, 1, 0, 0}, {0, 9, 2, 3, 4, 8, 6, 7, 1, 5, 10, 11},
             {0, 1, 0, 0, 0, 1, 0, 0, 1, 1, 0, 0}},
            {{0, 1, 3, 7, 4, 5, 2, 6}, {0, 0, 1, 2, 0, 0, 2, 1}, {0, 1, 2, 11, 4, 5, 6, 10, 8, 9, 3, 7},
             {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 1, 1}},
        };
        auto compose = [](const Q &a, const Q &b) {  // a then b (rubiks.hpp:324-338)
            Q r{};
            for (int i = 0; i < 8; ++i) {
                r.cf[i] = a.cf[b.cf[i]];
                r.co[i] = static_cast<std::uint8_t>((a.co[b.cf[i]] + b.co[i]) % 3);
            }
            for (int i = 0; i < 12; ++i) {
                r.ef[i] = a.ef[b.ef[i]];
                r.eo[i] = static_cast<std::uint8_t>((a.eo[b.ef[i]] + b.eo[i]) % 2);
            }
            return r;
        };
        RcShuffles t{};
        for (int f = 0; f < 6; ++f) {
            Q m[3];
            m[0] = q[f];
            m[1] = compose(q[f], q[f]);
            m[2] = compose(m[1], q[f]);
            for (int k = 0; k < 3; ++k) {
                const int a = f * 3 + k;
                const Q &x = m[k];
                for (int i = 0; i < 8; ++i) {
                    t.corner[a][i] = x.cf[i];
                    t.corner[a][8 + i] = static_cast<std::uint8_t>(8 + x.cf[i]);
                    t.corner_add[a][8 + i] = x.co[i];
                }
                // E0 = state bytes 16..31 = ep0..11, eo0..3;  E1 = bytes 24..39 = ep8..11, eo0..11
                for (int i = 0; i < 16; ++i)
                    t.e0_from0[a][i] = t.e0_from1[a][i] = t.e1_from0[a][i] = t.e1_from1[a][i] = 0x80;
                for (int i = 0; i < 12; ++i)
                    t.e0_from0[a][i] = x.ef[i];                                   // new ep[i] = ep[ef[i]]
                for (int i = 0; i < 4; ++i) {
                    t.e0_from1[a][12 + i] = static_cast<std::uint8_t>(4 + x.ef[i]);  // new eo[i] = eo[ef[i]]
                    t.e0_add[a][12 + i] = x.eo[i];
                }
                for (int i = 0; i < 4; ++i)
                    t.e1_from0[a][i] = x.ef[8 + i];
                for (int i = 0; i < 12; ++i) {
                    t.e1_from1[a][4 + i] = static_cast<std::uint8_t>(4 + x.ef[i]);
                    t.e1_add[a][4 + i] = x.eo[i];
                }
            }
        }
        return t;
    }();
    return t;
}

inline bool has_ssse3() {
#if defined(__x86_64__)
    static const bool yes = __builtin_cpu_supports("ssse3") && __builtin_cpu_supports("sse4.1");
    return yes;
#else
    return false;
#endif
}

#if defined(__x86_64__)
// true when done (orientation bytes in range), false to fall back
__attribute__((target("ssse3,sse4.1"))) inline bool rc_apply_simd(const bida::RubiksCube::State &s,
                                                                   std::uint8_t a,
                                                                   bida::RubiksCube::State &out) {
    static_assert(sizeof(bida::RubiksCube::State) == 40, "State layout cp[8] co[8] ep[12] eo[12]");
    const RcShuffles &t = rc_shuffles();
    const auto *p = reinterpret_cast<const std::uint8_t *>(&s);
    const __m128i V = _mm_loadu_si128(reinterpret_cast<const __m128i *>(p));
    const __m128i E0 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(p + 16));
    const __m128i E1 = _mm_loadu_si128(reinterpret_cast<const __m128i *>(p + 24));
    // range check (unsigned): co bytes (V 8..15) <= 2, eo bytes (E1 4..15) <= 1;
    // lanes holding cp / ep bytes compare against 0xFF and always pass
    const __m128i co_lim = _mm_set_epi8(2, 2, 2, 2, 2, 2, 2, 2, -1, -1, -1, -1, -1, -1, -1, -1);
    const __m128i eo_lim = _mm_set_epi8(1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, -1, -1, -1, -1);
    const __m128i ok = _mm_and_si128(_mm_cmpeq_epi8(_mm_max_epu8(V, co_lim), co_lim),
                                     _mm_cmpeq_epi8(_mm_max_epu8(E1, eo_lim), eo_lim));
    if (_mm_movemask_epi8(ok) != 0xFFFF)
        return false;
    const __m128i three = _mm_set_epi8(3, 3, 3, 3, 3, 3, 3, 3, 0, 0, 0, 0, 0, 0, 0, 0);
    __m128i c = _mm_shuffle_epi8(V, _mm_load_si128(reinterpret_cast<const __m128i *>(t.corner[a])));
    c = _mm_add_epi8(c, _mm_load_si128(reinterpret_cast<const __m128i *>(t.corner_add[a])));
    c = _mm_min_epu8(c, _mm_sub_epi8(c, three));  // co half: (co + twist) mod 3 for co + twist <= 4
    const __m128i one_hi = _mm_set_epi8(1, 1, 1, 1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1);
    __m128i o0 = _mm_or_si128(_mm_shuffle_epi8(E0, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e0_from0[a]))),
                              _mm_shuffle_epi8(E1, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e0_from1[a]))));
    o0 = _mm_and_si128(_mm_add_epi8(o0, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e0_add[a]))), one_hi);
    const __m128i one_lo = _mm_set_epi8(1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, -1, -1, -1, -1);
    __m128i o1 = _mm_or_si128(_mm_shuffle_epi8(E0, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e1_from0[a]))),
                              _mm_shuffle_epi8(E1, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e1_from1[a]))));
    o1 = _mm_and_si128(_mm_add_epi8(o1, _mm_load_si128(reinterpret_cast<const __m128i *>(t.e1_add[a]))), one_lo);
    auto *q = reinterpret_cast<std::uint8_t *>(&out);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(q), c);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(q + 16), o0);
    _mm_storeu_si128(reinterpret_cast<__m128i *>(q + 24), o1);
    return true;
}
#endif

// D::apply, with the shuffle path for the cube.
template <class D>
inline typename D::State apply(const typename D::State &s, typename D::Action a) {
#if defined(__x86_64__)
    if constexpr (std::is_same_v<D, bida::RubiksCube>) {
        if (a < 18 && has_ssse3()) {
            typename D::State out;
            if (rc_apply_simd(s, a, out))
                return out;
        }
    }
#endif
    return D::apply(s, a);
}

}  // namespace bida_fast
