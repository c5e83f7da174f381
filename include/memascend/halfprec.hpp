// fp32 <-> bf16 / fp16 conversions — drop-in for
// proj/include/memascend/halfprec.hpp:13-99.
//
// Host-side twins of the device casts in csrc/ma_device.cuh.  Both sides
// round to nearest even and agree with the reference bit-for-bit on all 2^32
// inputs (tests/test_gpu_parity.py::test_cast_exhaustive_vs_reference,
// tests/test_oracle_golden.py::test_half_narrowing_exhaustive).
#pragma once

#include <cstdint>
#include <cstring>

namespace memascend {

inline std::uint32_t float_bits(float f) {
    std::uint32_t u;
    std::memcpy(&u, &f, sizeof u);
    return u;
}

inline float bits_float(std::uint32_t u) {
    float f;
    std::memcpy(&f, &u, sizeof f);
    return f;
}

namespace detail {
// (x >> sh) rounded to nearest, ties to even
constexpr std::uint32_t shift_rne(std::uint32_t x, unsigned sh) {
    const std::uint32_t kept = x >> sh;
    const std::uint32_t dropped = x & ((1u << sh) - 1u);
    const std::uint32_t half = 1u << (sh - 1u);
    return kept + ((dropped > half || (dropped == half && (kept & 1u))) ? 1u : 0u);
}
}  // namespace detail

/// RNE to bf16; NaN keeps its payload's top bits and is quieted (| 0x0040).
inline std::uint16_t bf16_from_float(float f) {
    const std::uint32_t u = float_bits(f);
    const std::uint32_t mag = u & 0x7FFFFFFFu;
    if (mag > 0x7F800000u) return static_cast<std::uint16_t>((u >> 16) | 0x0040u);
    return static_cast<std::uint16_t>(detail::shift_rne(mag, 16) | ((u >> 16) & 0x8000u));
}

inline float bf16_to_float(std::uint16_t h) { return bits_float(std::uint32_t{h} << 16); }

/// RNE to IEEE half with subnormals; |f| >= 65520 -> inf; NaN -> sign|0x7E00.
inline std::uint16_t fp16_from_float(float f) {
    const std::uint32_t u = float_bits(f);
    const auto sign = static_cast<std::uint16_t>((u >> 16) & 0x8000u);
    const std::uint32_t mag = u & 0x7FFFFFFFu;
    if (mag > 0x7F800000u) return static_cast<std::uint16_t>(sign | 0x7E00u);
    if (mag >= 0x477FF000u) return static_cast<std::uint16_t>(sign | 0x7C00u);
    if (mag >= 0x38800000u) {  // normal half: exponent rebias 127 -> 15
        return static_cast<std::uint16_t>(sign | detail::shift_rne(mag - (112u << 23), 13));
    }
    if (mag < 0x33000000u) return sign;
    const std::uint32_t significand = (mag & 0x007FFFFFu) | 0x00800000u;
    return static_cast<std::uint16_t>(sign | detail::shift_rne(significand, 126u - (mag >> 23)));
}

inline float fp16_to_float(std::uint16_t h) {
    const std::uint32_t sign = std::uint32_t{h & 0x8000u} << 16;
    const std::uint32_t e = (h >> 10) & 0x1Fu;
    const std::uint32_t frac = h & 0x3FFu;
    if (e == 0x1Fu) return bits_float(sign | 0x7F800000u | (frac << 13));
    if (e != 0) return bits_float(sign | ((e + 112u) << 23) | (frac << 13));
    if (frac == 0) return bits_float(sign);
    const float mag = static_cast<float>(frac) * 0x1p-24f;  // exact
    return bits_float(sign | float_bits(mag));
}

}  // namespace memascend
