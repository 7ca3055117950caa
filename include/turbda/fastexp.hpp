// exp(x) for x <= 0 as the reference's weight kernel evaluates it
// (proj/include/turbda/fastexp.hpp:13-50): Cody-Waite split by ln 2, a
// degree-13 Taylor polynomial, exponent injection; x < -708 gives 0.  The
// fp64 faithful device kernel uses the same scheme (ensf_kernels.cu).
#pragma once

#include <cstdint>
#include <cstring>

namespace turbda {

inline double fast_exp_nonpos(double x) {
    const bool underflow = x < -708.0;
    if (underflow) x = 0.0;
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52: rounds to integer
    const double t = x * 1.4426950408889634074 + shifter;
    const double n_real = t - shifter;
    std::uint64_t t_bits;
    std::memcpy(&t_bits, &t, sizeof t_bits);
    const auto n = static_cast<std::int32_t>(t_bits & 0xffffffffu);
    double r = x - n_real * 6.93147180369123816490e-01;
    r -= n_real * 1.90821492927058770002e-10;
    static constexpr double c[13] = {1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0,
                                     1.0 / 362880.0,    1.0 / 40320.0,    1.0 / 5040.0,
                                     1.0 / 720.0,       1.0 / 120.0,      1.0 / 24.0,
                                     1.0 / 6.0,         0.5,              1.0,
                                     1.0};
    double p = c[0];
    for (int q = 1; q < 13; ++q) p = p * r + c[q];
    std::uint64_t p_bits;
    std::memcpy(&p_bits, &p, sizeof p_bits);
    p_bits += static_cast<std::uint64_t>(static_cast<std::int64_t>(n)) << 52;
    std::memcpy(&p, &p_bits, sizeof p);
    return underflow ? 0.0 : p;
}

}  // namespace turbda
