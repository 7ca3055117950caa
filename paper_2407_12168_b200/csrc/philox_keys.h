// Host-computable Philox round keys shared by the C-ABI (which fills them)
// and the kernels (which read them from the kernel parameters).
#pragma once
#include <cstdint>

namespace tb200 {

// The 10 round keys of a stream key, (k0 + r W0, k1 + r W1): computed once on
// the host and passed in the kernel parameters, so each round's key XOR reads
// a constant-bank operand instead of re-deriving the key schedule.
struct PhiloxKeys {
    uint32_t k[20];
};

inline PhiloxKeys philox_round_keys(uint32_t k0, uint32_t k1) {
    PhiloxKeys rk;
    for (int r = 0; r < 10; ++r) {
        rk.k[2 * r] = k0;
        rk.k[2 * r + 1] = k1;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return rk;
}

}  // namespace tb200
