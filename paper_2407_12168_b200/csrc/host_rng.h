// Host-side counter-based RNG shared by the C-ABI (minibatch tables, stream
// keys) and the C++ API's turbda::RngStream.  Same generator as the device
// (philox.cuh) and as the reference (proj/src/rng.cpp:8-84): Philox4x32-10
// keyed by splitmix64(seed ^ splitmix64(use)).
#pragma once
#include <array>
#include <cstdint>

namespace tb200 {

inline uint64_t splitmix64(uint64_t v) {
    v += 0x9E3779B97F4A7C15ull;
    v = (v ^ (v >> 30)) * 0xBF58476D1CE4E5B9ull;
    v = (v ^ (v >> 27)) * 0x94D049BB133111EBull;
    return v ^ (v >> 31);
}

inline std::array<uint32_t, 4> philox4x32_10(std::array<uint32_t, 4> c, std::array<uint32_t, 2> k) {
    for (int round = 0; round < 10; ++round) {
        const uint64_t m0 = uint64_t(0xD2511F53u) * c[0];
        const uint64_t m1 = uint64_t(0xCD9E8D57u) * c[2];
        c = {uint32_t(m1 >> 32) ^ c[1] ^ k[0], uint32_t(m1), uint32_t(m0 >> 32) ^ c[3] ^ k[1],
             uint32_t(m0)};
        k[0] += 0x9E3779B9u;
        k[1] += 0xBB67AE85u;
    }
    return c;
}

inline uint64_t stream_key(uint64_t seed, uint64_t use) { return splitmix64(seed ^ splitmix64(use)); }

// word-level view of a stream: word w lives in block w >> 2, lane w & 3
struct HostStream {
    uint32_t k0, k1, e0, e1;
    uint64_t block = 0;
    std::array<uint32_t, 4> buf{};
    int pos = 4;

    HostStream(uint64_t seed, uint64_t use, uint64_t entity) {
        const uint64_t k = stream_key(seed, use);
        k0 = uint32_t(k);
        k1 = uint32_t(k >> 32);
        e0 = uint32_t(entity);
        e1 = uint32_t(entity >> 32);
    }
    uint32_t next_u32() {
        if (pos >= 4) {
            buf = philox4x32_10({uint32_t(block), uint32_t(block >> 32), e0, e1}, {k0, k1});
            ++block;
            pos = 0;
        }
        return buf[pos++];
    }
    uint64_t next_u64() {
        const uint64_t lo = next_u32();
        const uint64_t hi = next_u32();
        return lo | (hi << 32);
    }
};

constexpr uint64_t kUseEnsfParticles = 6;  // StreamUse::ensf_particles
constexpr uint64_t kUseEnsfBatch = 7;      // StreamUse::ensf_batch

}  // namespace tb200
