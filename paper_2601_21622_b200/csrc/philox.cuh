// philox.cuh -- device Philox4x32-10 (Salmon et al., SC'11), the counter-based generator the
// verify step draws its uniforms from (reading C-8 in DESIGN.md).  Written independently of
// the oracle's C copy; both are pinned by the Random123 known-answer vectors.
#pragma once
#include <cstdint>

namespace sd {

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            key.x += 0x9E3779B9u;
            key.y += 0xBB67AE85u;
        }
        const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
        ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    }
    return ctr;
}

// counter (position, round lo, rid lo, rid hi), key = seed
__device__ __forceinline__ uint4 verify_words(uint64_t seed, uint32_t pos, uint64_t round,
                                              uint64_t rid) {
    return philox4x32_10(
        make_uint4(pos, static_cast<uint32_t>(round), static_cast<uint32_t>(rid),
                   static_cast<uint32_t>(rid >> 32)),
        make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)));
}

// 24-bit uniform on the grid k * 2^-24, exact in fp64
__device__ __forceinline__ double unit24(uint32_t w) {
    return static_cast<double>(w >> 8) * 5.9604644775390625e-08;
}

}  // namespace sd
