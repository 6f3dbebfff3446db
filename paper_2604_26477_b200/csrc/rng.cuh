// Device-side counter RNG: bit-exact restatement of momc::rng (rng.hpp) for sm_100a.
//
//   philox4x32_10   rng.hpp:22-38   (Random123 Philox4x32-10; round keys are warp-uniform)
//   derive_key      rng.hpp:54-57   (SplitMix64 finaliser mix64, rng.hpp:42-50)
//   stream ids      rng.hpp:107-111 counter = {block#, id_lo, id_mid, id_hi}
//   u01 / symmetric rng.hpp:131-146 (u64 >> 11) * 2^-53, h * (2u - 1)
//   normal          rng.hpp:156-185 128-layer ziggurat; tables are computed on the host by
//                   the same libm calls as rng.hpp:62-89 and uploaded (bit-identical).
// No cuRAND: its Philox state layout differs from the reference's counter layout.
#pragma once
#include <cstdint>

namespace momc_b200 {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kWeyl0 = 0x9E3779B9u;
constexpr uint32_t kWeyl1 = 0xBB67AE85u;

constexpr uint32_t kTagInitX = 1, kTagInitY = 2, kTagStepNoise = 3, kTagEdgePresence = 4,
                   kTagEdgeWeight = 5, kTagCorrelationNoise = 6, kTagProbePool = 7, kTagReferenceSample = 8;

__host__ __device__ __forceinline__ uint32_t tag_word(uint32_t tag, uint32_t step)
{
    return (tag << 26) | (step & 0x03FFFFFFu);
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z)
{
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__host__ __device__ __forceinline__ uint64_t derive_key(uint64_t seed, uint64_t ctx)
{
    return mix64(seed + 0x9E3779B97F4A7C15ull) ^ mix64(ctx * 0x9E3779B97F4A7C15ull + 1);
}

// solver.hpp:98-104
__host__ __device__ __forceinline__ uint64_t run_key(uint64_t seed, uint32_t run)
{
    return derive_key(derive_key(seed, 0x736F6C76u), run);
}

// 32x32 -> 64 product as one IMAD.WIDE.U32 (the C++ 64-bit multiply also adds a zero high
// term, one extra instruction per product)
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi)
{
    asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"(a), "r"(b));
}

// One Philox4x32-10 block. ctr = {c0 (block#), c1 (id_lo), c2 (id_mid), c3 (id_hi)}.
__device__ __forceinline__ uint4 philox(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t c2,
                                        uint32_t c3)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0, hi0, lo1, hi1;
        mul_wide(kPhiloxM0, c0, lo0, hi0);
        mul_wide(kPhiloxM1, c2, lo1, hi1);
        const uint32_t n0 = hi1 ^ c1 ^ (k0 + kWeyl0 * r);
        const uint32_t n2 = hi0 ^ c3 ^ (k1 + kWeyl1 * r);
        c1 = lo1;
        c3 = lo0;
        c0 = n0;
        c2 = n2;
    }
    return make_uint4(c0, c1, c2, c3);
}

__device__ __forceinline__ double u01_from(uint32_t lo, uint32_t hi)
{
    const uint64_t v = (static_cast<uint64_t>(hi) << 32) | lo;
    return static_cast<double>(v >> 11) * 0x1.0p-53;
}
__device__ __forceinline__ double u01_open_from(uint32_t lo, uint32_t hi)
{
    const uint64_t v = (static_cast<uint64_t>(hi) << 32) | lo;
    return static_cast<double>((v >> 11) + 1) * 0x1.0p-53;
}

// Sequential reader of one reference Stream (rng.hpp:113-121), for the cold paths.
struct DevStream {
    uint32_t k0, k1, lo, mid, hi;
    uint32_t block;  // next block index to generate
    uint32_t buf[4];
    int pos;
    __device__ __forceinline__ void init(uint64_t key, uint32_t id_hi, uint32_t id_mid, uint32_t id_lo)
    {
        k0 = static_cast<uint32_t>(key);
        k1 = static_cast<uint32_t>(key >> 32);
        hi = id_hi;
        mid = id_mid;
        lo = id_lo;
        block = 0;
        pos = 4;
    }
    __device__ __forceinline__ uint32_t next_u32()
    {
        if (pos == 4) {
            const uint4 b = philox(k0, k1, block, lo, mid, hi);
            buf[0] = b.x;
            buf[1] = b.y;
            buf[2] = b.z;
            buf[3] = b.w;
            ++block;
            pos = 0;
        }
        return buf[pos++];
    }
    __device__ __forceinline__ uint64_t next_u64()
    {
        const uint64_t a = next_u32();
        const uint64_t b = next_u32();
        return a | (b << 32);
    }
};

// Ziggurat tables (rng.hpp:62-89), uploaded from the host.
struct ZigTables {
    uint32_t kn[128];
    double wn[128];
    double fn[128];
};

// rng.hpp:156-185 over a DevStream (sequential; this path is not throughput-critical)
__device__ inline double normal_seq(DevStream& s, const ZigTables* __restrict__ z)
{
    for (;;) {
        const uint32_t u = s.next_u32();
        const int32_t hz = static_cast<int32_t>(u);
        const uint32_t iz = u & 127u;
        const uint32_t mag = hz < 0 ? static_cast<uint32_t>(-static_cast<int64_t>(hz)) : static_cast<uint32_t>(hz);
        if (mag < z->kn[iz]) return __dmul_rn(static_cast<double>(hz), z->wn[iz]);
        if (iz == 0) {
            const double r = 3.442619855899;
            for (;;) {
                const uint64_t a = s.next_u64();
                const double x = __ddiv_rn(-log(static_cast<double>((a >> 11) + 1) * 0x1.0p-53), r);
                const uint64_t b = s.next_u64();
                const double y = -log(static_cast<double>((b >> 11) + 1) * 0x1.0p-53);
                if (__dadd_rn(y, y) >= __dmul_rn(x, x)) return hz > 0 ? __dadd_rn(r, x) : -__dadd_rn(r, x);
            }
        }
        const double x = __dmul_rn(static_cast<double>(hz), z->wn[iz]);
        const uint64_t a = s.next_u64();
        const double u01 = static_cast<double>(a >> 11) * 0x1.0p-53;
        if (__dadd_rn(z->fn[iz], __dmul_rn(u01, __dsub_rn(z->fn[iz - 1], z->fn[iz]))) <
            exp(__dmul_rn(__dmul_rn(-0.5, x), x)))
            return x;
    }
}

}  // namespace momc_b200
