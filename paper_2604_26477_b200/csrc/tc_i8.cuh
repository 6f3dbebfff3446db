// tcgen05 (5th-generation tensor core) building blocks for the int8 J·sgn(X) contraction:
// shared-memory matrix descriptors, the kind::i8 instruction descriptor, TMEM allocation,
// MMA issue / commit, mbarrier waits and TMEM -> register loads. Inline PTX for sm_100a.
//
// Operand layout in shared memory (K-major, no swizzle, "interleaved" canonical form): a
// chunk of R rows x 128 int8 along K is stored as core matrices of 8 rows x 16 bytes
// (128 contiguous bytes, row r at +16 r); the 8 core matrices of one 8-row group along K
// are adjacent (leading byte offset 128), and 8-row groups follow each other every 1024
// bytes (stride byte offset). One MMA consumes K = 32 (two core matrices along K); the
// k-th MMA of a chunk starts 256 k bytes further.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace momc_b200 {
namespace tc {

constexpr int kChunkK = 128;            // int8 elements of K per staged chunk
constexpr int kGroupBytes = 1024;       // one 8-row group x 128 K bytes
constexpr uint32_t kLBO = 128;          // bytes between adjacent K core matrices
constexpr uint32_t kSBO = kGroupBytes;  // bytes between adjacent 8-row groups

// byte offset of (row, k) inside a staged chunk
__host__ __device__ __forceinline__ uint32_t chunk_offset(int row, int k)
{
    return static_cast<uint32_t>((row >> 3) * kGroupBytes + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// SM100 shared-memory matrix descriptor (no swizzle, version 1)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr)
{
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((kLBO >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((kSBO >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version (Blackwell)
    // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
    return d;
}

// kind::i8 instruction descriptor: signed int8 A and B, int32 accumulator, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N)
{
    return (2u << 4)                             // c_format = S32
           | (1u << 7)                           // a_format = signed int8
           | (1u << 10)                          // b_format = signed int8
           | (static_cast<uint32_t>(N >> 3) << 17)  // n_dim
           | (static_cast<uint32_t>(M >> 4) << 24); // m_dim
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}

__device__ __forceinline__ void commit(uint64_t* mbar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(mbar)));
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count));
}

// the waiting thread is suspended until the phase completes (or this many ns pass), so a
// waiter does not spin on the issue slots the compute warps need
constexpr uint32_t kSuspendHintNs = 1000000;
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(phase), "r"(kSuspendHintNs)
        : "memory");
}

__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// TMEM allocation by one full warp; the base address lands in *slot (shared memory)
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}

template <uint32_t kCols>
__device__ __forceinline__ void tmem_free(uint32_t base)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(kCols));
}

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (warp's quarter + i),
// columns [col, col + 32)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// ---- 128-byte-swizzled K-major operands loaded by TMA: a box of R rows x 128 bytes lands
// as R rows of 128 B with the 16-byte chunks XOR-swizzled by (row & 7); 8-row groups are
// 1024 B apart (stride byte offset), the leading byte offset is unused (1). The k-th MMA of
// a chunk (K = 32 bytes) starts 32 k bytes further: the hardware applies the swizzle to the
// full address, so the descriptor's start address simply advances. Tiles are 1024-aligned.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr)
{
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;                   // leading byte offset (unused)
    d |= static_cast<uint64_t>((1024 >> 4) & 0x3FFF) << 32;  // stride byte offset
    d |= 1ull << 46;                                       // version (Blackwell)
    d |= static_cast<uint64_t>(2) << 61;                   // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

// 2-D TMA tile load (coordinates: inner dimension first) completing on mbar
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* mbar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap)
{
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// 32 lanes x 8 columns of 32-bit (thread i of the warp: lane quarter + i)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// registers -> TMEM, 32 lanes x 32 columns of 32-bit (thread i of the warp writes lane
// quarter + i); completes before tcgen05.wait::st returns
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// kind::f16 instruction descriptor: bf16 A and B (both K-major), FP32 accumulator
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N)
{
    return (1u << 4)                                // c_format = F32
           | (1u << 7)                              // a_format = BF16
           | (1u << 10)                             // b_format = BF16
           | (static_cast<uint32_t>(N >> 3) << 17)  // n_dim
           | (static_cast<uint32_t>(M >> 4) << 24); // m_dim
}

// D[tmem] (+)= A[tmem] . B[smem]^T. A (M x K) sits in TMEM: row m in lane m, K packed along
// the columns (4 int8 or 2 bf16 per 32-bit column); the K step of one MMA is 32 bytes,
// i.e. 8 columns.
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}
// both operands in shared memory (kind::f16)
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

// mbarrier wait with a nanosleep back-off (for waiters that are not on the critical path:
// their polling would otherwise take issue slots from the compute warps of their SM
// sub-partition)
__device__ __forceinline__ bool mbar_test(uint64_t* mbar, uint32_t phase)
{
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(mbar)), "r"(phase)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* mbar, uint32_t phase, uint32_t max_ns = 2048)
{
    uint32_t ns = 64;
    while (!mbar_test(mbar, phase)) {
        __nanosleep(ns);
        ns = ns < max_ns ? 2 * ns : max_ns;
    }
}

// ---- CTA pairs (cta_group::2, __cluster_dims__(2, 1, 1)): rank 0 issues the MMAs of an
// M = 256 tile whose A rows and B columns are split between the two CTAs' shared memory
// (same offsets in both); each CTA's TMEM holds its 128 rows of the accumulator.
__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// the shared::cluster address of this CTA's shared variable at `addr` in CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// arrive on an mbarrier given by its shared::cluster address (this CTA's or the peer's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t caddr)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}
__device__ __forceinline__ void mma_f16_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            bool accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}
// completion of the pair's MMAs issued so far arrives on the mbarrier at this offset in every
// CTA of `mask`
__device__ __forceinline__ void commit_2sm(uint64_t* mbar, uint16_t mask)
{
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::
                     "r"(smem_u32(mbar)),
                 "h"(mask));
}
// 2-D TMA load into this CTA's shared memory, completing on the mbarrier at shared::cluster
// address `mbar_caddr` (rank 0's)
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const void* tmap, int c0, int c1, uint32_t mbar_caddr)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(mbar_caddr)
        : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* slot)
{
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_free_2sm(uint32_t base)
{
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(kCols));
}

}  // namespace tc
}  // namespace momc_b200
