// ssn_gemm_tc.cu -- exact mod-p share GEMM on the 5th-gen tensor cores (tcgen05, kind::i8).
//
// Replaces the object-dtype contraction of sss_linear (S/layers.py:252 conv, :254 dense).
// Field elements (< 2^(8L)) are split into L little-endian u8 limbs.  For a tile of
// 128 output rows (activation pixels) x 32 output columns (channels) the CTA keeps 2L-1
// int32 accumulators in TMEM, one per limb diagonal d = i + j:
//       D_d = sum_{i+j=d} A_i(128 x K) . B_j(32 x K)^T          (exact: <= L*K*255^2 < 2^32)
// fed by TMA (4-D tensor maps over [party][limb][row][K], 64-byte swizzle) through a
// 3-stage mbarrier pipeline; one elected thread issues, per 32-wide K slice, L tcgen05.mma
// of 128 x (L*32) x 32 -- A limb i against all B limbs stacked along N, written at TMEM
// column offset 32*i so each limb product lands on its diagonal.  The epilogue reads TMEM (tcgen05.ld), recombines sum_d D_d * (2^(8d) mod p) in
// 128-bit registers and reduces mod p (Barrett), writing canonical u64 shares straight into
// the [party][img][O][OH*OW] layout the protocol kernels consume.
//
// Operand preparation (also here): ssn_limb_split (row-major u64 -> K-major u8 limb planes:
// weights once per model, dense activations) and ssn_im2col_limbs (implicit conv unfold
// S/model.py:354-371 fused with the limb split, shared-memory transposed so both the gather
// and the plane writes are coalesced).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "ssn_field.cuh"
#include "ssn_lincomb.cuh"
#include "ssn.h"

namespace {

constexpr int BM = 128;        // UMMA_M: rows per tile
constexpr int BN = 32;         // UMMA_N: output channels per tile
constexpr int BK = 64;         // bytes of K per pipeline stage (= one 64B swizzle atom row)
constexpr int UK = 32;         // K per tcgen05.mma.kind::i8
constexpr int STAGES_MAX = 3;
template <int L> __host__ __device__ constexpr int stages_for() { return L >= 8 ? 2 : STAGES_MAX; }   // 227 KB smem cap
constexpr int MAXL = 8;

struct CdTable { u64 c[2 * MAXL - 1]; };

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// TMA loads multicast to the CTAs of ctaMask: the box lands at the same shared-memory offset in
// each of them and completes bytes on the mbarrier at the same offset in each.
__device__ __forceinline__ void tma_load_4d_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                               int c2, int c3, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1,
                                               int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;"
        ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor for an MN-major (M contiguous) operand, 128-byte swizzle:
// each K row holds 128 M-bytes, 8-row (1 KB) swizzle atoms stacked along K (SBO = 1 KB).
__device__ __forceinline__ uint64_t umma_desc_sw128_mn(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)0 << 16;                          // LBO: one atom along M (unused)
    d |= (uint64_t)(1024 >> 4) << 32;                // SBO: next 8 K rows
    d |= (uint64_t)1 << 46;                          // version (sm_100)
    d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
    return d;
}

// UMMA shared-memory descriptor: K-major, 64-byte swizzle, 8-row core groups 512 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)0 << 16;                          // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;                 // SBO
    d |= (uint64_t)1 << 46;                          // version (sm_100)
    d |= (uint64_t)4 << 61;                          // SWIZZLE_64B
    return d;
}

// instruction descriptor: D=S32, A=B=U8, K-major both, M=BM, N=n
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// arrive on the mbarrier at this offset in every CTA of ctaMask once the issued MMAs complete
__device__ __forceinline__ void mma_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
        ::"r"(smem_u32(bar)), "h"(mask) : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// (hi*2^64 + lo) mod p for p >= 2^40 (L >= 6): hi < 2^40 <= p, so hi*r64 is one mulmod.
// Not inlined: keeps the epilogue's SASS small enough to stay in the instruction cache.
__device__ __noinline__ u64 epi_reduce(u64 lo, u64 hi, SsnField f, u64 r64) {
    const u64 t = ssn_mulmod(hi, r64, f);
    return ssn_addmod(t, ssn_reduce_wide(0, lo, f), f.p);
}

template <int L>
__global__ void __launch_bounds__(128, 1)
k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, u64 *__restrict__ out,
          u64 out_pstride, u64 ohw, int O, int M, int nkb, SsnField f, u64 r64, CdTable cd) {
    constexpr int ND = 2 * L - 1;
    constexpr int STAGES = stages_for<L>();
    constexpr int A_BYTES = L * BM * BK;
    constexpr int B_BYTES = L * BN * BK;
    constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(base + STAGES * STAGE_BYTES);
    uint64_t *empty = full + STAGES;
    uint64_t *done = empty + STAGES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.y * BN, m0 = blockIdx.x * BM, party = blockIdx.z;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
            uint8_t *sa = base + s * STAGE_BYTES;
            tma_load_4d(sa, &tmA, &full[s], kb * BK, m0, 0, party);
            tma_load_4d(sa + A_BYTES, &tmB, &full[s], kb * BK, n0, 0, party);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer.  The L limb planes of B sit back to back in shared memory, so one
        // MMA with N = L*BN multiplies A limb i by ALL B limbs at once; writing its D at TMEM
        // column i*BN lands the product with B limb j on column block (i+j)*BN -- exactly the
        // limb diagonal d = i+j.  L MMAs of 128 x L*BN x 32 per K slice instead of L^2 of
        // 128 x BN x 32.  On the very first K slice diagonals >= L are not yet written, so
        // A limb i >= 1 splits into an accumulating N=(L-1)*BN part and a fresh N=BN part.
        constexpr uint32_t ID_ALL = idesc_i8(L * BN), ID_HEAD = idesc_i8((L - 1) * BN), ID_ONE = idesc_i8(BN);
        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            mbar_wait(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = smem_u32(base + s * STAGE_BYTES);
            const uint32_t sb = sa + A_BYTES;
#pragma unroll 1
            for (int kk = 0; kk < BK / UK; kk++) {
                const uint64_t bdesc = umma_desc_sw64(sb + kk * UK);
                const bool first = kb == 0 && kk == 0;
#pragma unroll 1
                for (int i = 0; i < L; i++) {
                    const uint64_t adesc = umma_desc_sw64(sa + i * BM * BK + kk * UK);
                    const uint32_t d = tmem + (uint32_t)(i * BN);
                    if (!first) {
                        mma_i8(d, adesc, bdesc, ID_ALL, 1u);
                    } else if (i == 0) {
                        mma_i8(d, adesc, bdesc, ID_ALL, 0u);
                    } else {
                        mma_i8(d, adesc, bdesc, ID_HEAD, 1u);
                        mma_i8(d + (uint32_t)((L - 1) * BN), adesc,
                               umma_desc_sw64(sb + (L - 1) * BN * BK + kk * UK), ID_ONE, 0u);
                    }
                }
            }
            mma_commit(&empty[s]);
        }
        mma_commit(done);
    }
    __syncwarp();

    // ---- epilogue: all 4 warps; warp w owns TMEM lanes 32w..32w+31 (tile rows) ----
    mbar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = m0 + warp * 32 + lane;
    const bool row_ok = row < M;
    const u64 img = row_ok ? (u64)row / ohw : 0;
    const u64 pix = row_ok ? (u64)row - img * ohw : 0;
    u64 *obase = out + (u64)party * out_pstride + img * (u64)O * ohw + pix;
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    // Kept as rolled loops: a fully unrolled epilogue is ~80 KB of SASS that each CTA runs
    // once, which made the kernel instruction-fetch bound (ncu: stalled_no_instruction).
    // sum_d D_d * w_d with w = wh*2^32 + wl:  S0 = sum D*wl (128-bit via carry count),
    // S1 = sum D*wh (< 2^61), total = S0 + S1*2^32.
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 8) {
        u64 s0[8], s1[8];
        uint32_t cy[8];
#pragma unroll
        for (int c = 0; c < 8; c++) {
            s0[c] = s1[c] = 0;
            cy[c] = 0;
        }
#pragma unroll 1
        for (int d = 0; d < ND; d++) {
            uint32_t r[8];
            tmem_ld8(lane_addr + (uint32_t)(d * BN + c0), r);
            const uint32_t wl = (uint32_t)cd.c[d], wh = (uint32_t)(cd.c[d] >> 32);
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const u64 t0 = (u64)r[c] * wl;
                s0[c] += t0;
                cy[c] += (s0[c] < t0);
                s1[c] += (u64)r[c] * wh;
            }
        }
        if (row_ok) {
#pragma unroll
            for (int c = 0; c < 8; c++) {
                const int col = n0 + c0 + c;
                const u64 lo = s0[c] + (s1[c] << 32);
                const u64 hi = (u64)cy[c] + (s1[c] >> 32) + (lo < s0[c]);
                if (col < O) obase[(u64)col * ohw] = epi_reduce(lo, hi, f, r64);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ============================================================================================
// Persistent, warp-specialised kernel for the default field p = 2^45 - 55 (L = 6 limbs).
//   warp 0      TMA producer (smem ring of A 128x64x6 + B BNx64x6 bytes per stage)
//   warp 1      TMEM allocator + MMA issuer: per 32-wide K slice, 6 MMAs of 128 x (6 BN) x 32
//   warps 2..   epilogue: TMEM -> registers -> mod-p recombination -> HBM
// The 11 limb-diagonal accumulators of a 128 x BN tile take 11 BN TMEM columns: one buffer at
// BN = 32, two (columns 0 and 256) at BN = 16 so the epilogue of tile t overlaps the MMAs of
// tile t+1.  Epilogue recombination is exact integer arithmetic specialised to p:
//   g0 = sum_{d<4} D_d 2^{8d},  g1 = sum_{4<=d<8} D_d 2^{8(d-4)},  g2 = sum_{d>=8} D_d 2^{8(d-8)}
//   (each one IMAD.WIDE per diagonal, all < 2^57), value = g0 + g1 2^32 + g2 2^64: g1 2^32 and
//   g2 2^64 are rewritten with 2^45 == 55 (mod p) into terms below 2^51, and the sum (< 2^57)
//   takes ONE fold.
namespace p45 {
constexpr int L = 6;
constexpr int ND = 2 * L - 1;            // 11 limb diagonals
constexpr int A_BYTES = L * BM * BK;     // 49152
constexpr u64 P = (1ull << 45) - 55;
constexpr u64 MASK45 = (1ull << 45) - 1;

__device__ __forceinline__ u64 lz(u64 x) { return (x >> 45) * 55 + (x & MASK45); }

// acc + a * b in ONE IMAD.WIDE.U32 (a shift-and-add compiles to four 32-bit ops)
__device__ __forceinline__ u64 mad_wide(uint32_t a, uint32_t b, u64 acc) {
    u64 r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(acc));
    return r;
}

// ---- wide variant: 128 x 32 tiles, N = 6 x 32 = 192 per MMA (A re-read from smem 6x less
// than with 16-wide tiles: ~107 B/clk of operand traffic per SM), one TMEM accumulator of
// 11 x 32 = 352 columns.  Eight epilogue warps (two per TMEM lane quarter, 16 columns each)
// drain TMEM into registers and release it BEFORE the mod-p recombination and the stores,
// so the next tile's MMAs overlap the arithmetic and the HBM writes.
namespace wide {
// Tile widths: BN = 32 (one 352-column TMEM accumulator, 3 smem stages: the MMA waits for the
// epilogue's drain) or BN = 16 (N = 96 per MMA, two 176-column accumulators 256 columns apart,
// 4 stages: the MMA of tile t+1 runs while the epilogue drains tile t -- what keeps the tensor
// pipe busy when co-scheduled chain warps take most of the issue slots).
template <int BN>
struct Cfg {
    static constexpr int NBUF = BN == 16 ? 2 : 1;
    static constexpr int ST = BN == 16 ? 4 : 3;
    static constexpr int B_BYTES = L * BN * BK;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int SMEM = ST * STAGE + 1024 + 256;
    static constexpr uint32_t TB = 256;                  // TMEM column offset of buffer 1
};
// Epilogue: 8 warps (two per TMEM lane quarter, 112 registers) or -- co-scheduled with the chain
// kernels (SSN_COSCHED, see ssn_chain.cu) -- 4 warps draining 8 columns per pass at <= 80
// registers, so one GEMM CTA (192 x 80 registers) always fits beside two chain blocks.
#ifndef SSN_COSCHED
#define SSN_COSCHED 0
#endif
#if SSN_COSCHED
constexpr int EPI_W = 4, EPI_COLS = 8;
#define SSN_GEMM_W_BOUNDS __maxnreg__(80)
#else
#ifndef SSN_GEMM_EPI_W
#define SSN_GEMM_EPI_W 8
#endif
#ifndef SSN_GEMM_MAXNREG
#define SSN_GEMM_MAXNREG 112
#endif
constexpr int EPI_W = SSN_GEMM_EPI_W, EPI_COLS = 16;
#define SSN_GEMM_W_BOUNDS __maxnreg__(SSN_GEMM_MAXNREG)
#endif
#ifndef SSN_GEMM_BN_DEFAULT
#define SSN_GEMM_BN_DEFAULT 32
#endif

// A operand modes: 0 = K-major limb planes [party][L][rows][Kpad] (explicit im2col / dense);
// 1 = channel-major planes [party*L][C][B*H*W] of a 1x1 stride-1 conv input (M-major, TMA 3-D);
// 2 = channel-major row-padded planes [3][party*L][C][B][H*Wp] (Wp >= W, Wp % 16 == 0) of a 3x3 stride-1
//     pad-1 conv input, copy dx holding the rows shifted by dx - 1 columns (zero where the shift
//     leaves the image): implicit GEMM, tap (dy, dx) reads copy dx at a flattened (y, x) offset
//     of (dy-1)*Wp; out-of-range rows are TMA zero fill -- the convolution's zero padding.
struct ConvGeom {
    int C, H, W, Wp, cblocks, ntf, nparty;   // ntf: 128-row tiles per image (mode 2)
};

// Reshare step 1 fused into the epilogue (SUB instantiation): instead of the product y of
// party `party`, write its nf RESHARE_OUT sub-shares  y + sum_e c_e * id_f^(e+1)  (front ranks
// f < nf, S/protocol.py:154-164) straight into the per-destination send buffers
//   sub[party * sub_pstride + f * sub_fstride + element],
// drawing c_e exactly as ssn_gen does (Philox4x32-10 of (seed, stream + party, element,
// 0x800 | pair), masked 45-bit words), so the fused and unfused paths are bit-identical.
struct EpiSub {
    u64 *sub;
    u64 sub_pstride, sub_fstride, seed, stream;
    int km1, nf;
    uint32_t pw[SSN_MAXK][SSN_MAXK];        // front id powers id_f^(e+1) (small, p45)
};

// tcgen05.ld of NC consecutive 32-bit TMEM columns of this warp's lane quarter (NC = 8 or 16)
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[NC]) {
    if constexpr (NC == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    }
}

// CL = 2: a cluster of two CTAs works on the two N tiles of one 128-row A tile in lockstep; each
// CTA loads three of the six A limb planes and multicasts them to both, halving the A operand's
// L2 -> SM traffic (A is 48 of the 60 KB a stage moves; at the tensor pipe's rate the unshared
// stream needs ~50 B/clk per SM, above the L2's share per SM).  The stage's `empty` barrier then
// waits for both CTAs' MMA warps (commit multicast to the pair).
template <int AMODE, int BN, bool SUB = false, int CL = 1, int EW = EPI_W>
__global__ void SSN_GEMM_W_BOUNDS
k_gemm_p45w(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, u64 *__restrict__ out,
            u64 out_pstride, uint32_t ohw, int O, int M, int nkb, int ntm, int ntn, int ntiles, ConvGeom geo,
            const __grid_constant__ EpiSub es) {
    using C = Cfg<BN>;
    constexpr int STW = C::ST, STAGE_W = C::STAGE, NBUF = C::NBUF;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(base + STW * STAGE_W);
    uint64_t *empty = full + STW;
    uint64_t *tfull = empty + STW;             // [NBUF]
    uint64_t *tempty = tfull + NBUF;           // [NBUF]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + NBUF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // 1-D grid, clusters of CL consecutive CTAs: the cluster rank is blockIdx.x % CL (read where it
    // is used: a rank held in a local also defeated the uniform datapath), and CTA b
    // takes tiles b, b + grid, ... -- the CL CTAs of a cluster hold the CL consecutive N tiles of
    // one A tile (ntn % CL == 0, grid % CL == 0).  The loops below start at blockIdx.x itself: a
    // copy in a local made ptxas treat the loop state as non-uniform (R2UR waterfalls around
    // every tcgen05.mma, 8% slower).
    if (threadIdx.x == 0) {
        for (int s = 0; s < STW; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CL);
        }
        for (int b = 0; b < NBUF; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if constexpr (CL > 1) cluster_sync_all();           // the peer's barriers exist before any multicast
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int nt = t % ntn, mt = (t / ntn) % ntm, party = t / (ntn * ntm);
                for (int kb = 0; kb < nkb; kb++, it++) {
                    const int s = it % STW;
                    mbar_wait(&empty[s], ((it / STW) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], STAGE_W);
                    uint8_t *sa = base + s * STAGE_W;
                    // CL = 2: this CTA's half of the limb planes, multicast to the pair
                    constexpr int LH = L / CL;
                    const int l0 = CL > 1 ? (int)(blockIdx.x % CL) * LH : 0;
                    uint8_t *sah = sa + l0 * BM * BK;
                    if (AMODE == 0) {
                        if constexpr (CL > 1) tma_load_4d_mc(sah, &tmA, &full[s], kb * BK, mt * BM, l0, party, 3);
                        else tma_load_4d(sa, &tmA, &full[s], kb * BK, mt * BM, 0, party);
                    } else if (AMODE == 1) {
                        if constexpr (CL > 1) tma_load_3d_mc(sah, &tmA, &full[s], mt * BM, kb * BK, party * L + l0, 3);
                        else tma_load_3d(sa, &tmA, &full[s], mt * BM, kb * BK, party * L);
                    } else {
                        const int tap = kb / geo.cblocks, cb = kb - tap * geo.cblocks;
                        const int dy = tap / 3, dx = tap - dy * 3;
                        const int img = mt / geo.ntf, ft = mt - img * geo.ntf;
                        // column shift dx - 1 comes from the dx-th pre-shifted copy (TMA inner
                        // coordinates must stay 16-byte aligned); the row shift is (dy - 1) * Wp
                        if constexpr (CL > 1)
                            tma_load_4d_mc(sah, &tmA, &full[s], ft * BM + (dy - 1) * geo.Wp, img, cb * BK,
                                           (dx * geo.nparty + party) * L + l0, 3);
                        else
                            tma_load_4d(sa, &tmA, &full[s], ft * BM + (dy - 1) * geo.Wp, img, cb * BK,
                                        (dx * geo.nparty + party) * L);
                    }
                    tma_load_4d(sa + A_BYTES, &tmB, &full[s], kb * BK, nt * BN, 0, party);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t AM = AMODE ? (1u << 15) : 0u;          // A major-ness: MN for conv planes
            constexpr uint32_t ID_ALL = idesc_i8(L * BN) | AM, ID_HEAD = idesc_i8((L - 1) * BN) | AM,
                               ID_ONE = idesc_i8(BN) | AM;
            int it = 0, lt = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
                const int buf = lt % NBUF;
                mbar_wait(&tempty[buf], ((lt / NBUF) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t dbase = tmem + (uint32_t)buf * C::TB;
                for (int kb = 0; kb < nkb; kb++, it++) {
                    const int s = it % STW;
                    mbar_wait(&full[s], (it / STW) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t sa = smem_u32(base + s * STAGE_W);
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < BK / UK; kk++) {
                        const uint64_t bdesc = umma_desc_sw64(sb + kk * UK);
                        const bool first = kb == 0 && kk == 0;
                        auto adesc_of = [&](int i) {
                            return AMODE ? umma_desc_sw128_mn(sa + i * BM * BK + kk * UK * BM)
                                         : umma_desc_sw64(sa + i * BM * BK + kk * UK);
                        };
                        if (!first) {
#pragma unroll
                            for (int i = 0; i < L; i++)
                                mma_i8(dbase + (uint32_t)(i * BN), adesc_of(i), bdesc, ID_ALL, 1u);
                        } else {
                            // first K slice: the accumulators start undefined.  Limb 0 initialises
                            // diagonals 0..L-1; limb L-1 then adds to diagonal L-1 (B limb 0, N = BN)
                            // and initialises L..2L-2 (B limbs 1.., N = (L-1) BN); limbs 1..L-2
                            // accumulate over fully initialised columns.  7 MMAs, one narrow.
                            mma_i8(dbase, adesc_of(0), bdesc, ID_ALL, 0u);
                            const uint64_t a5 = adesc_of(L - 1);
                            mma_i8(dbase + (uint32_t)((L - 1) * BN), a5, bdesc, ID_ONE, 1u);
                            mma_i8(dbase + (uint32_t)(L * BN), a5, umma_desc_sw64(sb + BN * BK + kk * UK), ID_HEAD, 0u);
#pragma unroll
                            for (int i = 1; i < L - 1; i++)
                                mma_i8(dbase + (uint32_t)(i * BN), adesc_of(i), bdesc, ID_ALL, 1u);
                        }
                    }
                    if constexpr (CL > 1) mma_commit_mc(&empty[s], 3);
                    else mma_commit(&empty[s]);
                }
                mma_commit(&tfull[buf]);
            }
        }
    } else {
        // epilogue warps: TMEM lane quarter = warp % 4; with 8 warps the two of a quarter take one
        // 16-column half each, with 4 warps one warp drains all 32 columns, EPI_COLS per pass
        const int q = warp & 3;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        constexpr int CPW = BN / (EW / 4);                  // columns per epilogue warp
        constexpr int ECOLS = EPI_COLS < CPW ? EPI_COLS : CPW;
        constexpr int NPASS = CPW / ECOLS;
        const int colbase = ((warp - 2) >> 2) * CPW;           // EW / 4 warps per lane quarter
        int lt = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, lt++) {
            const int nt = t % ntn, mt = (t / ntn) % ntm, party = t / (ntn * ntm);
            const int v = q * 32 + lane;
            bool ok;
            uint32_t img, pix;
            if (AMODE == 2) {
                img = (uint32_t)(mt / geo.ntf);
                const int f = (mt - (int)img * geo.ntf) * BM + v;
                const int y = f / geo.Wp, x = f - y * geo.Wp;
                ok = y < geo.H && x < geo.W;
                pix = (uint32_t)(y * geo.W + x);
            } else {
                const int row = mt * BM + v;
                ok = row < M;
                img = (uint32_t)row / ohw;
                pix = (uint32_t)row - img * ohw;
            }
            const int buf = lt % NBUF;
            mbar_wait(&tfull[buf], (lt / NBUF) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int pp = 0; pp < NPASS; pp++) {
                const int cb = colbase + pp * ECOLS;
                const uint32_t taddr = tmem + lane_off + (uint32_t)buf * C::TB + (uint32_t)cb;
                // running lazy residue per column, folded group by group (EPI_COLS live u64
                // instead of 3 x EPI_COLS partial sums)
                u64 s[ECOLS];
#pragma unroll
                for (int grp = 0; grp < 3; grp++) {
                    uint32_t r[4][ECOLS];
#pragma unroll
                    for (int dd = 0; dd < 4; dd++)
                        if (grp * 4 + dd < ND) tmem_ld_cols<ECOLS>(taddr + (uint32_t)((grp * 4 + dd) * BN), r[dd]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (grp == 2 && pp == NPASS - 1) {
                        // TMEM drained: hand it back to the MMA warp before the last fold and stores
                        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                        __syncwarp();
                        if (lane == 0)
                            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
                    }
#pragma unroll
                    for (int c = 0; c < ECOLS; c++) {
                        // diagonal dd = 0 of the group enters as a plain add: the epilogue is bound
                        // by the FMA-heavy pipe (IMAD.WIDE) on short-K tiles
                        u64 acc = r[0][c];
#pragma unroll
                        for (int dd = 1; dd < 4; dd++)
                            if (grp * 4 + dd < ND) acc = mad_wide(r[dd][c], 1u << (8 * dd), acc);
                        // acc carries weight 2^(32 grp): combine()'s fold, one group at a time
                        // no fold per group: with D_d < 2^32 the group sums stay below 2^56.1
                        // (groups 0, 1) and 2^48.1 (group 2), and the weighted total below 2^57,
                        // so ONE fold at the end replaces three (-15 instructions per output)
                        if (grp == 0) {
                            s[c] = acc;                                                // < 2^56.1
                        } else if (grp == 1) {
                            s[c] += (acc >> 13) * 55 + ((acc & 0x1FFF) << 32);         // acc * 2^32, < 2^50
                        } else {
                            // acc >> 26 < 2^22.1: its product with 55 is a 32-bit IMAD
                            const u64 z = (u64)((uint32_t)(acc >> 26) * 55u) + ((acc & 0x3FFFFFF) << 19); // acc * 2^19, < 2^45.1
                            const u64 tt = lz(s[c] + z * 55);                          // acc * 2^64; sum < 2^57
                            s[c] = tt >= P ? tt - P : tt;
                        }
                    }
                }
                const int c0 = nt * BN + cb;
                if (ok) {
                    const u64 e0 = ((u64)img * O + (u64)c0) * ohw + pix;     // element index in [img][O][ohw]
                    if constexpr (SUB) {
                        u64 *sb = es.sub + (u64)party * es.sub_pstride + e0;
#pragma unroll 1
                        for (int c = 0; c < ECOLS; c++) {
                            if (c0 + c >= O) break;
                            const u64 i = e0 + (u64)c * ohw;
                            u64 cf[SSN_MAXK];
#pragma unroll
                            for (int jp = 0; jp < SSN_MAXK / 2; jp++)
                                if (2 * jp < es.km1) {
                                    const ssn_u4 r = ssn_philox_at(es.seed, es.stream + party, i, 0x800u | jp);
                                    const u64 x0 = (((u64)r.x << 32) | r.y) & MASK45, x1 = (((u64)r.z << 32) | r.w) & MASK45;
                                    cf[2 * jp] = x0 >= P ? x0 - P : x0;
                                    cf[2 * jp + 1] = x1 >= P ? x1 - P : x1;
                                }
#pragma unroll 1
                            for (int f = 0; f < es.nf; f++) {
                                u64 acc = s[c];
#pragma unroll
                                for (int e = 0; e < SSN_MAXK; e++)
                                    if (e < es.km1) acc += ((u64)(uint32_t)(cf[e] >> 32) * es.pw[f][e] << 32) +
                                                           (u64)(uint32_t)cf[e] * es.pw[f][e];
                                const u64 t = lz(acc);
                                sb[(u64)f * es.sub_fstride + (u64)c * ohw] = t >= P ? t - P : t;
                            }
                        }
                    } else {
                        u64 *ob = out + (u64)party * out_pstride + e0;
#pragma unroll
                        for (int c = 0; c < ECOLS; c++)
                            if (c0 + c < O) ob[(u64)c * ohw] = s[c];
                    }
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // no CTA of a pair leaves while the other may still multicast into its shared memory
    if constexpr (CL > 1) cluster_sync_all();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}
}  // namespace wide
}  // namespace p45

// tile width of the p45 share GEMM for a K of `kpad` bytes: SSN_GEMM_BN=16 / 32 forces one;
// otherwise BN = 16 (two 176-column TMEM accumulators: the MMAs of tile t+1 run while the
// epilogue drains tile t) when K <= SSN_GEMM_BN16_K (default 0: off), else BN = 32.
static int p45_bn(int kpad) {
    static int bn = -1, kmax = 0;
    if (bn < 0) {
        const char *e = getenv("SSN_GEMM_BN");
        bn = (e && atoi(e) == 32) ? 32 : (e && atoi(e) == 16) ? 16 : 0;
        const char *k = getenv("SSN_GEMM_BN16_K");
        kmax = k ? atoi(k) : 0;
    }
    if (bn) return bn;
    return kpad <= kmax ? 16 : SSN_GEMM_BN_DEFAULT;
}

template <int AMODE, int BN, bool SUB = false, int CL = 1, int EW = p45::wide::EPI_W>
static int launch_wide_bn(int grid, cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb, u64 *out,
                          u64 out_pstride, uint32_t ohw, int O, int M, int nkb, int ntm, int ntn, int ntiles,
                          p45::wide::ConvGeom geo, const p45::wide::EpiSub &es) {
    using namespace p45::wide;
    auto kern = k_gemm_p45w<AMODE, BN, SUB, CL, EW>;
    constexpr int THREADS = 64 + 32 * EW;             // TMA, MMA, epilogue warps
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM) != cudaSuccess)
            return SSN_ERR_CUDA;
        attr = true;
    }
    SSN_COUNT_LAUNCH();
    if constexpr (CL == 1) {
        kern<<<grid, THREADS, Cfg<BN>::SMEM, st>>>(ma, mb, out, out_pstride, ohw, O, M, nkb, ntm, ntn, ntiles, geo, es);
        const cudaError_t e = cudaPeekAtLastError();
        if (e != cudaSuccess && getenv("SSN_DEBUG"))
            fprintf(stderr, "k_gemm_p45w<%d,%d,%d,%d> grid %d x %d smem %d: %s\n", AMODE, BN, (int)SUB, CL, grid,
                    THREADS, Cfg<BN>::SMEM, cudaGetErrorString(e));
    } else {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3((unsigned)(grid - grid % CL));
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = Cfg<BN>::SMEM;
        cfg.stream = st;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm, ntn, ntiles, geo, es) !=
            cudaSuccess)
            return SSN_ERR_CUDA;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

// A-operand multicast across a 2-CTA cluster (SSN_GEMM_CLUSTER=1 disables): needs an even number of
// N tiles (the pair shares the A tile) and the plain (non-fused) epilogue
static int p45_cluster() {
    static int cl = 0;
    if (!cl) {
        const char *e = getenv("SSN_GEMM_CLUSTER");
        cl = (e && atoi(e) == 1) ? 1 : 2;
    }
    return cl;
}

template <int AMODE>
static int launch_wide(int bn, int cl, int grid, cudaStream_t st, const CUtensorMap &ma, const CUtensorMap &mb,
                       u64 *out, u64 out_pstride, uint32_t ohw, int O, int M, int nkb, int ntm, int ntn, int ntiles,
                       p45::wide::ConvGeom geo, const p45::wide::EpiSub *es = nullptr) {
    const p45::wide::EpiSub none{};
    if (es) {                          // fused RESHARE_OUT epilogue: 128 x 32 tiles, K-major A only
        if constexpr (AMODE == 0)
            return launch_wide_bn<0, 32, true>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm, ntn, ntiles,
                                               geo, *es);
        return SSN_ERR_UNSUPPORTED;
    }
    if (cl == 2) {
        // the 3x3 implicit GEMMs are MMA-bound (epilogue warps idle ~85%): with SSN_GEMM_EW2=4 they
        // run 4 epilogue warps, a smaller CTA that leaves room for co-resident chain blocks
        if constexpr (AMODE == 2) {
            static const int ew2 = getenv("SSN_GEMM_EW2") ? atoi(getenv("SSN_GEMM_EW2")) : 8;
            if (ew2 == 4 && bn == 32)
                return launch_wide_bn<AMODE, 32, false, 2, 4>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm,
                                                              ntn, ntiles, geo, none);
        }
        return bn == 16 ? launch_wide_bn<AMODE, 16, false, 2>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm,
                                                              ntn, ntiles, geo, none)
                        : launch_wide_bn<AMODE, 32, false, 2>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm,
                                                              ntn, ntiles, geo, none);
    }
    return bn == 16 ? launch_wide_bn<AMODE, 16>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm, ntn, ntiles,
                                                geo, none)
                    : launch_wide_bn<AMODE, 32>(grid, st, ma, mb, out, out_pstride, ohw, O, M, nkb, ntm, ntn, ntiles,
                                                geo, none);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

int make_map(CUtensorMap *map, const uint8_t *planes, int Kpad, int rows, int L, int P, int box_rows,
             int box_limbs = 0) {
    auto enc = get_encode();
    if (!enc) return SSN_ERR_CUDA;
    cuuint64_t dims[4] = {(cuuint64_t)Kpad, (cuuint64_t)rows, (cuuint64_t)L, (cuuint64_t)P};
    cuuint64_t strides[3] = {(cuuint64_t)Kpad, (cuuint64_t)Kpad * rows, (cuuint64_t)Kpad * rows * L};
    cuuint32_t box[4] = {(cuuint32_t)BK, (cuuint32_t)box_rows, (cuuint32_t)(box_limbs ? box_limbs : L), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t *>(planes), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : SSN_ERR_CUDA;
}

template <int L>
int launch_tc(const uint8_t *a, const uint8_t *b, int nparty, int M, int O, int Kpad, u64 *out, u64 out_pstride,
              u64 ohw, u64 p, cudaStream_t st) {
    CUtensorMap ma, mb;
    if (make_map(&ma, a, Kpad, M, L, nparty, BM) || make_map(&mb, b, Kpad, O, L, nparty, BN)) return SSN_ERR_CUDA;
    constexpr int smem = stages_for<L>() * (L * BM * BK + L * BN * BK) + 1024 + 256;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(k_gemm_tc<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
            return SSN_ERR_CUDA;
        attr = true;
    }
    CdTable cd = {};
    unsigned __int128 w = 1;
    for (int d = 0; d < 2 * L - 1; d++) {
        cd.c[d] = (u64)(w % p);
        w = (w % p) << 8;
    }
    SsnField f = ssn_make_field(p);
    u64 r64 = (u64)((((unsigned __int128)1) << 64) % p);
    if ((O + BN - 1) / BN > 65535 || nparty > 65535) return SSN_ERR_UNSUPPORTED;
    dim3 grid((M + BM - 1) / BM, (O + BN - 1) / BN, nparty);          // row tiles on x (no 65535 cap)
    SSN_COUNT_LAUNCH();
    k_gemm_tc<L><<<grid, 128, smem, st>>>(ma, mb, out, out_pstride, ohw, O, M, (Kpad + BK - 1) / BK, f, r64, cd);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

static int num_sms() {
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        // experiments: cap the persistent GEMM's CTAs (leaves SMs to concurrent chain kernels)
        const char *e = getenv("SSN_GEMM_GRID");
        if (e && atoi(e) >= 2 && atoi(e) < nsm) nsm = atoi(e) & ~1;
    }
    return nsm;
}

int launch_p45(const uint8_t *a, const uint8_t *b, int nparty, int M, int O, int Kpad, u64 *out, u64 out_pstride,
               u64 ohw, cudaStream_t st, const p45::wide::EpiSub *es = nullptr) {
    using namespace p45;
    const int bn = es ? 32 : p45_bn(Kpad);
    const int ntm = (M + BM - 1) / BM, ntn = (O + bn - 1) / bn;
    const int cl = (!es && ntn % 2 == 0) ? p45_cluster() : 1;
    CUtensorMap ma, mb;
    if (make_map(&ma, a, Kpad, M, L, nparty, BM, L / cl) || make_map(&mb, b, Kpad, O, L, nparty, bn))
        return SSN_ERR_CUDA;
    if (ohw >= (1ull << 32) || (u64)M * 1 >= (1ull << 31)) return SSN_ERR_UNSUPPORTED;
    const long long ntiles = (long long)ntm * ntn * nparty;
    if (ntiles >= (1ll << 31)) return SSN_ERR_UNSUPPORTED;
    const int nsm = num_sms();
    const int grid = (int)(ntiles < nsm ? ntiles : nsm);
    return launch_wide<0>(bn, cl, grid, st, ma, mb, out, out_pstride, (uint32_t)ohw, O, M, (Kpad + BK - 1) / BK, ntm, ntn,
                          (int)ntiles, wide::ConvGeom{}, es);
}


// Implicit-GEMM convolution from channel-major limb planes (modes 1 and 2 of k_gemm_p45w).
int launch_cn(const uint8_t *a, int mode, int nimg, int C, int H, int W, int Wp, const uint8_t *b, int nparty, int O,
              u64 *out, u64 out_pstride, cudaStream_t st) {
    using namespace p45;
    auto enc = get_encode();
    if (!enc) return SSN_ERR_CUDA;
    if (C % BK) return SSN_ERR_UNSUPPORTED;
    const int taps = mode == 2 ? 9 : 1;
    const int Kpad = taps * C;
    const int bn = p45_bn(Kpad);
    const int cl = ((O + bn - 1) / bn) % 2 == 0 ? p45_cluster() : 1;
    CUtensorMap ma, mb;
    const cuuint64_t PL = (cuuint64_t)nparty * L;
    CUresult r;
    if (mode == 1) {
        const cuuint64_t bhw = (cuuint64_t)nimg * H * W;
        if (bhw % 16) return SSN_ERR_UNSUPPORTED;
        cuuint64_t dims[3] = {bhw, (cuuint64_t)C, PL};
        cuuint64_t strides[2] = {bhw, bhw * C};
        cuuint32_t box[3] = {(cuuint32_t)BM, (cuuint32_t)BK, (cuuint32_t)(L / cl)};
        cuuint32_t estr[3] = {1, 1, 1};
        r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t *>(a), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        if (Wp < W || Wp % 16 || ((u64)H * Wp) % 16) return SSN_ERR_UNSUPPORTED;
        const cuuint64_t hw = (cuuint64_t)H * Wp;
        cuuint64_t dims[4] = {hw, (cuuint64_t)nimg, (cuuint64_t)C, 3 * PL};
        cuuint64_t strides[3] = {hw, hw * nimg, hw * nimg * C};
        cuuint32_t box[4] = {(cuuint32_t)BM, 1, (cuuint32_t)BK, (cuuint32_t)(L / cl)};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t *>(a), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return SSN_ERR_CUDA;
    if (make_map(&mb, b, Kpad, O, L, nparty, bn)) return SSN_ERR_CUDA;
    wide::ConvGeom geo{C, H, W, Wp, C / BK, 0, nparty};
    const int M = nimg * H * W;
    int ntm;
    if (mode == 1) {
        ntm = (M + BM - 1) / BM;
    } else {
        geo.ntf = (H * Wp + BM - 1) / BM;
        ntm = nimg * geo.ntf;
    }
    const int ntn = (O + bn - 1) / bn;
    const long long ntiles = (long long)ntm * ntn * nparty;
    if (ntiles >= (1ll << 31)) return SSN_ERR_UNSUPPORTED;
    const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
    const uint32_t ohw = (uint32_t)(H * W);
    if (mode == 1)
        return launch_wide<1>(bn, cl, grid, st, ma, mb, out, out_pstride, ohw, O, M, taps * geo.cblocks, ntm, ntn,
                              (int)ntiles, geo);
    return launch_wide<2>(bn, cl, grid, st, ma, mb, out, out_pstride, ohw, O, M, taps * geo.cblocks, ntm, ntn, (int)ntiles,
                          geo);
}

// ---------------------------------------------------------------- int8 tensor-pipe peak probe
// One CTA per SM issues back-to-back tcgen05.mma.kind::i8 of 128 x 256 x 32 from one resident
// smem tile pair into one TMEM accumulator (no global traffic, no epilogue): the measured dense
// int8 rate that the share GEMM's roofline divides by (bench.py, MEASURED_INT8.json).
__global__ void __launch_bounds__(128, 1) k_mma_peak(int iters, unsigned long long *sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // A 128 x 32 B and B 256 x 32 B, K-major SW64 tiles (contents irrelevant for throughput)
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + 128 * 64 + 256 * 64);
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 256) * 64 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = i;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const uint64_t ad = umma_desc_sw64(smem_u32(base)), bd = umma_desc_sw64(smem_u32(base + 128 * 64));
        constexpr uint32_t ID = idesc_i8(256);
        for (int i = 0; i < iters; i++) mma_i8(tmem, ad, bd, ID, i > 0 ? 1u : 0u);
        mma_commit(bar);
        mbar_wait(bar, 0);
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t r[8];
        tmem_ld8(tmem + ((uint32_t)(threadIdx.x & 31) << 16), r);
        if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)r[0]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// Measurement only: the MMA issue pattern of the share GEMM from resident shared memory (no TMA,
// no epilogue).  mode 0: one A tile x one B tile (N = n) back to back into one accumulator;
// mode 1: the wide GEMM's K slice -- per 32-deep slice, 6 MMAs of 128 x n x 32, A limb i (six
// distinct 128 x 64 B tiles) against the stacked B limbs, D at TMEM column 32 i.
__global__ void __launch_bounds__(128, 1) k_mma_probe(int mode, int n, int iters, unsigned long long *sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int AB = 6 * 128 * 64, BB = 256 * 64;
    uint64_t *bar = reinterpret_cast<uint64_t *>(base + AB + BB);
    uint32_t *slot = reinterpret_cast<uint32_t *>(bar + 1);
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (AB + BB) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(base)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        const uint32_t sa = smem_u32(base), sb = smem_u32(base + AB);
        const uint32_t id = idesc_i8(n);
        if (mode == 0) {
            const uint64_t ad = umma_desc_sw64(sa), bd = umma_desc_sw64(sb);
            for (int i = 0; i < iters; i++) mma_i8(tmem, ad, bd, id, i > 0 ? 1u : 0u);
        } else {
            for (int it = 0; it < iters; it += 12) {
#pragma unroll
                for (int kk = 0; kk < 2; kk++) {
                    const uint64_t bd = umma_desc_sw64(sb + kk * 32);
#pragma unroll
                    for (int i = 0; i < 6; i++)
                        mma_i8(tmem + (uint32_t)(i * 32), umma_desc_sw64(sa + i * 128 * 64 + kk * 32), bd, id,
                               it > 0 ? 1u : 0u);
                }
            }
        }
        mma_commit(bar);
        mbar_wait(bar, 0);
    }
    __syncthreads();
    if (warp == 0) {
        uint32_t r[8];
        tmem_ld8(tmem + ((uint32_t)(threadIdx.x & 31) << 16), r);
        if (threadIdx.x == 0) atomicAdd(sink, (unsigned long long)r[0]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------- operand preparation
// x: [P][rows][K] u64 (row-major) -> planes [P][L][rows][Kpad] u8, zero padded in K.
__global__ void k_limb_split(const u64 *__restrict__ x, u64 rows, u64 K, u64 Kpad, int L, uint8_t *__restrict__ planes,
                             u64 x_pstride, u64 total_chunks) {
    const u64 chunks_per_row = Kpad / 8;
    for (u64 g = blockIdx.x * (u64)blockDim.x + threadIdx.x; g < total_chunks; g += (u64)gridDim.x * blockDim.x) {
        const u64 per_party = rows * chunks_per_row;
        const u64 party = g / per_party;
        const u64 rem = g - party * per_party;
        const u64 r = rem / chunks_per_row, kc = (rem - r * chunks_per_row) * 8;
        const u64 *src = x + party * x_pstride + r * K;
        u64 v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = (kc + q < K) ? src[kc + q] : 0;
        uint8_t *dst = planes + party * (u64)L * rows * Kpad + r * Kpad + kc;
        for (int l = 0; l < L; l++) {
            u64 packed = 0;
#pragma unroll
            for (int q = 0; q < 8; q++) packed |= ((v[q] >> (8 * l)) & 0xFF) << (8 * q);
            *reinterpret_cast<u64 *>(dst + (u64)l * rows * Kpad) = packed;
        }
    }
}

// conv: x [P][img][C][H][W] -> planes [P][L][img*OH*OW][Kpad], k = (c, i, j) like im2col.
// Block: 64 rows x 64 k.  Gather coalesced along rows (consecutive output pixels) into
// shared memory, then each thread emits one 16-byte vector per limb plane (16 k of one row).
constexpr int IC_ROWS = 64, IC_K = 64, IC_THREADS = 256;

__global__ void __launch_bounds__(IC_THREADS) k_im2col_limbs(const u64 *__restrict__ x, int C, int H, int W, int kh,
                                                              int kw, int stride, int pad, int OH, int OW, int L,
                                                              uint32_t rows, int K, int Kpad,
                                                              uint8_t *__restrict__ planes, u64 x_pstride) {
    __shared__ u64 sv[IC_ROWS][IC_K + 1];
    __shared__ int64_t s_off[IC_K];               // k -> c*H*W (or -1 past K), tap row/col - pad
    __shared__ int s_i[IC_K], s_j[IC_K];
    const int party = blockIdx.z;
    const uint32_t r0 = blockIdx.x * IC_ROWS;     // row tiles on x (up to 2^31 - 1 blocks)
    const int k0 = blockIdx.y * IC_K;
    const int t = threadIdx.x;
    const u64 *xp = x + (u64)party * x_pstride;
    const uint32_t ohw = (uint32_t)(OH * OW);
    const int khw = kh * kw;
    if (t < IC_K) {                               // the block's 64 k decompositions, once
        const int k = k0 + t;
        if (k < K) {
            const int c = k / khw, rem = k - c * khw;
            const int i = rem / kw;
            s_off[t] = (int64_t)c * H * W;
            s_i[t] = i - pad;
            s_j[t] = rem - i * kw - pad;
        } else {
            s_off[t] = -1;
        }
    }
    __syncthreads();
    {
        const int rr = t & (IC_ROWS - 1);
        const uint32_t r = r0 + rr;
        const bool rok = r < rows;
        uint32_t img = 0;
        int oy = 0, ox = 0;
        if (rok) {
            img = r / ohw;
            const int pix = (int)(r - img * ohw);
            oy = pix / OW;
            ox = pix - oy * OW;
        }
        const u64 *ximg = xp + (u64)img * C * H * W;
        const int oys = oy * stride, oxs = ox * stride;
#pragma unroll 4
        for (int kk = t / IC_ROWS; kk < IC_K; kk += IC_THREADS / IC_ROWS) {
            u64 v = 0;
            const int64_t off = s_off[kk];
            if (rok && off >= 0) {
                const int sy = oys + s_i[kk], sx = oxs + s_j[kk];
                if (sy >= 0 && sy < H && sx >= 0 && sx < W) v = ximg[off + (int64_t)sy * W + sx];
            }
            sv[rr][kk] = v;
        }
    }
    __syncthreads();
    {
        const int rr = t >> 2, kc = (t & 3) * 16;
        const uint32_t r = r0 + rr;
        if (r < rows && k0 + kc < Kpad) {
            uint8_t *dst = planes + (u64)party * L * rows * Kpad + (u64)r * Kpad + k0 + kc;
            u64 v[16];
#pragma unroll
            for (int q = 0; q < 16; q++) v[q] = sv[rr][kc + q];          // one pass over smem
#pragma unroll 1
            for (int l = 0; l < L; l++) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    // byte l of 4 consecutive elements -> one 32-bit word (PRMT-friendly)
                    const uint32_t b0 = (uint32_t)(v[4 * q] >> (8 * l)) & 0xFF;
                    const uint32_t b1 = (uint32_t)(v[4 * q + 1] >> (8 * l)) & 0xFF;
                    const uint32_t b2 = (uint32_t)(v[4 * q + 2] >> (8 * l)) & 0xFF;
                    const uint32_t b3 = (uint32_t)(v[4 * q + 3] >> (8 * l)) & 0xFF;
                    w[q] = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
                }
                *reinterpret_cast<uint4 *>(dst + (u64)l * rows * Kpad) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
}

// x [P][img][C][H][W] u64 -> channel-major limb planes [P][L][C][img][H][Wp] (Wp >= W; pad
// columns untouched: the caller zeroes the buffer once).  Wp == W gives the contiguous layout
// [P][L][C][img*H*W] of mode 1.
__global__ void k_planes_cn(const u64 *__restrict__ x, int nimg, int C, int H, int W, int Wp, int L,
                            uint8_t *__restrict__ planes, u64 x_pstride, u64 total, int copies, int nparty) {
    const u64 per_party = (u64)nimg * C * H * W;
    const u64 plane = (u64)C * nimg * H * Wp;
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        const u64 party = i / per_party;
        const u64 r = i - party * per_party;
        const uint32_t xx = (uint32_t)(r % W);
        const u64 r2 = r / W;
        const uint32_t y = (uint32_t)(r2 % H);
        const u64 r3 = r2 / H;
        const uint32_t c = (uint32_t)(r3 % C), img = (uint32_t)(r3 / C);
        const u64 v = x[party * x_pstride + r];
        for (int dx = 0; dx < copies; dx++) {
            const int xc = copies == 1 ? (int)xx : (int)xx + 1 - dx;     // copy dx holds column x + dx - 1
            if (xc < 0 || xc >= Wp) continue;
            uint8_t *dst = planes + ((u64)dx * nparty + party) * L * plane + (((u64)c * nimg + img) * H + y) * Wp + xc;
            for (int l = 0; l < L; l++) dst[(u64)l * plane] = (uint8_t)(v >> (8 * l));
        }
    }
}

// Mode-2 column copies from the unshifted copy: planes [3][rows][Wp] with rows = party*L*C*img*H;
// copy 0 at x = copy 1 at x - 1 (0 at x = 0), copy 2 at x = copy 1 at x + 1 (copy 1's pad
// columns x >= W are zero).  One thread per 16-byte chunk, funnel-shifted in registers.
__global__ void k_planes_shift(uint8_t *__restrict__ planes, u64 rows, int Wp) {
    const int cpr = Wp / 16;                                   // chunks per row
    const u64 total = rows * cpr;
    const u64 cs = rows * (u64)Wp;                             // copy stride
    for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < total; i += (u64)gridDim.x * blockDim.x) {
        const u64 row = i / cpr;
        const int ch = (int)(i - row * cpr);
        const uint8_t *src = planes + cs + row * Wp + ch * 16;
        const uint4 cur = *reinterpret_cast<const uint4 *>(src);
        const uint32_t prev = ch > 0 ? *reinterpret_cast<const uint32_t *>(src - 4) : 0u;          // bytes x-4..x-1
        const uint32_t next = ch + 1 < cpr ? *reinterpret_cast<const uint32_t *>(src + 16) : 0u;  // bytes x+16..
        // left shift by one byte (copy 0): out[j] = in[j-1]
        uint4 l, r;
        l.x = __funnelshift_l(prev, cur.x, 8);
        l.y = __funnelshift_l(cur.x, cur.y, 8);
        l.z = __funnelshift_l(cur.y, cur.z, 8);
        l.w = __funnelshift_l(cur.z, cur.w, 8);
        // right shift by one byte (copy 2): out[j] = in[j+1]
        r.x = __funnelshift_r(cur.x, cur.y, 8);
        r.y = __funnelshift_r(cur.y, cur.z, 8);
        r.z = __funnelshift_r(cur.z, cur.w, 8);
        r.w = __funnelshift_r(cur.w, next, 8);
        *reinterpret_cast<uint4 *>(planes + row * Wp + ch * 16) = l;
        *reinterpret_cast<uint4 *>(planes + 2 * cs + row * Wp + ch * 16) = r;
    }
}

}  // namespace

extern "C" int ssn_planes_shift(uint8_t *planes, uint64_t rows, int Wp, void *stream) {
    if (Wp < 16 || Wp % 16 || rows == 0) return SSN_ERR_ARG;
    const u64 total = rows * (Wp / 16);
    u64 blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    SSN_COUNT_LAUNCH();
    static const bool carve_k_planes_shift = (ssn_prefer_max_smem(k_planes_shift), true);
    (void)carve_k_planes_shift;
    k_planes_shift<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(planes, rows, Wp);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_planes_cn(const u64 *x, int nparty, int nimg, int C, int H, int W, int Wp, int L, uint8_t *planes,
                             u64 x_pstride, int copies, void *stream) {
    if (nparty < 1 || nimg < 1 || C < 1 || H < 1 || W < 1 || Wp < W || L < 1 || L > MAXL) return SSN_ERR_ARG;
    if (copies != 1 && (copies != 3 || Wp % 16)) return SSN_ERR_ARG;
    const u64 total = (u64)nparty * nimg * C * H * W;
    u64 blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    SSN_COUNT_LAUNCH();
    static const bool carve_k_planes_cn = (ssn_prefer_max_smem(k_planes_cn), true);
    (void)carve_k_planes_cn;
    k_planes_cn<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, nimg, C, H, W, Wp, L, planes, x_pstride, total,
                                                                     copies, nparty);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_limb_split(const u64 *x, u64 rows, u64 K, u64 Kpad, int L, uint8_t *planes, u64 x_pstride,
                              int nparty, void *stream) {
    if (L < 1 || L > MAXL || Kpad % 16 || Kpad < K || nparty < 1) return SSN_ERR_ARG;
    u64 total = (u64)nparty * rows * (Kpad / 8);
    if (total == 0) return 0;
    u64 blocks = (total + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    SSN_COUNT_LAUNCH();
    static const bool carve_k_limb_split = (ssn_prefer_max_smem(k_limb_split), true);
    (void)carve_k_limb_split;
    k_limb_split<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, rows, K, Kpad, L, planes, x_pstride, total);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_im2col_limbs(const u64 *x, int nparty, int nimg, int C, int H, int W, int kh, int kw, int stride,
                                int pad, int L, uint8_t *planes, u64 Kpad, u64 x_pstride, void *stream) {
    if (L < 1 || L > MAXL || Kpad % 16 || nparty < 1 || nimg < 1) return SSN_ERR_ARG;
    const int OH = (H + 2 * pad - kh) / stride + 1, OW = (W + 2 * pad - kw) / stride + 1;
    const int K = C * kh * kw;
    if ((u64)K > Kpad || OH < 1 || OW < 1) return SSN_ERR_ARG;
    const u64 rows = (u64)nimg * OH * OW;
    if (rows >= (1ull << 32)) return SSN_ERR_UNSUPPORTED;
    if ((Kpad + IC_K - 1) / IC_K > 65535 || nparty > 65535) return SSN_ERR_UNSUPPORTED;
    dim3 grid((unsigned)((rows + IC_ROWS - 1) / IC_ROWS), (unsigned)((Kpad + IC_K - 1) / IC_K), (unsigned)nparty);
    SSN_COUNT_LAUNCH();
    static const bool carve_k_im2col_limbs = (ssn_prefer_max_smem(k_im2col_limbs), true);
    (void)carve_k_im2col_limbs;
    k_im2col_limbs<<<grid, IC_THREADS, 0, (cudaStream_t)stream>>>(x, C, H, W, kh, kw, stride, pad, OH, OW, L,
                                                                  (uint32_t)rows, K, (int)Kpad, planes, x_pstride);
    return cudaGetLastError() == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_gemm_tc_conv(const uint8_t *a_planes, int mode, int nimg, int C, int H, int W, int Wp,
                                const uint8_t *b_planes, int nparty, int O, u64 *out, u64 out_pstride, u64 p,
                                void *stream) {
    if ((mode != 1 && mode != 2) || nimg < 1 || C < 1 || H < 1 || W < 1 || nparty < 1 || O < 1) return SSN_ERR_ARG;
    if (p != p45::P) return SSN_ERR_UNSUPPORTED;
    return launch_cn(a_planes, mode, nimg, C, H, W, Wp, b_planes, nparty, O, out, out_pstride, (cudaStream_t)stream);
}

// planes A [P][L][M][Kpad] (rows = activation pixels), B [P][L][O][Kpad] (weights);
// out [P] at out_pstride: element (row, col) -> out[(row / ohw) * O * ohw + col * ohw + row % ohw].
// Exactness requires L * K * 255^2 < 2^32 (host splits K otherwise).
extern "C" int ssn_gemm_tc(const uint8_t *a_planes, const uint8_t *b_planes, int nparty, int L, int M, int O,
                           u64 Kpad, u64 ohw, u64 *out, u64 out_pstride, u64 p, void *stream) {
    if (L < 1 || L > MAXL || Kpad % 16 || M < 1 || O < 1 || nparty < 1 || ohw < 1) return SSN_ERR_ARG;
    if ((unsigned __int128)L * Kpad * 65025 >= ((unsigned __int128)1 << 32)) return SSN_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (L == 6 && p == p45::P) return launch_p45(a_planes, b_planes, nparty, M, O, (int)Kpad, out, out_pstride, ohw, st);
    switch (L) {
        case 6: return launch_tc<6>(a_planes, b_planes, nparty, M, O, (int)Kpad, out, out_pstride, ohw, p, st);
        case 7: return launch_tc<7>(a_planes, b_planes, nparty, M, O, (int)Kpad, out, out_pstride, ohw, p, st);
        case 8: return launch_tc<8>(a_planes, b_planes, nparty, M, O, (int)Kpad, out, out_pstride, ohw, p, st);
        default: return SSN_ERR_UNSUPPORTED;
    }
}

extern "C" int ssn_gemm_tc_subshares(const uint8_t *a_planes, const uint8_t *b_planes, int nparty, int M, int O,
                                     u64 Kpad, u64 ohw, const ssn_subshare_desc *d, u64 p, void *stream) {
    if (!d || !d->sub || !d->front_ids || Kpad % 16 || M < 1 || O < 1 || nparty < 1 || ohw < 1 || d->km1 < 0 ||
        d->km1 > SSN_MAXK - 1 || d->nf < 1 || d->nf > SSN_MAXK)
        return SSN_ERR_ARG;
    if (p != p45::P || (unsigned __int128)6 * Kpad * 65025 >= ((unsigned __int128)1 << 32)) return SSN_ERR_UNSUPPORTED;
    p45::wide::EpiSub es{};
    es.sub = d->sub;
    es.sub_pstride = d->party_stride;
    es.sub_fstride = d->front_stride;
    es.seed = d->seed;
    es.stream = d->stream;
    es.km1 = d->km1;
    es.nf = d->nf;
    for (int f = 0; f < d->nf; f++) {
        unsigned __int128 acc = 1;
        for (int e = 0; e < d->km1; e++) {
            acc = acc * (d->front_ids[f] % p) % p;
            if (acc >= (1u << 13)) return SSN_ERR_UNSUPPORTED;      // small id powers (ids 1..k)
            es.pw[f][e] = (uint32_t)acc;
        }
    }
    return launch_p45(a_planes, b_planes, nparty, M, O, (int)Kpad, nullptr, 0, ohw, (cudaStream_t)stream, &es);
}

extern "C" int ssn_mma_peak(int iters, int ctas, float *ms, double *int8_ops, void *stream) {
    if (iters < 1 || ctas < 1 || !ms || !int8_ops) return SSN_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int smem = (128 + 256) * 64 + 1024 + 64;
    if (cudaFuncSetAttribute(k_mma_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SSN_ERR_CUDA;
    unsigned long long *sink = nullptr;
    if (cudaMallocAsync(&sink, sizeof(*sink), st) != cudaSuccess) return SSN_ERR_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mma_peak<<<ctas, 128, smem, st>>>(2, sink);          // warm-up
    cudaEventRecord(e0, st);
    SSN_COUNT_LAUNCH();
    k_mma_peak<<<ctas, 128, smem, st>>>(iters, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(sink, st);
    *int8_ops = 2.0 * 128 * 256 * 32 * (double)iters * ctas;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : SSN_ERR_CUDA;
}

extern "C" int ssn_mma_probe(int mode, int n, int iters, int ctas, float *ms, double *int8_ops, void *stream) {
    if (iters < 12 || ctas < 1 || !ms || !int8_ops || n < 16 || n > 256 || n % 16 || (mode == 1 && n > 192))
        return SSN_ERR_ARG;
    iters -= iters % 12;
    cudaStream_t st = (cudaStream_t)stream;
    const int smem = 6 * 128 * 64 + 256 * 64 + 1024 + 64;
    if (cudaFuncSetAttribute(k_mma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SSN_ERR_CUDA;
    unsigned long long *sink = nullptr;
    if (cudaMallocAsync(&sink, sizeof(*sink), st) != cudaSuccess) return SSN_ERR_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mma_probe<<<ctas, 128, smem, st>>>(mode, n, 12, sink);          // warm-up
    cudaEventRecord(e0, st);
    SSN_COUNT_LAUNCH();
    k_mma_probe<<<ctas, 128, smem, st>>>(mode, n, iters, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(sink, st);
    *int8_ops = 2.0 * 128 * n * 32 * (double)iters * ctas;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : SSN_ERR_CUDA;
}
