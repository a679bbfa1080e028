// lrbms_ns.cuh -- Newton-Schulz update of the coarse inverse on the 5th-generation tensor cores.
//
//   Xn = X + X R,   R = I - E X   (E = Z^T B Z the coarse operator of this step, X ~ E^-1)
//
// one step per time step keeps the deflation preconditioner's coarse inverse current (DESIGN.md,
// reduced solve).  X is kept exactly symmetric, so R^T = I - X E is formed row-wise (k_coarse_rt)
// and both GEMM operands are K-major: D = X * RT^T.  Only the upper-triangular 128 x 128 output
// tiles are computed; each is written to (I, J) and, transposed, to (J, I).
//
// Kernel anatomy (one output tile per CTA, 4 warps):
//   warp 0 / lane 0  TMA producer: 128 x 32 fp32 tiles of X and RT (128-byte swizzle) into a
//                    4-stage shared-memory ring, completion on mbarriers (expect_tx);
//   warp 1 / lane 0  MMA issuer: tcgen05.mma.cta_group::1.kind::tf32, M = N = 128, K = 8 per
//                    instruction, accumulator in TMEM (128 lanes x 128 fp32 columns);
//                    tcgen05.commit frees a ring slot / signals the epilogue;
//   warps 0-3        epilogue: tcgen05.ld (32 lanes x 32 columns per warp and chunk), + X, fp32
//                    stores of the tile and of its transpose.
// TF32 inputs (10-bit mantissa), fp32 accumulation: R is the one-step change of E^-1, so the
// rounding perturbs only the correction (error ~1e-3 |X R|).
#pragma once
#include <cuda.h>
#include <cstdint>

namespace lrbms {

constexpr int NS_TM = 128, NS_TK = 32, NS_STAGES = 6;   // 6-stage TMA ring: 30 vs 33 us with 4
constexpr int NS_TILE_BYTES = NS_TM * NS_TK * 4;                  // 16 KB per operand and stage
constexpr int NS_TC_SMEM = 2 * NS_STAGES * NS_TILE_BYTES + 1024;  // + 1 KB alignment slack

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n NS_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra NS_WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 bytes apart
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr & 0x3FFFF) >> 4;              // start address (16-byte units)
  d |= (uint64_t)1 << 16;                  // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                  // layout: SWIZZLE_128B
  return d;
}
// instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major, M = N = 128
constexpr uint32_t NS_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NS_TM >> 3) << 17) |
                              ((uint32_t)(NS_TM >> 4) << 24);

__global__ void __launch_bounds__(128, 1) k_ns_gemm_tc(const __grid_constant__ CUtensorMap mapX,
                                                       const __grid_constant__ CUtensorMap mapRT,
                                                       const float* __restrict__ X, float* __restrict__ Xn, int n,
                                                       const unsigned* __restrict__ guard, int* __restrict__ trip) {
  extern __shared__ uint8_t ns_raw[];
  __shared__ __align__(8) uint64_t full[NS_STAGES], empty[NS_STAGES], done;
  __shared__ uint32_t tmem_base;
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ns_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;                                   // [stage][128 rows][128 B]
  uint8_t* sB = sm + NS_STAGES * NS_TILE_BYTES;       // [stage][128 rows][128 B]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // upper-triangular tile (I <= J) of the nb x nb tile grid
  const int nb = (n + NS_TM - 1) / NS_TM;
  int t = blockIdx.x, I = 0;
  while (t >= nb - I) {
    t -= nb - I;
    ++I;
  }
  const int J = I + t;
  const int nk = n / NS_TK;

  if (warp == 0) {   // TMEM: 128 fp32 accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(NS_TM));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < NS_STAGES; ++s) {
      mbar_init_n(&full[s], 1);
      mbar_init_n(&empty[s], 1);
    }
    mbar_init_n(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0 && lane == 0) {   // TMA producer
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapX)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&mapRT)) : "memory");
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % NS_STAGES;
      if (kc >= NS_STAGES) mbar_wait_parity(&empty[s], ((kc / NS_STAGES) - 1) & 1);
      mbar_arrive_tx(&full[s], 2 * NS_TILE_BYTES);
      tma_load_2d(sA + s * NS_TILE_BYTES, &mapX, kc * NS_TK, I * NS_TM, &full[s]);
      tma_load_2d(sB + s * NS_TILE_BYTES, &mapRT, kc * NS_TK, J * NS_TM, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {   // MMA issuer
    for (int kc = 0; kc < nk; ++kc) {
      const int s = kc % NS_STAGES;
      mbar_wait_parity(&full[s], (kc / NS_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint64_t da = umma_desc_sw128(sA + s * NS_TILE_BYTES);
      const uint64_t db = umma_desc_sw128(sB + s * NS_TILE_BYTES);
#pragma unroll
      for (int kk = 0; kk < NS_TK / 8; ++kk) {   // K = 8 tf32 = 32 bytes per instruction
        const uint64_t adv = (uint64_t)((kk * 32) >> 4);
        const uint32_t acc = (kc > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(da + adv), "l"(db + adv), "r"(NS_IDESC), "r"(acc)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&done))
                 : "memory");
  }
  __syncwarp();

  // epilogue: warp w owns TMEM lanes (tile rows) 32 w .. 32 w + 31.  Guard: if max |I - E X| of this
  // step (k_coarse_rt*) is >= NS_GUARD_MAX or NaN, the iteration is not converging to E^-1: the
  // inverse is dropped (Xn = 0, the solve continues as block-Jacobi PCG, which the deflation variant
  // with a wrong coarse inverse would not) and the context is flagged; it rebuilds at its next call
  const float gmax = __uint_as_float(__ldcg(guard));
  const bool keep = gmax < NS_GUARD_MAX;
  if (!keep && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(trip, 1);
  mbar_wait_parity(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = I * NS_TM + 32 * warp + lane;
  for (int c0 = 0; c0 < NS_TM; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int col0 = J * NS_TM + c0;
    if (col0 < n) {   // n % 32 == 0: a 32-column chunk is entirely inside or outside
      if (I == J) {   // diagonal tile: the upper half, mirrored (exactly symmetric)
        if (row < n) {
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int col = col0 + q;
            if (col < row) continue;
            const float val = keep ? X[(size_t)col * n + row] + __uint_as_float(v[q]) : 0.f;
            Xn[(size_t)row * n + col] = val;
            Xn[(size_t)col * n + row] = val;
          }
        }
      } else {
        float val[32];
#pragma unroll
        for (int q = 0; q < 32; ++q)   // X symmetric: X[row][col] = X[col][row], read coalesced
          val[q] = (row < n && keep) ? X[(size_t)(col0 + q) * n + row] + __uint_as_float(v[q]) : 0.f;
        if (row < n) {
          float4* dst = reinterpret_cast<float4*>(Xn + (size_t)row * n + col0);
#pragma unroll
          for (int q4 = 0; q4 < 8; ++q4)
            dst[q4] = make_float4(val[4 * q4], val[4 * q4 + 1], val[4 * q4 + 2], val[4 * q4 + 3]);
#pragma unroll
          for (int q = 0; q < 32; ++q) Xn[(size_t)(col0 + q) * n + row] = val[q];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(NS_TM));
}

}  // namespace lrbms
