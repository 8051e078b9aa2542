// 5th-generation tensor cores (tcgen05 / UMMA, accumulator in TMEM) for the
// per-step weighted Gram matrix of the logistic-regression Hessian
// (targets.py:254-287): H_t = X^T diag(w_t) X, X (N x D <= 128), K = N.
//
// Operands are K-major 128 x 32 f32 tiles (one 128-byte swizzle row per
// operand row, SWIZZLE_128B), A = w_t . X^T and B = X^T staged by the CTA's
// threads from a transposed f32 copy XT (128 x Npad, L2-resident), two
// stages in flight; one elected thread issues kind::tf32 MMAs (M = N = 128,
// K = 8) into a 128-column f32 accumulator in TMEM, committing each stage back
// to its producers through an mbarrier; the epilogue reads the accumulator
// with tcgen05.ld (warp w -> TMEM lanes 32 (w % 4) ..) into shared memory.
#pragma once
#include "cs_common.cuh"
#include "cs_tma.cuh"

namespace cs {

constexpr int kUmmaTile = 128 * 32;          // f32 elements of one operand tile (16 KB)
constexpr int kUmmaStages = 3;
constexpr int kUmmaKB = 32;                  // K (data rows) per stage

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm100 layout:
// start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48),
// layout type [61,64) = 2); 8-row core-matrix groups are 1024 B apart
CS_D uint64_t umma_desc_sw128(const void *smem_tile) {
  const uint64_t a = (uint64_t)smem_u32(smem_tile);
  return ((a & 0x3FFFFull) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t kIdescTf32_128x128 = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

CS_D void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
CS_D void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
CS_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
CS_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 16 consecutive 32-bit columns of TMEM -> 16 registers per thread
CS_D void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// TMEM allocation by warp 0 (128 columns); every thread gets the base address
CS_D uint32_t tmem_alloc128(uint32_t *s_slot) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(s_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  return *(volatile uint32_t *)s_slot;
}
CS_D void tmem_free128(uint32_t base) {
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base) : "memory");
}

// Pipeline state carried across the steps a persistent CTA processes.
struct UmmaPipe {
  uint64_t *full;   // [kUmmaStages] count = staging threads (every one stored its share)
  uint64_t *empty;  // [kUmmaStages] count 1 (tcgen05.commit)
  uint64_t *done;   // [1] count 1: the accumulator of this step is complete
  uint32_t tmem;
  uint32_t kb;      // K-blocks staged so far (stage = kb % S, phase = (kb / S) & 1)
  uint32_t steps;   // accumulations completed (done-barrier phase)
};

CS_D void umma_pipe_init(UmmaPipe &p) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kUmmaStages; ++s) {
      mbar_init(&p.full[s], blockDim.x - 32);  // the staging threads (warps 1..)
      mbar_init(&p.empty[s], 1);
    }
    mbar_init(p.done, 1);
    fence_mbar_init();
  }
  p.kb = 0;
  p.steps = 0;
}

// Hs[i][j] (row stride ldh, f32) = sum_n w[n] X[n][i] X[n][j] for i, j < 128,
// exactly symmetric (upper triangle mirrored).  XT: f32 [128][ldx] (rows >= D
// and columns >= N zero), w: N weights in shared memory, tiles: 1024-aligned
// smem of kUmmaStages * 2 * kUmmaTile floats (may alias Hs: the epilogue
// starts after every MMA has completed).  Called by all threads of the CTA.
template <int NTHR>
CS_D void gram_tcgen05(UmmaPipe &p, const float *__restrict__ XT, int ldx, int N, const float *w, float *tiles,
                       float *Hs, int ldh) {
  // warp 0 only issues (lane 0: wait for a staged block, 4 MMAs, commit);
  // warps 1.. stage, running up to kUmmaStages blocks ahead of the MMAs
  constexpr int NS = NTHR - 32;                       // staging threads
  constexpr int PER = (128 * 8 + NS - 1) / NS;        // 16-byte chunks per staging thread per operand
  const int tid = threadIdx.x;
  const int nkb = (N + kUmmaKB - 1) / kUmmaKB;
  if (tid < 32) {
    if (tid == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const uint32_t g = p.kb + kb;
        const int s = (int)(g % kUmmaStages);
        mbar_wait(&p.full[s], (g / kUmmaStages) & 1);
        tc_fence_after();
        float *A = tiles + s * 2 * kUmmaTile, *B = A + kUmmaTile;
        const uint64_t da = umma_desc_sw128(A), db = umma_desc_sw128(B);
#pragma unroll
        for (int k = 0; k < kUmmaKB / 8; ++k)  // K = 8 tf32 = 32 B per MMA: advance the start address by 2 (x16 B)
          umma_tf32(p.tmem, da + 2 * k, db + 2 * k, kIdescTf32_128x128, (kb | k) != 0);
        umma_commit(&p.empty[s]);
      }
      umma_commit(p.done);
    }
    __syncwarp();
  } else {
    const int st = tid - 32;
    // X^T chunks are loaded into registers two K-blocks ahead of their store
    float4 xr[2][PER];
    auto load = [&](int kb, float4 (&dst)[PER]) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = st + i * NS, r = q >> 3, c = q & 7;
        dst[i] = (kb < nkb && q < 128 * 8) ? __ldg((const float4 *)(XT + (int64_t)r * ldx + kb * kUmmaKB + 4 * c))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    load(0, xr[0]);
    load(1, xr[1]);
#pragma unroll 2
    for (int kb = 0; kb < nkb; ++kb) {
      const uint32_t g = p.kb + kb;
      const int s = (int)(g % kUmmaStages);
      const uint32_t use = g / kUmmaStages;
      if (use > 0) mbar_wait(&p.empty[s], (use - 1) & 1);  // the MMAs that read this stage are done
      float *A = tiles + s * 2 * kUmmaTile, *B = A + kUmmaTile;
      // 128 rows x 8 chunks of 16 B per operand; chunk c of row r lands at c ^ (r & 7)
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int q = st + i * NS, r = q >> 3, c = q & 7, n0 = kb * kUmmaKB + 4 * c;
        if (q < 128 * 8) {
          const float4 x = xr[kb & 1][i];
          const float4 ww = *(const float4 *)(w + n0);
          const int off = r * 32 + ((c ^ (r & 7)) << 2);
          *(float4 *)(B + off) = x;
          *(float4 *)(A + off) = make_float4(x.x * ww.x, x.y * ww.y, x.z * ww.z, x.w * ww.w);
        }
      }
      if (kb + 2 < nkb) load(kb + 2, xr[kb & 1]);
      fence_proxy_async_smem();  // generic-proxy stores -> visible to the tensor core (async proxy)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p.full[s])) : "memory");
    }
  }
  p.kb += nkb;
  // epilogue: TMEM -> registers -> Hs (warp w: lanes 32 (w % 4) .., column half w / 4)
  mbar_wait(p.done, p.steps & 1);
  ++p.steps;
  tc_fence_after();
  const int wid = tid >> 5, lane = tid & 31;
  if (wid < 8) {
    const int row = 32 * (wid & 3) + lane, c0 = 64 * (wid >> 2);
#pragma unroll
    for (int cc = 0; cc < 64; cc += 16) {
      float v[16];
      tmem_ld16(p.tmem + ((uint32_t)(32 * (wid & 3)) << 16) + (uint32_t)(c0 + cc), v);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = c0 + cc + i;
        if (col >= row) {
          Hs[row * ldh + col] = v[i];
          Hs[col * ldh + row] = v[i];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
}

}  // namespace cs
