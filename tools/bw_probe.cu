// Streaming-read microbenchmark (development probe, not part of the library):
// how fast can one CTA per SM pull data through shared memory with 1-D bulk
// copies (cp.async.bulk + mbarrier) at a given stage size and depth, versus
// plain 16-byte loads?  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_spin(uint64_t *bar, unsigned parity) {
  unsigned ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// each CTA streams a contiguous range in stages of `stage` bytes, `depth` in flight,
// split into `pieces` bulk copies per stage
__global__ void k_tma(const char *src, size_t per_cta, int stage, int depth, int pieces, float *sink, int multi) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const char *base = src + (size_t)blockIdx.x * per_cta;
  const int nst = (int)(per_cta / stage);
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int s) {
    const int sl = s % depth;
    const int pb = stage / pieces;
    if (!multi || multi >= 8) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bars[sl], stage);
        for (int p = 0; p < pieces; ++p)
          bulk_g2s(sm + (size_t)sl * stage + p * pb, base + (size_t)s * stage + p * pb, pb, &bars[sl]);
      }
    } else {
      // piece p issued by lane p of warp 0 (multi=1) or by warp p (multi=2)
      const int who = multi == 1 ? (threadIdx.x < 32 ? (int)threadIdx.x : -1) : ((threadIdx.x & 31) == 0 ? (int)threadIdx.x / 32 : -1);
      if (threadIdx.x == 0) mbar_expect_tx(&bars[sl], stage);
      __syncwarp();
      if (who >= 0 && who < pieces) bulk_g2s(sm + (size_t)sl * stage + who * pb, base + (size_t)s * stage + who * pb, pb, &bars[sl]);
    }
  };
  for (int s = 0; s < depth - 1 && s < nst; ++s) issue(s);
  __syncthreads();
  float acc = 0.f;
  for (int s = 0; s < nst; ++s) {
    const int sl = s % depth;
    if (s + depth - 1 < nst) issue(s + depth - 1);
    if (multi >= 8) mbar_spin(&bars[sl], (s / depth) & 1);
    else mbar_wait(&bars[sl], (s / depth) & 1);
    const float *f = (const float *)(sm + (size_t)sl * stage);
    if (multi == 9) {  // no consumer work at all
    } else {
      for (int i = threadIdx.x; i < stage / 4; i += blockDim.x) acc += f[i];
    }
    __syncthreads();
  }
  if (acc == 123.456f) sink[0] = acc;
}

// cp.async (LDGSTS) ring: every thread copies 16-byte pieces of the stage
__global__ void k_cpa(const char *src, size_t per_cta, int stage, int depth, float *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const char *base = src + (size_t)blockIdx.x * per_cta;
  const int nst = (int)(per_cta / stage);
  auto issue = [&](int s) {
    const int sl = s % depth;
    for (int i = threadIdx.x * 16; i < stage; i += blockDim.x * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (size_t)sl * stage + i)),
                   "l"(base + (size_t)s * stage + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int s = 0; s < depth - 1; ++s) {
    if (s < nst) issue(s);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  float acc = 0.f;
  for (int s = 0; s < nst; ++s) {
    const int sl = s % depth;
    if (s + depth - 1 < nst) issue(s + depth - 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    // groups committed after stage s: depth-1 -> wait until at most depth-1 pending
    switch (depth) {
      case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
      case 4: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
      case 6: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
      default: asm volatile("cp.async.wait_group 7;" ::: "memory"); break;
    }
    __syncthreads();
    const float *f = (const float *)(sm + (size_t)sl * stage);
    for (int i = threadIdx.x; i < stage / 4; i += blockDim.x) acc += f[i];
    __syncthreads();
  }
  if (acc == 123.456f) sink[0] = acc;
}

__global__ void k_ldg(const float4 *src, size_t n4_per_cta, float *sink) {
  const float4 *b = src + (size_t)blockIdx.x * n4_per_cta;
  float acc = 0.f;
  for (size_t i = threadIdx.x; i < n4_per_cta; i += blockDim.x * 4) {
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (i + k * blockDim.x < n4_per_cta) ? __ldcs(b + i + k * blockDim.x) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 123.456f) sink[0] = acc;
}

// all copies issued up front, then waited: are a CTA's bulk copies concurrent?
__global__ void k_burst(const char *src, int copy, int ncopies, unsigned long long *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  const char *base = src + (size_t)blockIdx.x * copy * ncopies;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, copy * ncopies);
    for (int i = 0; i < ncopies; ++i) bulk_g2s(sm + (size_t)i * copy, base + (size_t)i * copy, copy, &bar);
  }
  mbar_wait(&bar, 0);
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main(int argc, char **argv) {
  const size_t total = (size_t)1 << 30;  // 1 GiB
  char *buf;
  float *sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 0, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_burst, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  {
    unsigned long long *d_out;
    cudaMalloc(&d_out, sizeof(unsigned long long) * 1024);
    struct B { int copy, n, grid; };
    for (B b : {B{4096, 1, 1}, B{4096, 8, 1}, B{4096, 32, 1}, B{16384, 1, 1}, B{16384, 8, 1}, B{32768, 4, 1},
                B{65536, 3, 1}, B{4096, 32, 148}, B{16384, 8, 148}, B{65536, 3, 148}}) {
      for (int rep = 0; rep < 3; ++rep) k_burst<<<b.grid, 128, (size_t)b.copy * b.n>>>(buf, b.copy, b.n, d_out);
      cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d_out, sizeof(unsigned long long) * b.grid, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0, sum = 0;
      for (int i = 0; i < b.grid; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
      printf("burst copy=%6d x %2d grid=%3d : mean %8.0f cyc  max %8llu cyc (%s)\n", b.copy, b.n, b.grid,
             (double)sum / b.grid, mx, cudaGetErrorString(cudaGetLastError()));
    }
  }
  struct Cfg { int stage, depth, pieces, ctas_per_sm, multi; };
  std::vector<Cfg> cfgs = {{16384, 4, 1, 1, 0}, {16384, 4, 1, 1, 8}, {16384, 4, 1, 1, 9}, {16384, 8, 1, 1, 9},
                           {8192, 8, 1, 1, 9},  {8192, 8, 1, 1, 8}, {32768, 4, 1, 1, 9}, {16384, 4, 2, 1, 9},
                           {8192, 4, 1, 2, 9},  {4096, 16, 1, 1, 9}};
  for (auto c : cfgs) {
    const int grid = sms * c.ctas_per_sm;
    const size_t per = (total / grid) / c.stage * c.stage;
    const size_t smem = (size_t)c.stage * c.depth;
    if (smem * c.ctas_per_sm > 220 * 1024) continue;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_tma<<<grid, 256, smem>>>(buf, per, c.stage, c.depth, c.pieces, sink, c.multi);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("bulk stage=%6d depth=%2d pieces=%d ctas/sm=%d multi=%d : %7.1f GB/s  (err=%s)\n", c.stage, c.depth,
           c.pieces, c.ctas_per_sm, c.multi, per * grid / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_cpa, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C2 { int stage, depth, cps; };
  for (C2 c : {C2{8192, 4, 2}, C2{16384, 4, 1}, C2{16384, 4, 2}, C2{16384, 6, 2}, C2{8192, 6, 4}, C2{8192, 8, 2},
               C2{32768, 4, 1}, C2{4096, 8, 4}}) {
    const int grid = sms * c.cps;
    const size_t per = (total / grid) / c.stage * c.stage;
    const size_t smem = (size_t)c.stage * c.depth;
    if (smem * c.cps > 220 * 1024) continue;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_cpa<<<grid, 256, smem>>>(buf, per, c.stage, c.depth, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("cp.async stage=%6d depth=%2d ctas/sm=%d : %7.1f GB/s (err=%s)\n", c.stage, c.depth, c.cps,
           per * grid / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  for (int cps : {1, 2, 4, 8}) {
    const int grid = sms * cps;
    const size_t n4 = total / 16 / grid;
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_ldg<<<grid, 256>>>((const float4 *)buf, n4, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    printf("ldg.128 x4 unroll ctas/sm=%d : %7.1f GB/s\n", cps, n4 * 16 * grid / best / 1e6);
  }
  return 0;
}
