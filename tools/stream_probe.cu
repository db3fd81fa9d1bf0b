// Per-SM DRAM -> shared memory streaming rate vs bytes in flight (bulk
// copies completing on mbarriers), the ceiling a weight-streaming (decode)
// GEMM producer can reach.  Each CTA streams its own contiguous region in
// CH-byte chunks through an S-stage ring; one thread issues, the CTA only
// waits for completion (no consumer work).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/stream_probe.cu
//   /tmp/stream_probe
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_stream(const char* src, size_t per_cta, int ch, int stages, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const char* base = src + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / ch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(ch) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf + (size_t)s * ch)),
        "l"(base + (size_t)i * ch), "r"(ch), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int i = 0; i < stages && i < nch; ++i) issue(i);
  for (int i = 0; i < nch; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * ch];
    if (i + stages < nch) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// L2-resident variant: CTA c streams per_cta bytes starting at
// (c * 1 MiB) mod (region - per_cta) of a region small enough to stay in L2
// (warmed by the previous launch), so the copies hit L2.
__global__ void k_stream_l2(const char* src, size_t per_cta, size_t region, int ch, int stages,
                            unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const char* base = src + ((size_t)blockIdx.x << 20) % (region - per_cta);
  const int nch = (int)(per_cta / ch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(ch) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf + (size_t)s * ch)),
        "l"(base + (size_t)i * ch), "r"(ch), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int i = 0; i < stages && i < nch; ++i) issue(i);
  for (int i = 0; i < nch; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * ch];
    if (i + stages < nch) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// Same ring with 2D tensor-map boxes (box_rows x 64 bf16, 128B swizzle):
// CTA c streams row panel c (box_rows rows) along K, or with tiled = 1 the
// map views the bytes as [rows*K/64][64] and the box walks contiguous 16 KB.
__global__ void k_stream2d(const __grid_constant__ CUtensorMap map, int kblocks, int box_rows,
                           int stages, int tiled, int boxes_per_stage, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const int bytes = box_rows * 128 * boxes_per_stage;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  const int nst = kblocks / boxes_per_stage;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    for (int q = 0; q < boxes_per_stage; ++q) {
      const int kb = i * boxes_per_stage + q;
      int c0, c1;
      if (tiled) { c0 = 0; c1 = (blockIdx.x * kblocks + kb) * box_rows; }
      else { c0 = kb * 64; c1 = blockIdx.x * box_rows; }
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(buf + (size_t)s * bytes + q * box_rows * 128)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar[s])), "r"(c0), "r"(c1)
          : "memory");
    }
  };
  for (int i = 0; i < stages && i < nst; ++i) issue(i);
  for (int i = 0; i < nst; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * bytes];
    if (i + stages < nst) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// L2-resident tensor-map boxes: a [rows][K] bf16 matrix of `region` bytes
// viewed 3D as (64 cols, rows, K/64 k-blocks) with box (64, box_rows, kb):
// one instruction brings kb consecutive 128B-swizzled [box_rows][128 B]
// k-block tiles (the grouped GEMM's operand tiles, kb of them at once).
// CTA c walks row panel (c % panels) along K, looping over the matrix.
__global__ void k_stream3d(const __grid_constant__ CUtensorMap map, int kblocks, int box_rows, int kb,
                           int stages, int panels, int iters, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const int bytes = box_rows * 128 * kb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  const int per_panel = kblocks / kb;
  const int nst = per_panel * iters;
  const int row0 = (blockIdx.x % panels) * box_rows;
  auto issue = [&](int i) {
    const int s = i % stages;
    const int k0 = (i % per_panel) * kb;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(buf + (size_t)s * bytes)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar[s])), "r"(0), "r"(row0), "r"(k0)
        : "memory");
  };
  for (int i = 0; i < stages && i < nst; ++i) issue(i);
  for (int i = 0; i < nst; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * bytes];
    if (i + stages < nst) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

// Same L2 stream with `np` issuing threads (lane 0 of warps 0..np-1), warp w
// owning the ring stages s = w (mod np): is the per-copy cost on the
// issuing thread (then more issuers help) or in the SM's TMA unit?
__global__ void k_stream3d_mp(const __grid_constant__ CUtensorMap map, int kblocks, int box_rows,
                              int stages, int panels, int iters, int np, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const int bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0 || w >= np) return;
  unsigned acc = 0;
  const int nst = kblocks * iters;
  const int row0 = (blockIdx.x % panels) * box_rows;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(buf + (size_t)s * bytes)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar[s])), "r"(0), "r"(row0), "r"(i % kblocks)
        : "memory");
  };
  for (int i = w; i < stages && i < nst; i += np) issue(i);
  for (int i = w; i < nst; i += np) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * bytes];
    if (i + stages < nst) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

static void run3d_mp(char* src, unsigned long long* sink, int g, int box_rows, int np) {
  const int K = 2048, kblocks = K / 64;
  const long long rows = (48LL << 20) / (K * 2);
  const int panels = (int)(rows / box_rows);
  CUtensorMap map;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)kblocks};
  cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1}, estr[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box,
                                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode3d failed %d\n", (int)r); return; }
  const int bytes = box_rows * 128, stages = 196608 / bytes, iters = 16;
  if (stages % np) return;  // each issuing warp must own whole ring positions
  const size_t smem = 1024 + (size_t)stages * bytes;
  cudaFuncSetAttribute(k_stream3d_mp, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w = 0; w < 2; ++w) k_stream3d_mp<<<g, 128, smem>>>(map, kblocks, box_rows, stages, panels, iters, np, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) k_stream3d_mp<<<g, 128, smem>>>(map, kblocks, box_rows, stages, panels, iters, np, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double sec = ms / 1e3 / it, per = (double)box_rows * K * 2 * iters;
  printf("L2 MP grid %3d box 64x%3d, %d issuing warps: %7.1f GB/s total, %6.1f per CTA\n", g, box_rows, np,
         per * g / sec / 1e9, per / sec / 1e9);
}

// 4 KB bulk copies (the pair pre-reduction's slot rows) from DRAM with
// `lanes` issuing lanes in each of `nw` warps: lane l of warp w owns ring
// slots s = w*lanes + l (mod stages) -- are several lanes of one warp
// several issuers?
__global__ void k_stream_lanes(const char* src, size_t per_cta, int stages, int lanes, int nw,
                               unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  unsigned char* buf = sm + 1024;
  const int ch = 4096;
  const char* base = src + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / ch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (w >= nw || l >= lanes) return;
  const int me = w * lanes + l, np = nw * lanes;
  unsigned acc = 0;
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(ch) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(buf + (size_t)s * ch)),
        "l"(base + (size_t)i * ch), "r"(ch), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int i = me; i < stages && i < nch; i += np) issue(i);
  for (int i = me; i < nch; i += np) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    acc += buf[(size_t)s * ch];
    if (i + stages < nch) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

static void run_lanes(char* src, unsigned long long* sink, int g, int lanes, int nw) {
  const int stages = 48;  // 192 KB of 4 KB slots
  if (stages % (lanes * nw)) return;  // each issuer must own whole ring positions
  const size_t per_cta = (size_t)4 << 20;
  const size_t smem = 1024 + (size_t)stages * 4096;
  cudaFuncSetAttribute(k_stream_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w = 0; w < 2; ++w) k_stream_lanes<<<g, 256, smem>>>(src, per_cta, stages, lanes, nw, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) k_stream_lanes<<<g, 256, smem>>>(src, per_cta, stages, lanes, nw, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double sec = ms / 1e3 / it;
  printf("4KB bulk grid %3d, %d warps x %d lanes issuing: %7.1f GB/s total, %6.1f per CTA\n", g, nw, lanes,
         per_cta * g / sec / 1e9, per_cta / sec / 1e9);
}

static void run3d(char* src, unsigned long long* sink, int g, int box_rows, int kb, int inflight) {
  const int K = 2048, kblocks = K / 64;
  const long long rows = (48LL << 20) / (K * 2);  // 48 MiB matrix: L2 resident
  const int panels = (int)(rows / box_rows);
  CUtensorMap map;
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)kblocks};
  cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)kb}, estr[3] = {1, 1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box,
                                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode3d failed %d\n", (int)r); return; }
  const int bytes = box_rows * 128 * kb, stages = inflight / bytes;
  if (stages < 1) return;
  const int iters = 16;
  const size_t smem = 1024 + (size_t)stages * bytes;
  cudaFuncSetAttribute(k_stream3d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w = 0; w < 2; ++w) k_stream3d<<<g, 32, smem>>>(map, kblocks, box_rows, kb, stages, panels, iters, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) k_stream3d<<<g, 32, smem>>>(map, kblocks, box_rows, kb, stages, panels, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double sec = ms / 1e3 / it, per = (double)box_rows * K * 2 * iters;
  printf("L2 3D grid %3d box 64x%3dx%d (%6d B/instr, %d stages): %7.1f GB/s total, %6.1f per CTA\n", g, box_rows,
         kb, bytes, stages, per * g / sec / 1e9, per / sec / 1e9);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

static void run2d(char* src, unsigned long long* sink, int g, int box_rows, int K, int stages,
                  int tiled, int bps) {
  CUtensorMap map;
  const long long rows = (long long)g * box_rows;
  cuuint64_t dims[2], strides[1];
  if (tiled) { dims[0] = 64; dims[1] = rows * (K / 64); strides[0] = 128; }
  else { dims[0] = K; dims[1] = rows; strides[0] = (cuuint64_t)K * 2; }
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows}, estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box,
                                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return; }
  const int kblocks = K / 64;
  const size_t smem = 1024 + (size_t)stages * box_rows * 128 * bps;
  cudaFuncSetAttribute(k_stream2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int w = 0; w < 2; ++w) k_stream2d<<<g, 32, smem>>>(map, kblocks, box_rows, stages, tiled, bps, sink);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) k_stream2d<<<g, 32, smem>>>(map, kblocks, box_rows, stages, tiled, bps, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double sec = ms / 1e3 / it, per = (double)box_rows * K * 2;
  printf("2D grid %3d box %3dx64 K %6d %s stages %2d x %d boxes (%6d B in flight): %7.1f GB/s total, %6.1f per CTA\n",
         g, box_rows, K, tiled ? "tiled " : "rowmaj", stages, bps, stages * box_rows * 128 * bps,
         per * g / sec / 1e9, per / sec / 1e9);
}

int main() {
  const size_t total = 1ull << 30;  // 1 GiB source, larger than L2
  char* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_stream_l2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (getenv("PROBE_LANES_ONLY")) {  // 4 KB bulk copies vs issuing lanes/warps only
    for (int nw : {1, 2, 4})
      for (int lanes : {1, 8, 16})
        run_lanes(src, sink, 148, lanes, nw);
    return 0;
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grids[] = {96, 148};
  const int chs[] = {4096, 16384, 32768};
  const int inflight[] = {32768, 65536, 131072, 196608};
  for (int g : grids)
    for (int ch : chs)
      for (int inf : inflight) {
        const int stages = inf / ch;
        if (stages < 1 || stages > 64) continue;
        const size_t per_cta = (size_t)4 << 20;  // 4 MiB per CTA
        if (per_cta * g > total) continue;
        const size_t smem = 1024 + (size_t)stages * ch;
        for (int w = 0; w < 2; ++w) k_stream<<<g, 32, smem>>>(src, per_cta, ch, stages, sink);
        cudaEventRecord(a);
        const int it = 5;
        for (int r = 0; r < it; ++r) k_stream<<<g, 32, smem>>>(src + 0, per_cta, ch, stages, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double sec = ms / 1e3 / it;
        printf("grid %3d  chunk %6d  stages %2d  in-flight %6d B: %7.1f GB/s total, %6.1f GB/s per CTA\n", g,
               ch, stages, stages * ch, per_cta * g / sec / 1e9, per_cta / sec / 1e9);
      }
  // L2 -> SMEM: every CTA streams a 4 MiB window of a 48 MiB region that
  // stays resident in L2 (CTA c starts at (c MiB) mod 44 MiB)
  {
    const size_t region = (size_t)48 << 20;
    for (int g : grids)
      for (int ch : {16384, 32768})
        for (int inf : {65536, 131072, 196608}) {
          const int stages = inf / ch;
          const size_t per_cta = (size_t)4 << 20;
          const size_t smem = 1024 + (size_t)stages * ch;
          for (int w = 0; w < 3; ++w) k_stream_l2<<<g, 32, smem>>>(src, per_cta, region, ch, stages, sink);
          cudaEventRecord(a);
          const int it = 5;
          for (int r = 0; r < it; ++r) k_stream_l2<<<g, 32, smem>>>(src, per_cta, region, ch, stages, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double sec = ms / 1e3 / it;
          printf("L2 grid %3d  chunk %6d  stages %2d  in-flight %6d B: %7.1f GB/s total, %6.1f GB/s per CTA\n", g,
                 ch, stages, stages * ch, per_cta * g / sec / 1e9, per_cta / sec / 1e9);
        }
  }
  for (int g : grids)
    for (int br : {128, 256})
      for (int kb : {1, 2, 4})
        run3d(src, sink, g, br, kb, 196608);
  for (int br : {128, 256})
    for (int np : {1, 2, 4})
      run3d_mp(src, sink, 148, br, np);
  for (int g : grids)
    for (int tiled = 0; tiled < 2; ++tiled) {
      run2d(src, sink, g, 128, 16384, 6, tiled, 1);   // the GEMM's B ring (BN=128)
      run2d(src, sink, g, 128, 16384, 12, tiled, 1);
      run2d(src, sink, g, 256, 8192, 6, tiled, 1);    // BN=256 boxes
      run2d(src, sink, g, 128, 16384, 3, tiled, 4);   // 4 boxes per stage (64 KB stages)
    }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
