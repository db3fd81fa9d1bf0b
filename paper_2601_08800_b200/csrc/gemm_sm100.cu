// gemm_sm100.cu -- K3: persistent grouped GEMM on 5th-gen tensor cores.
//
// D[rows of group g] = A[rows of g] . B_g^T, bf16 operands, fp32 accumulate
// in TMEM, for the expert FFN (the reference's _partial_expert_outputs
// stand-in, sim:535-562, made a real TP-sharded SwiGLU):
//   GEMM1  A = received rows [S_d, h],  B = w13_e [2*I/m, h] -> SwiGLU
//          epilogue (silu(gate) * up, bf16) -> act [S_d, I/m]
//   GEMM2  A = act [S_d, I/m],          B = w2_e [h, I/m]    -> TP partial
// Groups (= experts of this host) are contiguous row segments of A/D.
//
// Structure (one CTA per SM, persistent static tile schedule):
//   warp 0  TMA producer   cp.async.bulk.tensor 2D, 128B swizzle, mbarriers
//   warp 1  MMA issuer     tcgen05.mma.cta_group::1.kind::f16, M=128 N=BN K=16
//   warp 2  TMEM owner     tcgen05.alloc / dealloc (2 x BN fp32 columns)
//   warps 4-7 epilogue     tcgen05.ld 32x32b -> regs -> (SwiGLU) -> global
// Double-buffered TMEM accumulators let the epilogue of tile i overlap the
// MMAs of tile i+1; a STAGES-deep smem ring overlaps TMA with MMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mx_internal.cuh"

namespace mx {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;   // bf16 elements per k-block: 128 B rows, one SWIZZLE_128B atom wide
constexpr int BKB = 128; // bytes per k-block row (64 bf16 or 128 e4m3)
constexpr int NUM_THREADS = 256;      // CTA-pair kernel: 4 epilogue warps
constexpr int NUM_THREADS_1 = 384;    // single-CTA kernel: warps 4..11 = 8 epilogue warps
constexpr int GATHER_THREADS = 64;    // gathered A: warps 0 and 3 issue the row LDGSTS
constexpr int GATHER_LAG = 2;         // stages a gathering thread runs ahead of its arrive

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BKB;
  static constexpr int B_BYTES = BN * BKB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulator buffers
  static constexpr int STAGING = 8 * 32 * 64;  // per epilogue warp: 32 rows x 64 B
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 1024 /*barriers*/ + STAGING;
};

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 4 rows (row coordinates r0..r3, negative = zero fill) x 64 columns into
// 512 contiguous bytes of smem, 128B swizzle applied by the TMA unit.
// 16-byte LDGSTS (L2 only); src_bytes = 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row atoms of
// 1024 B stacked along M/N (SBO = 1024 B), sm100 version bits = 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);  // start address   [0,14)
  d |= (uint64_t)(16 >> 4) << 16;          // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO             [32,46)
  d |= (uint64_t)1 << 46;                  // version = 1     [46,48)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B    [61,64)
  return d;
}
// Instruction descriptor, kind::f16: D f32, A/B bf16, both K-major.
template <int BN>
__device__ __forceinline__ constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
// kind::f8f6f4 with A = B = E4M3 (format code 0), D f32.
template <int BN>
__device__ __forceinline__ constexpr uint32_t idesc_e4m3() {
  return (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_e4m3(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// SiLU with the approximate divide (<= 2 ulp; g very negative: the
// denominator overflows and the quotient is 0, the function's limit).  The
// IEEE-rounded '/' cost the epilogue ~6 us per 32-column chunk on the
// decode tiles and made the prefill GEMM1 epilogue-bound in part: 381 ->
// 367 us at config B (tools/runs/silu_ab.sh; MX_SILU_IEEE keeps it for A/B).
#ifdef MX_SILU_IEEE
__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }
#else
__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }
#endif

// FP8 dequantisation of 32 accumulator columns: v *= row_scale * col_scale[j]
__device__ __forceinline__ void scale_cols(uint32_t (&r)[32], float sa, const float* __restrict__ sb) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 b = __ldg(reinterpret_cast<const float4*>(sb) + i);
    r[4 * i + 0] = __float_as_uint(__uint_as_float(r[4 * i + 0]) * sa * b.x);
    r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) * sa * b.y);
    r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) * sa * b.z);
    r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) * sa * b.w);
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Stage one 32-row x 32-col bf16 chunk (64 B per row, thread = row) in the
// SWIZZLE_64B layout the D tensor map expects (16 B chunk j of row r lives
// at chunk j ^ ((r >> 1) & 3)), then one lane TMA-stores the 32x32 box.
// Rows are complete boxes only; partial boxes use direct stores.
template <int PENDING>  // 1: double-buffered staging, 0: single buffer
__device__ __forceinline__ void stage_store_chunk(unsigned char* stg, const uint32_t (&p)[16],
                                                  int lane, const CUtensorMap* map, int col,
                                                  int row0) {
  if (lane == 0) {  // this buffer's previous store has been read out of smem
    if constexpr (PENDING == 1) tma_store_wait_read1();
    else tma_store_wait_read0();
  }
  __syncwarp();
  unsigned char* rowp = stg + lane * 64;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t addr = smem_u32(rowp + ((j ^ ((lane >> 1) & 3)) << 4));
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(p[4 * j]),
                 "r"(p[4 * j + 1]), "r"(p[4 * j + 2]), "r"(p[4 * j + 3])
                 : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) tma_store_2d(map, stg, col, row0);
}

// w13 rows are interleaved in blocks of 64: packed row 128*b + j is gate row
// 64*b + j, packed row 128*b + 64 + j the matching up row (mx_swiglu_pack_w13).
// A BN-wide SwiGLU tile therefore yields BN/2 outputs; output column c of a
// tile reads gate accumulator column swiglu_gate_col(c) and up column +64.
__device__ __forceinline__ int swiglu_gate_col(int c) { return ((c >> 6) << 7) + (c & 63); }

struct Args {
  void* D;
  const int32_t* a_rows;  // GATHER: source row of every A row (row index table)
  const char* a_base;     // FP8: A rows (lda bytes each), fp32 row scale at byte K
  long long lda;          // FP8: A row stride in bytes
  const float* b_scales;  // FP8: per-B-row (output channel) scales, [G*N]
  int sync_wait, sync_signal;  // fused device barrier (SPMD forward)
  DevView sv;                  // rank view for the fused barrier
  const int32_t* offs;
  const int32_t* cnts;
  const int32_t* b_index;
  int G, N, K, ldd, out_f32;
  long long M_cap;
  // clock probe: CTA 0 records {SM cycles, %globaltimer ns} over its
  // lifetime -- the effective SM clock the GEMM ran at (power capping
  // lowers it under sustained tensor load; bench.py reports it)
  unsigned long long* clk;
  // debug timeline (MX_GEMM_TRACE=1): SM clock per CTA at entry [0], setup
  // done [1], last MMA issued [3], epilogue drained [4], exit [5]; wait
  // cycles [2] [6] [7] in MX_GEMM_WAITSTATS builds
  unsigned long long* trace;
  // decode regime (weight-streaming tiles): `early` -- the group tables and
  // the weights were written long before the predecessor kernel, so the
  // schedule is built and the first stages' B boxes are issued before the
  // PDL wait, which then only gates the A boxes; `trigger` -- let the next
  // kernel's CTAs launch (and do the same) on the SMs this grid leaves idle.
  // Invariant: some kernel between the layout (the tables' producer) and the
  // GEMMs triggers its dependents only at exit (the token dispatch), so the
  // GEMMs cannot start before the layout completed even when every other
  // phase kernel triggers at entry (tests/spmd_check.py "decode regime"
  // caught the cascade: wrong outputs before this rule)
  int early, trigger;
  // GATHER with TMA tile::gather4 (map_a: the source rows, 64 x 1 boxes):
  // 32 four-row gathers per k-block, issued by three threads in parallel
  int gather4;
};
// MX_GEMM_WAITSTATS (compile-time, variant builds only): cycles the
// producer spends waiting for free stages [6], the MMA issuer for a free
// accumulator [7] and for landed stages [2], summed per CTA into the trace
#ifdef MX_GEMM_WAITSTATS
#define WAITSTAT(i, stmt)                                                   \
  do {                                                                      \
    const long long w0_ = clock64();                                        \
    stmt;                                                                   \
    if (args.trace) args.trace[blockIdx.x * 16 + (i)] += clock64() - w0_;    \
  } while (0)
#else
#define WAITSTAT(i, stmt) stmt
#endif
#define GEMM_TRACE(i, cond) \
  do { if (args.trace && (cond)) args.trace[blockIdx.x * 16 + (i)] = clock64(); } while (0)
#define GEMM_TRACE_NS(i, cond) \
  do { if (args.trace && (cond)) args.trace[blockIdx.x * 16 + (i)] = globaltimer_ns(); } while (0)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Tile t -> (group, m-block, n-block) through the per-group tile prefix.
__device__ __forceinline__ void decode_tile(int t, const int* s_tstart, int G, int nN, int* g,
                                            int* mb, int* nb) {
  int lo = 0, hi = G - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_tstart[mid] <= t) lo = mid; else hi = mid - 1;
  }
  const int r = t - s_tstart[lo];
  *g = lo;
  *mb = r / nN;
  *nb = r % nN;
}

template <int BN, bool SWIGLU, bool GATHER, bool FP8>
__global__ void __launch_bounds__(NUM_THREADS_1, 1)
k_grouped_gemm(const __grid_constant__ CUtensorMap map_a,
               const __grid_constant__ CUtensorMap map_b,
               const __grid_constant__ CUtensorMap map_d, Args args) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  unsigned char* staging = smem + C::STAGES * C::STAGE_BYTES + 1024;  // 1 KiB aligned
  __shared__ uint32_t s_tmem;
  __shared__ int s_tstart[MX_EMAX + 1];
  __shared__ int s_off[MX_EMAX];
  __shared__ int s_cnt[MX_EMAX];
  __shared__ __align__(8) uint64_t s_done;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  GEMM_TRACE(0, threadIdx.x == 0);
  GEMM_TRACE_NS(8, threadIdx.x == 0);
  if (threadIdx.x == 0) {  // descriptors do not depend on earlier kernels
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    if (!args.out_f32) tma_prefetch(&map_d);
  }
  constexpr int KE = FP8 ? 128 : 64;  // elements per k-block (128 B)
  const int G = args.G, nN = args.N / BN, kblocks = args.K / KE;

  // group offsets/counts -> smem (parallel loads), then the per-group tile
  // prefix by one warp-scan pass (G <= MX_EMAX); no per-tile global reads
  const bool early = !GATHER && !FP8 && args.early && !args.sync_wait;
  if (!early) {
    pdl_wait();  // group offsets/counts and A are written by earlier kernels
    if (args.sync_wait) grid_wait(args.sv);  // peers' rows have landed
  }
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    s_off[g] = args.offs[g];
    s_cnt[g] = args.cnts[g];
  }
  __syncthreads();
  if (warp == 3) {
    int carry = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int tiles = g < G ? ((s_cnt[g] + BM - 1) / BM) * nN : 0;
      int incl = tiles;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (g < G) s_tstart[g] = carry + incl - tiles;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_tstart[G] = carry;
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      // GATHER: the B TMA arrive + one arrive per gathering thread
      mbar_init(&full[s], GATHER && !args.gather4 ? 1 + GATHER_THREADS : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // one arrive per epilogue warp
    }
    mbar_init(&s_done, 8);  // epilogue warps: every TMEM read and store drained
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const int total_tiles = s_tstart[G];
  if (args.trigger) pdl_trigger();
  const bool probe = args.clk && blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long clk0 = probe ? clock64() : 0, gt0 = probe ? globaltimer_ns() : 0;
  GEMM_TRACE(1, threadIdx.x == 0);

  if (warp == 0 || (GATHER && (warp == 3 || (args.gather4 && warp == 2)))) {
    if (GATHER && args.gather4) {
      if (lane == 0) {
        // ===== gather4 producers (lane 0 of warps 0, 2, 3): each k-block's
        // A tile = 32 tile::gather4 copies of 4 rows x 128 B (the TMA unit
        // applies the 128B swizzle by smem address, as for a 128-row box);
        // warp w issues gathers [q0, q1) -- one issuing thread capped the
        // feed (round 1: 964 us for GEMM1) -- warp 0 also the B box and the
        // stage's one arrival (expect_tx of A + B: the other issuers' copies
        // may complete first, the tx-count then dips below zero meanwhile).
        const int w = warp == 0 ? 0 : warp == 2 ? 1 : 2;
        const int q0 = (32 * w) / 3, q1 = (32 * (w + 1)) / 3;  // 0-10, 10-21, 21-32
        int stage = 0;
        uint32_t phase = 0;
        for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
          int g, mb, nb;
          decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
          const int bg = args.b_index ? args.b_index[g] : g;
          const int b_row = bg * args.N + nb * BN;
          const int cnt = s_cnt[g];
          int rows[11][4];
#pragma unroll
          for (int q = 0; q < 11; ++q)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int r_local = mb * BM + 4 * (q0 + q) + j;
              rows[q][j] = (q0 + q < q1 && r_local < cnt)
                               ? args.a_rows[(long long)s_off[g] + r_local] : -1;
            }
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (w == 0) {
              mbar_expect_tx(&full[stage], C::STAGE_BYTES);
              tma_load_2d(sB + stage * C::B_BYTES, &map_b, &full[stage], kb * KE, b_row);
            }
            const uint32_t dst = smem_u32(sA + stage * C::A_BYTES);
#pragma unroll
            for (int q = 0; q < 11; ++q)
              if (q0 + q < q1)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::"
                    "complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
                        dst + (q0 + q) * 512),
                    "l"(reinterpret_cast<uint64_t>(&map_a)), "r"(smem_u32(&full[stage])),
                    "r"(kb * KE), "r"(rows[q][0]), "r"(rows[q][1]), "r"(rows[q][2]), "r"(rows[q][3])
                    : "memory");
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    } else if constexpr (GATHER) {
      // ===== gathering producer (warps 0 and 3): A rows come from an
      // arbitrary row table (token rows of x / XBUF), so they are brought
      // with 16 B LDGSTS into the 128B-swizzled layout the UMMA descriptor
      // expects (row r at r*128, chunk c at (c ^ (r & 7)) * 16); B by TMA.
      // Thread pt owns rows pt and pt + 64.  LDGSTS writes are generic-proxy:
      // each thread waits for its group GATHER_LAG stages later, fences to
      // the async proxy and only then arrives on the stage's full barrier.
      const int pt = (warp == 0 ? 0 : 32) + lane;
      const char* abase = args.a_base;
      const long long lda = args.lda;
      int stage = 0;
      uint32_t phase = 0;
      int issued = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int g, mb, nb;
        decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
        const int bg = args.b_index ? args.b_index[g] : g;
        const int b_row = bg * args.N + nb * BN;
        const int cnt = s_cnt[g];
        const char* src[2];
        int sz[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r_local = mb * BM + pt + 64 * h;
          const int row = r_local < cnt ? args.a_rows[(long long)s_off[g] + r_local] : -1;
          src[h] = row >= 0 ? abase + (long long)row * lda : abase;
          sz[h] = row >= 0 ? 16 : 0;
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (pt == 0) {
            mbar_expect_tx(&full[stage], C::B_BYTES);
            tma_load_2d(sB + stage * C::B_BYTES, &map_b, &full[stage], kb * KE, b_row);
          }
          const uint32_t dst = smem_u32(sA + stage * C::A_BYTES);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = pt + 64 * h;
            const char* sp = src[h] + kb * 128;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              cp_async16(dst + r * 128 + ((c ^ (r & 7)) << 4), sp + c * 16, sz[h]);
          }
          cp_async_commit();
          if (issued >= GATHER_LAG) {
            cp_async_wait<GATHER_LAG>();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(&full[(stage + C::STAGES - GATHER_LAG) % C::STAGES]);
          }
          ++issued;
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
      cp_async_wait<0>();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int j = (issued < GATHER_LAG ? issued : GATHER_LAG); j >= 1; --j)
        mbar_arrive(&full[(stage + C::STAGES - j) % C::STAGES]);
    } else if (lane == 0) {
      // ===== TMA producer
      // early start: the first (fresh, empty) stages get their B boxes
      // before the PDL wait -- expect_tx without an arrival; the stage's one
      // arrival comes with its A box after the wait
      int pre = 0;
      if (early) {
        for (int t = blockIdx.x; t < total_tiles && pre < C::STAGES; t += gridDim.x) {
          int g, mb, nb;
          decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
          const int bg = args.b_index ? args.b_index[g] : g;
          for (int kb = 0; kb < kblocks && pre < C::STAGES; ++kb, ++pre) {
            asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(
                             smem_u32(&full[pre])), "r"((uint32_t)C::B_BYTES) : "memory");
            tma_load_2d(sB + pre * C::B_BYTES, &map_b, &full[pre], kb * KE, bg * args.N + nb * BN);
          }
        }
        pdl_wait();  // A rows are written by the predecessor
      }
      int stage = 0, issued = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int g, mb, nb;
        decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
        const int a_row = s_off[g] + mb * BM;
        const int bg = args.b_index ? args.b_index[g] : g;
        const int b_row = bg * args.N + nb * BN;
        for (int kb = 0; kb < kblocks; ++kb, ++issued) {
          WAITSTAT(6, mbar_wait(&empty[stage], phase ^ 1));
          if (issued < pre) {
            mbar_expect_tx(&full[stage], C::A_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &map_a, &full[stage], kb * KE, a_row);
          } else {
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &map_a, &full[stage], kb * KE, a_row);
            tma_load_2d(sB + stage * C::B_BYTES, &map_b, &full[stage], kb * KE, b_row);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (single thread)
      constexpr uint32_t idesc = FP8 ? idesc_e4m3<BN>() : idesc_bf16<BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        WAITSTAT(7, mbar_wait(&tempty[acc], acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          WAITSTAT(2, mbar_wait(&full[stage], phase));
          tc_fence_after();
          const uint64_t adesc = smem_desc_sw128(smem_u32(sA + stage * C::A_BYTES));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + stage * C::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            // +32 B per MMA (K=16 bf16 / K=32 e4m3) inside the 128 B swizzle atom (>>4 -> +2)
            if constexpr (FP8) mma_e4m3(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
            else mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
          }
          mma_commit(&empty[stage]);  // frees the smem slot when the MMAs retire
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      GEMM_TRACE(3, true);
    }
  } else if (warp >= 4) {
    // ===== epilogue: thread = accumulator row (TMEM lane); two warps per lane
    // quarter split the tile's columns (warps 4-7: first half, 8-11: second)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;
    const int row_in_tile = q * 32 + lane;
    unsigned char* my_stage = staging + (warp - 4) * (32 * 64);
    constexpr int buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      int g, mb, nb;
      decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
      const int cnt = s_cnt[g];
      const int r_local = mb * BM + row_in_tile;
      const long long row = (long long)s_off[g] + r_local;
      // rows past M_cap (a host over capacity, flagged by the layout) are
      // never written: TMA drops them from full boxes, direct stores skip them
      const bool valid = r_local < cnt && row < args.M_cap;
      // the warp's 32 rows all belong to this group -> TMA box store
      const bool full_box = !args.out_f32 && (mb * BM + q * 32 + 31) < cnt;
      const int row0 = s_off[g] + mb * BM + q * 32;
      // FP8: per-row activation scale (row tail) and the group's weight scales
      float sa = 1.f;
      int bg = g;
      if constexpr (FP8) {
        bg = args.b_index ? args.b_index[g] : g;
        if (valid) sa = *reinterpret_cast<const float*>(args.a_base + row * args.lda + args.K);
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
      // a warp whose 32 rows all lie past the group's rows (short tiles:
      // decode, expert tails) has nothing to store: skip its TMEM reads and math
      const bool warp_idle = mb * BM + q * 32 >= cnt;
      if (warp_idle) {
      } else if constexpr (SWIGLU) {
        // gate/up accumulator columns interleaved in blocks of 64 (w13 packing)
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.D) + row * args.ldd + nb * (BN / 2);
#pragma unroll 1
        for (int c = half * (BN / 4); c < (half + 1) * (BN / 4); c += 32) {
          const int gc = swiglu_gate_col(c);
          uint32_t gr[32], ur[32];
          tmem_ld32(tbase + gc, gr);
          tmem_ld32(tbase + gc + 64, ur);
          tmem_wait_ld();
          if constexpr (FP8) {
            scale_cols(gr, sa, args.b_scales + (size_t)bg * args.N + nb * BN + gc);
            scale_cols(ur, sa, args.b_scales + (size_t)bg * args.N + nb * BN + gc + 64);
          }
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = silu(__uint_as_float(gr[2 * i])) * __uint_as_float(ur[2 * i]);
            const float a1 = silu(__uint_as_float(gr[2 * i + 1])) * __uint_as_float(ur[2 * i + 1]);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
            packed[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if (full_box) {
            stage_store_chunk<0>(my_stage + buf * 2048, packed, lane, &map_d, nb * (BN / 2) + c, row0);
          } else if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          }
        }
      } else {
#pragma unroll 1
        for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + c, r);
          tmem_wait_ld();
          if constexpr (FP8) scale_cols(r, sa, args.b_scales + (size_t)bg * args.N + nb * BN + c);
          if (args.out_f32) {
            if (valid) {
              float4* dst = reinterpret_cast<float4*>(static_cast<float*>(args.D) + row * args.ldd +
                                                      nb * BN + c);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                     __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
            }
          } else {
            uint32_t packed[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              __nv_bfloat162 b2 =
                  __floats2bfloat162_rn(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
              packed[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
            if (full_box) {
              stage_store_chunk<0>(my_stage + buf * 2048, packed, lane, &map_d, nb * BN + c, row0);
            } else if (valid) {
              uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.D) +
                                                    row * args.ldd + nb * BN + c);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) {
      tma_store_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    GEMM_TRACE(4, warp == 4 && lane == 0);
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_done);
  }

  // End of work: the role branches run single lanes (producer, MMA issuer,
  // store waits), and the CTA barrier alone was measured not to hold the
  // non-epilogue warps until the epilogue finished (tools/decode_gemm_bench.py
  // --trace: thread 0 left it before the last MMA was issued).  Warps 0-3
  // wait on the epilogue's mbarrier, so the TMEM dealloc, the clock probe and
  // the fused-barrier signal all follow the last TMEM read and bulk store.
  if (warp < 4) mbar_wait(&s_done, 0);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  GEMM_TRACE(5, threadIdx.x == 0);
  GEMM_TRACE_NS(9, threadIdx.x == 0);
  if (probe) {
    args.clk[0] = clock64() - clk0;
    args.clk[1] = globaltimer_ns() - gt0;
  }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
  if (args.sync_signal) grid_signal(args.sv);  // D complete (bulk stores drained): publish
}

// ------------------------------------------------------------ CTA pair (2SM)
// tcgen05.mma.cta_group::2, M=256 x N=256 tiles: CTA rank c of the cluster
// pair loads A rows [c*128, c*128+128) and B rows [c*128, c*128+128) of the
// tile into its own shared memory; the leader (rank 0) issues every MMA,
// which reads both CTAs' operands, and each CTA's TMEM holds its 128 rows x
// 256 columns of the accumulator.  Per SM, a 512-cycle k-block needs 32 KB
// of operands instead of 48 KB (M=128 single-CTA) -- the single-CTA kernel
// is bound by that L2->SM feed (GEMM1 ran at the same time at 1.45 and
// 1.97 GHz, profiles/r01).
constexpr int P_STAGES = 6;
constexpr int P_A = 128 * BKB;              // per CTA: 128 A rows
constexpr int P_B = 128 * BKB;              // per CTA: 128 of the 256 B rows
constexpr int P_STAGE = P_A + P_B;
constexpr int P_STAGING = 4 * 2 * 32 * 64;
constexpr int P_SMEM = P_STAGES * P_STAGE + 1024 + 1024 + P_STAGING;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(saddr), "r"(rank));
  return out;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load that completes on the pair leader's mbarrier (same offset)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint64_t* bar,
                                                 int c0, int c1) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
      : "memory");
}

template <bool SWIGLU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
k_grouped_gemm_pair(const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_d, Args args) {
  constexpr int BN = 256, PM = 256;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sA = smem;
  unsigned char* sB = smem + P_STAGES * P_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2] (leader's are used)
  unsigned char* staging = smem + P_STAGES * P_STAGE + 1024;
  __shared__ uint32_t s_tmem;
  __shared__ int s_tstart[MX_EMAX + 1];
  __shared__ int s_off[MX_EMAX];
  __shared__ int s_cnt[MX_EMAX];
  __shared__ __align__(8) uint64_t s_done;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const int G = args.G, nN = args.N / BN, kblocks = args.K / BK;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  pdl_wait();  // group offsets/counts and A are written by earlier kernels
  if (args.sync_wait) grid_wait(args.sv);  // peers' rows have landed
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    s_off[g] = args.offs[g];
    s_cnt[g] = args.cnts[g];
  }
  __syncthreads();
  if (warp == 3) {
    int carry = 0;
    for (int base = 0; base < G; base += 32) {
      const int g = base + lane;
      const int tiles = g < G ? ((s_cnt[g] + PM - 1) / PM) * nN : 0;
      int incl = tiles;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (g < G) s_tstart[g] = carry + incl - tiles;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_tstart[G] = carry;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_d);
  }
  if (warp == 1 && lane == 0) {
    for (int st = 0; st < P_STAGES; ++st) {
      mbar_init(&full[st], 1);   // leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&empty[st], 1);  // one multicast commit per use
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy)
    }
    mbar_init(&s_done, 4);  // this CTA's epilogue warps, work drained
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(2 * BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const int total_tiles = s_tstart[G];

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs): own half of A rows and of B rows
      int stage = 0;
      uint32_t phase = 0;
      for (int t = pair; t < total_tiles; t += npairs) {
        int g, mb, nb;
        decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
        const int a_row = s_off[g] + mb * PM + (int)crank * 128;
        const int b_row = g * args.N + nb * BN + (int)crank * 128;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader) mbar_expect_tx(&full[stage], 2 * P_STAGE);
          tma_load_2d_pair(sA + stage * P_A, &map_a, &full[stage], kb * BK, a_row);
          tma_load_2d_pair(sB + stage * P_B, &map_b, &full[stage], kb * BK, b_row);
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===== MMA issuer (leader CTA, single thread), M=256 N=256 K=16
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                 ((uint32_t)(PM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = pair; t < total_tiles; t += npairs) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t adesc = smem_desc_sw128(smem_u32(sA + stage * P_A));
          const uint64_t bdesc = smem_desc_sw128(smem_u32(sB + stage * P_B));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
          mma_commit_pair(&empty[stage]);  // frees the slot in both CTAs
          if (++stage == P_STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair(&tfull[acc]);  // both CTAs' accumulators ready
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue (both CTAs): thread = row of this CTA's 128-row half
    const int q = warp & 3;
    const int row_in_half = q * 32 + lane;
    unsigned char* my_stage = staging + q * (2 * 32 * 64);
    const uint32_t tempty_leader0 = map_to_rank(smem_u32(&tempty[0]), 0);
    int buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = pair; t < total_tiles; t += npairs) {
      int g, mb, nb;
      decode_tile(t, s_tstart, G, nN, &g, &mb, &nb);
      const int cnt = s_cnt[g];
      const int r_local = mb * PM + (int)crank * 128 + row_in_half;
      const long long row = (long long)s_off[g] + r_local;
      // rows past M_cap (a host over capacity, flagged by the layout) are
      // never written: TMA drops them from full boxes, direct stores skip them
      const bool valid = r_local < cnt && row < args.M_cap;
      const bool full_box = (mb * PM + (int)crank * 128 + q * 32 + 31) < cnt;
      const int row0 = s_off[g] + mb * PM + (int)crank * 128 + q * 32;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
      if constexpr (SWIGLU) {
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(args.D) + row * args.ldd + nb * (BN / 2);
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          const int gc = swiglu_gate_col(c);
          uint32_t gr[32], ur[32];
          tmem_ld32(tbase + gc, gr);
          tmem_ld32(tbase + gc + 64, ur);
          tmem_wait_ld();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float a0 = silu(__uint_as_float(gr[2 * i])) * __uint_as_float(ur[2 * i]);
            const float a1 = silu(__uint_as_float(gr[2 * i + 1])) * __uint_as_float(ur[2 * i + 1]);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(a0, a1);
            packed[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if (full_box) {
            stage_store_chunk<1>(my_stage + buf * 2048, packed, lane, &map_d, nb * (BN / 2) + c, row0);
            buf ^= 1;
          } else if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(out + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + c, r);
          tmem_wait_ld();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 b2 =
                __floats2bfloat162_rn(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
            packed[i] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if (full_box) {
            stage_store_chunk<1>(my_stage + buf * 2048, packed, lane, &map_d, nb * BN + c, row0);
            buf ^= 1;
          } else if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(args.D) +
                                                  row * args.ldd + nb * BN + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);  // leader's tempty[acc]
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) {
      tma_store_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&s_done);
  }

  // as in k_grouped_gemm: the other warps wait for this CTA's epilogue
  if (warp < 4) mbar_wait(&s_done, 0);
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
  }
  if (args.sync_signal) grid_signal(args.sv);
}

// ------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static int make_map(CUtensorMap* map, const void* base, long long rows, int cols, int box_rows,
                    int box_cols = BK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                    bool fp8 = false, long long row_bytes = 0) {
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return MX_ERR_CUDA; }
  const int esz = fp8 ? 1 : 2;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(row_bytes ? row_bytes : (long long)cols * esz)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%d", (int)r, rows, cols);
    return MX_ERR_CUDA;
  }
  return MX_OK;
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Persistent CTAs per grouped GEMM: every SM, or MX_GEMM_CTAS when set (leaves
// SMs free for a concurrent micro-batch's communication kernels).
static int gemm_ctas() {
  static int n = 0;
  if (!n) {
    n = sm_count();
    const char* e = getenv("MX_GEMM_CTAS");
    if (e && atoi(e) > 0 && atoi(e) < n) n = atoi(e);
  }
  return n;
}

template <int BN, bool SWIGLU, bool GATHER, bool FP8 = false>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                  const Args& a, long long max_tiles, cudaStream_t s) {
  auto kern = k_grouped_gemm<BN, SWIGLU, GATHER, FP8>;
  static bool attr = false;
  if (!attr) {
    MX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM));
    attr = true;
  }
  long long grid = gemm_ctas();
  if (max_tiles < grid) grid = max_tiles < 1 ? 1 : max_tiles;
  pdl_launch(kern, (int)grid, NUM_THREADS_1, Cfg<BN>::SMEM, s, ma, mb, md, a);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

template <bool SWIGLU>
static int launch_pair(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
                       const Args& a, long long max_tiles, cudaStream_t s) {
  auto kern = k_grouped_gemm_pair<SWIGLU>;
  static bool attr = false;
  if (!attr) {
    MX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM));
    attr = true;
  }
  long long pairs = gemm_ctas() / 2;
  if (max_tiles < pairs) pairs = max_tiles < 1 ? 1 : max_tiles;
  pdl_launch(kern, (int)(2 * pairs), NUM_THREADS, P_SMEM, s, ma, mb, md, a);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

// MX_GEMM_TRACE=1: per-CTA phase timestamps of the last grouped GEMM
// (tools/decode_gemm_bench.py --trace reads them with mx_debug_gemm_trace)
static unsigned long long* g_trace = nullptr;
static unsigned long long* gemm_trace_buf() {
  static const bool on = [] { const char* e = getenv("MX_GEMM_TRACE"); return e && e[0] == '1'; }();
  if (on && !g_trace) {
    if (cudaMalloc(&g_trace, 1024 * 16 * 8) != cudaSuccess) g_trace = nullptr;
    else cudaMemset(g_trace, 0, 1024 * 16 * 8);
  }
  return on ? g_trace : nullptr;
}

// 0: never, 1: auto (dense single-group GEMMs, e.g. the shared expert),
// 2: always.  Measured (tools/gemm_bench.py): the pair kernel wins on dense
// shapes (1580 vs 1482 TF/s at 16384x4096x4096) but loses on ragged experts
// (256-row tiles pad ~25% of 512+-22-row experts vs ~12% with 128 rows).
static int pair_mode() {
  static const int v = [] {
    const char* e = getenv("MX_GEMM_PAIR");
    return e ? atoi(e) : 1;
  }();
  return v;
}
static bool use_pair(int G, long long M_total) {
  const int mode = pair_mode();
  return mode == 2 || (mode == 1 && G == 1 && M_total >= 512);
}

}  // namespace gemm

int grouped_gemm(const void* A, const void* B, void* D, int out_dtype, const int32_t* offs,
                 const int32_t* cnts, const int32_t* b_index, int G, long long M_total,
                 long long M_cap, int N, int K, int swiglu, cudaStream_t s,
                 const int32_t* a_rows, long long a_src_rows, const DevView* sync) {
  using namespace gemm;
  if (G < 1 || G > MX_EMAX) { set_error("grouped_gemm: G=%d outside [1, %d]", G, MX_EMAX); return MX_ERR_UNSUPPORTED; }
  if (K % BK != 0 || N % 128 != 0) { set_error("grouped_gemm: K %% 64 and N %% 128 must be 0 (K=%d N=%d)", K, N); return MX_ERR_UNSUPPORTED; }
  if (swiglu && (N % 256 != 0 || out_dtype != MX_BF16)) { set_error("grouped_gemm: SwiGLU needs N %% 256 == 0 and bf16 out"); return MX_ERR_UNSUPPORTED; }
  if (out_dtype != MX_BF16 && out_dtype != MX_F32) { set_error("grouped_gemm: out dtype"); return MX_ERR_UNSUPPORTED; }
  if (M_cap < 1) return MX_OK;
  // BN = 256 unless N forbids it -- or the GEMM is weight-streaming (decode:
  // at most 64 rows per group on average), where the finer 128-column tiles
  // spread the weight reads over more CTAs (a 128-wide SwiGLU tile holds one
  // 64-row gate block and its up block)
  const bool small_m = M_cap <= 64LL * G;
  const int bn = (N % 256 == 0 && !small_m) ? 256 : 128;
  CUtensorMap ma, mb, md;
  memset(&md, 0, sizeof(md));
  const bool gather = a_rows != nullptr;

  // B rows: every group's N rows (b_index may address any of them)
  long long b_rows = (long long)G * N;
  int rc = make_map(&mb, B, b_rows, K, bn);
  if (rc) return rc;
  // gathered A: LDGSTS through a_rows (no tensor map), or (MX_GATHER4=1)
  // tile::gather4 through a 64 x 1-row box map over the source rows
  const char* g4_env = getenv("MX_GATHER4");  // read per call (tests toggle it)
  const bool g4 = g4_env && g4_env[0] == '1';
  if (gather && g4) { if ((rc = make_map(&ma, A, a_src_rows, K, 1))) return rc; }
  else if (gather) ma = mb;
  else if ((rc = make_map(&ma, A, M_cap, K, BM))) return rc;
  if (out_dtype == MX_BF16) {  // 32x32 output boxes, 64 B swizzle (staged epilogue)
    rc = make_map(&md, D, M_cap, swiglu ? N / 2 : N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  Args a{};
  if (sync) {
    a.sv = *sync; a.sync_wait = sync->sync_wait; a.sync_signal = sync->sync_signal;
    a.clk = at<unsigned long long>(*sync, sync->rank, sync->off.stamps) + (swiglu ? 56 : 58);
  }
  a.trace = gemm_trace_buf();
  // decode regime: start early (B boxes before the PDL wait), and let GEMM2
  // start early behind GEMM1 (MX_GEMM_EARLY=0 disables, for A/B runs)
  static const bool early_on = [] { const char* e = getenv("MX_GEMM_EARLY"); return !(e && e[0] == '0'); }();
  static const bool early_all = [] { const char* e = getenv("MX_GEMM_EARLY_ALL"); return e && e[0] == '1'; }();
  // multi-GPU prefill too: the next GEMM's CTAs fill the SMs of the previous
  // kernel's last wave (N=4: EP4 0.2922 -> 0.2886 ms, TP2xEP2 0.3165 ->
  // 0.3117; N=2 -0.25%, N=1 neutral -- profiles/r02_early_all_*)
  const bool spmd = sync && sync->W > 1;
  a.early = early_on && (small_m || early_all || spmd) && !gather;
  a.trigger = a.early && (swiglu || (sync && sync->early));
  a.D = D; a.offs = offs; a.cnts = cnts; a.b_index = b_index; a.a_rows = a_rows;
  if (gather) { a.a_base = static_cast<const char*>(A); a.lda = (long long)K * 2; a.gather4 = g4; }
  a.G = G; a.N = N; a.K = K; a.ldd = swiglu ? N / 2 : N; a.out_f32 = out_dtype == MX_F32;
  a.M_cap = M_cap;
  // upper bound on tiles (host does not know the per-group counts)
  const long long max_tiles = ((M_total + BM - 1) / BM + G) * (N / bn);
  if (gather) {
    if (bn == 256) return swiglu ? launch<256, true, true>(ma, mb, md, a, max_tiles, s)
                                 : launch<256, false, true>(ma, mb, md, a, max_tiles, s);
    return swiglu ? launch<128, true, true>(ma, mb, md, a, max_tiles, s)
                  : launch<128, false, true>(ma, mb, md, a, max_tiles, s);
  }
  if (bn == 256 && out_dtype == MX_BF16 && use_pair(G, M_total)) {
    // CTA-pair kernel: A box 128 rows (each CTA its half of the 256-row tile),
    // B box 128 rows (each CTA half of the 256 output columns)
    CUtensorMap mb2;
    rc = make_map(&mb2, B, b_rows, K, 128);
    if (rc) return rc;
    const long long pair_tiles = ((M_total + 255) / 256 + G) * (N / 256);
    return swiglu ? launch_pair<true>(ma, mb2, md, a, pair_tiles, s)
                  : launch_pair<false>(ma, mb2, md, a, pair_tiles, s);
  }
  if (bn == 256) return swiglu ? launch<256, true, false>(ma, mb, md, a, max_tiles, s)
                               : launch<256, false, false>(ma, mb, md, a, max_tiles, s);
  return swiglu ? launch<128, true, false>(ma, mb, md, a, max_tiles, s)
                : launch<128, false, false>(ma, mb, md, a, max_tiles, s);
}

// e4m3 x e4m3 -> f32 grouped GEMM with per-row activation scales (fp32 at
// byte K of every A row, rows lda bytes apart) and per-output-channel weight
// scales; D = bf16 (optionally SwiGLU).  The dequantised product equals
// sum_k (qa*sa) (qb*sb) exactly as the CPU replica computes it.
int grouped_gemm_fp8(const void* A, long long lda, const void* B, const float* b_scales, void* D,
                     const int32_t* offs, const int32_t* cnts, const int32_t* b_index, int G,
                     long long M_total, long long M_cap, int N, int K, int swiglu, cudaStream_t s,
                     const DevView* sync) {
  using namespace gemm;
  if (G < 1 || G > MX_EMAX) { set_error("grouped_gemm_fp8: G=%d outside [1, %d]", G, MX_EMAX); return MX_ERR_UNSUPPORTED; }
  if (K % 128 != 0 || N % 256 != 0) { set_error("grouped_gemm_fp8: K %% 128 and N %% 256 must be 0 (K=%d N=%d)", K, N); return MX_ERR_UNSUPPORTED; }
  if (lda < K + 4 || lda % 16 != 0) { set_error("grouped_gemm_fp8: lda must hold K bytes + fp32 scale, 16 B aligned"); return MX_ERR_UNSUPPORTED; }
  if (M_cap < 1) return MX_OK;
  CUtensorMap ma, mb, md;
  int rc = make_map(&ma, A, M_cap, K, BM, 128, CU_TENSOR_MAP_SWIZZLE_128B, true, lda);
  if (rc) return rc;
  rc = make_map(&mb, B, (long long)G * N, K, 256, 128, CU_TENSOR_MAP_SWIZZLE_128B, true);
  if (rc) return rc;
  rc = make_map(&md, D, M_cap, swiglu ? N / 2 : N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  Args a{};
  if (sync) {
    a.sv = *sync; a.sync_wait = sync->sync_wait; a.sync_signal = sync->sync_signal;
    a.clk = at<unsigned long long>(*sync, sync->rank, sync->off.stamps) + (swiglu ? 60 : 62);
  }
  a.D = D; a.offs = offs; a.cnts = cnts; a.b_index = b_index;
  a.a_base = static_cast<const char*>(A); a.lda = lda; a.b_scales = b_scales;
  a.G = G; a.N = N; a.K = K; a.ldd = swiglu ? N / 2 : N; a.out_f32 = 0;
  a.M_cap = M_cap;
  const long long max_tiles = ((M_total + BM - 1) / BM + G) * (N / 256);
  return swiglu ? launch<256, true, false, true>(ma, mb, md, a, max_tiles, s)
                : launch<256, false, false, true>(ma, mb, md, a, max_tiles, s);
}

// fp8 experts of one rank (BASELINE config C): e4m3 GEMM1 + SwiGLU -> bf16
// act -> per-row e4m3 re-quantisation -> e4m3 GEMM2 -> bf16 TP partial; the
// shared expert runs the same two GEMMs on the group's own tokens (one
// "group" of T rows) into part_s, which the combine adds.
int launch_expert_fp8(const DevView& v, const mx_expert_params& ep, int stage, cudaStream_t s) {
  const int e0 = first_expert(v.group, v.n, v.E), e1 = first_expert(v.group + 1, v.n, v.E);
  const int El = e1 - e0;
  const int32_t* offs = at<int32_t>(v, v.rank, v.off.exp_off) + e0;
  const int32_t* cnts = at<int32_t>(v, v.rank, v.off.exp_cnt) + e0;
  const int32_t* sh = at<int32_t>(v, v.rank, v.off.sh_meta);
  const int* host_rows = at<int>(v, v.rank, v.off.host_rows) + v.group;
  const bool shared = v.Is_t && v.T > 0;
  // fused barrier: the first GEMM of the stage waits, the last one signals
  DevView first = v, last = v, none = v;
  first.sync_signal = 0;
  last.sync_wait = 0;
  none.sync_wait = none.sync_signal = 0;
  const bool routed_first = El > 0;
  int rc = MX_OK;
  if (stage != 2) {
    if (El > 0) {
      rc = grouped_gemm_fp8(at<char>(v, v.rank, v.off.recv), v.wrow, ep.w13, ep.w13_scale,
                            at<char>(v, v.rank, v.off.act), offs, cnts, nullptr, El, v.cap, v.cap,
                            2 * v.I_t, v.h, 1, s, &first);
      if (rc) return rc;
      rc = quant_rows_e4m3(at<char>(v, v.rank, v.off.act), v.I_t, at<char>(v, v.rank, v.off.actq),
                           v.I_t + 16, v.cap, host_rows, v.I_t, s);
      if (rc) return rc;
    }
    if (shared) {
      rc = grouped_gemm_fp8(at<char>(v, v.rank, v.off.xq), v.wrow, ep.w13_shared, ep.w13_shared_scale,
                            at<char>(v, v.rank, v.off.act_s), sh, sh + 1, nullptr, 1, v.T, v.T,
                            2 * v.Is_t, v.h, 1, s, routed_first ? &none : &first);
      if (rc) return rc;
      rc = quant_rows_e4m3(at<char>(v, v.rank, v.off.act_s), v.Is_t,
                           at<char>(v, v.rank, v.off.actq_s), v.Is_t + 16, v.T, nullptr, v.Is_t, s);
      if (rc) return rc;
    }
  }
  if (stage != 1) {
    if (El > 0) {
      rc = grouped_gemm_fp8(at<char>(v, v.rank, v.off.actq), v.I_t + 16, ep.w2, ep.w2_scale,
                            at<char>(v, v.rank, v.off.partial), offs, cnts, nullptr, El, v.cap,
                            v.cap, v.h, v.I_t, 0, s, shared ? &none : &last);
      if (rc) return rc;
    }
    if (shared) {
      rc = grouped_gemm_fp8(at<char>(v, v.rank, v.off.actq_s), v.Is_t + 16, ep.w2_shared,
                            ep.w2_shared_scale, at<char>(v, v.rank, v.off.part_s), sh, sh + 1,
                            nullptr, 1, v.T, v.T, v.h, v.Is_t, 0, s, &last);
      if (rc) return rc;
    }
  }
  return rc;
}

// Expert FFN of one rank: GEMM1 (+SwiGLU) then GEMM2 over its host's experts
// -- all rows, or (sub = 1 / 2) only the own group's / the other groups'
// sub-blocks of every expert segment (the overlapped forward runs the two
// halves around the NVLink phases; same tiles' arithmetic, so the same bits).
int launch_expert_swiglu(const DevView& v, const void* w13, const void* w2, int stage,
                         cudaStream_t s, int sub) {
  const int e0 = first_expert(v.group, v.n, v.E), e1 = first_expert(v.group + 1, v.n, v.E);
  const int El = e1 - e0;
  if (El == 0) return MX_OK;
  const int32_t* offs = at<int32_t>(v, v.rank, v.off.exp_off) + e0;
  const int32_t* cnts = at<int32_t>(v, v.rank, v.off.exp_cnt) + e0;
  const int32_t* bidx = nullptr;
  int G = El;
  if (sub) {
    const int32_t* t = at<int32_t>(v, v.rank, v.off.sub);
    const int S = 2 * v.E;
    if (sub == 1) { offs = t; cnts = t + S; }
    else { offs = t + 2 * S; cnts = t + 3 * S; bidx = t + 4 * S; G = 2 * El; }
  }
  DevView first = v, last = v;  // fused barrier: GEMM1 waits, GEMM2 signals
  first.sync_signal = 0;
  last.sync_wait = 0;
  if (stage != 2) {
    // GEMM1 A operand: gathered token rows (row table + source buffer) when
    // the layout provides them, else the materialised expert-major RECV
    const void* A = v.a_src ? v.a_src : at<char>(v, v.rank, v.off.recv);
    const int32_t* rows = v.a_src ? at<int32_t>(v, v.rank, v.off.recv_src) : nullptr;
    int rc = grouped_gemm(A, w13, at<char>(v, v.rank, v.off.act), MX_BF16, offs, cnts, bidx, G,
                          v.cap, v.cap, 2 * v.I_t, v.h, 1, s, rows, v.a_src_rows, &first);
    if (rc || stage == 1) return rc;
  }
  return grouped_gemm(at<char>(v, v.rank, v.off.act), w2, at<char>(v, v.rank, v.off.partial),
                      MX_BF16, offs, cnts, bidx, G, v.cap, v.cap, v.h, v.I_t, 0, s, nullptr, 0,
                      &last);
}

}  // namespace mx

extern "C" __attribute__((visibility("default"))) int mx_debug_gemm_trace(unsigned long long* host, int ctas) {
  if (!mx::gemm::g_trace || ctas < 1 || ctas > 1024) return -1;
  if (cudaMemcpy(host, mx::gemm::g_trace, (size_t)ctas * 16 * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return cudaMemset(mx::gemm::g_trace, 0, 1024 * 16 * 8) == cudaSuccess ? 0 : -1;  // next launch starts clean
}
