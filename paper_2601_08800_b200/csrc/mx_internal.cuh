// mx_internal.cuh -- shared types, heap layout and PTX helpers.
//
// Every rank owns one symmetric heap (identical offsets on all ranks), so a
// kernel reaches buffer B of rank r as heap[r] + off.B.  In SPMD mode
// heap[r] for r != self is a CUDA-IPC mapping of the peer's heap (NVLink 5
// through NVSwitch); in emulated mode all heaps live on one device.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/mixserve_b200.h"

#define MX_MAXW 64         // max ranks in one cluster view
#define MX_CHUNK 128       // tokens per router chunk (one CTA)
#define MX_KMAX 32         // max top-k handled by the kernels
#define MX_EMAX 1024       // max experts
#define MX_STAMPS 64
#define MX_NMAX 64         // max groups

namespace mx {

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define MX_CUDA(call)                                                      \
  do {                                                                     \
    cudaError_t _e = (call);                                               \
    if (_e != cudaSuccess) return ::mx::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)
#define MX_LAUNCH_CHECK() MX_CUDA(cudaGetLastError())

// ---------------------------------------------------------------- layout
struct Offsets {
  size_t flags;       // uint64 [MX_MAXW]   barrier epochs written by peers
  size_t cnt_all;     // int32 [n][E]       pushed by every group (symmetric)
  size_t recv;        // act [cap][h]       written by peers (dispatch)
  size_t partial;     // act [cap][h]       read by peers (combine)
  size_t y;           // act [T][h]         written by TP peers (final AG)
  size_t act;         // bf16 [cap][I_t]    SwiGLU activation (local)
  size_t ids;         // int32 [T][k]
  size_t w;           // AccT [T][k]
  size_t slot_pos;    // int32 [T][k]
  size_t slot_tm;     // int32 [T][k]
  size_t slot_rank;   // int32 [T][k]  rank among chunk tokens of the expert
  size_t slot_tmr;    // int32 [T][k]  token-major rank inside the chunk/host
  size_t chunk_hist;  // int32 [C][E]  -> exclusive chunk base after route
  size_t chunk_host;  // int32 [C][n]  -> exclusive chunk base after route
  size_t exp_off;     // int32 [E]
  size_t exp_cnt;     // int32 [E]
  size_t grp_off;     // int32 [n][E]
  size_t send;        // int32 [n][n]
  size_t tm_off;      // int32 [n][n]
  size_t host_rows;   // int32 [n]
  // (token, host) pairs -- wire TOKEN (dispatch dedup / pre-reduced combine)
  size_t ucnt_all;    // int32 [n][n]  U[j][d]: tokens of group j with an expert on d (symmetric)
  size_t poff;        // int32 [n][n]  exclusive over j of U[j][d]
  size_t host_pairs;  // int32 [n]
  size_t chunk_pair;  // int32 [n][C]  -> exclusive chunk base after route
  size_t tok_pair_rank;  // int32 [T][n] rank among chunk tokens hitting d (-1: none)
  size_t upos;        // int32 [T][n]  row of (token, d) in d's xbuf (-1: none)
  size_t xbuf;        // act [T*n][h]  deduplicated rows (peers write)
  size_t recv_src;    // int32 [cap]   source row (token / xbuf pair) of every expert-major row
  size_t pair_p;      // int32 [T*n][KH] slot rows of a pair (peers write)
  size_t pair_w;      // AccT [T*n][KH]  slot weights of a pair (peers write)
  size_t pair_n;      // int32 [T*n]     slots of a pair (peers write)
  size_t pair_tok;    // int32 [T*n]     owner token (group*T + t) of a pair (peers write)
  size_t zin;         // act [n][m][T][h/m] pre-reduced TP partials pushed by every
                      //   host TP rank into the owner's shard (peers write)
  // fp8 experts (SWIGLU_FP8) and the shared expert
  size_t xq;          // [T][wrow]       this group's tokens, e4m3 + row scale
  size_t actq;        // [cap][I_t+16]   e4m3 activation + row scale (GEMM2 A)
  size_t act_s;       // bf16 [T][Is_t]  shared expert activation
  size_t actq_s;      // [T][Is_t+16]
  size_t part_s;      // bf16 [T][h]     shared expert TP partial (peers read)
  size_t sh_meta;     // int32 [4]       {0, T} offs/cnt of the shared "group"
  // source-group sub-blocks of this host's expert segments (overlapped
  // forward): [0] own-group offs, [1] own-group counts (El each), [2]/[3]
  // offs/counts of the rows before and after the own sub-block (2*El), [4]
  // their local expert (GEMM b_index); stride 2*E ints
  size_t sub;
  size_t counters;    // int32 [16]  [0]=route CTA counter [2..3]=u64 barrier epoch
  size_t err;         // int32 [16]  [0]=capacity [1]=bad id [2]=timeout
  size_t stamps;      // uint64 [MX_STAMPS] %globaltimer ns written by mx_stamp
  size_t total;
};

struct DevView {
  int rank, group, tp_rank, n, m, W;
  int T, h, E, k, I_t, C;
  int elt;            // bytes per hidden element on the wire
  int renorm;
  int router;         // mx_router: 0 softmax top-k, 1 sigmoid group-limited
  int r_groups, r_topk_groups;  // group-limited router: groups, groups kept
  float r_scaling;    // routed scaling factor (group-limited router)
  const float* r_bias;  // [E] score-correction bias (device)
  int wire;           // mx_wire
  int KH;             // max slots of one token on one host
  int welt;           // bytes per element on the wire (1: e4m3)
  int wrow;           // bytes per row on the wire (h*welt [+16 scale tail])
  int fp8;            // SWIGLU_FP8 plan
  int Is_t;           // shared expert intermediate per TP rank (0: none)
  int sync_signal;    // fused barrier: this kernel's last CTA publishes the epoch
  int sync_wait;      // fused barrier: every CTA waits for all peers' epoch at entry
  int early;          // decode regime: phase kernels trigger their dependents at entry
  const void* a_src;  // GEMM1 gathers A rows from here (x or XBUF), nullptr: RECV
  long long a_src_rows;
  long long cap;
  Offsets off;
  char* heap[MX_MAXW];
};

template <class T>
__host__ __device__ __forceinline__ T* at(const DevView& v, int r, size_t off) {
  return reinterpret_cast<T*>(v.heap[r] + off);
}

__host__ __device__ __forceinline__ int home_of(int e, int n, int E) {
  return (e * n) / E;  // sim:210-212 (e*n < 2^16 for E <= 1024, n <= 64)
}
// first expert hosted on group d: smallest e with e*n//E == d
__host__ __device__ __forceinline__ int first_expert(int d, int n, int E) {
  return (int)(((long long)d * E + n - 1) / n);
}
// array_split column shards (sim:317-323)
__host__ __device__ __forceinline__ void col_shard(int h, int m, int t, int* c0, int* c1) {
  int base = h / m, rem = h % m;
  *c0 = t * base + (t < rem ? t : rem);
  *c1 = *c0 + base + (t < rem ? 1 : 0);
}

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}

// shared-memory mbarriers (TMA / bulk-copy completion, producer-consumer rings)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a), "r"(parity) : "memory");
}
// 1D bulk copy global -> shared (TMA engine), completion as tx bytes on bar
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: every kernel of the layer is launched with
// programmatic stream serialisation and waits (griddepcontrol.wait) before
// reading its predecessor's outputs; dependents are released as each CTA
// exits (implicit trigger), so a kernel's launch and prologue overlap the
// previous kernel's tail (also inside the captured CUDA graph).  An explicit
// trigger at entry was measured to hurt: the persistent GEMM's early CTAs
// squat registers while the multi-wave dispatch is still running.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t pdl_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- fused barriers
// The device barrier between phases, folded into the kernels (SPMD, W > 1):
// the producer kernel's last CTA to finish bumps the rank's epoch and
// publishes it to every peer's flag slot (release, system scope); the
// consumer kernel's CTAs wait at entry until every peer published it.  The
// epoch counter is the same one k_barrier uses, so fused and standalone
// barriers interleave consistently.  Watchdog: error flag, no hang.
__device__ __forceinline__ unsigned long long* epoch_ctr(const DevView& v) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<int*>(v.heap[v.rank] + v.off.counters) + 2);
}
// Arrival per CTA with acq_rel at GPU scope (the CTA's writes, local and
// remote, happen-before the last arriver's system-scope release to the
// peers, which is cumulative over them): one system fence on the critical
// path, as in the lean device barrier (api.cu k_barrier_lean).
__device__ __forceinline__ int arrive_acq_rel_gpu(int* ctr) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
  return old;
}
__device__ __forceinline__ void grid_signal(const DevView& v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int* ctr = reinterpret_cast<int*>(v.heap[v.rank] + v.off.counters) + 4;
    if (arrive_acq_rel_gpu(ctr) == (int)(gridDim.x * gridDim.y) - 1) {
      *ctr = 0;
      const unsigned long long e = ++(*epoch_ctr(v));
      for (int r = 0; r < v.W; ++r)
        st_release_sys(reinterpret_cast<unsigned long long*>(v.heap[r] + v.off.flags) + v.rank, e);
    }
  }
}
__device__ __forceinline__ void grid_wait(const DevView& v) {
  if ((int)threadIdx.x < v.W) {
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(epoch_ctr(v));
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(v.heap[v.rank] + v.off.flags) + threadIdx.x;
    const long long t0 = clock64();
    while (ld_acquire_sys(mine) < e) {
      if (clock64() - t0 > 20000000000LL) {
        atomicOr(reinterpret_cast<int*>(v.heap[v.rank] + v.off.err) + 2, 1);
        break;
      }
    }
  }
  __syncthreads();
}
// combine's tail: publish, then the last CTA waits for every peer, so the
// kernel completes only when every TP peer's output shard has landed
__device__ __forceinline__ void grid_signal_and_wait(const DevView& v) {
  __syncthreads();
  __shared__ int s_is_last;
  if (threadIdx.x == 0) {
    int* ctr = reinterpret_cast<int*>(v.heap[v.rank] + v.off.counters) + 4;
    s_is_last = arrive_acq_rel_gpu(ctr) == (int)(gridDim.x * gridDim.y) - 1;
    if (s_is_last) {
      *ctr = 0;
      const unsigned long long e = ++(*epoch_ctr(v));
      for (int r = 0; r < v.W; ++r)
        st_release_sys(reinterpret_cast<unsigned long long*>(v.heap[r] + v.off.flags) + v.rank, e);
    }
  }
  __syncthreads();
  if (s_is_last) grid_wait(v);
}

// ---------------------------------------------------------------- dtypes
template <int DT> struct Elt;
template <> struct Elt<MX_F64> { using T = double; using Acc = double; static constexpr int V = 2; };
template <> struct Elt<MX_F32> { using T = float; using Acc = float; static constexpr int V = 4; };
template <> struct Elt<MX_BF16> { using T = __nv_bfloat16; using Acc = float; static constexpr int V = 8; };

__device__ __forceinline__ double to_acc(double x) { return x; }
__device__ __forceinline__ float to_acc(float x) { return x; }
__device__ __forceinline__ float to_acc(__nv_bfloat16 x) { return __bfloat162float(x); }
template <class T> __device__ __forceinline__ T from_acc(double x);
template <class T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ double from_acc<double>(double x) { return x; }
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) {
  return __float2bfloat16_rn(x);
}
// Uncontracted arithmetic: the f64 path reproduces the reference's numpy
// association exactly (no FMA fusion), sim:433-441 / sim:506-520.
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }

// ---------------------------------------------------------------- host plan
struct Comm;
struct Plan;

// kernels (launchers live next to their kernels)
int launch_route(const DevView& v, const float* logits, const int32_t* ids,
                 const void* w, cudaStream_t s);
int launch_layout(const DevView& v, cudaStream_t s);
int launch_dispatch(const DevView& v, const void* x, cudaStream_t s);
int launch_expert_affine(const DevView& v, const void* scales, const void* biases,
                         cudaStream_t s);
// sub: 0 every row of the host's experts, 1 the own group's sub-blocks,
// 2 the other groups' sub-blocks (Offsets::sub)
int launch_expert_swiglu(const DevView& v, const void* w13, const void* w2, int stage,
                         cudaStream_t s, int sub = 0);
int launch_expert_fp8(const DevView& v, const mx_expert_params& ep, int stage, cudaStream_t s);
int launch_combine(const DevView& v, cudaStream_t s);
// part: 0 every (token, host) pair, 1 the own group's pairs (local rows),
// 2 the other groups' pairs (NVLink).  coresident: one 128-thread CTA per
// SM, sized to share the SM with a running grouped-GEMM CTA (no shared
// memory, <= 128 registers) -- the overlapped forward's side stream.
int launch_dispatch_token(const DevView& v, const void* x, cudaStream_t s, int part = 0,
                          bool coresident = false);
int launch_expand(const DevView& v, cudaStream_t s, bool coresident = false);
int launch_pair_reduce(const DevView& v, cudaStream_t s, int part = 0, bool coresident = false);
int launch_combine_token(const DevView& v, cudaStream_t s);
int launch_reduce_combine(const DevView& v, cudaStream_t s);
bool reduce_combine_ok(const DevView& v);
int launch_barrier(const DevView& v, cudaStream_t s, bool group_only = false);
int launch_stamp(const DevView& v, int slot, cudaStream_t s);
int launch_baseline_dispatch_pack(const DevView& v, const void* x, void* send,
                                  int32_t* counts, cudaStream_t s);
int launch_baseline_dispatch_unpack(const DevView& v, const void* recv, cudaStream_t s);
int launch_baseline_combine_pack(const DevView& v, void* send, int32_t* counts,
                                 cudaStream_t s);
int launch_baseline_combine_unpack(const DevView& v, const void* recv, void* y,
                                   cudaStream_t s);
int grouped_gemm(const void* A, const void* B, void* D, int out_dtype,
                 const int32_t* offs, const int32_t* cnts, const int32_t* b_index,
                 int G, long long M_total, long long M_cap, int N, int K, int swiglu,
                 cudaStream_t s, const int32_t* a_rows = nullptr, long long a_src_rows = 0,
                 const DevView* sync = nullptr);
int grouped_gemm_fp8(const void* A, long long lda, const void* B, const float* b_scales, void* D,
                     const int32_t* offs, const int32_t* cnts, const int32_t* b_index, int G,
                     long long M_total, long long M_cap, int N, int K, int swiglu, cudaStream_t s,
                     const DevView* sync = nullptr);
int quant_rows_e4m3(const void* src, long long lds, void* dst, long long ldd, long long rows,
                    const int32_t* rows_dev, int cols, cudaStream_t s);
int launch_rowsrc_slot(const DevView& v, cudaStream_t s);
int launch_rowsrc_token(const DevView& v, cudaStream_t s);
int launch_nvlink_probe(const DevView& v, size_t bytes, cudaStream_t s);
int launch_prefetch_experts(const DevView& v, const void* w13, const void* w2, size_t b13,
                            size_t b2, long long budget, cudaStream_t s);

}  // namespace mx
