/*
 * mixserve_b200.h -- C ABI of the B200-native TP-EP hybrid MoE layer.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/moeplan/simcluster.py, "sim" below).  The
 * reference is a pure-Python API with no FFI; the Python package
 * paper_2601_08800_b200 binds these entry points with ctypes (see
 * INTEGRATION.md) and re-creates the reference signatures on top of them.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch types.  Device pointers are
 *     CUDA device memory, host pointers are marked "host".
 *   - Every call returns int: MX_OK (0) or a negative MX_ERR_* code; the
 *     message is available from mx_last_error() (thread-local).  The Python
 *     shim maps MX_ERR_INVALID -> StrategyError, MX_ERR_CAPACITY ->
 *     CapacityError (sim:346-351), everything else -> RuntimeError, as the
 *     reference does with its exception hierarchy (errors.py:16-41).
 *   - Stream-ordered: kernels are enqueued on the given cudaStream_t
 *     (passed as void* so the header needs no CUDA include).
 *   - A "rank" is global rank r = group*tp + tp_rank (node-major, sim:63-67).
 *     In emulated mode one process holds every rank of the cluster on one
 *     device and rank = -1 means "all ranks, phase by phase"; in SPMD mode
 *     (one process per GPU) rank must equal the process's own rank.
 */
#ifndef MIXSERVE_B200_H
#define MIXSERVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MX_ABI_VERSION 3

#if defined(__GNUC__)
#define MX_API __attribute__((visibility("default")))
#else
#define MX_API
#endif

#define MX_OK 0
#define MX_ERR_INVALID -1     /* shape / divisibility / cluster mismatch   */
#define MX_ERR_CAPACITY -2    /* a host's slots exceed the receive capacity */
#define MX_ERR_CUDA -3        /* CUDA runtime / driver failure             */
#define MX_ERR_UNSUPPORTED -4 /* configuration the kernels do not cover    */
#define MX_ERR_TIMEOUT -5     /* peer-flag watchdog expired                */

typedef enum { MX_F64 = 0, MX_F32 = 1, MX_BF16 = 2 } mx_dtype;
/* SWIGLU_FP8: e4m3 experts with per-output-channel weight scales; tokens are
 * quantised per row (e4m3 + fp32 scale) before dispatch, so the wire carries
 * h+16 bytes per row; activations are re-quantised between the GEMMs.  The
 * layer's input and output stay bf16 (act_dtype MX_BF16).                */
typedef enum { MX_EXPERT_AFFINE = 0, MX_EXPERT_SWIGLU = 1, MX_EXPERT_SWIGLU_FP8 = 2 } mx_expert_kind;
/* Wire format between groups.  SLOT: one row per routed slot both ways, the
 * reference's A2A layout (sim:366-369, sim:458-475).  TOKEN: one row per
 * (token, host group) pair -- dispatch dedup and combine pre-reduced per
 * (token, host) before the pull; the routing tables and
 * send/recv slot lists are identical, only the bytes on NVLink shrink.   */
typedef enum { MX_WIRE_SLOT = 0, MX_WIRE_TOKEN = 1 } mx_wire;

/* Gate applied by mx_route when it is given logits.
 * SOFTMAX: Qwen3-MoE -- fp32 softmax over E, top-k by logit, optional
 *   renormalisation (transformers modeling_qwen3_moe.py router).
 * GROUP_LIMITED: DeepSeek-V3 -- sigmoid scores, key = score + correction
 *   bias, top-2-sum group scores, keep router_topk_groups of router_groups,
 *   top-k of the masked key, weights = score (/ (sum + 1e-20) when
 *   renormalize) * routed_scaling (transformers modeling_deepseek_v3.py
 *   DeepseekV3MoE.route_tokens_to_experts).  Lowest index wins every tie. */
typedef enum { MX_ROUTER_SOFTMAX = 0, MX_ROUTER_GROUP_LIMITED = 1 } mx_router;

/* Buffers a plan exposes (for zero-copy views and parity inspection). */
typedef enum {
  MX_BUF_RECV = 0,     /* [capacity, h] act: expert-major received rows      */
  MX_BUF_PARTIAL = 1,  /* [capacity, h] act: TP-partial expert outputs       */
  MX_BUF_Y = 2,        /* [T, h] act: combined output of this rank's group   */
  MX_BUF_IDS = 3,      /* [T, k] int32: top-k expert ids (selection order)   */
  MX_BUF_WEIGHTS = 4,  /* [T, k] f64 (act f64) or f32: top-k weights         */
  MX_BUF_SLOT_POS = 5, /* [T, k] int32: row of the slot in host's RECV       */
  MX_BUF_SLOT_TM = 6,  /* [T, k] int32: index in host's token-major table    */
  MX_BUF_CNT_ALL = 7,  /* [n, E] int32: per-group per-expert token counts    */
  MX_BUF_EXP_OFF = 8,  /* [E] int32: first RECV row of each expert (its host)*/
  MX_BUF_EXP_CNT = 9,  /* [E] int32: rows of each expert summed over groups  */
  MX_BUF_SEND = 10,    /* [n, n] int32: S[j][d] slots of group j on host d   */
  MX_BUF_ACT = 11,     /* [capacity, I/tp] bf16: SwiGLU activation           */
  MX_BUF_UPOS = 12,    /* [T, n] int32: (token, host) pair row in host's XBUF */
  MX_BUF_XBUF = 13,    /* [T*n, h] act: deduplicated rows (wire TOKEN)       */
  MX_BUF_STAMPS = 14,  /* [64] uint64: %globaltimer ns written by mx_stamp   */
  MX_BUF_COUNT_ = 15
} mx_buffer;

typedef struct mx_comm mx_comm;
typedef struct mx_plan mx_plan;

typedef struct {
  int n_group;        /* n: groups (the paper's nodes, sim:41-67)            */
  int tp;             /* m: TP ranks per group                               */
  int tokens;         /* T: tokens per group (T_global / n, sim:574-580)     */
  int hidden;         /* h                                                   */
  int num_experts;    /* E (placement e*n//E, sim:210-212)                   */
  int top_k;          /* k                                                   */
  int inter;          /* I: full expert intermediate size (SwiGLU only)      */
  int act_dtype;      /* mx_dtype of hidden states on the wire               */
  int expert_kind;    /* mx_expert_kind                                      */
  int renormalize;    /* top-k weights renormalised over the k (logits mode) */
  int wire;           /* mx_wire                                             */
  int shared_inter;   /* shared expert intermediate size (0: none), SWIGLU_FP8 */
  long long capacity; /* receive rows per host; <=0: worst case T*n*min(k,E/n+1) */
  /* gate (zero-initialised: SOFTMAX) */
  int router;              /* mx_router                                      */
  int router_groups;       /* GROUP_LIMITED: expert groups (E % groups == 0) */
  int router_topk_groups;  /* GROUP_LIMITED: groups kept per token           */
  float routed_scaling;    /* GROUP_LIMITED: weight scale (0 -> 1.0)         */
  const float* router_bias;/* GROUP_LIMITED: [E] fp32 device, may be NULL    */
} mx_plan_desc;

/* Expert parameters for one rank (device pointers). */
typedef struct {
  /* MX_EXPERT_AFFINE: ExpertSpec (sim:189-207), per expert scale/bias,
   * f64 when act_dtype is MX_F64, otherwise f32.  Length E.            */
  const void* scales;
  const void* biases;
  /* MX_EXPERT_SWIGLU: this rank's TP shard of its host's experts, bf16.
   * w13: [E/n, 2*I/tp, h] rows interleaved in blocks of 64 (64 gate rows,
   *      the matching 64 up rows, ...) -- see mx_swiglu_pack_w13.
   * w2:  [E/n, h, I/tp].                                                 */
  const void* w13;
  const void* w2;
  /* MX_EXPERT_SWIGLU_FP8: e4m3 w13/w2 as above plus fp32 per-output-channel
   * scales [E/n, 2*I/tp] and [E/n, h]; the shared expert's TP shard
   * (w13_shared [2*Is/tp, h] interleaved like w13, w2_shared [h, Is/tp]).  */
  const float* w13_scale;
  const float* w2_scale;
  const void* w13_shared;
  const void* w2_shared;
  const float* w13_shared_scale;
  const float* w2_shared_scale;
} mx_expert_params;

/* ----- library ---------------------------------------------------------- */
MX_API int mx_abi_version(void);
MX_API const char* mx_last_error(void);
MX_API int mx_device_sm_count(int device, int* out);

/* ----- communicator: one symmetric heap per rank -----------------------
 * Replaces the in-process cluster of sim:41-67 (SimCluster/SimRank, whose
 * inbox is never used) with real peer-mapped device memory.              */
MX_API int mx_comm_create(int n_group, int tp, int rank, int emulate,
                   size_t heap_bytes_per_rank, mx_comm** out);
/* SPMD: export this rank's heap as a 64-byte CUDA IPC handle (host out). */
MX_API int mx_comm_ipc_handle(mx_comm* c, void* handle64);
/* SPMD: open every peer's heap from world*64 bytes of handles (host).    */
MX_API int mx_comm_open_peers(mx_comm* c, const void* handles);
MX_API int mx_comm_heap(mx_comm* c, int rank, void** base, size_t* bytes);
MX_API int mx_comm_destroy(mx_comm* c);
/* Device-side barrier over all ranks (SPMD; no-op when emulated).        */
/* The device barrier in two halves that never spin, for ranks that share
 * ONE GPU as separate processes (tests; kernels of different processes are
 * not guaranteed to run concurrently): half 1 publishes this rank's next
 * epoch to every peer (or TP-group peer), the caller then synchronizes the
 * processes on the host, half 2 checks every peer's flag and sets the
 * watchdog error word (reported by mx_plan_check) if one is missing.     */
MX_API int mx_comm_barrier_split(mx_comm* c, int half, int group_only, void* stream);
MX_API int mx_comm_barrier(mx_comm* c, void* stream);

/* ----- layer plan ------------------------------------------------------ */
/* Bytes of symmetric heap a plan needs per rank.                         */
MX_API int mx_plan_heap_bytes(const mx_plan_desc* d, size_t* out);
MX_API int mx_plan_create(mx_comm* c, const mx_plan_desc* d, mx_plan** out);
MX_API int mx_plan_destroy(mx_plan* p);
MX_API int mx_plan_buffer(mx_plan* p, int rank, int which, void** ptr, size_t* bytes);

/* K1 router.  Exactly one of (logits) or (ids, weights) is non-NULL.
 * logits [T, E] f32 -> fused softmax/top-k; ids [T, k] int32 with weights
 * [T, k] (f64 when act is f64 else f32) -> explicit RouterSpec routing
 * (sim:143-186).  Then per-expert counting, chunk prefix sums and the
 * publish of this group's count row to every rank (replaces the Python
 * loop of build_routing_table, sim:236-251).  In emulated mode the inputs
 * hold all n groups ([n*T, ...]).                                         */
MX_API int mx_route(mx_plan* p, int rank, const float* logits, const int32_t* ids,
             const void* weights, void* stream);
/* Expert-major / token-major slot positions and host segment offsets
 * (sim:249-250, sim:326-327, sim:528-532).  Requires every group's counts
 * (barrier after mx_route in SPMD).  Reports MX_ERR_CAPACITY after a sync
 * when check_capacity is set.                                             */
MX_API int mx_layout(mx_plan* p, int rank, int check_capacity, void* stream);
/* K2 fused AG-dispatch (sim:330-407): column shard tp_rank of each remote
 * slot row is stored into the receive buffer of every TP rank of the host
 * group (the intra-group all-gather fused into the inter-group send); the
 * local block is a local row gather.  x: [T, h] act of this rank's group
 * (emulated: [n*T, h]).                                                   */
MX_API int mx_dispatch(mx_plan* p, int rank, const void* x, void* stream);
/* K3 expert compute on this rank's received rows -> TP partials
 * (affine stand-in sim:535-562, or the SwiGLU grouped GEMM).             */
MX_API int mx_expert(mx_plan* p, int rank, const mx_expert_params* ep, void* stream);
/* The same expert compute split in its launches, for per-kernel timing:
 * 0 = everything below in order; 1 = GEMM1 + SwiGLU epilogue (or the affine
 * kernel); 2 = GEMM2; 3 = wire-TOKEN expand (XBUF -> RECV); 4 = wire-TOKEN
 * pair pre-reduction (PARTIAL -> z).  0 runs 3, 1, 2, 4.                 */
MX_API int mx_expert_stage(mx_plan* p, int rank, const mx_expert_params* ep, int stage,
                           void* stream);
/* K4 fused RS-combine (sim:410-521): the owner pulls its column shard of
 * every slot's TP partials (rank-ascending sum = the intra reduce-scatter),
 * weights and accumulates in the reference's host arrival order, and
 * pushes the finished shard to every TP rank of its group (the final
 * all-gather).  y_out: optional [T, h] act copy target (NULL: MX_BUF_Y). */
MX_API int mx_combine(mx_plan* p, int rank, void* y_out, void* stream);

/* Measured-trace export: write the device clock
 * (%globaltimer, ns) into stamp slot [0, 64) of the rank's heap, ordered
 * after every earlier launch on the stream.  Read with MX_BUF_STAMPS.    */
MX_API int mx_stamp(mx_plan* p, int rank, int slot, void* stream);
/* Whole layer: route -> layout -> dispatch -> expert -> combine, with the
 * device barriers between phases in SPMD mode (run_moe_block, sim:565).  */
MX_API int mx_forward(mx_plan* p, int rank, const void* x, const float* logits,
               const int32_t* ids, const void* weights,
               const mx_expert_params* ep, void* y_out, void* stream);
/* Error words of the last launches (the forward itself never syncs):
 * synchronizes the stream, then reports and clears the rank's device error
 * flags -- MX_ERR_CAPACITY "node d receives N routed slots, capacity C"
 * (sim:346-351; rows past capacity are never written, the slot wire skips
 * them and the token wire drops them from expand / pre-reduction),
 * MX_ERR_INVALID for an expert id out of range, MX_ERR_TIMEOUT when a
 * peer barrier's watchdog expired.  MoELayer.forward calls it after every
 * eager forward; a captured forward checks with CapturedForward.check(). */
MX_API int mx_plan_check(mx_plan* p, int rank, void* stream);
/* NVLink ceiling probe (bench.py's same-run denominator): this rank copies
 * bytes_per_peer (rounded down to 4 KB) of its PARTIAL region into every
 * peer's RECV region, 16 B loads from local HBM and 16 B stores over
 * NVLink, all peers at once.  SPMD, W > 1; every rank should run it
 * between the same barriers.  Clobbers RECV/PARTIAL: between forwards. */
MX_API int mx_nvlink_probe(mx_plan* p, size_t bytes_per_peer, void* stream);

/* ----- NCCL AR+A2A baseline helpers (value path of sim:598-680) -------
 * The baseline moves FULL-width rows with torch.distributed/NCCL
 * all_to_all_single from every TP rank (sim:617-640), runs the same expert
 * kernel, returns full-width TP partials with a second all_to_all
 * (sim:652-658) and finishes with a TP all_reduce (sim:659-666).  These
 * kernels only pack/unpack around the NCCL calls.  Block order on the wire:
 * by peer group ascending, inside a block by (expert, token).              */
/* send[.] <- x rows of this group's slots, blocks by destination host;
 * counts_out (device, [n] int32) = rows per destination host.             */
MX_API int mx_baseline_dispatch_pack(mx_plan* p, int rank, const void* x,
                              void* send, int32_t* counts_out, void* stream);
/* recv blocks (by source group) -> expert-major MX_BUF_RECV.              */
MX_API int mx_baseline_dispatch_unpack(mx_plan* p, int rank, const void* recv,
                                void* stream);
/* MX_BUF_PARTIAL -> blocks by owner group; counts_out [n] rows per owner. */
MX_API int mx_baseline_combine_pack(mx_plan* p, int rank, void* send,
                             int32_t* counts_out, void* stream);
/* blocks by host group -> y[t] = sum_slots w*row (host order j-1..j).    */
MX_API int mx_baseline_combine_unpack(mx_plan* p, int rank, const void* recv,
                               void* y, void* stream);

/* ----- utilities -------------------------------------------------------- */
/* Interleave [E_l, I_t, h] gate and up shards into the w13 layout:
 * packed row 128*b + j = gate row 64*b + j, 128*b + 64 + j = up row 64*b + j.
 * (ABI v3: the interleave was 128 rows in v2.)                            */
MX_API int mx_swiglu_pack_w13(const void* gate, const void* up, void* w13, int E_l,
                       int I_t, int h, void* stream);
/* Dense single-device MoE (moe_oracle, sim:302-310) on the GPU, computed
 * independently of the fused path: y[t] = sum_{e asc} w*expert_e(x[t]).  */
MX_API int mx_dense_moe(int T, int h, int E, int k, int act_dtype, int expert_kind,
                 int inter, const void* x, const int32_t* ids,
                 const void* weights, const void* scales, const void* biases,
                 const void* w_gate, const void* w_up, const void* w_down,
                 void* y, void* stream);
/* Standalone tcgen05 grouped GEMM (bf16 in, fp32 accumulate):
 * D[rows of group g] = A[rows] . B_g^T for g in [0, G); rows of group g
 * are [offs[g], offs[g]+cnts[g]) of A (M_total x K, row-major) and D
 * (M_total x N, out_dtype).  B: [G, N, K].  Used by tests and the bench. */
MX_API int mx_grouped_gemm(const void* A, const void* B, void* D, int out_dtype,
                    const int32_t* offs, const int32_t* cnts, int G,
                    long long M_total, int N, int K, int swiglu, void* stream);

/* fp8 (e4m3) expert path (BASELINE config C).  Rows carry their fp32
 * scale: row r = cols e4m3 bytes, then the scale at byte `cols`; stride
 * ld >= cols + 16 (16 B aligned).  scale = amax/448, RNE, saturating.    */
MX_API int mx_quant_rows_e4m3(const void* src_bf16, long long lds_elems, void* dst,
                              long long ldd_bytes, long long rows, int cols, void* stream);
/* e4m3 grouped GEMM: A rows as above (lda bytes), B [G, N, K] e4m3 with
 * b_scales [G, N] fp32 per output channel, D bf16 [M, N] (or [M, N/2]
 * with the SwiGLU epilogue); f32 accumulation on tcgen05 kind::f8f6f4.   */
MX_API int mx_grouped_gemm_fp8(const void* A, long long lda, const void* B,
                               const float* b_scales, void* D, const int32_t* offs,
                               const int32_t* cnts, int G, long long M_total, int N, int K,
                               int swiglu, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MIXSERVE_B200_H */
