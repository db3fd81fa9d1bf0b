// api.cu -- the extern "C" boundary (include/mixserve_b200.h): symmetric
// heap communicator, layer plan, phase sequencing and the device barrier.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "mx_internal.cuh"

namespace mx {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  set_error("CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e),
            file, line, what);
  return MX_ERR_CUDA;
}

// ---------------------------------------------------------------- barrier
// All ranks: publish the epoch into every peer's flag slot (release, system
// scope), then wait until every peer has published it into ours (acquire).
// One thread per peer.  A watchdog turns a lost peer into an error flag
// instead of a hang (SURVEY.md §5 failure detection).
// Ranks [r0, r0 + nr) take part (the whole world, or one TP group); every
// rank still advances its epoch, so full and group barriers interleave.
__global__ void k_barrier(DevView v, int r0, int nr) {
  pdl_wait();  // predecessor's outputs are visible after this
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    // epochs live on the device so the barrier can be replayed in a CUDA graph;
    // every rank runs the same barrier sequence, so the counters agree
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(
        at<int>(v, v.rank, v.off.counters) + 2);
    s_epoch = ++(*ctr);
  }
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const int r = r0 + threadIdx.x;
  if ((int)threadIdx.x < nr) {
    __threadfence_system();
    st_release_sys(at<unsigned long long>(v, r, v.off.flags) + v.rank, epoch);
    const unsigned long long* mine = at<unsigned long long>(v, v.rank, v.off.flags) + r;
    long long t0 = clock64();
    while (ld_acquire_sys(mine) < epoch) {
      if (clock64() - t0 > (long long)20000000000LL) {  // ~10 s at 2 GHz
        atomicOr(at<int>(v, v.rank, v.off.err) + 2, 1);
        break;
      }
    }
  }
  __syncthreads();
  __threadfence_system();
}

// Lean form (default): the flag store's release.sys is the one fence
// (release is cumulative over everything the previous kernels wrote, local
// and remote, since they happen-before this kernel), and the acquire loads
// need no trailing fence -- later kernels are ordered after this one.
// tools/barrier_probe.py at 2 GPUs: 3.2 vs 5.1 us per barrier (graph
// replay, kernel boundary 0.46 us).  MX_BARRIER=0 selects k_barrier above.
__global__ void k_barrier_lean(DevView v, int r0, int nr) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  // one read and one bump of the epoch counter per barrier, broadcast by a
  // shuffle (one warp: worlds up to 32 ranks) or through shared memory
  __shared__ unsigned long long s_epoch;
  unsigned long long e0 = 0;
  if (threadIdx.x == 0) {
    unsigned long long* ctr =
        reinterpret_cast<unsigned long long*>(at<int>(v, v.rank, v.off.counters) + 2);
    e0 = *reinterpret_cast<volatile unsigned long long*>(ctr) + 1;
    *ctr = e0;
    s_epoch = e0;
  }
  unsigned long long epoch;
  if (blockDim.x <= 32) {
    epoch = __shfl_sync(0xffffffffu, e0, 0);
  } else {
    __syncthreads();
    epoch = s_epoch;
  }
  const int r = r0 + threadIdx.x;
  if ((int)threadIdx.x < nr) {
    st_release_sys(at<unsigned long long>(v, r, v.off.flags) + v.rank, epoch);
    const unsigned long long* mine = at<unsigned long long>(v, v.rank, v.off.flags) + r;
    long long t0 = clock64();
    while (ld_acquire_sys(mine) < epoch) {
      if (clock64() - t0 > (long long)20000000000LL) {  // ~10 s at 2 GHz
        atomicOr(at<int>(v, v.rank, v.off.err) + 2, 1);
        break;
      }
    }
  }
}

static bool barrier_lean() {
  static const bool b = [] {
    const char* e = getenv("MX_BARRIER");
    return !(e && e[0] == '0');
  }();
  return b;
}

// The barrier split in halves that never spin, for ranks that share ONE GPU
// as separate processes (tests): nothing guarantees that kernels of
// different processes run at the same time on one GPU, so a rank spinning
// on a peer's flag may never see it (B200_PROFILING.md: Xid 109).  arrive
// bumps the epoch and publishes it to the peers' flag slots; the host then
// synchronizes the processes; verify checks (no waiting) that every peer's
// flag holds the epoch and raises the error word otherwise.
__global__ void k_barrier_arrive(DevView v, int r0, int nr) {
  pdl_wait();
  if (threadIdx.x == 0) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(
        at<int>(v, v.rank, v.off.counters) + 2);
    const unsigned long long epoch = ++(*ctr);
    __threadfence_system();
    for (int r = r0; r < r0 + nr; ++r)
      st_release_sys(at<unsigned long long>(v, r, v.off.flags) + v.rank, epoch);
  }
}

__global__ void k_barrier_verify(DevView v, int r0, int nr) {
  pdl_wait();
  const unsigned long long epoch =
      *reinterpret_cast<volatile unsigned long long*>(at<int>(v, v.rank, v.off.counters) + 2);
  const int r = r0 + threadIdx.x;
  if ((int)threadIdx.x < nr &&
      ld_acquire_sys(at<unsigned long long>(v, v.rank, v.off.flags) + r) < epoch)
    atomicOr(at<int>(v, v.rank, v.off.err) + 2, 1);
  __syncthreads();
  __threadfence_system();
}

int launch_barrier(const DevView& v, cudaStream_t s, bool group_only) {
  const int r0 = group_only ? v.group * v.m : 0, nr = group_only ? v.m : v.W;
  if (barrier_lean()) pdl_launch(k_barrier_lean, 1, (nr + 31) / 32 * 32, 0, s, v, r0, nr);
  else pdl_launch(k_barrier, 1, 64, 0, s, v, r0, nr);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static int elt_bytes(int dt) { return dt == MX_F64 ? 8 : dt == MX_F32 ? 4 : 2; }

static long long default_capacity(const mx_plan_desc& d) {
  // worst case: every token of every group lands on one host with
  // min(k, experts on that host) slots each
  const int per_host = (d.num_experts + d.n_group - 1) / d.n_group;
  const int kk = d.top_k < per_host ? d.top_k : per_host;
  return (long long)d.tokens * d.n_group * kk;
}

static int validate(const mx_plan_desc& d) {
  if (d.n_group < 1 || d.tp < 1) { set_error("cluster needs at least one node and one device"); return MX_ERR_INVALID; }
  if (d.n_group * d.tp > MX_MAXW) { set_error("world size %d exceeds %d", d.n_group * d.tp, MX_MAXW); return MX_ERR_UNSUPPORTED; }
  if (d.n_group > MX_NMAX) { set_error("n_group %d exceeds %d", d.n_group, MX_NMAX); return MX_ERR_UNSUPPORTED; }
  if (d.tokens < 0 || d.hidden < 1) { set_error("bad tokens/hidden"); return MX_ERR_INVALID; }
  if (d.num_experts < 1 || d.num_experts > MX_EMAX) { set_error("num_experts %d outside [1, %d]", d.num_experts, MX_EMAX); return MX_ERR_UNSUPPORTED; }
  if (d.top_k < 1 || d.top_k > d.num_experts) { set_error("top_k must be in [1, num_experts]"); return MX_ERR_INVALID; }
  if (d.top_k > MX_KMAX) { set_error("top_k %d exceeds %d", d.top_k, MX_KMAX); return MX_ERR_UNSUPPORTED; }
  if (d.act_dtype < MX_F64 || d.act_dtype > MX_BF16) { set_error("bad act_dtype"); return MX_ERR_INVALID; }
  if (d.wire != MX_WIRE_SLOT && d.wire != MX_WIRE_TOKEN) { set_error("bad wire format"); return MX_ERR_INVALID; }
  if (d.router == MX_ROUTER_GROUP_LIMITED) {
    const int G = d.router_groups;
    if (G < 1 || G > 32 || d.num_experts % G != 0 || d.num_experts / G < 2) {
      set_error("group-limited router: groups must divide E into groups of >= 2 experts, at most 32 groups");
      return MX_ERR_INVALID;
    }
    if (d.router_topk_groups < 1 || d.router_topk_groups > G) { set_error("router_topk_groups must be in [1, groups]"); return MX_ERR_INVALID; }
    if (d.top_k > d.router_topk_groups * (d.num_experts / G)) { set_error("top_k exceeds the experts of the kept groups"); return MX_ERR_INVALID; }
  } else if (d.router != MX_ROUTER_SOFTMAX) {
    set_error("bad router"); return MX_ERR_INVALID;
  }
  if (d.expert_kind == MX_EXPERT_SWIGLU_FP8) {
    if (d.act_dtype != MX_BF16) { set_error("fp8 experts take bf16 tokens"); return MX_ERR_UNSUPPORTED; }
    if (d.inter % d.tp != 0 || (d.inter / d.tp) % 128 != 0) { set_error("inter/tp must be a multiple of 128"); return MX_ERR_UNSUPPORTED; }
    if (d.hidden % 256 != 0) { set_error("fp8 experts need hidden %% 256 == 0"); return MX_ERR_UNSUPPORTED; }
    if (d.shared_inter < 0 || d.shared_inter % d.tp != 0 || (d.shared_inter / d.tp) % 128 != 0) {
      set_error("shared_inter/tp must be a multiple of 128"); return MX_ERR_UNSUPPORTED;
    }
    if ((d.hidden / d.tp) % 16 != 0) { set_error("fp8 wire needs (h/tp) %% 16 == 0"); return MX_ERR_UNSUPPORTED; }
    if (d.shared_inter > 0 && d.top_k > 8) { set_error("shared expert needs top_k <= 8"); return MX_ERR_UNSUPPORTED; }
  } else if (d.shared_inter != 0) {
    set_error("shared experts are supported with SWIGLU_FP8 experts"); return MX_ERR_UNSUPPORTED;
  }
  if (d.expert_kind == MX_EXPERT_SWIGLU_FP8) {
  } else if (d.expert_kind == MX_EXPERT_SWIGLU) {
    if (d.act_dtype != MX_BF16) { set_error("SwiGLU experts run in bf16"); return MX_ERR_UNSUPPORTED; }
    if (d.inter % d.tp != 0 || (d.inter / d.tp) % 128 != 0) { set_error("inter/tp must be a multiple of 128"); return MX_ERR_UNSUPPORTED; }
    if (d.hidden % 128 != 0) { set_error("hidden must be a multiple of 128 for the grouped GEMM"); return MX_ERR_UNSUPPORTED; }
  } else if (d.expert_kind != MX_EXPERT_AFFINE) {
    set_error("bad expert_kind"); return MX_ERR_INVALID;
  }
  return MX_OK;
}

static int kh_of(const mx_plan_desc& d) {
  const int per_host = (d.num_experts + d.n_group - 1) / d.n_group;
  return d.top_k < per_host ? d.top_k : per_host;
}

static Offsets compute_offsets(const mx_plan_desc& d, long long cap) {
  Offsets o{};
  size_t p = 0;
  auto take = [&](size_t bytes) { size_t at = p; p = align_up(p + bytes, 1024); return at; };
  const size_t T = d.tokens, k = d.top_k, E = d.num_experts, n = d.n_group, h = d.hidden;
  const size_t C = (T + MX_CHUNK - 1) / MX_CHUNK;
  const size_t elt = elt_bytes(d.act_dtype);
  const size_t wsz = d.act_dtype == MX_F64 ? 8 : 4;
  const bool fp8 = d.expert_kind == MX_EXPERT_SWIGLU_FP8;
  const size_t It = d.expert_kind != MX_EXPERT_AFFINE ? d.inter / d.tp : 0;
  const size_t Ist = fp8 ? d.shared_inter / d.tp : 0;
  const size_t wrow = fp8 ? h + 16 : h * elt;  // bytes per row on the wire
  o.flags = take(8 * MX_MAXW);
  o.cnt_all = take(4 * n * E);
  o.counters = take(4 * 16);
  o.err = take(4 * 16);
  o.stamps = take(8 * MX_STAMPS);
  o.recv = take((size_t)cap * wrow);
  o.partial = take((size_t)cap * h * elt);
  o.y = take(T * h * elt);
  o.act = take((size_t)cap * It * 2);
  o.ids = take(4 * T * k);
  o.w = take(wsz * T * k);
  o.slot_pos = take(4 * T * k);
  o.slot_tm = take(4 * T * k);
  o.slot_rank = take(4 * T * k);
  o.slot_tmr = take(4 * T * k);
  o.chunk_hist = take(4 * C * E);
  o.chunk_host = take(4 * C * n);
  o.exp_off = take(4 * E);
  o.exp_cnt = take(4 * E);
  o.grp_off = take(4 * n * E);
  o.send = take(4 * n * n);
  o.tm_off = take(4 * n * n);
  o.host_rows = take(4 * n);
  o.ucnt_all = take(4 * n * n);
  o.poff = take(4 * n * n);
  o.host_pairs = take(4 * n);
  o.chunk_pair = take(4 * C * n);
  o.tok_pair_rank = take(4 * T * n);
  o.upos = take(4 * T * n);
  const bool tok = d.wire == MX_WIRE_TOKEN;
  const size_t U = tok ? T * n : 0;
  const size_t KH = kh_of(d);
  o.xbuf = take(U * wrow);
  o.recv_src = take(4 * (size_t)cap);
  o.pair_p = take(2 * wsz * U * KH);  // packed {row, weight} entries
  o.pair_w = take(0);
  o.pair_n = take(4 * U);
  o.pair_tok = take(4 * U);
  o.zin = take(tok ? (size_t)n * d.tp * T * ((h + d.tp - 1) / d.tp) * elt : 0);
  o.xq = take(fp8 ? T * wrow : 0);
  o.actq = take(fp8 ? (size_t)cap * (It + 16) : 0);
  o.act_s = take(T * Ist * 2);
  o.actq_s = take(Ist ? T * (Ist + 16) : 0);
  o.part_s = take(Ist ? T * h * 2 : 0);
  o.sh_meta = take(16);
  o.sub = take(4 * 5 * 2 * E);
  o.total = p;
  return o;
}

}  // namespace mx

using namespace mx;

struct mx_comm {
  int n = 0, m = 0, W = 0, rank = 0, emulate = 0, device = 0;
  size_t heap_bytes = 0;
  char* heap[MX_MAXW] = {};
  bool owned[MX_MAXW] = {};
  unsigned long long epoch = 0;
  Offsets off{};       // of the plan using this heap (flags live at 0)
  bool has_plan = false;
};

struct mx_plan {
  mx_comm* comm = nullptr;
  mx_plan_desc d{};
  long long cap = 0;
  Offsets off{};
  DevView base{};
  // per rank: where GEMM1 gathers its A rows from (set by dispatch; cleared
  // by the baseline's unpack, which materialises RECV instead)
  const void* a_src[MX_MAXW] = {};
  long long a_src_rows[MX_MAXW] = {};
  // fused device barrier flags for the next phase (mx_forward, SPMD only)
  int sync_signal = 0, sync_wait = 0;
  // overlapped forward: the side stream the NVLink phases run on, and the
  // fork/join events (created on first use, capturable into a CUDA graph)
  cudaStream_t side = nullptr;
  cudaEvent_t ev[4] = {};
  bool pf_forked = false;  // decode weight prefetch branch open on `side`
};

// Decode regime (the grouped GEMMs stream weights: at most 64 rows per
// local expert on average): the SPMD phase kernels trigger their dependents
// at entry, so each next phase's CTAs are already resident, waiting in
// griddepcontrol.wait, when its predecessor completes (MX_PDL_EARLY=0
// disables, for A/B runs).
static bool decode_regime(const mx_plan* p, const DevView& v) {
  static const bool on = [] {
    const char* e = getenv("MX_PDL_EARLY");
    return !(e && e[0] == '0');
  }();
  static const bool all = [] {
    const char* e = getenv("MX_PDL_EARLY_ALL");
    return e && e[0] == '1';
  }();
  const int El = first_expert(v.group + 1, v.n, v.E) - first_expert(v.group, v.n, v.E);
  // (at 1-2 tokens per group the parked CTAs cost more than the launches
  // they hide: EP2 T_g = 2 77.0 vs 74.3 us, profiles/r02_decode_diag_n4.log)
  return on && !p->comm->emulate && !v.sync_signal && !v.sync_wait && El > 0 &&
         ((v.cap <= 64LL * El && v.T >= 4) || (all && v.W > 1));
}

static DevView view_for(const mx_plan* p, int r) {
  DevView v = p->base;
  v.rank = r;
  v.group = r / p->d.tp;
  v.tp_rank = r % p->d.tp;
  v.a_src = p->a_src[r];
  v.a_src_rows = p->a_src_rows[r];
  v.sync_signal = p->sync_signal;
  v.sync_wait = p->sync_wait;
  v.early = decode_regime(p, v) ? 1 : 0;
  return v;
}

// GEMM1 gathers its A rows through a row table (16 B LDGSTS in the GEMM
// producer) instead of reading a materialised expert-major copy: SwiGLU
// experts, and either one group (rows straight from x, no dispatch copy) or
// the TOKEN wire (rows from the XBUF, no expand).  Opt-in (MX_GATHER=1,
// read per call): measured on B200 at config B N=1, GEMM1 takes 613 us with
// the gathering producer vs 354 us on the TMA-tiled copy, which outweighs
// the 60 us dispatch copy it removes (the old TMA tile::gather4 producer:
// 964 us).  Two stages of 128 scattered rows in flight per CTA cannot hide
// L2 latency; the tiled TMA path keeps four 48 KB stages in flight.
static bool gathers(const mx_plan* p) {
  const char* e = getenv("MX_GATHER");
  const bool enabled = e && e[0] == '1';
  return enabled && p->d.expert_kind == MX_EXPERT_SWIGLU &&
         (p->d.wire == MX_WIRE_TOKEN || p->d.n_group == 1);
}

extern "C" {

int mx_abi_version(void) { return MX_ABI_VERSION; }
const char* mx_last_error(void) { return g_err.c_str(); }

int mx_device_sm_count(int device, int* out) {
  MX_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device));
  return MX_OK;
}

int mx_comm_create(int n_group, int tp, int rank, int emulate, size_t heap_bytes,
                   mx_comm** out) {
  if (n_group < 1 || tp < 1) { set_error("cluster needs at least one node and one device"); return MX_ERR_INVALID; }
  const int W = n_group * tp;
  if (W > MX_MAXW) { set_error("world size %d exceeds %d", W, MX_MAXW); return MX_ERR_UNSUPPORTED; }
  if (!emulate && (rank < 0 || rank >= W)) { set_error("rank %d outside world %d", rank, W); return MX_ERR_INVALID; }
  mx_comm* c = new mx_comm();
  c->n = n_group; c->m = tp; c->W = W; c->rank = emulate ? -1 : rank; c->emulate = emulate;
  c->heap_bytes = align_up(heap_bytes < 4096 ? 4096 : heap_bytes, 2 << 20);
  cudaGetDevice(&c->device);
  const int first = emulate ? 0 : rank, last = emulate ? W : rank + 1;
  for (int r = first; r < last; ++r) {
    void* ptr = nullptr;
    cudaError_t e = cudaMalloc(&ptr, c->heap_bytes);
    if (e != cudaSuccess) {
      for (int q = first; q < r; ++q) cudaFree(c->heap[q]);
      delete c;
      return cuda_fail(e, "cudaMalloc(heap)", __FILE__, __LINE__);
    }
    cudaMemset(ptr, 0, c->heap_bytes);
    c->heap[r] = static_cast<char*>(ptr);
    c->owned[r] = true;
  }
  MX_CUDA(cudaDeviceSynchronize());
  *out = c;
  return MX_OK;
}

int mx_comm_ipc_handle(mx_comm* c, void* handle64) {
  if (c->emulate) { set_error("emulated communicator has no IPC handle"); return MX_ERR_INVALID; }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "ipc handle size");
  cudaIpcMemHandle_t hd;
  MX_CUDA(cudaIpcGetMemHandle(&hd, c->heap[c->rank]));
  memcpy(handle64, &hd, 64);
  return MX_OK;
}

int mx_comm_open_peers(mx_comm* c, const void* handles) {
  if (c->emulate) return MX_OK;
  const char* hs = static_cast<const char*>(handles);
  for (int r = 0; r < c->W; ++r) {
    if (r == c->rank || c->heap[r]) continue;
    cudaIpcMemHandle_t hd;
    memcpy(&hd, hs + 64 * r, 64);
    void* ptr = nullptr;
    MX_CUDA(cudaIpcOpenMemHandle(&ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    c->heap[r] = static_cast<char*>(ptr);
    c->owned[r] = false;
  }
  return MX_OK;
}

int mx_comm_heap(mx_comm* c, int rank, void** base, size_t* bytes) {
  if (rank < 0 || rank >= c->W) { set_error("bad rank"); return MX_ERR_INVALID; }
  *base = c->heap[rank];
  *bytes = c->heap_bytes;
  return MX_OK;
}

int mx_comm_destroy(mx_comm* c) {
  if (!c) return MX_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < c->W; ++r) {
    if (!c->heap[r]) continue;
    if (c->owned[r]) cudaFree(c->heap[r]);
    else cudaIpcCloseMemHandle(c->heap[r]);
  }
  delete c;
  return MX_OK;
}

int mx_plan_heap_bytes(const mx_plan_desc* d, size_t* out) {
  int rc = validate(*d);
  if (rc) return rc;
  const long long cap = d->capacity > 0 ? d->capacity : default_capacity(*d);
  *out = compute_offsets(*d, cap).total;
  return MX_OK;
}

int mx_plan_create(mx_comm* c, const mx_plan_desc* d, mx_plan** out) {
  int rc = validate(*d);
  if (rc) return rc;
  if (d->n_group != c->n || d->tp != c->m) {
    set_error("plan cluster %dx%d mismatches communicator %dx%d", d->n_group, d->tp, c->n, c->m);
    return MX_ERR_INVALID;
  }
  mx_plan* p = new mx_plan();
  p->comm = c;
  p->d = *d;
  p->cap = d->capacity > 0 ? d->capacity : default_capacity(*d);
  p->off = compute_offsets(*d, p->cap);
  if (p->off.total > c->heap_bytes) {
    set_error("plan needs %zu heap bytes, communicator has %zu", p->off.total, c->heap_bytes);
    delete p;
    return MX_ERR_INVALID;
  }
  DevView& v = p->base;
  v.n = d->n_group; v.m = d->tp; v.W = c->W;
  v.T = d->tokens; v.h = d->hidden; v.E = d->num_experts; v.k = d->top_k;

  v.C = (d->tokens + MX_CHUNK - 1) / MX_CHUNK;
  v.elt = elt_bytes(d->act_dtype);
  v.renorm = d->renormalize;
  v.router = d->router;
  v.r_groups = d->router_groups;
  v.r_topk_groups = d->router_topk_groups;
  v.r_scaling = d->routed_scaling != 0.f ? d->routed_scaling : 1.f;
  v.r_bias = d->router_bias;
  v.wire = d->wire;
  v.KH = kh_of(*d);
  v.fp8 = d->expert_kind == MX_EXPERT_SWIGLU_FP8;
  v.welt = v.fp8 ? 1 : v.elt;
  v.wrow = v.fp8 ? d->hidden + 16 : d->hidden * v.elt;
  v.Is_t = v.fp8 ? d->shared_inter / d->tp : 0;
  v.I_t = d->expert_kind != MX_EXPERT_AFFINE ? d->inter / d->tp : 0;
  v.cap = p->cap;
  v.off = p->off;
  for (int r = 0; r < c->W; ++r) v.heap[r] = c->heap[r];
  c->off = p->off;
  c->has_plan = true;
  {
    const int meta[4] = {0, d->tokens, 0, 0};
    for (int r = 0; r < c->W; ++r)
      if (c->owned[r]) MX_CUDA(cudaMemcpy(c->heap[r] + p->off.sh_meta, meta, sizeof(meta), cudaMemcpyHostToDevice));
  }
  *out = p;
  return MX_OK;
}

int mx_plan_destroy(mx_plan* p) {
  if (p && p->side) {
    cudaStreamSynchronize(p->side);
    for (cudaEvent_t e : p->ev) if (e) cudaEventDestroy(e);
    cudaStreamDestroy(p->side);
  }
  delete p;
  return MX_OK;
}

int mx_plan_buffer(mx_plan* p, int rank, int which, void** ptr, size_t* bytes) {
  const mx_plan_desc& d = p->d;
  if (rank < 0 || rank >= p->comm->W || !p->comm->heap[rank]) { set_error("bad rank %d", rank); return MX_ERR_INVALID; }
  const Offsets& o = p->off;
  const size_t T = d.tokens, k = d.top_k, E = d.num_experts, n = d.n_group, h = d.hidden;
  const size_t elt = elt_bytes(d.act_dtype);
  size_t off = 0, len = 0;
  switch (which) {
    case MX_BUF_RECV: off = o.recv; len = p->cap * (size_t)p->base.wrow; break;
    case MX_BUF_PARTIAL: off = o.partial; len = p->cap * h * elt; break;
    case MX_BUF_Y: off = o.y; len = T * h * elt; break;
    case MX_BUF_IDS: off = o.ids; len = 4 * T * k; break;
    case MX_BUF_WEIGHTS: off = o.w; len = (d.act_dtype == MX_F64 ? 8 : 4) * T * k; break;
    case MX_BUF_SLOT_POS: off = o.slot_pos; len = 4 * T * k; break;
    case MX_BUF_SLOT_TM: off = o.slot_tm; len = 4 * T * k; break;
    case MX_BUF_CNT_ALL: off = o.cnt_all; len = 4 * n * E; break;
    case MX_BUF_EXP_OFF: off = o.exp_off; len = 4 * E; break;
    case MX_BUF_EXP_CNT: off = o.exp_cnt; len = 4 * E; break;
    case MX_BUF_SEND: off = o.send; len = 4 * n * n; break;
    case MX_BUF_ACT: off = o.act; len = p->cap * (size_t)p->base.I_t * 2; break;
    case MX_BUF_UPOS: off = o.upos; len = 4 * T * n; break;
    case MX_BUF_XBUF: off = o.xbuf; len = (d.wire == MX_WIRE_TOKEN ? T * n : 0) * (size_t)p->base.wrow; break;
    case MX_BUF_STAMPS: off = o.stamps; len = 8 * MX_STAMPS; break;
    default: set_error("bad buffer id %d", which); return MX_ERR_INVALID;
  }
  *ptr = p->comm->heap[rank] + off;
  *bytes = len;
  return MX_OK;
}

int mx_comm_barrier_split(mx_comm* c, int half, int group_only, void* stream) {
  if (c->emulate || c->W == 1) return MX_OK;
  if (!c->has_plan) { set_error("barrier needs a plan on the heap"); return MX_ERR_INVALID; }
  if (half != 1 && half != 2) { set_error("half must be 1 (arrive) or 2 (verify)"); return MX_ERR_INVALID; }
  DevView v{};
  v.rank = c->rank; v.W = c->W; v.off = c->off;
  for (int r = 0; r < c->W; ++r) v.heap[r] = c->heap[r];
  const int r0 = group_only ? c->rank / c->m * c->m : 0, nr = group_only ? c->m : c->W;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (half == 1) pdl_launch(k_barrier_arrive, 1, 32, 0, s, v, r0, nr);
  else pdl_launch(k_barrier_verify, 1, 64, 0, s, v, r0, nr);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int mx_comm_barrier(mx_comm* c, void* stream) {
  if (c->emulate || c->W == 1) return MX_OK;
  if (!c->has_plan) { set_error("barrier needs a plan on the heap"); return MX_ERR_INVALID; }
  DevView v{};
  v.rank = c->rank; v.W = c->W; v.off = c->off;
  for (int r = 0; r < c->W; ++r) v.heap[r] = c->heap[r];
  return launch_barrier(v, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// ------------------------------------------------------------ phases
namespace {

struct RankIter {
  int first, last;
};

int ranks_for(const mx_plan* p, int rank, RankIter* it) {
  const mx_comm* c = p->comm;
  if (c->emulate) {
    if (rank < 0) { it->first = 0; it->last = c->W; return MX_OK; }
    if (rank >= c->W) { set_error("rank %d outside world %d", rank, c->W); return MX_ERR_INVALID; }
    it->first = rank; it->last = rank + 1; return MX_OK;
  }
  if (rank >= 0 && rank != c->rank) { set_error("SPMD process of rank %d asked for rank %d", c->rank, rank); return MX_ERR_INVALID; }
  it->first = c->rank; it->last = c->rank + 1;
  return MX_OK;
}

// In emulated mode per-group inputs are stacked [n*T, ...].
const char* group_ptr(const mx_plan* p, const void* base, int group, size_t per_token_bytes) {
  if (!base) return nullptr;
  if (!p->comm->emulate) return static_cast<const char*>(base);
  return static_cast<const char*>(base) + (size_t)group * p->d.tokens * per_token_bytes;
}

int barrier(mx_plan* p, cudaStream_t s, bool group_only = false) {
  mx_comm* c = p->comm;
  if (c->emulate || c->W == 1) return MX_OK;
  DevView v = view_for(p, c->rank);
  return launch_barrier(v, s, group_only);
}

// Reads (and clears) the rank's device error words: err[0] the largest host
// row count over capacity (k_layout), err[1] an expert id out of range
// (k_route), err[2] the barrier watchdog, err[3] a slot row past capacity.
// Every word is cleared whichever fired, so a plan reused after an error
// (simcluster caches plans) reports only its own later failures.
int check_errors(mx_plan* p, int first, int last) {
  for (int r = first; r < last; ++r) {
    int err[4];
    MX_CUDA(cudaMemcpy(err, p->comm->heap[r] + p->off.err, sizeof(err), cudaMemcpyDeviceToHost));
    if (!(err[0] | err[1] | err[2] | err[3])) continue;
    int rows[MX_NMAX] = {};
    MX_CUDA(cudaMemcpy(rows, p->comm->heap[r] + p->off.host_rows, 4 * p->d.n_group, cudaMemcpyDeviceToHost));
    const int zero[4] = {0, 0, 0, 0};
    MX_CUDA(cudaMemcpy(p->comm->heap[r] + p->off.err, zero, sizeof(zero), cudaMemcpyHostToDevice));
    if (err[1]) { set_error("expert id out of range"); return MX_ERR_INVALID; }
    if (err[0] || err[3]) {
      // the first host over capacity with its slot count (sim:346-351)
      for (int d = 0; d < p->d.n_group; ++d)
        if (rows[d] > p->cap) {
          set_error("node %d receives %d routed slots, capacity %lld", d, rows[d], p->cap);
          return MX_ERR_CAPACITY;
        }
      set_error("routed slots exceed capacity %lld", p->cap);
      return MX_ERR_CAPACITY;
    }
    if (err[2]) { set_error("peer barrier watchdog expired"); return MX_ERR_TIMEOUT; }
  }
  return MX_OK;
}

}  // namespace

extern "C" {

int mx_route(mx_plan* p, int rank, const float* logits, const int32_t* ids, const void* weights,
             void* stream) {
  if ((logits == nullptr) == (ids == nullptr)) { set_error("pass exactly one of logits or ids"); return MX_ERR_INVALID; }
  if (ids && !weights) { set_error("ids need weights"); return MX_ERR_INVALID; }
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t wsz = p->d.act_dtype == MX_F64 ? 8 : 4;
  for (int r = it.first; r < it.last; ++r) {
    DevView v = view_for(p, r);
    rc = launch_route(v, reinterpret_cast<const float*>(group_ptr(p, logits, v.group, 4 * (size_t)p->d.num_experts)),
                      reinterpret_cast<const int32_t*>(group_ptr(p, ids, v.group, 4 * (size_t)p->d.top_k)),
                      group_ptr(p, weights, v.group, wsz * p->d.top_k), s);
    if (rc) return rc;
  }
  return MX_OK;
}

int mx_layout(mx_plan* p, int rank, int check_capacity, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = it.first; r < it.last; ++r) {
    rc = launch_layout(view_for(p, r), s);
    if (rc) return rc;
  }
  if (check_capacity) {
    MX_CUDA(cudaStreamSynchronize(s));
    return check_errors(p, it.first, it.last);
  }
  return MX_OK;
}

int mx_dispatch(mx_plan* p, int rank, const void* x, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t row = (size_t)p->d.hidden * elt_bytes(p->d.act_dtype);
  for (int r = it.first; r < it.last; ++r) {
    DevView v = view_for(p, r);
    const char* xg = group_ptr(p, x, v.group, row);
    if (v.fp8) {  // e4m3 rows + scale: the wire and GEMM1 operate on these
      char* xq = p->comm->heap[r] + p->off.xq;
      rc = quant_rows_e4m3(xg, v.h, xq, v.wrow, v.T, nullptr, v.h, s);
      if (rc) return rc;
      xg = xq;
    }
    if (p->d.wire == MX_WIRE_TOKEN) {
      // decided before the launch: without the gathered GEMM1 the dispatch
      // writes own-group rows straight into RECV (and expand skips them)
      p->a_src[r] = gathers(p) ? static_cast<const void*>(p->comm->heap[r] + p->off.xbuf) : nullptr;
      p->a_src_rows[r] = (long long)p->d.tokens * p->d.n_group;
      v.a_src = p->a_src[r];
      rc = launch_dispatch_token(v, xg, s);
    } else if (gathers(p)) {
      rc = launch_rowsrc_slot(v, s);  // n == 1: no row copies at all
      p->a_src[r] = xg;
      p->a_src_rows[r] = p->d.tokens;
    } else {
      rc = launch_dispatch(v, xg, s);
      p->a_src[r] = nullptr;
    }
    if (rc) return rc;
  }
  return MX_OK;
}

int mx_expert_stage(mx_plan* p, int rank, const mx_expert_params* ep, int stage, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  if (stage < 0 || stage > 4) { set_error("stage must be in [0, 4]"); return MX_ERR_INVALID; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = it.first; r < it.last; ++r) {
    DevView v = view_for(p, r);
    const bool tok = p->d.wire == MX_WIRE_TOKEN;
    // fused barrier (stage 0 only): the stage's first kernel waits, its last
    // one signals -- expand / pair_reduce on the token wire, else the
    // expert kernels themselves
    DevView vfirst = v, vlast = v;
    vfirst.sync_signal = 0;
    vlast.sync_wait = 0;
    if (tok) v.sync_wait = v.sync_signal = 0;
    if (tok && (stage == 0 || stage == 3)) {
      // gathered GEMM1 only needs the row table; otherwise expand into RECV
      rc = v.a_src ? launch_rowsrc_token(vfirst, s) : launch_expand(vfirst, s);
      if (rc) return rc;
    }
    if (stage == 3 || stage == 4) {
      if (tok && stage == 4 && (rc = launch_pair_reduce(v, s))) return rc;
      continue;
    }
    if (p->d.expert_kind == MX_EXPERT_AFFINE) {
      if (stage != 2) rc = launch_expert_affine(v, ep->scales, ep->biases, s);
    } else if (v.fp8) {
      mx_expert_params e = *ep;
      if (p->comm->emulate) {  // per-rank shards stacked rank-major
        const size_t El = (v.E + v.n - 1) / v.n;
        e.w13 = static_cast<const char*>(ep->w13) + r * El * 2 * v.I_t * v.h;
        e.w2 = static_cast<const char*>(ep->w2) + r * El * v.h * v.I_t;
        e.w13_scale = ep->w13_scale + r * El * 2 * v.I_t;
        e.w2_scale = ep->w2_scale + r * El * v.h;
        if (v.Is_t) {
          e.w13_shared = static_cast<const char*>(ep->w13_shared) + (size_t)r * 2 * v.Is_t * v.h;
          e.w2_shared = static_cast<const char*>(ep->w2_shared) + (size_t)r * v.h * v.Is_t;
          e.w13_shared_scale = ep->w13_shared_scale + (size_t)r * 2 * v.Is_t;
          e.w2_shared_scale = ep->w2_shared_scale + (size_t)r * v.h;
        }
      }
      rc = launch_expert_fp8(v, e, stage, s);
    } else {
      // emulated: per-rank weight shards stacked rank-major
      const int Elmax = (v.E + v.n - 1) / v.n;
      const size_t w13_rank = (size_t)Elmax * 2 * v.I_t * v.h * 2;
      const size_t w2_rank = (size_t)Elmax * v.h * v.I_t * 2;
      const int slot = p->comm->emulate ? r : 0;
      rc = launch_expert_swiglu(v, static_cast<const char*>(ep->w13) + slot * w13_rank,
                                static_cast<const char*>(ep->w2) + slot * w2_rank, stage, s);
    }
    if (rc) return rc;
    if (tok && stage == 0 && (rc = launch_pair_reduce(vlast, s))) return rc;
  }
  return MX_OK;
}

int mx_expert(mx_plan* p, int rank, const mx_expert_params* ep, void* stream) {
  return mx_expert_stage(p, rank, ep, 0, stream);
}

int mx_combine(mx_plan* p, int rank, void* y_out, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int r = it.first; r < it.last; ++r) {
    rc = p->d.wire == MX_WIRE_TOKEN ? launch_combine_token(view_for(p, r), s)
                                    : launch_combine(view_for(p, r), s);
    if (rc) return rc;
  }
  if (y_out) {
    rc = barrier(p, s);  // y is complete only after every TP peer pushed
    if (rc) return rc;
    const size_t bytes = (size_t)p->d.tokens * p->d.hidden * elt_bytes(p->d.act_dtype);
    for (int r = it.first; r < it.last; ++r) {
      const int g = r / p->d.tp;
      if (p->comm->emulate && (r % p->d.tp) != 0) continue;
      char* dst = static_cast<char*>(y_out) + (p->comm->emulate ? (size_t)g * bytes : 0);
      MX_CUDA(cudaMemcpyAsync(dst, p->comm->heap[r] + p->off.y, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  return MX_OK;
}

// Optionally (MX_FUSE_BARRIER_T = max tokens per group, default 0 = off) the
// inter-phase barriers are folded into the phase kernels (SPMD, W > 1, every
// phase guaranteed to launch on every rank): the producer's last CTA
// publishes the epoch, the consumer's CTAs wait for it at entry, combine's
// last CTA publishes and waits (y complete, buffers reusable).  Measured on
// B200 it is slower than the standalone barrier kernels at every size --
// config B N=4 prefill 0.442 vs 0.395 ms, decode T_g=64 162.6 vs 143.0 us --
// per-CTA system-scope fences and every CTA polling peer flags cost more
// than the launches they save.  Kept opt-in for persistent-kernel work.
static bool fused_barriers(const mx_plan* p) {
  static const long long limit = [] {
    const char* e = getenv("MX_FUSE_BARRIER_T");
    return e ? atoll(e) : 0LL;
  }();
  const mx_comm* c = p->comm;
  return !c->emulate && c->W > 1 && p->d.tokens > 0 && p->d.tokens <= limit && p->cap >= 1 &&
         p->d.num_experts >= p->d.n_group && !gathers(p);
}

namespace {
struct SyncFlags {  // sets the plan's fused-barrier flags for one phase
  mx_plan* p;
  SyncFlags(mx_plan* p_, bool on, int wait, int sig) : p(p_) {
    p->sync_wait = on ? wait : 0;
    p->sync_signal = on ? sig : 0;
  }
  ~SyncFlags() { p->sync_wait = p->sync_signal = 0; }
};
}  // namespace

// ---------------------------------------------------------------- overlap
// The overlapped forward (SPMD, wire TOKEN, bf16 SwiGLU experts, n > 1):
// the NVLink phases run on a side stream under the grouped GEMMs of rows
// that do not depend on them -- the pairwise rounds of Alg. 1/2 (sim:363-393,
// sim:448-504) feeding compute without waiting for the whole exchange.
//
//   main stream                         side stream
//   route, barrier, layout
//   dispatch part 1 (own rows -> RECV)  -- fork -->
//   GEMM1 on own-group sub-blocks        dispatch part 2 (pairs -> peers' XBUF,
//                                          NVLink), barrier (rows landed), expand
//   <-- join --
//   GEMM1 + GEMM2 on the other groups' sub-blocks
//                                        -- fork -->
//   GEMM2 on own-group sub-blocks        pre-reduce + push the other groups'
//   pre-reduce own pairs                   pairs into their owners' ZIN (NVLink)
//   <-- join --
//   barrier, combine, TP-group barrier
//
// Side-stream kernels use one 128-thread CTA per SM and no shared memory,
// so they run on the same SMs as the persistent GEMM CTAs (213 KB smem,
// 384 threads) instead of waiting for them.  Every row's arithmetic is the
// non-overlapped forward's (same tiles, same sums): identical output bits.
//
// Opt-in (MX_OVERLAP=1): measured SLOWER at config B, 2 GPUs EP2 -- 0.504
// vs 0.439 ms sequential (profiles/r02_n2_overlap_timeline.json).  Splitting
// each grouped GEMM by source group streams every expert's weights twice
// (403 MB per rank for GEMM1 at EP2): GEMM1 on the other groups' rows alone
// took 124 us with nothing beside it, against ~175 us for all rows at once,
// and the co-resident side kernels slowed the own-group halves further.
// With ~512 rows per expert the weight traffic a split adds outweighs the
// ~60 us of NVLink time it hides.
static bool overlap_forward(const mx_plan* p) {
  const char* e = getenv("MX_OVERLAP");
  if (!(e && e[0] == '1')) return false;
  const mx_comm* c = p->comm;
  return !c->emulate && c->W > 1 && p->d.n_group > 1 && p->d.wire == MX_WIRE_TOKEN &&
         p->d.expert_kind == MX_EXPERT_SWIGLU && p->d.act_dtype == MX_BF16 && !gathers(p) &&
         p->d.tokens > 0 && !fused_barriers(p);
}

// Decode regime: prefetch the active local experts' weights into L2 on the
// side stream while the dispatch, its barrier and the expand run (see
// k_prefetch_experts).  Applies when the grouped GEMMs stream weights (at
// most 64 rows per local expert on average, the GEMM's own decode criterion),
// SPMD only (one rank per process and device).  MX_PREFETCH_MB: byte budget
// (default 0 = off: together with the early-launched phase kernels the
// side-stream branch cost ~130 us per decode forward on some boxes,
// tools/runs/decode_diag.sh; 64 for the measured A/B).
static int prefetch_weights(mx_plan* p, const mx_expert_params* ep, cudaStream_t s) {
  p->pf_forked = false;
  static const long long budget = [] {
    const char* e = getenv("MX_PREFETCH_MB");
    return (e ? atoll(e) : 0LL) << 20;
  }();
  mx_comm* c = p->comm;
  if (budget <= 0 || c->emulate || !ep) return MX_OK;
  const bool swiglu = p->d.expert_kind == MX_EXPERT_SWIGLU || p->d.expert_kind == MX_EXPERT_SWIGLU_FP8;
  if (!swiglu || !ep->w13 || !ep->w2) return MX_OK;
  DevView v = view_for(p, c->rank);
  const int El = first_expert(v.group + 1, v.n, v.E) - first_expert(v.group, v.n, v.E);
  if (El < 1 || v.cap > 64LL * El) return MX_OK;
  if (!p->side) {
    MX_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    for (cudaEvent_t& e : p->ev) MX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const size_t wb = p->d.expert_kind == MX_EXPERT_SWIGLU_FP8 ? 1 : 2;
  const size_t b13 = (size_t)2 * v.I_t * v.h * wb, b2 = (size_t)v.h * v.I_t * wb;
  MX_CUDA(cudaEventRecord(p->ev[2], s));
  MX_CUDA(cudaStreamWaitEvent(p->side, p->ev[2], 0));
  int rc = launch_prefetch_experts(v, ep->w13, ep->w2, b13, b2, budget, p->side);
  if (rc) return rc;
  MX_CUDA(cudaEventRecord(p->ev[3], p->side));
  p->pf_forked = true;
  return MX_OK;
}

static int forward_overlapped(mx_plan* p, int rank, const void* x, const float* logits,
                              const int32_t* ids, const void* weights, const mx_expert_params* ep,
                              cudaStream_t s) {
  mx_comm* c = p->comm;
  if (!p->side) {
    MX_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    for (cudaEvent_t& e : p->ev) MX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t side = p->side;
  int rc;
  // MX_OVERLAP_STAMPS=1: %globaltimer stamps after each step on its stream
  // (stamp slots 30..45) for tools/overlap_timeline.py
  const char* st_env = getenv("MX_OVERLAP_STAMPS");
  const bool stamps = st_env && st_env[0] == '1';
  const char* co_env = getenv("MX_OVERLAP_CORES");  // 0: full-grid side kernels (experiments)
  const bool cores = !(co_env && co_env[0] == '0');
  int slot = 30;
  auto stamp = [&](cudaStream_t q) {
    return stamps ? launch_stamp(view_for(p, c->rank), slot++, q) : MX_OK;
  };
  if ((rc = stamp(s))) return rc;
  if ((rc = mx_route(p, rank, logits, ids, weights, s))) return rc;
  if ((rc = barrier(p, s))) return rc;  // every group's counts published
  if ((rc = mx_layout(p, rank, 0, s))) return rc;
  const int r = c->rank;
  p->a_src[r] = nullptr;
  p->a_src_rows[r] = 0;
  const DevView v = view_for(p, r);
  const void* w13 = ep->w13;
  const void* w2 = ep->w2;
  if ((rc = stamp(s))) return rc;                                        // 31 layout done
  if ((rc = launch_dispatch_token(v, x, s, 1, false))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 32 own rows
  MX_CUDA(cudaEventRecord(p->ev[0], s));
  MX_CUDA(cudaStreamWaitEvent(side, p->ev[0], 0));
  if ((rc = launch_dispatch_token(v, x, side, 2, cores))) return rc;
  if ((rc = stamp(side))) return rc;                                     // 33 pushes issued
  if ((rc = barrier(p, side))) return rc;  // every pair row landed
  if ((rc = stamp(side))) return rc;                                     // 34 rows landed
  if ((rc = launch_expand(v, side, cores))) return rc;
  if ((rc = stamp(side))) return rc;                                     // 35 expanded
  MX_CUDA(cudaEventRecord(p->ev[1], side));
  if ((rc = launch_expert_swiglu(v, w13, w2, 1, s, 1))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 36 GEMM1 own
  MX_CUDA(cudaStreamWaitEvent(s, p->ev[1], 0));
  if ((rc = launch_expert_swiglu(v, w13, w2, 1, s, 2))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 37 GEMM1 other
  if ((rc = launch_expert_swiglu(v, w13, w2, 2, s, 2))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 38 GEMM2 other
  MX_CUDA(cudaEventRecord(p->ev[2], s));
  MX_CUDA(cudaStreamWaitEvent(side, p->ev[2], 0));
  if ((rc = launch_pair_reduce(v, side, 2, cores))) return rc;
  if ((rc = stamp(side))) return rc;                                     // 39 other pairs pushed
  MX_CUDA(cudaEventRecord(p->ev[3], side));
  if ((rc = launch_expert_swiglu(v, w13, w2, 2, s, 1))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 40 GEMM2 own
  if ((rc = launch_pair_reduce(v, s, 1, false))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 41 own pairs
  MX_CUDA(cudaStreamWaitEvent(s, p->ev[3], 0));
  if ((rc = barrier(p, s))) return rc;  // every owner's ZIN written
  if ((rc = stamp(s))) return rc;                                        // 42 ZIN complete
  if ((rc = launch_combine_token(v, s))) return rc;
  if ((rc = stamp(s))) return rc;                                        // 43 combined
  if (p->d.tp > 1 && (rc = barrier(p, s, true))) return rc;  // y complete (TP group)
  if ((rc = stamp(s))) return rc;                                        // 44 y complete
  return MX_OK;
}

int mx_forward(mx_plan* p, int rank, const void* x, const float* logits, const int32_t* ids,
               const void* weights, const mx_expert_params* ep, void* y_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool fuse = fused_barriers(p);
  int rc;
  if (overlap_forward(p)) {
    RankIter it;
    if ((rc = ranks_for(p, rank, &it))) return rc;
    if ((rc = forward_overlapped(p, rank, x, logits, ids, weights, ep, s))) return rc;
    if (y_out) {
      const size_t bytes = (size_t)p->d.tokens * p->d.hidden * elt_bytes(p->d.act_dtype);
      MX_CUDA(cudaMemcpyAsync(y_out, p->comm->heap[p->comm->rank] + p->off.y, bytes,
                              cudaMemcpyDeviceToDevice, s));
    }
    return MX_OK;
  }
  {
    SyncFlags f(p, fuse, 0, 1);
    if ((rc = mx_route(p, rank, logits, ids, weights, stream))) return rc;
  }
  if (!fuse && (rc = barrier(p, s))) return rc;  // every group's counts published
  {
    SyncFlags f(p, fuse, 1, 0);
    if ((rc = mx_layout(p, rank, 0, stream))) return rc;
  }
  const bool pf = (rc = prefetch_weights(p, ep, s)) == MX_OK && p->pf_forked;
  if (rc) return rc;
  {
    SyncFlags f(p, fuse, 0, 1);
    if ((rc = mx_dispatch(p, rank, x, stream))) return rc;
  }
  if (!fuse && (rc = barrier(p, s))) return rc;  // every row landed
  // opt-in (MX_FUSED_COMBINE=1): the token wire's combine side as one
  // persistent kernel (pre-reduction, exchange barrier, combine:
  // k_reduce_combine) where it applies.  Bit-identical to the three
  // launches and measured equal at config B, 2 GPUs EP2 (0.4421 vs 0.4420
  // ms): the two kernel boundaries it removes cost what its cooperative
  // launch (no programmatic dependent launch) and in-kernel barrier add.
  const char* rc_env = getenv("MX_FUSED_COMBINE");
  const bool fused_combine = !fuse && (rc_env && rc_env[0] == '1') && !p->comm->emulate &&
                             p->d.wire == MX_WIRE_TOKEN && reduce_combine_ok(view_for(p, p->comm->rank));
  if (fused_combine) {
    for (int st : {3, 1, 2})
      if ((rc = mx_expert_stage(p, rank, ep, st, stream))) return rc;
    if ((rc = launch_reduce_combine(view_for(p, p->comm->rank), s))) return rc;
    if (p->d.tp > 1 && (rc = barrier(p, s, true))) return rc;  // y complete (TP group)
    if (pf) {
      MX_CUDA(cudaStreamWaitEvent(s, p->ev[3], 0));
      p->pf_forked = false;
    }
    if (y_out) {
      const size_t bytes = (size_t)p->d.tokens * p->d.hidden * elt_bytes(p->d.act_dtype);
      MX_CUDA(cudaMemcpyAsync(y_out, p->comm->heap[p->comm->rank] + p->off.y, bytes,
                              cudaMemcpyDeviceToDevice, s));
    }
    return MX_OK;
  }
  {
    SyncFlags f(p, fuse, 1, 1);
    if ((rc = mx_expert(p, rank, ep, stream))) return rc;
  }
  if (!fuse && (rc = barrier(p, s))) return rc;  // every partial written
  {
    // the combine's closing publish-and-wait makes y complete; without TP
    // peers (m == 1) this rank wrote all of y itself
    SyncFlags f(p, fuse, 1, p->d.tp > 1 ? 1 : 0);
    if ((rc = mx_combine(p, rank, nullptr, stream))) return rc;
  }
  // y complete: every TP peer of the group pushed its shard.  Group-local --
  // nothing of another group is touched before the next forward's first
  // full barrier (its route only writes count rows read after that barrier);
  // without TP peers (m == 1) y is written by this rank alone: no barrier
  if (!fuse && p->d.tp > 1 && (rc = barrier(p, s, true))) return rc;
  if (pf) {  // join the prefetch branch (long finished: it only issues hints)
    MX_CUDA(cudaStreamWaitEvent(s, p->ev[3], 0));
    p->pf_forked = false;
  }
  if (y_out) {
    RankIter it;
    if ((rc = ranks_for(p, rank, &it))) return rc;
    const size_t bytes = (size_t)p->d.tokens * p->d.hidden * elt_bytes(p->d.act_dtype);
    for (int r = it.first; r < it.last; ++r) {
      if (p->comm->emulate && (r % p->d.tp) != 0) continue;
      char* dst = static_cast<char*>(y_out) + (p->comm->emulate ? (size_t)(r / p->d.tp) * bytes : 0);
      MX_CUDA(cudaMemcpyAsync(dst, p->comm->heap[r] + p->off.y, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  return MX_OK;
}

// Device timestamp (%globaltimer, ns) into the rank's stamp slot, ordered
// after every earlier launch on the stream: the measured-trace export
// brackets each phase with these.
int mx_stamp(mx_plan* p, int rank, int slot, void* stream) {
  if (slot < 0 || slot >= MX_STAMPS) { set_error("stamp slot %d outside [0, %d)", slot, MX_STAMPS); return MX_ERR_INVALID; }
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  for (int r = it.first; r < it.last; ++r) {
    rc = launch_stamp(view_for(p, r), slot, static_cast<cudaStream_t>(stream));
    if (rc) return rc;
  }
  return MX_OK;
}

int mx_baseline_dispatch_pack(mx_plan* p, int rank, const void* x, void* send,
                              int32_t* counts_out, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  if (it.last - it.first != 1) { set_error("baseline helpers take one rank"); return MX_ERR_INVALID; }
  DevView v = view_for(p, it.first);
  const size_t row = (size_t)p->d.hidden * elt_bytes(p->d.act_dtype);
  return launch_baseline_dispatch_pack(v, group_ptr(p, x, v.group, row), send, counts_out,
                                       static_cast<cudaStream_t>(stream));
}

int mx_baseline_dispatch_unpack(mx_plan* p, int rank, const void* recv, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  if (it.last - it.first != 1) { set_error("baseline helpers take one rank"); return MX_ERR_INVALID; }
  p->a_src[it.first] = nullptr;  // RECV is materialised by the unpack
  return launch_baseline_dispatch_unpack(view_for(p, it.first), recv, static_cast<cudaStream_t>(stream));
}

int mx_baseline_combine_pack(mx_plan* p, int rank, void* send, int32_t* counts_out, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  if (it.last - it.first != 1) { set_error("baseline helpers take one rank"); return MX_ERR_INVALID; }
  return launch_baseline_combine_pack(view_for(p, it.first), send, counts_out,
                                      static_cast<cudaStream_t>(stream));
}

int mx_baseline_combine_unpack(mx_plan* p, int rank, const void* recv, void* y, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  if (it.last - it.first != 1) { set_error("baseline helpers take one rank"); return MX_ERR_INVALID; }
  return launch_baseline_combine_unpack(view_for(p, it.first), recv, y,
                                        static_cast<cudaStream_t>(stream));
}

int mx_plan_check(mx_plan* p, int rank, void* stream) {
  RankIter it;
  int rc = ranks_for(p, rank, &it);
  if (rc) return rc;
  MX_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  return check_errors(p, it.first, it.last);
}

int mx_nvlink_probe(mx_plan* p, size_t bytes_per_peer, void* stream) {
  mx_comm* c = p->comm;
  if (c->emulate || c->W < 2) { set_error("the NVLink probe runs in SPMD mode with peers"); return MX_ERR_INVALID; }
  bytes_per_peer &= ~(size_t)4095;
  const size_t recv_bytes = p->off.partial - p->off.recv, part_bytes = p->off.y - p->off.partial;
  if (bytes_per_peer == 0 || bytes_per_peer * c->W > recv_bytes || bytes_per_peer > part_bytes) {
    set_error("probe needs 4 KB <= bytes_per_peer <= %zu", recv_bytes / c->W < part_bytes ? recv_bytes / c->W : part_bytes);
    return MX_ERR_INVALID;
  }
  return launch_nvlink_probe(view_for(p, c->rank), bytes_per_peer, static_cast<cudaStream_t>(stream));
}

int mx_grouped_gemm(const void* A, const void* B, void* D, int out_dtype, const int32_t* offs,
                    const int32_t* cnts, int G, long long M_total, int N, int K, int swiglu,
                    void* stream) {
  return grouped_gemm(A, B, D, out_dtype, offs, cnts, nullptr, G, M_total, M_total, N, K, swiglu,
                      static_cast<cudaStream_t>(stream));
}

}  // extern "C"
