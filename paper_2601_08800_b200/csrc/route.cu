// route.cu -- K1: fused top-k gate + per-expert counting + stable ranks +
// chunk prefix sums, and the layout pass that turns them into expert-major
// and token-major slot positions.
//
// Replaces the reference's O(T*k) Python loops:
//   RouterSpec (sim:143-186)            -> ids/weights (or the fused gate)
//   build_routing_table (sim:236-251)   -> token-major table index (slot_tm)
//   _slot_rows_from (sim:326-327)       -> send counts S[j][d] + tm offsets
//   _expert_rows (sim:528-532)          -> expert-major row (slot_pos)
//
// Order contracts (bit-exact with the reference):
//   host d's token-major table = all (token, expert) with home(expert)=d,
//   sorted by (global token, expert); expert-major = experts ascending,
//   inside an expert tokens ascending.  Groups own contiguous token blocks,
//   so both orders decompose into per-group contiguous sub-blocks whose
//   offsets only need the [n][E] count matrix.
#include "mx_internal.cuh"

namespace mx {

// Warp-wide fp32 max in one instruction (CREDUX.MAX.F32, sm_100a).
__device__ __forceinline__ float warp_max_f32(float v) {
  float m;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(v));
  return m;
}

// Fused softmax + top-k gate: one warp per token over all SMs.  Lane owns
// experts e = 128*i + 4*lane + q (128-bit coalesced row loads).  Selection
// key: fp32 logit descending, lowest id on ties (exact compares, so ids are
// bit-exact with the oracle).  Each lane sorts its candidates once; a round
// is two warp reductions -- the max key (redux.sync.max.f32) and the lowest
// id holding it (redux.sync.min) -- and a pop of the winning lane's list.
template <class WT, int EV>
__global__ void __launch_bounds__(256)
k_gate(DevView v, const float* __restrict__ logits) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const long long tok = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (tok >= v.T) return;
  const int E = v.E, k = v.k;
  int* ids = at<int>(v, v.rank, v.off.ids);
  WT* w = at<WT>(v, v.rank, v.off.w);
  const float* row = logits + (size_t)tok * E;
  float val[EV * 4];
#pragma unroll
  for (int i = 0; i < EV; ++i) {
    const int e0 = 128 * i + 4 * lane;
    if ((E % 4) == 0 && e0 < E) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(row + e0));
      val[4 * i] = f.x; val[4 * i + 1] = f.y; val[4 * i + 2] = f.z; val[4 * i + 3] = f.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) val[4 * i + q] = (e0 + q < E) ? __ldg(row + e0 + q) : -INFINITY;
    }
  }
  // each lane sorts its candidates once (key descending, lowest id first on
  // ties); a round then only advances the winning lane's list
  constexpr int NV = EV * 4;
  int se[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int e = 128 * (i >> 2) + 4 * lane + (i & 3);
    se[i] = e < E ? e : 0x7fffffff;
    if (e >= E) val[i] = -INFINITY;
  }
#pragma unroll
  for (int i = 1; i < NV; ++i) {
#pragma unroll
    for (int j = i; j > 0; --j) {
      const bool before = val[j] > val[j - 1] || (val[j] == val[j - 1] && se[j] < se[j - 1]);
      const float tv = before ? val[j - 1] : val[j];
      const int te = before ? se[j - 1] : se[j];
      val[j - 1] = before ? val[j] : val[j - 1];
      se[j - 1] = before ? se[j] : se[j - 1];
      val[j] = tv;
      se[j] = te;
    }
  }
  // softmax denominator over every expert (renormalize off): before the
  // rounds pop the winners out of the lists
  const float row_max = warp_max_f32(val[0]);
  float sacc = 0.f;
  if (!v.renorm) {
#pragma unroll
    for (int i = 0; i < NV; ++i) sacc += expf(val[i] - row_max);  // -inf pads add 0
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  }
  int my_e = 0;
  float my_v = 0.f;
  for (int r = 0; r < k; ++r) {
    const float bv = warp_max_f32(val[0]);
    const int be = (int)__reduce_min_sync(0xffffffffu, val[0] == bv ? (unsigned)se[0] : 0xffffffffu);
    if (lane == r) { my_e = be; my_v = bv; }
    if (be == se[0]) {  // this lane owned the winner: pop its list head
#pragma unroll
      for (int i = 0; i + 1 < NV; ++i) {
        val[i] = val[i + 1];
        se[i] = se[i + 1];
      }
      val[NV - 1] = -INFINITY;
      se[NV - 1] = 0x7fffffff;
    }
  }
  const float ex = (lane < k) ? expf(my_v - row_max) : 0.f;
  float denom;
  if (v.renorm) {
    denom = ex;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
  } else {
    denom = sacc;
  }
  if (lane < k) {
    ids[(size_t)tok * k + lane] = my_e;
    w[(size_t)tok * k + lane] = (WT)(ex / denom);
  }
}

// DeepSeek-V3 group-limited router (transformers modeling_deepseek_v3.py
// DeepseekV3MoE.route_tokens_to_experts), one warp per
// token, same lane ownership as k_gate.  s = sigmoid(logit) (evaluated in
// f64, rounded once to fp32 -- the oracle's definition), key c = s + bias;
// group score = sum of the group's top-2 c (a warp top-2 reduction per
// group); the r_topk_groups best groups stay (lowest group id on ties), c of
// every other expert becomes 0.0 (masked_fill, not -inf); top-k of that key
// (lowest id on ties); weight = s / (sum_r s_r + 1e-20) * scaling, the sum
// running in selection order.
template <class WT, int EV>
__global__ void __launch_bounds__(256)
k_gate_grouped(DevView v, const float* __restrict__ logits) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const long long tok = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (tok >= v.T) return;
  const int E = v.E, k = v.k, G = v.r_groups, gs = E / G;
  int* ids = at<int>(v, v.rank, v.off.ids);
  WT* w = at<WT>(v, v.rank, v.off.w);
  const float* row = logits + (size_t)tok * E;
  float key[EV * 4], sv[EV * 4];
#pragma unroll
  for (int i = 0; i < EV * 4; ++i) {
    const int e = 128 * (i >> 2) + 4 * lane + (i & 3);
    if (e < E) {
      const float x = __ldg(row + e);
      sv[i] = (float)(1.0 / (1.0 + exp(-(double)x)));
      key[i] = __fadd_rn(sv[i], v.r_bias ? __ldg(v.r_bias + e) : 0.f);
    } else {
      sv[i] = 0.f;
      key[i] = -INFINITY;
    }
  }
  // group scores: top-2 sum of the choice key per group
  unsigned keep = 0;
  {
    float gsc[32];
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      float m1 = -INFINITY, m2 = -INFINITY;
#pragma unroll
      for (int i = 0; i < EV * 4; ++i) {
        const int e = 128 * (i >> 2) + 4 * lane + (i & 3);
        if (e < E && e / gs == g) {
          const float c = key[i];
          if (c > m1) { m2 = m1; m1 = c; } else if (c > m2) { m2 = c; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float o1 = __shfl_xor_sync(0xffffffffu, m1, o);
        const float o2 = __shfl_xor_sync(0xffffffffu, m2, o);
        if (o1 >= m1) { m2 = fmaxf(m1, o2); m1 = o1; } else { m2 = fmaxf(m2, o1); }
      }
      gsc[g < 32 ? g : 31] = __fadd_rn(m1, m2);
    }
#pragma unroll 1
    for (int g = 0; g < G; ++g) {
      int rank = 0;
      for (int g2 = 0; g2 < G; ++g2)
        rank += (gsc[g2] > gsc[g] || (gsc[g2] == gsc[g] && g2 < g)) ? 1 : 0;
      if (rank < v.r_topk_groups) keep |= 1u << g;
    }
  }
#pragma unroll
  for (int i = 0; i < EV * 4; ++i) {
    const int e = 128 * (i >> 2) + 4 * lane + (i & 3);
    if (e < E && !((keep >> (e / gs)) & 1u)) key[i] = 0.f;
  }
  unsigned taken = 0;
  float cv, cs;
  int ce;
  auto rescan = [&]() {
    cv = -INFINITY;
    cs = 0.f;
    ce = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < EV * 4; ++i) {
      const int e = 128 * (i >> 2) + 4 * lane + (i & 3);
      if (e < E && !((taken >> i) & 1u) && (key[i] > cv || (key[i] == cv && e < ce))) {
        cv = key[i];
        cs = sv[i];
        ce = e;
      }
    }
  };
  rescan();
  int my_e = 0;
  float my_s = 0.f;
  for (int r = 0; r < k; ++r) {
    const float bv = warp_max_f32(cv);
    const int be = (int)__reduce_min_sync(0xffffffffu, cv == bv ? (unsigned)ce : 0xffffffffu);
    const unsigned own = __ballot_sync(0xffffffffu, be == ce);
    const float ws = __shfl_sync(0xffffffffu, cs, __ffs(own) - 1);
    if (lane == r) { my_e = be; my_s = ws; }
    if (be == ce) {  // this lane owned the winner
      taken |= 1u << (4 * (be >> 7) + (be & 3));
      rescan();
    }
  }
  float wt = my_s;
  if (v.renorm) {
    float den = 0.f;
    for (int r = 0; r < k; ++r) den = __fadd_rn(den, __shfl_sync(0xffffffffu, my_s, r));
    den = __fadd_rn(den, 1e-20f);
    wt = __fdiv_rn(my_s, den);
  }
  wt = __fmul_rn(wt, v.r_scaling);
  if (lane < k) {
    ids[(size_t)tok * k + lane] = my_e;
    w[(size_t)tok * k + lane] = (WT)wt;
  }
}

// One CTA per chunk of MX_CHUNK tokens of this rank's group.
template <class WT>
__global__ void __launch_bounds__(512)
k_route(DevView v, const float* __restrict__ logits, const int32_t* __restrict__ ids_in,
        const WT* __restrict__ w_in) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = v.T, E = v.E, k = v.k, n = v.n;
  const int c = blockIdx.x, t0 = c * MX_CHUNK;
  const int nt = min(MX_CHUNK, T - t0);
  int* s_ids = reinterpret_cast<int*>(smem);                      // [CHUNK*k]
  unsigned* s_mask = reinterpret_cast<unsigned*>(s_ids + MX_CHUNK * k);  // [E][4]
  int* s_hc = reinterpret_cast<int*>(s_mask + E * 4);             // [CHUNK][n]
  int* s_home = s_hc + MX_CHUNK * n;                              // [E]
  int* s_hp = s_home + E;                                         // [CHUNK][n]

  int* ids = at<int>(v, v.rank, v.off.ids);
  WT* w = at<WT>(v, v.rank, v.off.w);
  int* slot_rank = at<int>(v, v.rank, v.off.slot_rank);
  int* slot_tmr = at<int>(v, v.rank, v.off.slot_tmr);
  int* chunk_hist = at<int>(v, v.rank, v.off.chunk_hist);
  int* chunk_host = at<int>(v, v.rank, v.off.chunk_host);
  int* chunk_pair = at<int>(v, v.rank, v.off.chunk_pair);
  int* tok_pair_rank = at<int>(v, v.rank, v.off.tok_pair_rank);
  int* err = at<int>(v, v.rank, v.off.err);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;

  for (int i = threadIdx.x; i < E * 4; i += blockDim.x) s_mask[i] = 0;
  for (int i = threadIdx.x; i < MX_CHUNK * n; i += blockDim.x) s_hc[i] = 0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_home[e] = home_of(e, n, E);

  if (logits != nullptr) {
    // gate already ran (k_gate): ids/weights are in this rank's buffers
    for (int i = threadIdx.x; i < nt * k; i += blockDim.x) s_ids[i] = ids[(size_t)t0 * k + i];
  } else {
    // ---- explicit routing (RouterSpec ids/weights, sim:143-166)
    for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
      const size_t si = (size_t)t0 * k + i;
      int e = ids_in[si];
      if (e < 0 || e >= E) { atomicOr(err + 1, 1); e = 0; }
      ids[si] = e;
      w[si] = w_in[si];
      s_ids[i] = e;
    }
  }
  __syncthreads();

  // ---- per-expert token bitmaps of this chunk
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
    const int e = s_ids[i], tl = i / k;
    atomicOr(&s_mask[e * 4 + (tl >> 5)], 1u << (tl & 31));
  }
  __syncthreads();

  // ---- stable rank of each slot among the chunk's tokens of its expert,
  //      and per-token host counts (token-major table order); thread per slot
  for (int i = threadIdx.x; i < nt * k; i += blockDim.x) {
    const int tl = i / k, base = tl * k;
    const int e = s_ids[i];
    const int d = s_home[e];
    int rk = 0;
    for (int wd = 0; wd < (tl >> 5); ++wd) rk += __popc(s_mask[e * 4 + wd]);
    rk += __popc(s_mask[e * 4 + (tl >> 5)] & ((1u << (tl & 31)) - 1u));
    int within = 0;  // experts of this token on host d with a smaller id
    for (int i2 = 0; i2 < k; ++i2) {
      const int e2 = s_ids[base + i2];
      within += (e2 < e && s_home[e2] == d) ? 1 : 0;
    }
    const size_t si = (size_t)t0 * k + i;
    slot_rank[si] = rk;
    slot_tmr[si] = within;
    atomicAdd(&s_hc[tl * n + d], 1);
  }
  __syncthreads();
  // exclusive scans over the chunk's tokens (4 per lane) of (a) the slot
  // counts per host (token-major table index) and (b) the indicator "token
  // has an expert on host d" ((token, host) pair index, wire TOKEN)
  for (int d = warp; d < n; d += nw) {
    int a[4], run = 0, pa[4], prun = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tl = 4 * lane + q;
      a[q] = (tl < nt) ? s_hc[tl * n + d] : 0;
      pa[q] = a[q] > 0 ? 1 : 0;
      run += a[q];
      prun += pa[q];
    }
    int incl = run, pincl = prun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      const int py = __shfl_up_sync(0xffffffffu, pincl, o);
      if (lane >= o) { incl += y; pincl += py; }
    }
    int ex = incl - run, pex = pincl - prun;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tl = 4 * lane + q;
      s_hc[tl * n + d] = ex;
      s_hp[tl * n + d] = pa[q] ? pex : -1;
      ex += a[q];
      pex += pa[q];
    }
    if (lane == 31) {
      chunk_host[d * v.C + c] = incl;
      chunk_pair[d * v.C + c] = pincl;
    }
  }
  __syncthreads();
  if (threadIdx.x < nt) {
    const int tl = threadIdx.x;
    for (int i = 0; i < k; ++i) {
      const int e = s_ids[tl * k + i];
      const size_t si = (size_t)(t0 + tl) * k + i;
      slot_tmr[si] += s_hc[tl * n + s_home[e]];
    }
    for (int d = 0; d < n; ++d) tok_pair_rank[(size_t)(t0 + tl) * n + d] = s_hp[tl * n + d];
  }
  if (v.C > 1) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      chunk_hist[e * v.C + c] = __popc(s_mask[e * 4]) + __popc(s_mask[e * 4 + 1]) +
                                __popc(s_mask[e * 4 + 2]) + __popc(s_mask[e * 4 + 3]);
    }
    return;
  }
  // one chunk (decode-sized groups): the chunk scans of k_route_scan are
  // trivial -- every exclusive prefix is 0 and the totals are this CTA's
  // counts -- so they are done here and the scan kernel is not launched
  __syncthreads();  // chunk_host / chunk_pair of this chunk are written above
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int tot = __popc(s_mask[e * 4]) + __popc(s_mask[e * 4 + 1]) +
                    __popc(s_mask[e * 4 + 2]) + __popc(s_mask[e * 4 + 3]);
    chunk_hist[e] = 0;
    for (int r = 0; r < v.W; ++r) at<int>(v, r, v.off.cnt_all)[v.group * E + e] = tot;
  }
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    const int u = chunk_pair[d];
    chunk_host[d] = 0;
    chunk_pair[d] = 0;
    for (int r = 0; r < v.W; ++r) at<int>(v, r, v.off.ucnt_all)[v.group * n + d] = u;
  }
  if (v.sync_signal) grid_signal(v);  // counts published: barrier #1
}

// Exclusive prefix of the chunk counts, one warp per expert (and per host),
// coalesced over the expert-major [E][C] layout; publishes the group's
// per-expert totals into every rank's count matrix (peer stores in SPMD).
__global__ void __launch_bounds__(256) k_route_scan(DevView v) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int E = v.E, n = v.n, C = v.C;
  int* row = nullptr;
  if (w < E) row = at<int>(v, v.rank, v.off.chunk_hist) + (size_t)w * C;
  else if (w < E + n) row = at<int>(v, v.rank, v.off.chunk_host) + (size_t)(w - E) * C;
  else if (w < E + 2 * n) row = at<int>(v, v.rank, v.off.chunk_pair) + (size_t)(w - E - n) * C;
  int carry = 0;
  for (int base = 0; row && base < C; base += 32) {
    const int c = base + lane;
    const int x = (c < C) ? row[c] : 0;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (c < C) row[c] = carry + incl - x;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (w < E && lane < v.W) {
    at<int>(v, lane, v.off.cnt_all)[v.group * E + w] = carry;
  }
  if (w < E && v.W > 32) {
    for (int r = 32 + lane; r < v.W; r += 32) at<int>(v, r, v.off.cnt_all)[v.group * E + w] = carry;
  }
  if (row && w >= E + n) {  // (token, host) pair totals U[group][d], published like the counts
    const int d = w - E - n;
    for (int r = lane; r < v.W; r += 32) at<int>(v, r, v.off.ucnt_all)[v.group * n + d] = carry;
  }
  if (v.sync_signal) grid_signal(v);  // counts published: barrier #1
}


// Layout in one launch: every CTA rebuilds the offset tables it needs from
// the gathered [n][E] count matrix in shared memory (a few KB), CTA 0 also
// publishes the global tables (exp_off/exp_cnt/grp_off/send/...) for later kernels;
// then the grid writes every slot's expert-major row and token-major index
// and every (token, host) pair row.
__global__ void __launch_bounds__(512) k_layout(DevView v) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);  // every group's counts have landed
  extern __shared__ int sm[];
  const int n = v.n, E = v.E, k = v.k, j = v.group;
  int* s_cnt = sm;                   // [n][E]
  int* s_exp_off = s_cnt + n * E;    // [E]
  int* s_grp_off = s_exp_off + E;    // [E] rows of groups < j, per expert
  int* s_send = s_grp_off + E;       // [n][n]
  int* s_tm = s_send + n * n;        // [n]  tm_off[j][d]
  int* s_po = s_tm + n;              // [n]  poff[j][d]
  int* s_part = s_po + n;            // [blockDim] scan partials
  const int* cnt = at<int>(v, v.rank, v.off.cnt_all);
  const int* ucnt = at<int>(v, v.rank, v.off.ucnt_all);
  const bool pub = blockIdx.x == 0;
  // this thread's first slot, loaded under the table prologue below
  const long long q_first = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int pf_e = 0, pf_r = 0, pf_m = 0;
  if (q_first < (long long)v.T * k) {
    pf_e = at<int>(v, v.rank, v.off.ids)[q_first];
    pf_r = at<int>(v, v.rank, v.off.slot_rank)[q_first];
    pf_m = at<int>(v, v.rank, v.off.slot_tmr)[q_first];
  }
  for (int i = threadIdx.x; i < n * E; i += blockDim.x) s_cnt[i] = cnt[i];
  __syncthreads();
  // per-expert totals, own-group offsets, host-segmented exclusive scan
  const int per = (E + blockDim.x - 1) / blockDim.x;
  const int e_lo = threadIdx.x * per, e_hi = min(E, e_lo + per);
  int run = 0;
  for (int e = e_lo; e < e_hi; ++e) {
    int tot = 0, mine = 0;
    for (int g = 0; g < n; ++g) {
      if (g == j) mine = tot;
      if (pub) at<int>(v, v.rank, v.off.grp_off)[g * E + e] = tot;
      tot += s_cnt[g * E + e];
    }
    s_grp_off[e] = mine;
    s_exp_off[e] = tot;  // holds totals until the scan below
    if (pub) at<int>(v, v.rank, v.off.exp_cnt)[e] = tot;
    run += tot;
  }
  {  // block-wide exclusive scan of the per-thread totals (warp shuffles)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_part[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int nw = blockDim.x >> 5;
      const int x = lane < nw ? s_part[lane] : 0;
      int wincl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, wincl, o);
        if (lane >= o) wincl += y;
      }
      if (lane < nw) s_part[lane] = wincl - x;
    }
    __syncthreads();
    run = s_part[wid] + incl - run;
    __syncthreads();
  }
  for (int e = e_lo; e < e_hi; ++e) {  // global exclusive prefix of totals
    const int tot = s_exp_off[e];
    s_exp_off[e] = run;
    run += tot;
  }
  __syncthreads();
  // host-segmented: subtract the prefix at the first expert of each host
  int* tmp = s_part;  // reuse: host segment bases (n <= blockDim)
  for (int d = threadIdx.x; d < n; d += blockDim.x) tmp[d] = s_exp_off[first_expert(d, n, E)];
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_exp_off[e] -= tmp[home_of(e, n, E)];
  }
  __syncthreads();
  if (pub) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) at<int>(v, v.rank, v.off.exp_off)[e] = s_exp_off[e];
    // source-group sub-blocks of this host's expert segments (rows grouped
    // by source group inside each expert): the own group's block, and the
    // blocks before / after it (the other groups' rows)
    const int e0 = first_expert(j, n, E), e1 = first_expert(j + 1, n, E), S = 2 * E;
    int* sub = at<int>(v, v.rank, v.off.sub);
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int i = e - e0, base = s_exp_off[e], before = s_grp_off[e], own = s_cnt[j * E + e];
      int tot = 0;
      for (int g = 0; g < n; ++g) tot += s_cnt[g * E + e];
      sub[i] = base + before;
      sub[S + i] = own;
      sub[2 * S + 2 * i] = base;
      sub[3 * S + 2 * i] = before;
      sub[4 * S + 2 * i] = i;
      sub[2 * S + 2 * i + 1] = base + before + own;
      sub[3 * S + 2 * i + 1] = tot - before - own;
      sub[4 * S + 2 * i + 1] = i;
    }
  }
  // send counts, token-major offsets, pair offsets
  for (int jd = threadIdx.x; jd < n * n; jd += blockDim.x) {
    const int g = jd / n, d = jd % n;
    const int e0 = first_expert(d, n, E), e1 = first_expert(d + 1, n, E);
    int sum = 0;
    for (int x = e0; x < e1; ++x) sum += s_cnt[g * E + x];
    s_send[jd] = sum;
    if (pub) at<int>(v, v.rank, v.off.send)[jd] = sum;
  }
  __syncthreads();
  for (int jd = threadIdx.x; jd < n * n; jd += blockDim.x) {
    const int g = jd / n, d = jd % n;
    int tm = 0, po = 0;
    for (int g2 = 0; g2 < g; ++g2) { tm += s_send[g2 * n + d]; po += ucnt[g2 * n + d]; }
    if (g == j) { s_tm[d] = tm; s_po[d] = po; }
    if (pub) {
      at<int>(v, v.rank, v.off.tm_off)[jd] = tm;
      at<int>(v, v.rank, v.off.poff)[jd] = po;
      if (g == n - 1) {
        at<int>(v, v.rank, v.off.host_pairs)[d] = po + ucnt[jd];
        const int rows = tm + s_send[jd];
        at<int>(v, v.rank, v.off.host_rows)[d] = rows;
        if ((long long)rows > v.cap) atomicMax(at<int>(v, v.rank, v.off.err) + 0, rows);
      }
    }
  }
  __syncthreads();
  // slot positions
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const int* slot_rank = at<int>(v, v.rank, v.off.slot_rank);
  const int* slot_tmr = at<int>(v, v.rank, v.off.slot_tmr);
  const int* chunk_hist = at<int>(v, v.rank, v.off.chunk_hist);
  const int* chunk_host = at<int>(v, v.rank, v.off.chunk_host);
  int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  int* slot_tm = at<int>(v, v.rank, v.off.slot_tm);
  int* err = at<int>(v, v.rank, v.off.err);
  const long long total = (long long)v.T * k;
  for (long long q = q_first; q < total; q += (long long)gridDim.x * blockDim.x) {
    const bool first = q == q_first;
    const int t = (int)(q / k);
    const int e = first ? pf_e : ids[q];
    const int d = home_of(e, n, E);
    const int c = t / MX_CHUNK;
    const long long pos = (long long)s_exp_off[e] + s_grp_off[e] + chunk_hist[e * v.C + c] +
                          (first ? pf_r : slot_rank[q]);
    if (pos >= v.cap) atomicOr(err + 3, 1);
    slot_pos[q] = (int)pos;
    slot_tm[q] = s_tm[d] + chunk_host[d * v.C + c] + (first ? pf_m : slot_tmr[q]);
  }
  const int* tpr = at<int>(v, v.rank, v.off.tok_pair_rank);
  const int* chunk_pair = at<int>(v, v.rank, v.off.chunk_pair);
  int* upos = at<int>(v, v.rank, v.off.upos);
  const long long tn = (long long)v.T * n;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < tn;
       q += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(q / n), d = (int)(q % n);
    const int r = tpr[q];
    upos[q] = r < 0 ? -1 : s_po[d] + chunk_pair[d * v.C + t / MX_CHUNK] + r;
  }
}

template <class WT, int EV>
static void launch_gate_ev(const DevView& v, const float* logits, cudaStream_t s) {
  if (v.router == MX_ROUTER_GROUP_LIMITED)
    pdl_launch(k_gate_grouped<WT, EV>, (v.T + 7) / 8, 256, 0, s, v, logits);
  else
    pdl_launch(k_gate<WT, EV>, (v.T + 7) / 8, 256, 0, s, v, logits);
}

template <class WT>
static int launch_route_wt(const DevView& v, int C, size_t smem, const float* logits,
                           const int32_t* ids, const void* w, cudaStream_t s) {
  if (logits) {
    if (v.E <= 128) launch_gate_ev<WT, 1>(v, logits, s);
    else if (v.E <= 256) launch_gate_ev<WT, 2>(v, logits, s);
    else if (v.E <= 512) launch_gate_ev<WT, 4>(v, logits, s);
    else launch_gate_ev<WT, 8>(v, logits, s);
    MX_LAUNCH_CHECK();
  }
  static bool attr = false;
  if (!attr) {
    MX_CUDA(cudaFuncSetAttribute(k_route<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  pdl_launch(k_route<WT>, C, 512, smem, s, v, logits, ids, static_cast<const WT*>(w));
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_route(const DevView& v, const float* logits, const int32_t* ids,
                 const void* w, cudaStream_t s) {
  const int C = v.C;
  if (C == 0) return MX_OK;
  const size_t smem = (size_t)MX_CHUNK * v.k * 4 + (size_t)v.E * 16 + (size_t)MX_CHUNK * v.n * 8 +
                      (size_t)v.E * 4;
  int rc = v.elt == 8 ? launch_route_wt<double>(v, C, smem, logits, ids, w, s)
                      : launch_route_wt<float>(v, C, smem, logits, ids, w, s);
  if (rc) return rc;
  if (C == 1) return MX_OK;  // k_route did the (trivial) scans itself
  const int warps = v.E + 2 * v.n;
  pdl_launch(k_route_scan, (warps + 7) / 8, 256, 0, s, v);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_layout(const DevView& v, cudaStream_t s) {
  const size_t smem = ((size_t)v.n * v.E + 2 * v.E + (size_t)v.n * v.n + 2 * v.n + 512) * 4;
  static bool attr = false;
  if (!attr) {
    MX_CUDA(cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  if (smem > 200 * 1024) { set_error("layout tables exceed shared memory (n*E too large)"); return MX_ERR_UNSUPPORTED; }
  const long long work = (long long)v.T * (v.k > v.n ? v.k : v.n);
  long long blocks = (work + 511) / 512;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 2) blocks = 148 * 2;
  pdl_launch(k_layout, (int)blocks, 512, smem, s, v);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
