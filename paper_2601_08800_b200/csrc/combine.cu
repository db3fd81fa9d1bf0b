// combine.cu -- K4: fused RS-combine (Alg. 1; sim:410-521).
//
// Reference schedule per destination: the host group reduce-scatters its TP
// partials (sim:436-441, sim:455-457), ships each reduced shard back to the
// token owner (sim:458-475), the owner accumulates w*row (sim:476-483,
// sim:508-520) and finally all-gathers its shards (sim:500-504).
//
// B200 form: owner rank (j,t) PULLS column shard t of every slot's partial
// from the m TP ranks of the slot's host over NVLink and sums them
// rank-ascending -- that is the reduce-scatter and the pairwise return in
// one hop, with the same bytes on the wire -- weights and accumulates in the
// reference's order (hosts j-1, j-2, ..., j; rows ascending, i.e. experts
// ascending within a token), then PUSHES the finished shard to every TP rank
// of its group (the final all-gather).  f64 is uncontracted and therefore
// bit-identical to the reference.
#include "mx_internal.cuh"

namespace mx {

// KU > 0: unrolled fast path for k <= KU -- every slot's load of a column
// vector is issued before any is consumed (KU x 16 B in flight per lane).
template <int DT, bool VEC, int KU>
__global__ void __launch_bounds__(256, 2) k_combine(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);  // every host's partials are written
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = VEC ? Elt<DT>::V : 1;  // elements per 16 B vector
  __shared__ int s_pos[8][MX_KMAX];
  __shared__ int s_src[8][MX_KMAX];  // first rank of the slot's host group
  __shared__ A s_w[8][MX_KMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = v.n, m = v.m, k = v.k, h = v.h, E = v.E, j = v.group;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const A* wts = at<A>(v, v.rank, v.off.w);
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  int c0, c1;
  col_shard(h, m, v.tp_rank, &c0, &c1);
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long tl = gw; tl < v.T; tl += nwarps) {
    int e = 0, key = 0x7fffffff, pos = 0;
    A w = (A)0;
    if (lane < k) {
      const size_t si = (size_t)tl * k + lane;
      e = ids[si];
      w = wts[si];
      pos = slot_pos[si];
      if (pos >= v.cap) { pos = 0; w = (A)0; }  // past capacity: never computed (mx_plan_check)
      const int d = home_of(e, n, E);
      key = (j - d - 1 + n) % n;  // arrival order (j-1, j-2, ..., j)
    }
    // rank of this slot in (arrival key, expert) order
    int rk = 0;
    for (int o = 0; o < k; ++o) {
      const int ok = __shfl_sync(0xffffffffu, key, o);
      const int oe = __shfl_sync(0xffffffffu, e, o);
      rk += (ok < key || (ok == key && oe < e)) ? 1 : 0;
    }
    if (lane < k) {
      s_pos[warp][rk] = pos;
      s_src[warp][rk] = home_of(e, n, E) * m;
      s_w[warp][rk] = w;
    }
    __syncwarp();
    if constexpr (KU > 0) {
      // exact mode (f64) keeps the reference association: per slot the TP
      // partials are summed rank-ascending first, then weighted (sim:436-441,
      // sim:519); the fp32-accumulating modes fold w into each partial,
      // which halves the live registers.
      constexpr bool EXACT = DT == MX_F64;
      A ws[KU];
      const T* bp[KU];  // slot rows on the host's TP rank 0 (tt = 0)
#pragma unroll
      for (int s = 0; s < KU; ++s) {
        const int ss = s < k ? s : 0;
        ws[s] = s_w[warp][ss];
        bp[s] = at<T>(v, s_src[warp][ss], v.off.partial) + (size_t)s_pos[warp][ss] * h;
      }
      for (int c = c0 + lane * V; c < c1; c += 32 * V) {
        A red[EXACT ? KU : 1][V];
        A acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = (A)0;
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
          if (tt >= m) break;
          uint4 raw[KU];
#pragma unroll
          for (int s = 0; s < KU; ++s) {
            if (s < k) {
              const T* p = tt == 0 ? bp[s] + c
                                   : at<T>(v, s_src[warp][s] + tt, v.off.partial) +
                                         (size_t)s_pos[warp][s] * h + c;
              if constexpr (VEC) raw[s] = ld_v4(p);
              else { T one = *p; raw[s].x = 0; *reinterpret_cast<T*>(&raw[s]) = one; }
            }
          }
#pragma unroll
          for (int s = 0; s < KU; ++s) {
            if (s < k) {
              const T* pv = reinterpret_cast<const T*>(&raw[s]);
#pragma unroll
              for (int q = 0; q < V; ++q) {
                if constexpr (EXACT)
                  red[s][q] = tt == 0 ? to_acc(pv[q]) : add_rn(red[s][q], to_acc(pv[q]));
                else
                  acc[q] = fmaf(ws[s], to_acc(pv[q]), acc[q]);
              }
            }
          }
        }
        if constexpr (EXACT) {
#pragma unroll
          for (int s = 0; s < KU; ++s)
            if (s < k) {
#pragma unroll
              for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], mul_rn(ws[s], red[s][q]));
            }
        }
        if (v.Is_t)  // shared expert: TP partials of the group's own tokens
          for (int tt = 0; tt < m; ++tt) {
            const uint4 raw = ld_v4(at<T>(v, j * m + tt, v.off.part_s) + (size_t)tl * h + c);
            const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
          }
        // final intra-group all-gather: push the shard to every TP rank
        for (int tt = 0; tt < m; ++tt) {
          T* y = at<T>(v, j * m + tt, v.off.y) + (size_t)tl * h + c;
          if constexpr (VEC) {
            T outv[V];
#pragma unroll
            for (int q = 0; q < V; ++q) outv[q] = from_acc<T>(acc[q]);
            st_v4(y, *reinterpret_cast<uint4*>(outv));
          } else {
            y[0] = from_acc<T>(acc[0]);
          }
        }
      }
    } else {
      for (int c = c0 + lane * V; c < c1; c += 32 * V) {
        A acc[V];
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = (A)0;
        for (int s = 0; s < k; ++s) {
          const size_t off = (size_t)s_pos[warp][s] * h + c;
          const int r0 = s_src[warp][s];
          A red[V];
          if constexpr (VEC) {
            uint4 raw = ld_v4(at<T>(v, r0, v.off.partial) + off);
            const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int q = 0; q < V; ++q) red[q] = to_acc(pv[q]);
            for (int tt = 1; tt < m; ++tt) {
              uint4 r2 = ld_v4(at<T>(v, r0 + tt, v.off.partial) + off);
              const T* p2 = reinterpret_cast<const T*>(&r2);
#pragma unroll
              for (int q = 0; q < V; ++q) red[q] = add_rn(red[q], to_acc(p2[q]));
            }
          } else {
            red[0] = to_acc(at<T>(v, r0, v.off.partial)[off]);
            for (int tt = 1; tt < m; ++tt)
              red[0] = add_rn(red[0], to_acc(at<T>(v, r0 + tt, v.off.partial)[off]));
          }
          const A ws = s_w[warp][s];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], mul_rn(ws, red[q]));
        }
        for (int tt = 0; tt < m; ++tt) {
          T* y = at<T>(v, j * m + tt, v.off.y) + (size_t)tl * h + c;
          if constexpr (VEC) {
            T outv[V];
#pragma unroll
            for (int q = 0; q < V; ++q) outv[q] = from_acc<T>(acc[q]);
            st_v4(y, *reinterpret_cast<uint4*>(outv));
          } else {
            y[0] = from_acc<T>(acc[0]);
          }
        }
      }
    }
    __syncwarp();
  }
  if (v.sync_signal) grid_signal_and_wait(v);  // y complete on every TP rank: barrier #4
}

// One group, no TP (the single-GPU layer): every slot row is a local
// PARTIAL row.  Warp per token; the token's slots are ordered experts
// ascending (k_combine's order for n = 1, so the sums are the same bits)
// and held as row pointers + weights in registers; each lane issues the
// loads of a column vector of every slot (k x 16 B in flight) before
// accumulating.  Registers bound the loads in flight: one column vector per
// slot per iteration (k x 16 B per lane) at three CTAs per SM (24 warps,
// ~96 KB in flight per SM) beats two vectors per slot at one CTA per SM
// (153 registers; capping it at 128 spills).
template <int KU>
__global__ void __launch_bounds__(256, 3) k_combine_local(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  using T = __nv_bfloat16;
  constexpr int V = 8;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int k = v.k, h = v.h;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const float* wts = at<float>(v, v.rank, v.off.w);
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  const T* part = at<T>(v, v.rank, v.off.partial);
  const T* part_s = at<T>(v, v.rank, v.off.part_s);
  T* y = at<T>(v, v.rank, v.off.y);
  for (long long t = gw; t < v.T; t += nwarps) {
    int e = 0x7fffffff, pos = 0;
    float w = 0.f;
    if (lane < k) {
      e = ids[t * k + lane];
      w = wts[t * k + lane];
      pos = slot_pos[t * k + lane];
      if (pos >= v.cap) { pos = 0; w = 0.f; }  // past capacity: never computed (mx_plan_check)
    }
    int rk = 0;  // rank of this slot among the token's experts (ascending)
    for (int o = 0; o < k; ++o) {
      const int oe = __shfl_sync(0xffffffffu, e, o);
      rk += oe < e ? 1 : 0;
    }
    unsigned rp[KU];  // slot rows (32-bit: registers are the budget here)
    float ws[KU];
#pragma unroll
    for (int s = 0; s < KU; ++s) {
      const unsigned who = __ballot_sync(0xffffffffu, lane < k && rk == s);
      const int src = who ? __ffs(who) - 1 : 0;
      const int p = __shfl_sync(0xffffffffu, pos, src);
      const float ww = __shfl_sync(0xffffffffu, w, src);
      rp[s] = (unsigned)p;
      ws[s] = who ? ww : 0.f;
    }
    int c = lane * V;
    for (; c < h; c += 32 * V) {
      uint4 raw[KU];
#pragma unroll
      for (int s = 0; s < KU; ++s)
        if (s < k) raw[s] = ld_v4(part + (size_t)rp[s] * h + c);
      float acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = 0.f;
#pragma unroll
      for (int s = 0; s < KU; ++s)
        if (s < k) {
          const T* pv = reinterpret_cast<const T*>(&raw[s]);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = fmaf(ws[s], to_acc(pv[q]), acc[q]);
        }
      if (v.Is_t) {  // shared expert (weight 1), after the routed slots as in k_combine
        const uint4 sraw = ld_v4(part_s + (size_t)t * h + c);
        const T* pv = reinterpret_cast<const T*>(&sraw);
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
      }
      T out[V];
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
      st_v4(y + (size_t)t * h + c, *reinterpret_cast<uint4*>(out));
    }
  }
}

template <int DT>
static void launch_combine_dt(const DevView& v, int blocks, cudaStream_t s) {
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  const bool vec = ((size_t)c0 * v.elt) % 16 == 0 && ((size_t)(c1 - c0) * v.elt) % 16 == 0 &&
                   ((size_t)v.h * v.elt) % 16 == 0;
  if (DT == MX_BF16 && vec && v.n == 1 && v.m == 1 && v.k <= 8 && !v.sync_wait &&
      !v.sync_signal) {
    long long b = (v.T + 7) / 8;
    pdl_launch(k_combine_local<8>, (int)(b < 148 * 8 ? b : 148 * 8), 256, 0, s, v);
  } else if (vec && v.k <= 8 && v.m <= 8) pdl_launch(k_combine<DT, true, 8>, blocks, 256, 0, s, v);
  else if (vec) pdl_launch(k_combine<DT, true, 0>, blocks, 256, 0, s, v);
  else pdl_launch(k_combine<DT, false, 0>, blocks, 256, 0, s, v);
}

int launch_combine(const DevView& v, cudaStream_t s) {
  if (v.T == 0) return MX_OK;
  if (v.k > MX_KMAX) return MX_ERR_UNSUPPORTED;
  long long blocks = (v.T + 7) / 8;
  if (blocks > 148 * 16) blocks = 148 * 16;
  switch (v.elt) {
    case 8: launch_combine_dt<MX_F64>(v, (int)blocks, s); break;
    case 4: launch_combine_dt<MX_F32>(v, (int)blocks, s); break;
    default: launch_combine_dt<MX_BF16>(v, (int)blocks, s);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
