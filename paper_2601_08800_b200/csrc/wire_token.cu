// wire_token.cu -- TOKEN wire format: one row per (token, host group) pair.
//
// The reference ships one row per routed slot in both directions: a token
// routed to several experts of the same remote group crosses the link once
// per expert (sim:366-369, sim:403-405), and the combine
// returns one TP-reduced row per slot (sim:458-475).  The routing table, the
// per-(src, dst) slot lists and the send counts stay exactly the reference's
// (K1 computes them); only the bytes on NVLink change:
//   dispatch: each (token, host) row crosses NVLink once into the host's
//             XBUF; the host expands XBUF rows into its expert-major RECV
//             (local HBM copy) before the grouped GEMM;
//   combine:  each host TP rank pre-reduces z[u] = sum_i w_i * partial[p_i]
//             over the token's slots on that host (experts ascending) and
//             pushes z's column shards straight into the owners' ZIN; the
//             owner sums its local ZIN planes.
// NVLink bytes per token drop from k rows to (#hosts hit) rows each way.
#include "mx_internal.cuh"

namespace mx {

constexpr int DSPLIT = 2;  // warps per token in the dispatch

// One pair-list entry: expert-major row of the slot and its top-k weight,
// written with a single remote store.
template <class WT> struct PairEnt;
template <> struct __align__(8) PairEnt<float> { int p; float w; };
template <> struct __align__(16) PairEnt<double> { int p; int pad; double w; };

__device__ __forceinline__ void copy_row(char* dst, const char* src, size_t nbytes, int lane) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes) & 15) == 0) {
    const size_t nv = nbytes >> 4;
    size_t i = lane;
    for (; i + 32 < nv; i += 64) {
      const uint4 a = ld_v4(src + (i << 4));
      const uint4 b = ld_v4(src + ((i + 32) << 4));
      st_v4(dst + (i << 4), a);
      st_v4(dst + ((i + 32) << 4), b);
    }
    for (; i < nv; i += 32) st_v4(dst + (i << 4), ld_v4(src + (i << 4)));
  } else {
    for (size_t i = lane; i < nbytes; i += 32) dst[i] = src[i];
  }
}

// Warp per token: ship the row (column shard tp_rank, or the full row to the
// own group) once per host it hits, then publish per-slot metadata to the TP
// peer on that host: the pair's packed (slot row, weight) list and its length.
template <class WT>
__global__ void __launch_bounds__(256) k_dispatch_token(DevView v, const char* __restrict__ x) {
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  // DSPLIT warps per token, each moving its slice of the row's 16 B vectors
  // (more stores in flight per SM); warp 0 of a token also writes metadata
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int sub = (int)(gw % DSPLIT);
  const int n = v.n, m = v.m, k = v.k, E = v.E;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const WT* wts = at<WT>(v, v.rank, v.off.w);
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  const int* upos = at<int>(v, v.rank, v.off.upos);
  const size_t row_bytes = (size_t)v.wrow;
  const size_t body = (size_t)v.h * v.welt;
  int c0, c1;
  col_shard(v.h, m, v.tp_rank, &c0, &c1);
  const size_t sh_off = (size_t)c0 * v.welt, sh_bytes = (size_t)(c1 - c0) * v.welt;
  const bool tail = v.tp_rank == 0 && row_bytes > body;
  // own-group rows go straight to their expert-major RECV rows (the local
  // hop needs no dedup); the XBUF keeps them only for the gathered GEMM1
  const bool aligned = ((sh_off | sh_bytes | row_bytes) & 15) == 0;
  const bool direct_local = v.a_src == nullptr && aligned;
  const size_t nv_row = row_bytes >> 4, nv_sh = sh_bytes >> 4;
  const size_t r_lo = sub * nv_row / DSPLIT, r_hi = (sub + 1) * nv_row / DSPLIT;
  const size_t s_lo = sub * nv_sh / DSPLIT, s_hi = (sub + 1) * nv_sh / DSPLIT;
  for (long long t = gw / DSPLIT; t < v.T; t += nwarps / DSPLIT) {
    const char* row = x + (size_t)t * row_bytes;
    for (int d = 0; d < n; ++d) {
      const int u = upos[t * n + d];
      if (u < 0) continue;
      if (d == v.group && direct_local) {
        // rows of this token's slots on the own host (pos < cap: layout-checked)
        int pos = -1;
        if (lane < k) {
          const int e = ids[t * k + lane];
          const int p = slot_pos[t * k + lane];
          if (home_of(e, n, E) == d && p < v.cap) pos = p;
        }
        const unsigned mine = __ballot_sync(0xffffffffu, pos >= 0);
        char* recv = at<char>(v, v.rank, v.off.recv);
        // warp-uniform passes (the slot broadcast below is a full-warp
        // shuffle), each lane predicated on its own vectors
        for (size_t base = r_lo; base < r_hi; base += 128) {
          uint4 val[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const size_t i = base + lane + 32 * q;
            if (i < r_hi) val[q] = ld_v4(row + (i << 4));
          }
          for (unsigned b = mine; b; b &= b - 1) {
            const int p = __shfl_sync(0xffffffffu, pos, __ffs(b) - 1);
            char* dst = recv + (size_t)p * row_bytes;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const size_t i = base + lane + 32 * q;
              if (i < r_hi) st_v4(dst + (i << 4), val[q]);
            }
          }
        }
      } else if (d == v.group) {
        if (sub == 0)
          copy_row(at<char>(v, v.rank, v.off.xbuf) + (size_t)u * row_bytes, row, row_bytes, lane);
      } else if (aligned) {
        // the shard is loaded once and stored to every TP rank of host d
        const char* src = row + sh_off;
        for (size_t i = s_lo + lane; i < s_hi; i += 128) {
          uint4 val[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (i + 32 * q < s_hi) val[q] = ld_v4(src + ((i + 32 * q) << 4));
          for (int tt = 0; tt < m; ++tt) {
            char* dst = at<char>(v, d * m + tt, v.off.xbuf) + (size_t)u * row_bytes + sh_off;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (i + 32 * q < s_hi) st_v4(dst + ((i + 32 * q) << 4), val[q]);
          }
        }
        if (tail && sub == 0)
          for (int tt = 0; tt < m; ++tt)
            copy_row(at<char>(v, d * m + tt, v.off.xbuf) + (size_t)u * row_bytes + body,
                     row + body, row_bytes - body, lane);
      } else if (sub == 0) {
        for (int tt = 0; tt < m; ++tt) {
          char* dst = at<char>(v, d * m + tt, v.off.xbuf) + (size_t)u * row_bytes;
          copy_row(dst + sh_off, row + sh_off, sh_bytes, lane);
          if (tail) copy_row(dst + body, row + body, row_bytes - body, lane);
        }
      }
    }
    if (sub != 0) continue;
    // metadata: lane i carries slot i
    int e = 0, d = -1;
    if (lane < k) {
      e = ids[t * k + lane];
      d = home_of(e, n, E);
    }
    int idx = 0, cnt = 0;
    for (int o = 0; o < k; ++o) {
      const int oe = __shfl_sync(0xffffffffu, e, o);
      const int od = __shfl_sync(0xffffffffu, d, o);
      if (od == d) {
        ++cnt;
        if (oe < e) ++idx;
      }
    }
    if (lane < k) {
      const int u = upos[t * n + d];
      const int p = slot_pos[t * k + lane];
      const int dst = d * m + v.tp_rank;  // the TP peer that reads this metadata
      PairEnt<WT> ent;
      ent.p = p;
      ent.w = wts[t * k + lane];
      reinterpret_cast<PairEnt<WT>*>(at<char>(v, dst, v.off.pair_p))[(size_t)u * v.KH + idx] = ent;
      if (idx == 0) {
        at<int>(v, dst, v.off.pair_n)[u] = cnt;
        at<int>(v, dst, v.off.pair_tok)[u] = v.group * v.T + (int)t;
      }
    }
  }
  if (v.sync_signal) grid_signal(v);  // rows + pair lists landed: barrier #2
}

// Host side: expert-major RECV rows from the deduplicated XBUF (local HBM),
// warp per pair: each 512 B column chunk of the pair's row is loaded once and
// stored to every slot row of the pair.
template <class WT>
__global__ void __launch_bounds__(256) k_expand(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int pairs = at<int>(v, v.rank, v.off.host_pairs)[v.group];
  const int* pn = at<int>(v, v.rank, v.off.pair_n);
  const PairEnt<WT>* pe = reinterpret_cast<const PairEnt<WT>*>(at<char>(v, v.rank, v.off.pair_p));
  const size_t row_bytes = (size_t)v.wrow;
  const char* xbuf = at<char>(v, v.rank, v.off.xbuf);
  char* recv = at<char>(v, v.rank, v.off.recv);
  // own-group pairs were written straight into RECV by the dispatch
  long long skip0 = 0, skip1 = 0;
  if (v.a_src == nullptr && (row_bytes & 15) == 0) {
    const int g = v.group;
    skip0 = at<int>(v, v.rank, v.off.poff)[g * v.n + g];
    skip1 = skip0 + at<int>(v, v.rank, v.off.ucnt_all)[g * v.n + g];
  }
  // warps walk only the pairs left to expand (the own-group block skipped)
  const long long todo = pairs - (skip1 - skip0);
  for (long long r = gw; r < todo; r += nwarps) {
    const long long u = r < skip0 ? r : r + (skip1 - skip0);
    const int cnt = pn[u];
    int rows[MX_KMAX];
    for (int i = 0; i < cnt; ++i) rows[i] = pe[u * v.KH + i].p;
    const char* src = xbuf + (size_t)u * row_bytes;
    size_t o = (size_t)lane * 16;
    for (; o + 3 * 512 < row_bytes; o += 4 * 512) {  // 4 x 16 B loads in flight per lane
      uint4 val[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) val[q] = ld_v4(src + o + q * 512);
      for (int i = 0; i < cnt; ++i) {
        char* dst = recv + (size_t)rows[i] * row_bytes + o;
#pragma unroll
        for (int q = 0; q < 4; ++q) st_v4(dst + q * 512, val[q]);
      }
    }
    for (; o < row_bytes; o += 512) {
      const uint4 val = ld_v4(src + o);
      for (int i = 0; i < cnt; ++i) st_v4(recv + (size_t)rows[i] * row_bytes + o, val);
    }
  }
}

// Destination of column c of pair-reduced row z (owner token tok = j*T + t)
// in the owner's shard: TP rank tt of group j owns columns [c0, c1) and keeps
// one [T][sw] plane per (host, host TP rank) in its ZIN.
template <class T>
__device__ __forceinline__ T* zin_dst(const DevView& v, int tok, int c, int sw) {
  const int j = tok / v.T, t = tok - j * v.T;
  int tt = 0, c0 = 0, c1 = 0;
  for (; tt < v.m; ++tt) {
    col_shard(v.h, v.m, tt, &c0, &c1);
    if (c < c1) break;
  }
  return at<T>(v, j * v.m + tt, v.off.zin) +
         (((size_t)v.group * v.m + v.tp_rank) * v.T + t) * sw + (c - c0);
}

// z = sum over the pair's slots (experts ascending) of w * partial[p], pushed
// straight into the owners' shards over NVLink (the reduce-scatter of the
// combine fused into the pre-reduction: the owner then only reads local
// memory); all slot loads of a column vector are issued before use.

template <int DT, class WT>
__global__ void __launch_bounds__(256, 2) k_pair_reduce(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = Elt<DT>::V;
  constexpr int KU = 8;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int pairs = at<int>(v, v.rank, v.off.host_pairs)[v.group];
  const int* pn = at<int>(v, v.rank, v.off.pair_n);
  const PairEnt<WT>* pe = reinterpret_cast<const PairEnt<WT>*>(at<char>(v, v.rank, v.off.pair_p));
  const T* part = at<T>(v, v.rank, v.off.partial);
  const int* ptok = at<int>(v, v.rank, v.off.pair_tok);
  const int h = v.h, sw = (h + v.m - 1) / v.m;
  for (long long u = gw; u < pairs; u += nwarps) {
    const int cnt = pn[u];
    const int tok = ptok[u];
    const T* rp[KU];
    A w[KU];
#pragma unroll
    for (int i = 0; i < KU; ++i) {
      const PairEnt<WT> e = pe[u * v.KH + (i < cnt ? i : 0)];
      rp[i] = part + (size_t)e.p * h;
      w[i] = (A)e.w;
    }
    int c = lane * V;
    if (cnt <= KU) {
      for (; c + 32 * V < h; c += 64 * V) {  // two column vectors per lane: 2 x cnt loads in flight
        uint4 raw[2][KU];
#pragma unroll
        for (int i = 0; i < KU; ++i)
          if (i < cnt) {
            raw[0][i] = ld_v4(rp[i] + c);
            raw[1][i] = ld_v4(rp[i] + c + 32 * V);
          }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          A acc[V];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = (A)0;
#pragma unroll
          for (int i = 0; i < KU; ++i)
            if (i < cnt) {
              const T* pv = reinterpret_cast<const T*>(&raw[hh][i]);
#pragma unroll
              for (int q = 0; q < V; ++q) {
                if constexpr (DT == MX_F64)  // reference association, uncontracted
                  acc[q] = add_rn(acc[q], mul_rn(w[i], to_acc(pv[q])));
                else
                  acc[q] = fmaf(w[i], to_acc(pv[q]), acc[q]);
              }
            }
          T out[V];
#pragma unroll
          for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
          st_v4(zin_dst<T>(v, tok, c + hh * 32 * V, sw), *reinterpret_cast<uint4*>(out));
        }
      }
    }
    for (; c < h; c += 32 * V) {
      A acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = (A)0;
      for (int i = 0; i < cnt; ++i) {
        const PairEnt<WT> e = pe[u * v.KH + i];
        const uint4 raw = ld_v4(part + (size_t)e.p * h + c);
        const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], mul_rn((A)e.w, to_acc(pv[q])));
      }
      T out[V];
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
      st_v4(zin_dst<T>(v, tok, c, sw), *reinterpret_cast<uint4*>(out));
    }
  }
  if (v.sync_signal) grid_signal(v);  // every owner's ZIN written: barrier #3
}

// Owner (j, t): y[tok, cols t] = sum over host TP ranks (ascending) and hosts
// (j-1, ..., j) of the pre-reduced partials the hosts pushed into this rank's
// ZIN; then push the shard to every TP rank of the group (final all-gather).
template <int DT>
__global__ void __launch_bounds__(256) k_combine_token(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);  // every host's pushes into ZIN have landed
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = Elt<DT>::V;
  constexpr int HMAX = 8;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int n = v.n, m = v.m, h = v.h, j = v.group;
  const int* upos = at<int>(v, v.rank, v.off.upos);
  int c0, c1;
  col_shard(h, m, v.tp_rank, &c0, &c1);
  // this rank's ZIN: one [T][sw] plane per (host, host TP rank), written by
  // the hosts' pair pre-reductions -- local reads only
  const int sw = (h + m - 1) / m;
  const T* zin = at<T>(v, v.rank, v.off.zin) - c0;
  for (long long t = gw; t < v.T; t += nwarps) {
    int hs[HMAX], nh = 0;
    for (int i = 1; i <= n; ++i) {
      const int d = (j - i + n) % n;  // arrival order j-1, ..., j
      const int u = upos[t * n + d];
      if (u >= 0 && nh < HMAX) hs[nh++] = d;
    }
    int c = c0 + lane * V;
    if (m * nh <= 4) {
      // fast path: every (host TP rank, host) ZIN load of two column vectors
      // is issued before any is consumed; the sum keeps the TP-rank-major,
      // arrival-order association
      const T* src[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int tt = i / (nh > 0 ? nh : 1), a = i % (nh > 0 ? nh : 1);
        src[i] = i < m * nh ? zin + (((size_t)hs[a] * m + tt) * v.T + t) * sw : nullptr;
      }
      for (; c + 32 * V < c1; c += 64 * V) {
        uint4 r0[4], r1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < m * nh) {
            r0[i] = ld_v4(src[i] + c);
            r1[i] = ld_v4(src[i] + c + 32 * V);
          }
        A a0[V], a1[V];
#pragma unroll
        for (int q = 0; q < V; ++q) a0[q] = a1[q] = (A)0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < m * nh) {
            const T* p0 = reinterpret_cast<const T*>(&r0[i]);
            const T* p1 = reinterpret_cast<const T*>(&r1[i]);
#pragma unroll
            for (int q = 0; q < V; ++q) {
              a0[q] = add_rn(a0[q], to_acc(p0[q]));
              a1[q] = add_rn(a1[q], to_acc(p1[q]));
            }
          }
        if (v.Is_t)
          for (int tt = 0; tt < m; ++tt) {
            const T* ps = at<T>(v, j * m + tt, v.off.part_s) + (size_t)t * h + c;
            const uint4 s0 = ld_v4(ps), s1 = ld_v4(ps + 32 * V);
            const T* q0 = reinterpret_cast<const T*>(&s0);
            const T* q1 = reinterpret_cast<const T*>(&s1);
#pragma unroll
            for (int q = 0; q < V; ++q) {
              a0[q] = add_rn(a0[q], to_acc(q0[q]));
              a1[q] = add_rn(a1[q], to_acc(q1[q]));
            }
          }
        T o0[V], o1[V];
#pragma unroll
        for (int q = 0; q < V; ++q) {
          o0[q] = from_acc<T>(a0[q]);
          o1[q] = from_acc<T>(a1[q]);
        }
        for (int tt = 0; tt < m; ++tt) {
          T* y = at<T>(v, j * m + tt, v.off.y) + (size_t)t * h + c;
          st_v4(y, *reinterpret_cast<uint4*>(o0));
          st_v4(y + 32 * V, *reinterpret_cast<uint4*>(o1));
        }
      }
    }
    for (; c < c1; c += 32 * V) {
      A acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = (A)0;
      for (int tt = 0; tt < m; ++tt) {
        uint4 raw[HMAX];
#pragma unroll
        for (int a = 0; a < HMAX; ++a)
          if (a < nh) raw[a] = ld_v4(zin + (((size_t)hs[a] * m + tt) * v.T + t) * sw + c);
#pragma unroll
        for (int a = 0; a < HMAX; ++a)
          if (a < nh) {
            const T* pv = reinterpret_cast<const T*>(&raw[a]);
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
          }
      }
      if (v.Is_t)  // shared expert: TP partials of the group's own tokens
        for (int tt = 0; tt < m; ++tt) {
          const uint4 raw = ld_v4(at<T>(v, j * m + tt, v.off.part_s) + (size_t)t * h + c);
          const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
        }
      T out[V];
#pragma unroll
      for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
      for (int tt = 0; tt < m; ++tt)
        st_v4(at<T>(v, j * m + tt, v.off.y) + (size_t)t * h + c, *reinterpret_cast<uint4*>(out));
    }
  }
  if (v.sync_signal) grid_signal_and_wait(v);  // y complete on every TP rank: barrier #4
}

// Gathered GEMM1 (SwiGLU): the row table replaces the expansion copy --
// recv_src[p] = u for every slot row p of pair u.
template <class WT>
__global__ void k_rowsrc_token(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);
  const int pairs = at<int>(v, v.rank, v.off.host_pairs)[v.group];
  const int* pn = at<int>(v, v.rank, v.off.pair_n);
  const PairEnt<WT>* pe = reinterpret_cast<const PairEnt<WT>*>(at<char>(v, v.rank, v.off.pair_p));
  int* src = at<int>(v, v.rank, v.off.recv_src);
  const long long total = (long long)pairs * v.KH;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long u = q / v.KH;
    const int i = (int)(q % v.KH);
    if (i < pn[u]) src[pe[q].p] = (int)u;
  }
}

static int blocks_for(long long warps) {
  long long b = (warps + 7) / 8;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

static int check_vec(const DevView& v) {
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  if (((size_t)c0 * v.elt) % 16 || ((size_t)(c1 - c0) * v.elt) % 16 || ((size_t)v.h * v.elt) % 16) {
    set_error("wire TOKEN needs 16-byte aligned column shards (h*elt/m %% 16 == 0)");
    return MX_ERR_UNSUPPORTED;
  }
  if (v.n > 8) { set_error("wire TOKEN supports up to 8 groups"); return MX_ERR_UNSUPPORTED; }
  return MX_OK;
}

int launch_dispatch_token(const DevView& v, const void* x, cudaStream_t s) {
  int rc = check_vec(v);
  if (rc) return rc;
  if (v.T == 0) return MX_OK;
  const int g = blocks_for((long long)v.T * DSPLIT);
  if (v.elt == 8) pdl_launch(k_dispatch_token<double>, g, 256, 0, s, v, static_cast<const char*>(x));
  else pdl_launch(k_dispatch_token<float>, g, 256, 0, s, v, static_cast<const char*>(x));
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_expand(const DevView& v, cudaStream_t s) {
  if (v.elt == 8) pdl_launch(k_expand<double>, blocks_for((long long)v.T * v.n), 256, 0, s, v);
  else pdl_launch(k_expand<float>, blocks_for((long long)v.T * v.n), 256, 0, s, v);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_rowsrc_token(const DevView& v, cudaStream_t s) {
  long long blocks = ((long long)v.T * v.n * v.KH + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (v.elt == 8) pdl_launch(k_rowsrc_token<double>, (int)blocks, 256, 0, s, v);
  else pdl_launch(k_rowsrc_token<float>, (int)blocks, 256, 0, s, v);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_pair_reduce(const DevView& v, cudaStream_t s) {
  const int g = blocks_for((long long)v.T * v.n);
  switch (v.elt) {
    case 8: pdl_launch(k_pair_reduce<MX_F64, double>, g, 256, 0, s, v); break;
    case 4: pdl_launch(k_pair_reduce<MX_F32, float>, g, 256, 0, s, v); break;
    default: pdl_launch(k_pair_reduce<MX_BF16, float>, g, 256, 0, s, v);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_combine_token(const DevView& v, cudaStream_t s) {
  int rc = check_vec(v);
  if (rc) return rc;
  if (v.T == 0) return MX_OK;
  const int g = blocks_for(v.T);
  switch (v.elt) {
    case 8: pdl_launch(k_combine_token<MX_F64>, g, 256, 0, s, v); break;
    case 4: pdl_launch(k_combine_token<MX_F32>, g, 256, 0, s, v); break;
    default: pdl_launch(k_combine_token<MX_BF16>, g, 256, 0, s, v);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
