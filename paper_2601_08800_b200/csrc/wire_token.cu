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

#ifndef MX_DSPLIT
#define MX_DSPLIT 2
#endif
constexpr int DSPLIT = MX_DSPLIT;  // warps per token in the dispatch

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
// part: 0 every pair, 1 the own group's (local RECV rows + metadata), 2 the
// other groups' (NVLink rows + metadata) -- the overlapped forward runs part
// 1, then part 2 on a side stream under the own group's GEMM1.
template <class WT>
__global__ void __launch_bounds__(256, 2) k_dispatch_token(DevView v, const char* __restrict__ x,
                                                           int part) {
  // no early trigger here (DevView::early): the grouped GEMMs read the
  // layout's tables before their PDL wait, which is only safe if some kernel
  // between the layout and them triggers at exit -- this one (its exit
  // implies its own wait, i.e. the layout's completion)
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
    // the token's routing, one load round: lane d holds its pair row on host
    // d, lane i (< k) slot i's expert, host, RECV row and weight
    const int u_l = lane < n ? upos[t * n + lane] : -1;
    int e_l = 0, d_l = -1, p_l = 0;
    WT w_l = 0;
    if (lane < k) {
      e_l = ids[t * k + lane];
      d_l = home_of(e_l, n, E);
      p_l = slot_pos[t * k + lane];
      if (sub == 0) w_l = wts[t * k + lane];
    }
    // with three or more hosts, the remote ones first (their NVLink stores
    // are in flight while the own host's local RECV rows are written):
    // EP4 dispatch 47.1 vs 51.7-52.0 us, layer 0.2794-0.2801 vs 0.2841-0.2845
    // ms; with two hosts measured equal or slightly slower, so ascending
    // there (profiles/r02_dispatch_order_ab.log)
    const int d0 = n >= 3 ? v.group + 1 : 0;
    for (int dd = 0; dd < n; ++dd) {
      const int d = (d0 + dd) % n;
      const int u = __shfl_sync(0xffffffffu, u_l, d);
      if (u < 0 || (part == 1 && d != v.group) || (part == 2 && d == v.group)) continue;
      if (d == v.group && direct_local) {
        // rows of this token's slots on the own host (pos < cap: layout-checked)
        const int pos = (d_l == d && p_l < v.cap) ? p_l : -1;
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
    const int e = e_l, d = d_l;
    const int ud = __shfl_sync(0xffffffffu, u_l, d < 0 ? 0 : d);
    int idx = 0, cnt = 0;
    for (int o = 0; o < k; ++o) {
      const int oe = __shfl_sync(0xffffffffu, e, o);
      const int od = __shfl_sync(0xffffffffu, d, o);
      if (od == d) {
        ++cnt;
        if (oe < e) ++idx;
      }
    }
    if (lane < k && (part == 0 || (d == v.group) == (part == 1))) {
      const int u = ud;
      const int dst = d * m + v.tp_rank;  // the TP peer that reads this metadata
      PairEnt<WT> ent;
      ent.p = p_l;
      ent.w = w_l;
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
__global__ void __launch_bounds__(256) k_expand(DevView v, int trigger) {
  // decode regime: the grouped GEMM1 behind this kernel may launch at once
  // and stream its first weight boxes while the rows are expanded
  if (trigger) pdl_trigger();
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
  // warps walk only the pairs left to expand (the own-group block skipped);
  // lane i holds slot i's row, the next pair's count and rows are loaded
  // while the current pair is copied, and a lane's whole 4 KB share of the
  // row (8 x 16 B) is in flight at once
  const long long todo = pairs - (skip1 - skip0);
  const int KH = v.KH;
  auto pair_of = [&](long long r) { return r < skip0 ? r : r + (skip1 - skip0); };
  int cnt = 0, row_l = 0;
  if (gw < todo) {
    const long long u = pair_of(gw);
    cnt = pn[u];
    if (lane < KH) row_l = pe[u * KH + lane].p;
  }
  for (long long r = gw; r < todo; r += nwarps) {
    const long long u = pair_of(r);
    int ncnt = 0, nrow_l = 0;
    if (r + nwarps < todo) {
      const long long un = pair_of(r + nwarps);
      ncnt = pn[un];
      if (lane < KH) nrow_l = pe[un * KH + lane].p;
    }
    const char* src = xbuf + (size_t)u * row_bytes;
    for (size_t base = 0; base < row_bytes; base += 8 * 512) {  // warp-uniform (shfl below)
      const size_t o = base + (size_t)lane * 16;
      uint4 val[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (o + q * 512 < row_bytes) val[q] = ld_v4(src + o + q * 512);
      for (int i = 0; i < cnt; ++i) {
        const int row = __shfl_sync(0xffffffffu, row_l, i);
        if (row >= v.cap) continue;  // flagged by the layout (mx_plan_check); never written
        char* dst = recv + (size_t)row * row_bytes + o;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (o + q * 512 < row_bytes) st_v4(dst + q * 512, val[q]);
      }
    }
    cnt = ncnt;
    row_l = nrow_l;
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

// The bulk-copy kernel's form: a lane's columns only grow along a row, so
// the cursor advances the shard incrementally (no division or shard search
// per store).
template <class T>
struct ZinCursor {
  int j, tt, c0, c1;
  size_t rowoff;
  T* base;
  __device__ __forceinline__ ZinCursor(const DevView& v, int tok, int sw) {
    j = tok / v.T;
    const int t = tok - j * v.T;
    rowoff = (((size_t)v.group * v.m + v.tp_rank) * v.T + t) * sw;
    tt = 0;
    col_shard(v.h, v.m, 0, &c0, &c1);
    base = at<T>(v, j * v.m, v.off.zin) + rowoff;
  }
  __device__ __forceinline__ T* operator()(const DevView& v, int c) {
    while (c >= c1 && tt + 1 < v.m) {
      ++tt;
      col_shard(v.h, v.m, tt, &c0, &c1);
      base = at<T>(v, j * v.m + tt, v.off.zin) + rowoff;
    }
    return base + (c - c0);
  }
};

// z = sum over the pair's slots (experts ascending) of w * partial[p], pushed
// straight into the owners' shards over NVLink (the reduce-scatter of the
// combine fused into the pre-reduction: the owner then only reads local
// memory); all slot loads of a column vector are issued before use.

// Pair index range of a part (pairs on this host are ordered by source
// group): 0 all, 1 the own group's [own0, own1), 2 every other group's
// (the own range skipped).
struct PairRange {
  long long todo, own0, own1;
  int part;
  __device__ PairRange(const DevView& v, int part_) : part(part_) {
    const int g = v.group, pairs = at<int>(v, v.rank, v.off.host_pairs)[g];
    own0 = at<int>(v, v.rank, v.off.poff)[g * v.n + g];
    own1 = own0 + at<int>(v, v.rank, v.off.ucnt_all)[g * v.n + g];
    todo = part == 0 ? pairs : part == 1 ? own1 - own0 : pairs - (own1 - own0);
  }
  __device__ long long operator()(long long r) const {
    return part == 0 ? r : part == 1 ? own0 + r : (r < own0 ? r : r + (own1 - own0));
  }
};

// S warps per pair (column split, a power of two dividing the warps per
// CTA): sub-warp s takes every S-th 32-vector column chunk, so a decode
// batch's few pairs keep all their loads in flight at once instead of
// walking the row in a chain of dependent rounds (same arithmetic per
// column, same bits).
template <int DT, class WT>
__global__ void __launch_bounds__(256, 2) k_pair_reduce(DevView v, int part, int S) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = Elt<DT>::V;
  constexpr int KU = 8;
  const int lane = threadIdx.x & 31;
  const long long gw0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int sub = (int)(gw0 % S);
  const long long gw = gw0 / S;
  const long long nwarps = (((long long)gridDim.x * blockDim.x) >> 5) / S;
  const int cstep = S * 32 * V;
  const PairRange pr(v, part);
  const int* pn = at<int>(v, v.rank, v.off.pair_n);
  const PairEnt<WT>* pe = reinterpret_cast<const PairEnt<WT>*>(at<char>(v, v.rank, v.off.pair_p));
  const T* prt = at<T>(v, v.rank, v.off.partial);
  const int* ptok = at<int>(v, v.rank, v.off.pair_tok);
  const int h = v.h, sw = (h + v.m - 1) / v.m;
  for (long long r = gw; r < pr.todo; r += nwarps) {
    const long long u = pr(r);
    const int cnt = pn[u];
    const int tok = ptok[u];
    const T* rp[KU];
    A w[KU];
#pragma unroll
    for (int i = 0; i < KU; ++i) {
      const PairEnt<WT> e = pe[u * v.KH + (i < cnt ? i : 0)];
      const bool ok = e.p < v.cap;  // rows past capacity were never computed
      rp[i] = prt + (size_t)(ok ? e.p : 0) * h;
      w[i] = ok ? (A)e.w : (A)0;
    }
    int c = (sub * 32 + lane) * V;
    if (cnt <= KU) {
      for (; c + cstep < h; c += 2 * cstep) {  // two column vectors per lane: 2 x cnt loads in flight
        uint4 raw[2][KU];
#pragma unroll
        for (int i = 0; i < KU; ++i)
          if (i < cnt) {
            raw[0][i] = ld_v4(rp[i] + c);
            raw[1][i] = ld_v4(rp[i] + c + cstep);
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
          st_v4(zin_dst<T>(v, tok, c + hh * cstep, sw), *reinterpret_cast<uint4*>(out));
        }
      }
    }
    for (; c < h; c += cstep) {
      A acc[V];
#pragma unroll
      for (int q = 0; q < V; ++q) acc[q] = (A)0;
      for (int i = 0; i < cnt; ++i) {
        const PairEnt<WT> e = pe[u * v.KH + i];
        if (e.p >= v.cap) continue;
        const uint4 raw = ld_v4(prt + (size_t)e.p * h + c);
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

// Bulk-copy pre-reduction (bf16 / f32 rows, at most 8 slots per pair read
// from shared memory; larger pairs straight from HBM).  A register-only
// kernel keeps only as many slot rows in flight as its registers hold (a
// persistent variant at one CTA per SM: 12% warps active, 51 us for one
// config-B rank's 134 MB on the emulated cluster, tools/emu_layer.py under
// ncu).  Here the TMA engine streams the rows into a ring of row slots in
// shared memory and registers only hold the sums (43-46 us emulated; 60.1
// vs 66-67 us for the register kernel above inside the 4-GPU layer, where
// the NVLink pushes bound it):
//   warp 0      producer: walks the CTA's contiguous range of pairs, four at
//               a time (lane l: entry l&7 of pair l>>3, two batches ahead),
//               writes each pair's header (count, owner token, first slot,
//               weights) and issues one cp.async.bulk per slot row,
//               completing on the slot's full barrier;
//   warps 1..15 consumers: pair i goes to warp 1 + i%15, which sums its rows
//               from shared memory (experts ascending, as above), pushes the
//               result into the owners' ZIN and frees the slots.  A single
//               consumer is issue-latency bound (ncu: 5.8 cycles per issued
//               instruction), hence many consumers and the ZinCursor.
constexpr int PRB_WARPS = 16, PRB_NC = PRB_WARPS - 1, PRB_NP = 32, PRB_KU = 8;
struct PrbHdr {
  int cnt, tok;
  unsigned q0;
  int u;
  float w[PRB_KU];
};

__host__ __device__ inline int prb_slots(size_t row_bytes) {
  const long long n = (200LL * 1024) / (long long)row_bytes;
  return (int)(n > 64 ? 64 : n);
}
__host__ __device__ inline size_t prb_smem(size_t row_bytes) {
  const int ns = prb_slots(row_bytes);
  return 128 + (size_t)ns * row_bytes + (2 * ns + 2 * PRB_NP) * 8 + PRB_NP * sizeof(PrbHdr);
}

template <int DT>
__device__ __forceinline__ void prb_body(const DevView& v, int part) {
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = Elt<DT>::V;
  extern __shared__ __align__(128) unsigned char prb_raw[];
  const int h = v.h, sw = (h + v.m - 1) / v.m;
  const uint32_t row_bytes = (uint32_t)h * sizeof(T);
  const int NS = prb_slots(row_bytes);
  unsigned char* slots = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(prb_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + (size_t)NS * row_bytes);
  uint64_t* empty = full + NS;
  uint64_t* pfull = empty + NS;
  uint64_t* pempty = pfull + PRB_NP;
  PrbHdr* hdr = reinterpret_cast<PrbHdr*>(pempty + PRB_NP);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < PRB_NP; ++i) {
      mbar_init(&pfull[i], 1);
      mbar_init(&pempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const PairRange pr(v, part);  // part 0 or 1: a contiguous pair range
  const long long base = pr(0), pairs = pr.todo;
  const long long u0 = base + pairs * blockIdx.x / gridDim.x;
  const long long u1 = base + pairs * (blockIdx.x + 1) / gridDim.x;
  const int* pn = at<int>(v, v.rank, v.off.pair_n);
  const PairEnt<float>* pe = reinterpret_cast<const PairEnt<float>*>(at<char>(v, v.rank, v.off.pair_p));
  const T* prt = at<T>(v, v.rank, v.off.partial);
  if (warp == 0) {
    const int* ptok = at<int>(v, v.rank, v.off.pair_tok);
    unsigned q = 0;
    // metadata of batch b (4 pairs; lane l: pair l>>3, entry l&7), loaded
    // two batches ahead of its bulk copies
    struct Meta {
      int cnt, tok;
      PairEnt<float> e;
    };
    auto load_meta = [&](long long b) {
      Meta mt{0, 0, {}};
      const long long ub = b + (lane >> 3);
      const int j = lane & 7;
      if (ub < u1) {
        mt.cnt = pn[ub];
        mt.tok = ptok[ub];
        if (j < v.KH) mt.e = pe[ub * v.KH + j];
      }
      return mt;
    };
    Meta m0 = load_meta(u0), m1 = load_meta(u0 + 4);
    for (long long b = u0; b < u1; b += 4) {
      const Meta m2 = load_meta(b + 8);
      const int j = lane & 7;
      const int cnt_l = m0.cnt, tok_l = m0.tok;
      const PairEnt<float> e = m0.e;
      for (int pb = 0; pb < 4; ++pb) {
        if (b + pb >= u1) break;
        const int cnt = __shfl_sync(0xffffffffu, cnt_l, pb * 8);
        const int tok = __shfl_sync(0xffffffffu, tok_l, pb * 8);
        const int ep_raw = __shfl_sync(0xffffffffu, e.p, pb * 8 + j);
        const bool ok = ep_raw < v.cap;  // rows past capacity: weight 0, row 0 read
        const int ep = ok ? ep_raw : 0;
        const float ew_raw = __shfl_sync(0xffffffffu, e.w, pb * 8 + j);
        const float ew = ok ? ew_raw : 0.f;
        const long long i = b + pb - u0;
        const int pi = (int)(i % PRB_NP);
        mbar_wait(&pempty[pi], (uint32_t)((i / PRB_NP) & 1) ^ 1u);
        const bool staged = cnt <= PRB_KU;
        if (staged && lane < cnt) {
          const unsigned qs = q + lane;
          const int sl = (int)(qs % NS);
          mbar_wait(&empty[sl], ((qs / NS) & 1) ^ 1u);
          mbar_expect_tx(&full[sl], row_bytes);
          bulk_load(slots + (size_t)sl * row_bytes, prt + (size_t)ep * h, row_bytes, &full[sl]);
        }
        if (lane < PRB_KU) hdr[pi].w[lane] = ew;
        if (lane == 0) {
          hdr[pi].cnt = cnt;
          hdr[pi].tok = tok;
          hdr[pi].q0 = q;
          hdr[pi].u = (int)(b + pb);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[pi]);
        if (staged) q += cnt;
      }
      m0 = m1;
      m1 = m2;
    }
  } else {
    for (long long i = warp - 1; i < u1 - u0; i += PRB_NC) {
      const int pi = (int)(i % PRB_NP);
      mbar_wait(&pfull[pi], (uint32_t)((i / PRB_NP) & 1));
      const int cnt = hdr[pi].cnt, tok = hdr[pi].tok, u = hdr[pi].u;
      const unsigned q0 = hdr[pi].q0;
      A w[PRB_KU];
#pragma unroll
      for (int jj = 0; jj < PRB_KU; ++jj) w[jj] = (A)hdr[pi].w[jj];
      __syncwarp();
      if (lane == 0) mbar_arrive(&pempty[pi]);
      ZinCursor<T> zc(v, tok, sw);
      if (cnt <= PRB_KU) {
        for (int jj = 0; jj < cnt; ++jj) {
          const unsigned qs = q0 + jj;
          mbar_wait(&full[qs % NS], (qs / NS) & 1);
        }
        for (int c = lane * V; c < h; c += 32 * V) {
          A acc[V];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = (A)0;
#pragma unroll
          for (int jj = 0; jj < PRB_KU; ++jj)
            if (jj < cnt) {
              const unsigned qs = q0 + jj;
              const uint4 raw = *reinterpret_cast<const uint4*>(
                  slots + (size_t)(qs % NS) * row_bytes + (size_t)c * sizeof(T));
              const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
              for (int q = 0; q < V; ++q) acc[q] = fmaf(w[jj], to_acc(pv[q]), acc[q]);
            }
          T out[V];
#pragma unroll
          for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
          st_v4(zc(v, c), *reinterpret_cast<uint4*>(out));
        }
        __syncwarp();
        if (lane < cnt) mbar_arrive(&empty[(q0 + lane) % NS]);
      } else {  // more slots than the staging handles: straight from HBM
        for (int c = lane * V; c < h; c += 32 * V) {
          A acc[V];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = (A)0;
          for (int jj = 0; jj < cnt; ++jj) {
            const PairEnt<float> e = pe[(long long)u * v.KH + jj];
            if (e.p >= v.cap) continue;
            const uint4 raw = ld_v4(prt + (size_t)e.p * h + c);
            const T* pv = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], mul_rn((A)e.w, to_acc(pv[q])));
          }
          T out[V];
#pragma unroll
          for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
          st_v4(zc(v, c), *reinterpret_cast<uint4*>(out));
        }
      }
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(PRB_WARPS * 32, 1) k_pair_reduce_bulk(DevView v, int part) {
  pdl_wait();  // predecessor's outputs are visible after this
  prb_body<DT>(v, part);
  if (v.sync_signal) grid_signal(v);  // every owner's ZIN written: barrier #3
}

// Owner (j, t): y[tok, cols t] = sum over host TP ranks (ascending) and hosts
// (j-1, ..., j) of the pre-reduced partials the hosts pushed into this rank's
// ZIN; then push the shard to every TP rank of the group (final all-gather).
// S warps per token (column split, as in k_pair_reduce).
template <int DT>
__device__ __forceinline__ void combine_token_body(const DevView& v, int S = 1) {
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  constexpr int V = Elt<DT>::V;
  constexpr int HMAX = 8;
  const int lane = threadIdx.x & 31;
  const long long gw0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int sub = (int)(gw0 % S);
  const long long gw = gw0 / S;
  const long long nwarps = (((long long)gridDim.x * blockDim.x) >> 5) / S;
  const int cstep = S * 32 * V;
  const int n = v.n, m = v.m, h = v.h, j = v.group;
  const int* upos = at<int>(v, v.rank, v.off.upos);
  int c0, c1;
  col_shard(h, m, v.tp_rank, &c0, &c1);
  // this rank's ZIN: one [T][sw] plane per (host, host TP rank), written by
  // the hosts' pair pre-reductions -- local reads only
  const int sw = (h + m - 1) / m;
  const T* zin = at<T>(v, v.rank, v.off.zin) - c0;
  for (long long t = gw; t < v.T; t += nwarps) {
    // lane l: the token's pair on host j-1-l (arrival order j-1, ..., j),
    // all n loaded in one round
    int u_l = -1;
    if (lane < n) u_l = upos[t * n + (j - (lane + 1) + n) % n];
    const unsigned hm = __ballot_sync(0xffffffffu, u_l >= 0);
    const int nh = __popc(hm);
    int hs[HMAX];
    {
      unsigned bits = hm;
#pragma unroll
      for (int a = 0; a < HMAX; ++a) {
        hs[a] = bits ? (j - __ffs(bits) + n) % n : 0;
        bits &= bits - 1;
      }
    }
    int c = c0 + (sub * 32 + lane) * V;
    if (m * nh <= 4) {
      // fast path: every (host TP rank, host) ZIN load of CG column
      // vectors is issued before any is consumed; the sum keeps the
      // TP-rank-major, arrival-order association
      const T* src[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int tt = i / (nh > 0 ? nh : 1), a = i % (nh > 0 ? nh : 1);
        int ha = hs[0];
#pragma unroll
        for (int q = 1; q < 4; ++q)
          if (q == a) ha = hs[q];
        src[i] = i < m * nh ? zin + (((size_t)ha * m + tt) * v.T + t) * sw : nullptr;
      }
      constexpr int CG = 2;
      for (; c + (CG - 1) * cstep < c1; c += CG * cstep) {
        uint4 r[4][CG];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < m * nh)
#pragma unroll
            for (int g = 0; g < CG; ++g) r[i][g] = ld_v4(src[i] + c + g * cstep);
#pragma unroll
        for (int g = 0; g < CG; ++g) {
          A acc[V];
#pragma unroll
          for (int q = 0; q < V; ++q) acc[q] = (A)0;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (i < m * nh) {
              const T* pv = reinterpret_cast<const T*>(&r[i][g]);
#pragma unroll
              for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
            }
          const int cg = c + g * cstep;
          if (v.Is_t)
            for (int tt = 0; tt < m; ++tt) {
              const uint4 sraw = ld_v4(at<T>(v, j * m + tt, v.off.part_s) + (size_t)t * h + cg);
              const T* pv = reinterpret_cast<const T*>(&sraw);
#pragma unroll
              for (int q = 0; q < V; ++q) acc[q] = add_rn(acc[q], to_acc(pv[q]));
            }
          T out[V];
#pragma unroll
          for (int q = 0; q < V; ++q) out[q] = from_acc<T>(acc[q]);
          for (int tt = 0; tt < m; ++tt)
            st_v4(at<T>(v, j * m + tt, v.off.y) + (size_t)t * h + cg,
                  *reinterpret_cast<uint4*>(out));
        }
      }
    }
    for (; c < c1; c += cstep) {
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
}

template <int DT>
__global__ void __launch_bounds__(256) k_combine_token(DevView v, int S) {
  if (v.early) pdl_trigger();  // decode: the next phase launches now, waits in griddepcontrol.wait
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);  // every host's pushes into ZIN have landed
  combine_token_body<DT>(v, S);
  if (v.sync_signal) grid_signal_and_wait(v);  // y complete on every TP rank: barrier #4
}

// The combine side as ONE persistent kernel (one CTA per SM, all resident):
// the pair pre-reduction pushes every pair row's column shards into the
// owners' ZIN over NVLink, the grid meets at an exchange barrier -- the last
// CTA to finish publishes this rank's epoch to every peer and alone polls
// the peers' flags, the other CTAs poll one local flag it raises -- and the
// same CTAs then sum their local ZIN planes and push y's shard to the TP
// peers.  Replaces pre-reduction kernel -> barrier kernel -> combine kernel
// (two kernel boundaries and the standalone barrier's launch).
__device__ __forceinline__ void exchange_barrier(const DevView& v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    int* cnt = reinterpret_cast<int*>(v.heap[v.rank] + v.off.counters) + 4;
    unsigned long long* go = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<int*>(v.heap[v.rank] + v.off.counters) + 8);
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(epoch_ctr(v)) + 1;
    const long long t0 = clock64();
    // arrival with acq_rel at GPU scope: this CTA's pushes (after the CTA
    // barrier above) happen-before the last arriver's system-scope release
    // to the peers, which is cumulative over them -- one fence on the
    // critical path instead of a system fence per CTA plus two in the last
    // (the lean device barrier's reasoning, api.cu k_barrier_lean)
    int arrived;
    asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(arrived) : "l"(cnt) : "memory");
    if (arrived == (int)gridDim.x - 1) {
      *cnt = 0;
      *epoch_ctr(v) = e;
      for (int r = 0; r < v.W; ++r)
        st_release_sys(reinterpret_cast<unsigned long long*>(v.heap[r] + v.off.flags) + v.rank, e);
      const unsigned long long* mine = reinterpret_cast<const unsigned long long*>(v.heap[v.rank] + v.off.flags);
      for (int r = 0; r < v.W; ++r)
        while (ld_acquire_sys(mine + r) < e)
          if (clock64() - t0 > 20000000000LL) { atomicOr(reinterpret_cast<int*>(v.heap[v.rank] + v.off.err) + 2, 1); break; }
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(go), "l"(e) : "memory");
    } else {
      unsigned long long g = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(g) : "l"(go) : "memory");
        if (clock64() - t0 > 20000000000LL) { atomicOr(reinterpret_cast<int*>(v.heap[v.rank] + v.off.err) + 2, 1); break; }
      } while (g < e);
    }
  }
  __syncthreads();
}

template <int DT>
__global__ void __launch_bounds__(PRB_WARPS * 32, 1) k_reduce_combine(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  prb_body<DT>(v, 0);
  exchange_barrier(v);  // every host's pushes into this rank's ZIN have landed
  combine_token_body<DT>(v);
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
    if (i < pn[u] && pe[q].p < v.cap) src[pe[q].p] = (int)u;
  }
}

static int blocks_for(long long warps) {
  long long b = (warps + 7) / 8;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return (int)b;
}

// Warps per row for the warp-per-row kernels (k_pair_reduce,
// k_combine_token): split a row's columns over up to 8 warps while the rows
// alone would not fill one 8-warp CTA per SM (decode batches).
static int col_split(long long rows) {
  int S = 1;
  while (S < 8 && rows * S * 2 <= 148LL * 8) S *= 2;
  return S;
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

int launch_dispatch_token(const DevView& v, const void* x, cudaStream_t s, int part,
                          bool coresident) {
  int rc = check_vec(v);
  if (rc) return rc;
  if (v.T == 0) return MX_OK;
  const int threads = coresident ? 128 : 256;
  const int g = coresident ? 148 : blocks_for((long long)v.T * DSPLIT);
  if (v.elt == 8) pdl_launch(k_dispatch_token<double>, g, threads, 0, s, v, static_cast<const char*>(x), part);
  else pdl_launch(k_dispatch_token<float>, g, threads, 0, s, v, static_cast<const char*>(x), part);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_expand(const DevView& v, cudaStream_t s, bool coresident) {
  const int threads = coresident ? 128 : 256;
  const int g = coresident ? 148 : blocks_for((long long)v.T * v.n);
  const int El = first_expert(v.group + 1, v.n, v.E) - first_expert(v.group, v.n, v.E);
  static const bool early_on = [] { const char* e = getenv("MX_GEMM_EARLY"); return !(e && e[0] == '0'); }();
  static const bool early_all = [] { const char* e = getenv("MX_GEMM_EARLY_ALL"); return e && e[0] == '1'; }();
  const int trigger = early_on && v.elt != 8 && El > 0 && (v.cap <= 64LL * El || early_all || v.W > 1);
  if (v.elt == 8) pdl_launch(k_expand<double>, g, threads, 0, s, v, trigger);
  else pdl_launch(k_expand<float>, g, threads, 0, s, v, trigger);
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

int launch_pair_reduce(const DevView& v, cudaStream_t s, int part, bool coresident) {
  const size_t row_bytes = (size_t)v.h * v.elt;
  // The ring pays off for many short pairs (k/n slots per pair on
  // average): config B, 4 GPUs (k/n = 4) 60.1 vs 62.6-66 us in the layer.
  // With one host (n = 1: every pair holds all k slots) the register kernel
  // is faster: 67.6 vs 90.3 us at 2 GPUs, k = 8.  Batches too small to give
  // every SM 32 pairs (decode) keep the register kernel's single latency
  // chain per pair.  Its ~200 KB ring cannot share an SM with a GEMM CTA, so
  // co-resident launches and the non-contiguous part 2 use the register kernel.
  // The ring must also hold several pairs' rows: config C's 14 KB rows leave
  // 14 slots (fewer than two full pairs) and the register kernel is faster
  // there (TP2xEP2 at 4 GPUs: 192 vs 330 us, layer 1.554 vs 1.681 ms;
  // profiles/r02_prb_wide_rows_ab.log).  MX_PRB=0 forces the register kernel.
  static const int prb_env = [] { const char* e = getenv("MX_PRB"); return e ? atoi(e) : -1; }();
  if (prb_env != 0 && !coresident && part != 2 && v.elt != 8 && v.k <= 4 * v.n &&
      (long long)v.T * v.n >= 148LL * 32 && prb_slots(row_bytes) >= 3 * PRB_KU) {
    auto kern = v.elt == 4 ? k_pair_reduce_bulk<MX_F32> : k_pair_reduce_bulk<MX_BF16>;
    static bool attr[2] = {false, false};
    if (!attr[v.elt == 4]) {
      MX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr[v.elt == 4] = true;
    }
    pdl_launch(kern, 148, PRB_WARPS * 32, prb_smem(row_bytes), s, v, part);  // one CTA per SM
    MX_LAUNCH_CHECK();
    return MX_OK;
  }
  // f64 (reference association), long pairs, rows too wide to stage
  const int threads = coresident ? 128 : 256;
  const int S = coresident ? 1 : col_split((long long)v.T * v.n);
  const int g = coresident ? 148 : blocks_for((long long)v.T * v.n * S);
  switch (v.elt) {
    case 8: pdl_launch(k_pair_reduce<MX_F64, double>, g, threads, 0, s, v, part, S); break;
    case 4: pdl_launch(k_pair_reduce<MX_F32, float>, g, threads, 0, s, v, part, S); break;
    default: pdl_launch(k_pair_reduce<MX_BF16, float>, g, threads, 0, s, v, part, S);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

// The fused combine side (k_reduce_combine) where the bulk pre-reduction
// applies; returns MX_ERR_UNSUPPORTED otherwise (the caller then launches
// pre-reduction, barrier and combine separately).  Cooperative launch: the
// exchange barrier needs every CTA resident.
bool reduce_combine_ok(const DevView& v) {
  const size_t row_bytes = (size_t)v.h * v.elt;
  return !(v.elt == 8 || v.k > 4 * v.n || (long long)v.T * v.n < 148LL * 32 ||
           prb_slots(row_bytes) < 3 * PRB_KU || v.T == 0 || v.W < 2);
}

int launch_reduce_combine(const DevView& v, cudaStream_t s) {
  const size_t row_bytes = (size_t)v.h * v.elt;
  if (!reduce_combine_ok(v)) return MX_ERR_UNSUPPORTED;
  int rc = check_vec(v);
  if (rc) return rc;
  auto kern = v.elt == 4 ? k_reduce_combine<MX_F32> : k_reduce_combine<MX_BF16>;
  static bool attr[2] = {false, false};
  if (!attr[v.elt == 4]) {
    MX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr[v.elt == 4] = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(PRB_WARPS * 32);
  cfg.dynamicSmemBytes = prb_smem(row_bytes);
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeCooperative;
  attrs[0].val.cooperative = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  MX_CUDA(cudaLaunchKernelEx(&cfg, kern, v));
  return MX_OK;
}

int launch_combine_token(const DevView& v, cudaStream_t s) {
  int rc = check_vec(v);
  if (rc) return rc;
  if (v.T == 0) return MX_OK;
  const int S = col_split(v.T);
  const int g = blocks_for((long long)v.T * S);
  switch (v.elt) {
    case 8: pdl_launch(k_combine_token<MX_F64>, g, 256, 0, s, v, S); break;
    case 4: pdl_launch(k_combine_token<MX_F32>, g, 256, 0, s, v, S); break;
    default: pdl_launch(k_combine_token<MX_BF16>, g, 256, 0, s, v, S);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
