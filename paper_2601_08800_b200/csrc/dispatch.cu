// dispatch.cu -- K2: fused AG-dispatch (Alg. 2; sim:330-407).
//
// Reference schedule: rank (j,t) isends column shard t of every slot row
// destined to group d=(j+i) mod n to rank (d,t) (sim:363-381), then group d
// all-gathers the m shards (sim:385-393); the locally hosted block is not
// communicated because x is replicated across the TP group (sim:383-384).
//
// On one NVSwitch box every peer is one hop away at full bandwidth, so the
// two hops collapse into one: rank (j,t) stores its column shard directly
// into the receive buffer of EVERY TP rank of the host group -- the
// intra-group all-gather is fused into the inter-group send.  Per-GPU
// ingress is unchanged (R_d rows x h), the staging buffer and the second
// round trip disappear.  Rows land at their expert-major position, so the
// grouped GEMM reads contiguous expert segments.  Values are byte copies:
// bit-exact with sim:395-406.
#include "mx_internal.cuh"

namespace mx {

// Warp-cooperative byte copy with the widest vector the alignment allows.
__device__ __forceinline__ void warp_copy(char* dst, const char* src, size_t nbytes, int lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes;
  if ((a & 15) == 0) {
    const size_t nv = nbytes >> 4;
    size_t i = lane;
    for (; i + 96 < nv; i += 128) {  // 4 x 16 B in flight per lane
      uint4 r0 = ld_nc_v4(src + (i << 4));
      uint4 r1 = ld_nc_v4(src + ((i + 32) << 4));
      uint4 r2 = ld_nc_v4(src + ((i + 64) << 4));
      uint4 r3 = ld_nc_v4(src + ((i + 96) << 4));
      st_v4(dst + (i << 4), r0);
      st_v4(dst + ((i + 32) << 4), r1);
      st_v4(dst + ((i + 64) << 4), r2);
      st_v4(dst + ((i + 96) << 4), r3);
    }
    for (; i < nv; i += 32) st_v4(dst + (i << 4), ld_nc_v4(src + (i << 4)));
  } else if ((a & 7) == 0) {
    const uint2* s = reinterpret_cast<const uint2*>(src);
    uint2* d = reinterpret_cast<uint2*>(dst);
    for (size_t i = lane; i < (nbytes >> 3); i += 32) d[i] = s[i];
  } else if ((a & 3) == 0) {
    const unsigned* s = reinterpret_cast<const unsigned*>(src);
    unsigned* d = reinterpret_cast<unsigned*>(dst);
    for (size_t i = lane; i < (nbytes >> 2); i += 32) d[i] = s[i];
  } else {
    for (size_t i = lane; i < nbytes; i += 32) dst[i] = src[i];
  }
}

__global__ void __launch_bounds__(256) k_dispatch(DevView v, const char* __restrict__ x) {
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  const size_t row_bytes = (size_t)v.wrow;  // wire row (e4m3 rows carry a scale tail)
  const size_t body = (size_t)v.h * v.welt;
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  const size_t sh_off = (size_t)c0 * v.welt, sh_bytes = (size_t)(c1 - c0) * v.welt;
  const bool tail = v.tp_rank == 0 && row_bytes > body;  // TP rank 0 ships the scale
  const long long total = (long long)v.T * v.k;
  for (long long s = gw; s < total; s += nwarps) {
    const int t = (int)(s / v.k);
    const int e = ids[s];
    const int d = home_of(e, v.n, v.E);
    const long long pos = slot_pos[s];
    if (pos >= v.cap) continue;  // flagged by k_slotpos; never write out of bounds
    const char* row = x + (size_t)t * row_bytes;
    if (d == v.group) {
      // locally hosted block: input replicated in the TP group (sim:383-384)
      warp_copy(at<char>(v, v.rank, v.off.recv) + pos * row_bytes, row, row_bytes, lane);
    } else {
      for (int tt = 0; tt < v.m; ++tt) {
        char* dst = at<char>(v, d * v.m + tt, v.off.recv) + pos * row_bytes;
        warp_copy(dst + sh_off, row + sh_off, sh_bytes, lane);
        if (tail) warp_copy(dst + body, row + body, row_bytes - body, lane);
      }
    }
  }
  if (v.sync_signal) grid_signal(v);  // rows landed (fused barrier)
}

// Token-major form for rows of at most VPL x 512 B: warp per token, the row
// is loaded into registers once (VPL x 16 B per lane) and stored to every
// one of the token's k slot rows (full row locally, column shard to each TP
// rank of a remote host).  Same destinations and bytes as k_dispatch.
template <int VPL>
__global__ void __launch_bounds__(256) k_dispatch_rows(DevView v, const char* __restrict__ x) {
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  const size_t row_bytes = (size_t)v.wrow;
  const int nvec = (int)(row_bytes >> 4);
  const size_t body = (size_t)v.h * v.welt;
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  const int v0 = (int)(((size_t)c0 * v.welt) >> 4), v1 = (int)(((size_t)c1 * v.welt) >> 4);
  const int vt = (int)(body >> 4);  // first vector of the scale tail
  const bool tail = v.tp_rank == 0 && row_bytes > body;
  for (long long t = gw; t < v.T; t += nwarps) {
    int e = 0, pos = 0;
    if (lane < v.k) {
      e = ids[t * v.k + lane];
      pos = slot_pos[t * v.k + lane];
    }
    uint4 val[VPL];
    const char* row = x + (size_t)t * row_bytes;
#pragma unroll
    for (int q = 0; q < VPL; ++q)
      if (q * 32 + lane < nvec) val[q] = ld_nc_v4(row + ((size_t)(q * 32 + lane) << 4));
    for (int sl = 0; sl < v.k; ++sl) {
      const int es = __shfl_sync(0xffffffffu, e, sl);
      const long long p = __shfl_sync(0xffffffffu, pos, sl);
      if (p >= v.cap) continue;  // flagged by the layout; never write out of bounds
      const int d = home_of(es, v.n, v.E);
      if (d == v.group) {
        char* dst = at<char>(v, v.rank, v.off.recv) + p * row_bytes;
#pragma unroll
        for (int q = 0; q < VPL; ++q)
          if (q * 32 + lane < nvec) st_v4(dst + ((size_t)(q * 32 + lane) << 4), val[q]);
      } else {
        for (int tt = 0; tt < v.m; ++tt) {
          char* dst = at<char>(v, d * v.m + tt, v.off.recv) + p * row_bytes;
#pragma unroll
          for (int q = 0; q < VPL; ++q) {
            const int vi = q * 32 + lane;
            if ((vi >= v0 && vi < v1) || (tail && vi >= vt && vi < nvec))
              st_v4(dst + ((size_t)vi << 4), val[q]);
          }
        }
      }
    }
  }
  if (v.sync_signal) grid_signal(v);  // rows landed (fused barrier)
}

int launch_dispatch(const DevView& v, const void* x, cudaStream_t s) {
  const long long total = (long long)v.T * v.k;
  if (total == 0) return MX_OK;
  const char* xp = static_cast<const char*>(x);
  const size_t row_bytes = (size_t)v.wrow;
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  const bool aligned = (row_bytes % 16) == 0 && ((size_t)c0 * v.welt) % 16 == 0 &&
                       ((size_t)c1 * v.welt) % 16 == 0 && ((size_t)v.h * v.welt) % 16 == 0 &&
                       v.k <= 32;
  if (aligned && row_bytes <= 8 * 512) {
    long long blocks = (v.T + 7) / 8;  // warp per token
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (row_bytes <= 2 * 512) pdl_launch(k_dispatch_rows<2>, (int)blocks, 256, 0, s, v, xp);
    else if (row_bytes <= 4 * 512) pdl_launch(k_dispatch_rows<4>, (int)blocks, 256, 0, s, v, xp);
    else pdl_launch(k_dispatch_rows<8>, (int)blocks, 256, 0, s, v, xp);
    MX_LAUNCH_CHECK();
    return MX_OK;
  }
  long long blocks = (total + 7) / 8;  // 8 warps per CTA, one slot per warp
  if (blocks > 148 * 16) blocks = 148 * 16;
  pdl_launch(k_dispatch, (int)blocks, 256, 0, s, v, xp);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

// Single group (n == 1): every slot is local, so instead of copying rows into
// the expert-major RECV the grouped GEMM gathers them straight from x; this
// kernel only writes the row table recv_src[p] = token of slot p.
__global__ void k_rowsrc_slot(DevView v) {
  pdl_wait();  // predecessor's outputs are visible after this
  const int* slot_pos = at<int>(v, v.rank, v.off.slot_pos);
  int* src = at<int>(v, v.rank, v.off.recv_src);
  const long long total = (long long)v.T * v.k;
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < total;
       s += (long long)gridDim.x * blockDim.x) {
    const int p = slot_pos[s];
    if (p < v.cap) src[p] = (int)(s / v.k);
  }
}

int launch_rowsrc_slot(const DevView& v, cudaStream_t s) {
  const long long total = (long long)v.T * v.k;
  if (total == 0) return MX_OK;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  pdl_launch(k_rowsrc_slot, (int)blocks, 256, 0, s, v);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
