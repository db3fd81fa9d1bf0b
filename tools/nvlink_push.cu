// NVLink peer store / load micro-benchmark (diagnostic, not product code).
// One process drives every GPU with peer access enabled; each GPU moves 4 KB
// rows between its own HBM and its peers' with 16-byte vector accesses, the
// access pattern of the token wire's dispatch, pre-reduction push and
// combine.  Built on the box by tools/nvlink_bench.py:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <stdint.h>

namespace {
constexpr int ROW = 4096;             // bytes per row (h = 2048 bf16)
constexpr int VPR = ROW / 16;         // 16 B vectors per row
constexpr int VPL = VPR / 32;         // vectors per lane

struct Peers {
  char* p[8];
  int n;
};

__device__ __forceinline__ uint4 ldv(const char* p) {
  uint4 r;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stv(char* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w) : "memory");
}

// mode 0: push   row r of src -> peer (r % n), row r / n
// mode 1: pull   row r / n of peer (r % n) -> local row r
// mode 2: bcast  row r of src -> row r of every peer (dispatch to TP ranks)
// mode 3: local  row r of src -> local row r (HBM sanity check)
// mode 4: mixed  row r of src -> peer (r % n) and to 4 local rows (the
//                dispatch's own-group RECV rows), one warp does both
// mode 5: split  as mode 4, one warp stores a row to the peer, the next
//                warp stores it to the 4 local rows
// mode 6: reduce four local rows -> peer (r % n): the pre-reduction's shape
// mode 7: scatter  source row and destination rows permuted; the row's two
//                  2 KB halves go to two different peers (the pre-reduction's
//                  column shards to the owner group's TP ranks)
// HALF: each lane moves half its vectors per pass (fewer bytes in flight)
__device__ __forceinline__ char* pick(const Peers& pe, int i) {
  char* p = pe.p[0];
#pragma unroll
  for (int j = 1; j < 8; ++j)
    if (j == i) p = pe.p[j];
  return p;
}

template <int MODE, int HALF>
__global__ void __launch_bounds__(256) k_move(Peers pe, const char* __restrict__ src,
                                              char* __restrict__ local, long long rows) {
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr int PASS = HALF ? VPL / 2 : VPL;
  const long long R = MODE == 5 ? 2 * rows : rows;
  for (long long r = gw; r < R; r += nw) {
    const char* s = src + r * ROW;
    char* d = local + r * ROW;
    if (MODE == 0) d = pick(pe, (int)(r % pe.n)) + (r / pe.n) * ROW;
    if (MODE == 1) s = pick(pe, (int)(r % pe.n)) + (r / pe.n) * ROW;
    if (MODE == 7) {
      const long long rs = (r * 2654435761LL) & (rows - 1);         // rows: power of 2
      const long long rd = ((r / pe.n) * 40503LL) & (rows / pe.n - 1);
      const int p0 = (int)(r % pe.n), p1 = (p0 + 1) % pe.n;
      s = src + rs * ROW;
      uint4 v[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) v[q] = ldv(s + ((size_t)(lane + 32 * q) << 4));
#pragma unroll
      for (int q = 0; q < VPL; ++q) {
        char* pd = pick(pe, q < VPL / 2 ? p0 : p1) + rd * ROW;
        stv(pd + ((size_t)(lane + 32 * q) << 4), v[q]);
      }
      continue;
    }
    if (MODE == 6) {
      char* pd = pick(pe, (int)(r % pe.n)) + (r / pe.n) * ROW;
#pragma unroll
      for (int b = 0; b < VPL; b += 4) {
        uint4 v[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            v[j][q] = ldv(src + ((r * 4 + j) % rows) * ROW + ((size_t)(lane + 32 * (b + q)) << 4));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o = v[0][q];
#pragma unroll
          for (int j = 1; j < 4; ++j) {
            o.x += v[j][q].x; o.y += v[j][q].y; o.z += v[j][q].z; o.w += v[j][q].w;
          }
          stv(pd + ((size_t)(lane + 32 * (b + q)) << 4), o);
        }
      }
      continue;
    }
    if (MODE == 4 || MODE == 5) {
      const long long rr = MODE == 5 ? r >> 1 : r;
      const int role = MODE == 5 ? (int)(r & 1) : 2;  // 0 peer, 1 local, 2 both
      char* pd = pick(pe, (int)(rr % pe.n)) + (rr / pe.n) * ROW;
      s = src + rr * ROW;
      uint4 v[VPL];
#pragma unroll
      for (int q = 0; q < VPL; ++q) v[q] = ldv(s + ((size_t)(lane + 32 * q) << 4));
      if (role != 1)
#pragma unroll
        for (int q = 0; q < VPL; ++q) stv(pd + ((size_t)(lane + 32 * q) << 4), v[q]);
      if (role != 0)
        for (int j = 0; j < 4; ++j) {
          char* ld = local + ((rr * 4 + j) % rows) * ROW;
#pragma unroll
          for (int q = 0; q < VPL; ++q) stv(ld + ((size_t)(lane + 32 * q) << 4), v[q]);
        }
      continue;
    }
#pragma unroll
    for (int b = 0; b < VPL; b += PASS) {
      uint4 v[PASS];
#pragma unroll
      for (int q = 0; q < PASS; ++q) v[q] = ldv(s + ((size_t)(lane + 32 * (b + q)) << 4));
      if (MODE == 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < pe.n)
#pragma unroll
            for (int q = 0; q < PASS; ++q)
              stv(pe.p[i] + r * ROW + ((size_t)(lane + 32 * (b + q)) << 4), v[q]);
      } else {
#pragma unroll
        for (int q = 0; q < PASS; ++q) stv(d + ((size_t)(lane + 32 * (b + q)) << 4), v[q]);
      }
    }
  }
}
}  // namespace

extern "C" {
int nb_enable_peers(int n) {
  for (int a = 0; a < n; ++a) {
    if (cudaSetDevice(a) != cudaSuccess) return 1;
    for (int b = 0; b < n; ++b) {
      if (a == b) continue;
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return 2;
      cudaGetLastError();
    }
  }
  return 0;
}

int nb_launch(int dev, int mode, void** peers, int npeers, const void* src, void* local,
              long long rows, int blocks, int half, void* stream) {
  if (npeers < 1 || npeers > 8) return 3;
  if (cudaSetDevice(dev) != cudaSuccess) return 1;
  Peers pe;
  pe.n = npeers;
  for (int i = 0; i < 8; ++i) pe.p[i] = static_cast<char*>(peers[i < npeers ? i : 0]);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const char* sp = static_cast<const char*>(src);
  char* lp = static_cast<char*>(local);
#define NB_CASE(M)                                                         \
  case M:                                                                  \
    if (half) k_move<M, 1><<<blocks, 256, 0, s>>>(pe, sp, lp, rows);       \
    else k_move<M, 0><<<blocks, 256, 0, s>>>(pe, sp, lp, rows);            \
    break;
  switch (mode) {
    NB_CASE(0)
    NB_CASE(1)
    NB_CASE(2)
    NB_CASE(3)
    NB_CASE(4)
    NB_CASE(5)
    NB_CASE(6)
    NB_CASE(7)
    default: return 3;
  }
#undef NB_CASE
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
}
