// baseline.cu -- pack/unpack kernels around the NCCL AR+A2A baseline
// (value path of _run_baseline, sim:598-680).  The baseline ships FULL-width
// rows with all_to_all from every TP rank (sim:617-640), computes, ships
// full-width TP partials back (sim:652-658) and all-reduces over the TP group
// (sim:659-666).  Wire order: blocks by peer group ascending, inside a block
// by (expert, token) -- so a slot's row index in its block is fixed by the
// [n][E] count matrix and the chunk ranks of K1.
#include "mx_internal.cuh"

namespace mx {

// exclusive prefix over experts of group j's per-expert counts, into smem
__device__ void excl_experts(const DevView& v, int j, int* s_pre) {
  const int* cnt = at<int>(v, v.rank, v.off.cnt_all) + (size_t)j * v.E;
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < v.E; ++e) { s_pre[e] = run; run += cnt[e]; }
    s_pre[v.E] = run;
  }
  __syncthreads();
}

__device__ __forceinline__ void warp_copy_rows(char* dst, const char* src, size_t nbytes, int lane) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | nbytes) & 15) == 0) {
    for (size_t i = (size_t)lane * 16; i < nbytes; i += 512) st_v4(dst + i, ld_v4(src + i));
  } else {
    for (size_t i = lane; i < nbytes; i += 32) dst[i] = src[i];
  }
}

// slot's row in the (host, expert, token)-ordered block layout of group j
__device__ __forceinline__ int block_pos(const DevView& v, const int* s_pre, int t, int i) {
  const size_t si = (size_t)t * v.k + i;
  const int e = at<int>(v, v.rank, v.off.ids)[si];
  const int c = t / MX_CHUNK;
  return s_pre[e] + at<int>(v, v.rank, v.off.chunk_hist)[e * v.C + c] +
         at<int>(v, v.rank, v.off.slot_rank)[si];
}

__global__ void k_bl_dispatch_pack(DevView v, const char* x, char* send, int32_t* counts) {
  __shared__ int s_pre[MX_EMAX + 1];
  excl_experts(v, v.group, s_pre);
  const int lane = threadIdx.x & 31;
  const size_t row = (size_t)v.h * v.elt;
  if (blockIdx.x == 0)
    for (int d = threadIdx.x; d < v.n; d += blockDim.x)
      counts[d] = at<int>(v, v.rank, v.off.send)[v.group * v.n + d];
  const long long total = (long long)v.T * v.k;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long s = gw; s < total; s += nw) {
    const int t = (int)(s / v.k), i = (int)(s % v.k);
    warp_copy_rows(send + (size_t)block_pos(v, s_pre, t, i) * row, x + (size_t)t * row, row, lane);
  }
}

__global__ void k_bl_dispatch_unpack(DevView v, const char* recv) {
  // rows arrive as blocks from source groups j = 0..n-1, each (expert, token)
  extern __shared__ int s_dyn[];  // [n][El+1] per-source prefix over local experts
  const int d = v.group;
  const int e0 = first_expert(d, v.n, v.E), e1 = first_expert(d + 1, v.n, v.E);
  const int El = e1 - e0;
  const int* cnt = at<int>(v, v.rank, v.off.cnt_all);
  const int* tm_off = at<int>(v, v.rank, v.off.tm_off);
  const int* exp_off = at<int>(v, v.rank, v.off.exp_off);
  const int* grp_off = at<int>(v, v.rank, v.off.grp_off);
  for (int j = threadIdx.x; j < v.n; j += blockDim.x) {
    int run = 0;
    for (int e = 0; e < El; ++e) { s_dyn[j * (El + 1) + e] = run; run += cnt[j * v.E + e0 + e]; }
    s_dyn[j * (El + 1) + El] = run;
  }
  __syncthreads();
  const int rows = (int)min((long long)at<int>(v, v.rank, v.off.host_rows)[d], v.cap);
  const size_t row = (size_t)v.h * v.elt;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long q = gw; q < rows; q += nw) {
    int j = 0;
    while (j + 1 < v.n && tm_off[(j + 1) * v.n + d] <= q) ++j;
    const int i = (int)(q - tm_off[j * v.n + d]);
    const int* pre = s_dyn + j * (El + 1);
    int lo = 0, hi = El - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int e = e0 + lo;
    const long long pos = (long long)exp_off[e] + grp_off[j * v.E + e] + (i - pre[lo]);
    warp_copy_rows(at<char>(v, v.rank, v.off.recv) + pos * row, recv + q * row, row, lane);
  }
}

__global__ void k_bl_combine_pack(DevView v, char* send, int32_t* counts) {
  // expert-major partial rows -> blocks by owner group j, each (expert, token)
  extern __shared__ int s_dyn[];
  const int d = v.group;
  const int e0 = first_expert(d, v.n, v.E), e1 = first_expert(d + 1, v.n, v.E);
  const int El = e1 - e0;
  const int* cnt = at<int>(v, v.rank, v.off.cnt_all);
  const int* tm_off = at<int>(v, v.rank, v.off.tm_off);
  const int* exp_off = at<int>(v, v.rank, v.off.exp_off);
  const int* grp_off = at<int>(v, v.rank, v.off.grp_off);
  int* s_off = s_dyn + v.n * (El + 1);
  for (int j = threadIdx.x; j < v.n; j += blockDim.x) {
    int run = 0;
    for (int e = 0; e < El; ++e) { s_dyn[j * (El + 1) + e] = run; run += cnt[j * v.E + e0 + e]; }
    s_dyn[j * (El + 1) + El] = run;
  }
  for (int e = threadIdx.x; e < El; e += blockDim.x) s_off[e] = exp_off[e0 + e];
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < v.n; j += blockDim.x)
      counts[j] = at<int>(v, v.rank, v.off.send)[j * v.n + d];
  __syncthreads();
  const int rows = (int)min((long long)at<int>(v, v.rank, v.off.host_rows)[d], v.cap);
  const size_t row = (size_t)v.h * v.elt;
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long p = gw; p < rows; p += nw) {
    int lo = 0, hi = El - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int e = e0 + lo;
    const int r = (int)(p - s_off[lo]);
    int j = 0;
    while (j + 1 < v.n && grp_off[(j + 1) * v.E + e] <= r) ++j;
    const int i = r - grp_off[j * v.E + e];
    const long long q = (long long)tm_off[j * v.n + d] + s_dyn[j * (El + 1) + lo] + i;
    warp_copy_rows(send + q * row, at<char>(v, v.rank, v.off.partial) + p * row, row, lane);
  }
}

template <int DT>
__global__ void k_bl_combine_unpack(DevView v, const char* recv, char* yout) {
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  __shared__ int s_pre[MX_EMAX + 1];
  __shared__ int s_pos[8][MX_KMAX];
  __shared__ A s_w[8][MX_KMAX];
  excl_experts(v, v.group, s_pre);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = v.n, k = v.k, h = v.h, E = v.E, j = v.group;
  const int* ids = at<int>(v, v.rank, v.off.ids);
  const A* wts = at<A>(v, v.rank, v.off.w);
  const T* src = reinterpret_cast<const T*>(recv);
  T* y = reinterpret_cast<T*>(yout);
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long tl = gw; tl < v.T; tl += nw) {
    int e = 0, key = 0x7fffffff, pos = 0;
    A w = (A)0;
    if (lane < k) {
      e = ids[tl * k + lane];
      w = wts[tl * k + lane];
      pos = block_pos(v, s_pre, (int)tl, lane);
      key = (j - home_of(e, n, E) - 1 + n) % n;
    }
    int rk = 0;
    for (int o = 0; o < k; ++o) {
      const int ok = __shfl_sync(0xffffffffu, key, o);
      const int oe = __shfl_sync(0xffffffffu, e, o);
      rk += (ok < key || (ok == key && oe < e)) ? 1 : 0;
    }
    if (lane < k) { s_pos[warp][rk] = pos; s_w[warp][rk] = w; }
    __syncwarp();
    for (int c = lane; c < h; c += 32) {
      A acc = (A)0;
      for (int s = 0; s < k; ++s)
        acc = add_rn(acc, mul_rn(s_w[warp][s], to_acc(src[(size_t)s_pos[warp][s] * h + c])));
      y[tl * h + c] = from_acc<T>(acc);
    }
    __syncwarp();
  }
}

static int grid_for(long long work_items_per_warp_unit) {
  long long b = (work_items_per_warp_unit + 7) / 8;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return (int)b;
}

int launch_baseline_dispatch_pack(const DevView& v, const void* x, void* send, int32_t* counts,
                                  cudaStream_t s) {
  k_bl_dispatch_pack<<<grid_for((long long)v.T * v.k), 256, 0, s>>>(
      v, static_cast<const char*>(x), static_cast<char*>(send), counts);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

static size_t unpack_smem(const DevView& v) {
  const int El = first_expert(v.group + 1, v.n, v.E) - first_expert(v.group, v.n, v.E);
  return (size_t)(v.n * (El + 1) + El + 1) * 4;
}

int launch_baseline_dispatch_unpack(const DevView& v, const void* recv, cudaStream_t s) {
  k_bl_dispatch_unpack<<<grid_for(v.cap), 256, unpack_smem(v), s>>>(v, static_cast<const char*>(recv));
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_baseline_combine_pack(const DevView& v, void* send, int32_t* counts, cudaStream_t s) {
  k_bl_combine_pack<<<grid_for(v.cap), 256, unpack_smem(v), s>>>(v, static_cast<char*>(send), counts);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int launch_baseline_combine_unpack(const DevView& v, const void* recv, void* y, cudaStream_t s) {
  const int g = grid_for(v.T);
  switch (v.elt) {
    case 8: k_bl_combine_unpack<MX_F64><<<g, 256, 0, s>>>(v, static_cast<const char*>(recv), static_cast<char*>(y)); break;
    case 4: k_bl_combine_unpack<MX_F32><<<g, 256, 0, s>>>(v, static_cast<const char*>(recv), static_cast<char*>(y)); break;
    default: k_bl_combine_unpack<MX_BF16><<<g, 256, 0, s>>>(v, static_cast<const char*>(recv), static_cast<char*>(y));
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
