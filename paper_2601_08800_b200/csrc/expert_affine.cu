// expert_affine.cu -- K3 (affine mode): the reference's TP-sharded expert
// stand-in, _partial_expert_outputs (sim:535-562), on expert-major rows.
//
// Rank (d,t) writes scale_e*x into its column shard t and adds bias_e/m to
// every column, so the rank-ascending TP sum equals scale_e*x + bias_e.
// f64 uses uncontracted IEEE ops, reproducing numpy's
// (scale*x) + bias/m exactly.
#include "mx_internal.cuh"

namespace mx {

template <int DT>
__global__ void __launch_bounds__(256)
k_expert_affine(DevView v, const typename Elt<DT>::Acc* __restrict__ scales,
                const typename Elt<DT>::Acc* __restrict__ biases) {
  pdl_wait();  // predecessor's outputs are visible after this
  if (v.sync_wait) grid_wait(v);  // fused barrier: every peer's rows have landed
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  __shared__ int s_off[MX_EMAX + 1];
  const int d = v.group;
  const int e0 = first_expert(d, v.n, v.E), e1 = first_expert(d + 1, v.n, v.E);
  const int ne = e1 - e0;
  const int* exp_off = at<int>(v, v.rank, v.off.exp_off);
  // rows past capacity were never received (flagged by the layout)
  const int rows = (int)min((long long)at<int>(v, v.rank, v.off.host_rows)[d], v.cap);
  for (int i = threadIdx.x; i < ne; i += blockDim.x) s_off[i] = exp_off[e0 + i];
  __syncthreads();
  int c0, c1;
  col_shard(v.h, v.m, v.tp_rank, &c0, &c1);
  const T* recv = at<T>(v, v.rank, v.off.recv);
  T* part = at<T>(v, v.rank, v.off.partial);
  const long long total = (long long)rows * v.h;
  const A m = (A)v.m;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int p = (int)(idx / v.h), c = (int)(idx % v.h);
    // expert of row p: last local expert whose segment starts at or before p
    int lo = 0, hi = ne - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= p) lo = mid; else hi = mid - 1;
    }
    const int e = e0 + lo;
    A val = (c >= c0 && c < c1) ? mul_rn(scales[e], to_acc(recv[idx])) : (A)0;
    val = add_rn(val, biases[e] / m);
    part[idx] = from_acc<T>(val);
  }
  if (v.sync_signal) grid_signal(v);
}

int launch_expert_affine(const DevView& v, const void* scales, const void* biases,
                         cudaStream_t s) {
  const long long work = (v.cap < 1 ? 1 : v.cap) * (long long)v.h;
  long long blocks = (work + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  switch (v.elt) {
    case 8:
      pdl_launch(k_expert_affine<MX_F64>, (int)blocks, 256, 0, s, 
          v, static_cast<const double*>(scales), static_cast<const double*>(biases));
      break;
    case 4:
      pdl_launch(k_expert_affine<MX_F32>, (int)blocks, 256, 0, s, 
          v, static_cast<const float*>(scales), static_cast<const float*>(biases));
      break;
    default:
      pdl_launch(k_expert_affine<MX_BF16>, (int)blocks, 256, 0, s, 
          v, static_cast<const float*>(scales), static_cast<const float*>(biases));
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
