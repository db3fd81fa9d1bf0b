// misc.cu -- weight packing and the independent dense GPU reference used by
// the API's moe_oracle mirror (sim:302-310).  Neither is on the fused path.
#include "mx_internal.cuh"

namespace mx {

// w13[e][256*b + r] = gate[e][128*b + r] (r < 128), up[e][128*b + r-128]
__global__ void k_pack_w13(const __nv_bfloat16* gate, const __nv_bfloat16* up, __nv_bfloat16* w13,
                           int E_l, int I_t, int h) {
  const long long rows = (long long)E_l * 2 * I_t;
  for (long long rr = blockIdx.x; rr < rows; rr += gridDim.x) {
    const int e = (int)(rr / (2 * I_t)), r = (int)(rr % (2 * I_t));
    const int b = r / 128, q = r % 128;  // blocks of 64 gate rows, then 64 up rows
    const __nv_bfloat16* src = (q < 64 ? gate : up) + ((size_t)e * I_t + b * 64 + (q & 63)) * h;
    __nv_bfloat16* dst = w13 + (size_t)rr * h;
    for (int c = threadIdx.x; c < h; c += blockDim.x) dst[c] = src[c];
  }
}

// One CTA per token; slots visited in ascending expert id (sim:306-309).
template <int DT>
__global__ void k_dense_affine(int h, int k, const typename Elt<DT>::T* x, const int32_t* ids,
                               const typename Elt<DT>::Acc* w, const typename Elt<DT>::Acc* sc,
                               const typename Elt<DT>::Acc* bi, typename Elt<DT>::T* y) {
  using T = typename Elt<DT>::T;
  using A = typename Elt<DT>::Acc;
  const int t = blockIdx.x;
  __shared__ int s_ord[MX_KMAX];
  if (threadIdx.x < k) {
    const int e = ids[(size_t)t * k + threadIdx.x];
    int rk = 0;
    for (int o = 0; o < k; ++o) rk += ids[(size_t)t * k + o] < e ? 1 : 0;
    s_ord[rk] = threadIdx.x;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    const A xv = to_acc(x[(size_t)t * h + c]);
    A acc = (A)0;
    for (int s = 0; s < k; ++s) {
      const int i = s_ord[s];
      const int e = ids[(size_t)t * k + i];
      acc = add_rn(acc, mul_rn(w[(size_t)t * k + i], add_rn(mul_rn(sc[e], xv), bi[e])));
    }
    y[(size_t)t * h + c] = from_acc<T>(acc);
  }
}

__global__ void k_dense_swiglu(int h, int k, int I, const __nv_bfloat16* x, const int32_t* ids,
                               const float* w, const __nv_bfloat16* wg, const __nv_bfloat16* wu,
                               const __nv_bfloat16* wd, float* y) {
  extern __shared__ float s_buf[];  // x row [h] + act [I]
  float* s_x = s_buf;
  float* s_a = s_buf + h;
  __shared__ int s_ord[MX_KMAX];
  const int t = blockIdx.x;
  for (int c = threadIdx.x; c < h; c += blockDim.x) s_x[c] = __bfloat162float(x[(size_t)t * h + c]);
  if (threadIdx.x < k) {
    const int e = ids[(size_t)t * k + threadIdx.x];
    int rk = 0;
    for (int o = 0; o < k; ++o) rk += ids[(size_t)t * k + o] < e ? 1 : 0;
    s_ord[rk] = threadIdx.x;
  }
  for (int c = threadIdx.x; c < h; c += blockDim.x) y[(size_t)t * h + c] = 0.f;
  __syncthreads();
  for (int s = 0; s < k; ++s) {
    const int i = s_ord[s];
    const int e = ids[(size_t)t * k + i];
    const float ws = w[(size_t)t * k + i];
    for (int r = threadIdx.x; r < I; r += blockDim.x) {
      const __nv_bfloat16* g = wg + ((size_t)e * I + r) * h;
      const __nv_bfloat16* u = wu + ((size_t)e * I + r) * h;
      float ga = 0.f, ua = 0.f;
      for (int c = 0; c < h; ++c) {
        ga = fmaf(s_x[c], __bfloat162float(g[c]), ga);
        ua = fmaf(s_x[c], __bfloat162float(u[c]), ua);
      }
      const float a = ga / (1.f + expf(-ga)) * ua;
      s_a[r] = __bfloat162float(__float2bfloat16_rn(a));  // product rounding point
    }
    __syncthreads();
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      const __nv_bfloat16* d = wd + ((size_t)e * h + c) * I;
      float o = 0.f;
      for (int r = 0; r < I; ++r) o = fmaf(s_a[r], __bfloat162float(d[r]), o);
      y[(size_t)t * h + c] += ws * o;
    }
    __syncthreads();
  }
}

}  // namespace mx

using namespace mx;

extern "C" {

int mx_swiglu_pack_w13(const void* gate, const void* up, void* w13, int E_l, int I_t, int h,
                       void* stream) {
  if (I_t % 128 != 0) { set_error("I/tp must be a multiple of 128"); return MX_ERR_UNSUPPORTED; }
  const long long rows = (long long)E_l * 2 * I_t;
  if (rows == 0) return MX_OK;
  k_pack_w13<<<(int)(rows < 65535 ? rows : 65535), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(gate), static_cast<const __nv_bfloat16*>(up),
      static_cast<__nv_bfloat16*>(w13), E_l, I_t, h);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

int mx_dense_moe(int T, int h, int E, int k, int act_dtype, int expert_kind, int inter,
                 const void* x, const int32_t* ids, const void* weights, const void* scales,
                 const void* biases, const void* w_gate, const void* w_up, const void* w_down,
                 void* y, void* stream) {
  (void)E;
  if (T == 0) return MX_OK;
  if (k > MX_KMAX) { set_error("top_k exceeds %d", MX_KMAX); return MX_ERR_UNSUPPORTED; }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (expert_kind == MX_EXPERT_AFFINE) {
    switch (act_dtype) {
      case MX_F64:
        k_dense_affine<MX_F64><<<T, 128, 0, s>>>(h, k, (const double*)x, ids, (const double*)weights,
                                                 (const double*)scales, (const double*)biases, (double*)y);
        break;
      case MX_F32:
        k_dense_affine<MX_F32><<<T, 128, 0, s>>>(h, k, (const float*)x, ids, (const float*)weights,
                                                 (const float*)scales, (const float*)biases, (float*)y);
        break;
      default:
        k_dense_affine<MX_BF16><<<T, 128, 0, s>>>(h, k, (const __nv_bfloat16*)x, ids,
                                                  (const float*)weights, (const float*)scales,
                                                  (const float*)biases, (__nv_bfloat16*)y);
    }
  } else {
    if (act_dtype != MX_BF16) { set_error("dense SwiGLU reference takes bf16"); return MX_ERR_UNSUPPORTED; }
    const size_t smem = (size_t)(h + inter) * 4;
    if (smem > 200 * 1024) { set_error("dense SwiGLU reference: h+I too large"); return MX_ERR_UNSUPPORTED; }
    static bool attr = false;
    if (!attr) {
      MX_CUDA(cudaFuncSetAttribute(k_dense_swiglu, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    k_dense_swiglu<<<T, 256, smem, s>>>(h, k, inter, (const __nv_bfloat16*)x, ids,
                                        (const float*)weights, (const __nv_bfloat16*)w_gate,
                                        (const __nv_bfloat16*)w_up, (const __nv_bfloat16*)w_down,
                                        (float*)y);
  }
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // extern "C"

namespace mx {

// ---------------------------------------------------------------- stamps
__global__ void k_stamp(DevView v, int slot) {
  pdl_wait();  // every earlier launch on the stream has completed
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  at<unsigned long long>(v, v.rank, v.off.stamps)[slot] = t;
}

int launch_stamp(const DevView& v, int slot, cudaStream_t s) {
  pdl_launch(k_stamp, 1, 32, 0, s, v, slot);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx

namespace mx {

// ---------------------------------------------------------------- NVLink probe
// Same-run NVLink denominator for bench.py: every rank copies `bytes` of its
// own PARTIAL region into every peer's RECV region (slot `rank`), 16 B
// vector loads from local HBM and 16 B stores over NVLink -- the access mix
// of the layer's dispatch and pre-reduction pushes.  A warp moves one 4 KB
// chunk at a time, chunks dealt round-robin over the peers so every link
// is busy at once.  Scratch use of RECV/PARTIAL: call between forwards only.
__global__ void __launch_bounds__(256) k_nvlink_probe(DevView v, size_t bytes) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int peers = v.W - 1;
  const long long per_peer = (long long)(bytes >> 12);  // 4 KB chunks per peer
  const long long chunks = per_peer * peers;
  const char* src = at<char>(v, v.rank, v.off.partial);
  for (long long c = gw; c < chunks; c += nwarps) {
    const int p = (int)(c % peers);
    const int dst_rank = (v.rank + 1 + p) % v.W;
    const size_t off = (size_t)(c / peers) << 12;
    char* dst = at<char>(v, dst_rank, v.off.recv) + (size_t)v.rank * bytes + off;
    uint4 val[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) val[q] = ld_v4(src + off + (size_t)(q * 32 + lane) * 16);
#pragma unroll
    for (int q = 0; q < 8; ++q) st_v4(dst + (size_t)(q * 32 + lane) * 16, val[q]);
  }
}

int launch_nvlink_probe(const DevView& v, size_t bytes, cudaStream_t s) {
  if (v.W < 2) { set_error("NVLink probe needs peers"); return MX_ERR_INVALID; }
  pdl_launch(k_nvlink_probe, 148 * 4, 256, 0, s, v, bytes);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx

namespace mx {

// ------------------------------------------------------- expert weight prefetch
// Decode regime (weight-streaming GEMMs): once the layout has published the
// per-expert row counts, the weights of this rank's active experts are
// prefetched into L2 (cp.async.bulk.prefetch) on a side stream while the
// dispatch, its barrier and the expand run -- the GEMMs then find the first
// part of their weights in L2 instead of streaming all of it from HBM after
// the communication.  GEMM1's w13 first, then w2, up to `budget` bytes.
// Chunks are dealt round-robin over every thread of the grid (the bulk
// prefetches of one SM alone would serialise in its TMA unit).
__global__ void __launch_bounds__(128) k_prefetch_experts(DevView v, const char* w13,
                                                          const char* w2, size_t b13, size_t b2,
                                                          long long budget) {
  __shared__ int s_act[MX_EMAX];
  __shared__ int s_na;
  const int e0 = first_expert(v.group, v.n, v.E), e1 = first_expert(v.group + 1, v.n, v.E);
  const int* cnt = at<int>(v, v.rank, v.off.exp_cnt);
  if (threadIdx.x == 0) {
    int na = 0;
    for (int e = e0; e < e1; ++e)
      if (cnt[e] > 0) s_act[na++] = e - e0;
    s_na = na;
  }
  __syncthreads();
  const long long na = s_na;
  const long long t13 = na * (long long)b13, total0 = t13 + na * (long long)b2;
  const long long total = total0 < budget ? total0 : budget;
  constexpr long long CH = 32 * 1024;
  const long long nch = (total + CH - 1) / CH;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nch;
       c += (long long)gridDim.x * blockDim.x) {
    long long o = c * CH;
    const char* base;
    long long left;
    if (o < t13) {
      const long long a = o / (long long)b13, in = o - a * (long long)b13;
      base = w13 + (size_t)s_act[a] * b13 + in;
      left = (long long)b13 - in;
    } else {
      o -= t13;
      const long long a = o / (long long)b2, in = o - a * (long long)b2;
      base = w2 + (size_t)s_act[a] * b2 + in;
      left = (long long)b2 - in;
    }
    long long sz = CH < left ? CH : left;
    if (sz > total - c * CH) sz = total - c * CH;
    sz &= ~15LL;
    if (sz > 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base), "r"((unsigned)sz)
                   : "memory");
  }
}

int launch_prefetch_experts(const DevView& v, const void* w13, const void* w2, size_t b13,
                            size_t b2, long long budget, cudaStream_t s) {
  if (!w13 || !w2 || budget <= 0) return MX_OK;
  k_prefetch_experts<<<148, 128, 0, s>>>(v, static_cast<const char*>(w13),
                                         static_cast<const char*>(w2), b13, b2, budget);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx
