// quant.cu -- bf16 -> e4m3 row quantisation for the fp8 expert path.
//
// Each row gets one fp32 scale = amax / 448 (e4m3 max finite); the e4m3
// bytes (round-to-nearest-even, saturating) are followed in the same row by
// the fp32 scale at byte `cols`, so a row travels over NVLink and into the
// GEMM's TMA tile with its scale (row stride ldd >= cols + 16).
#include <cuda_fp8.h>

#include "mx_internal.cuh"

namespace mx {

__global__ void __launch_bounds__(256)
k_quant_rows(const __nv_bfloat16* __restrict__ src, long long lds, unsigned char* __restrict__ dst,
             long long ldd, long long rows, const int32_t* rows_dev, int cols) {
  pdl_wait();  // predecessor's outputs are visible after this
  const int lane = threadIdx.x & 31;
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  // rows_dev: the live row count (a host's routed rows), clamped to the buffer's
  const long long R = rows_dev ? min((long long)*rows_dev, rows) : rows;
  for (long long r = gw; r < R; r += nw) {
    const __nv_bfloat16* s = src + r * lds;
    float amax = 0.f;
    for (int c = lane * 8; c < cols; c += 256) {
      const uint4 raw = ld_v4(s + c);
      const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
      for (int q = 0; q < 8; ++q) amax = fmaxf(amax, fabsf(__bfloat162float(v[q])));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const float scale = amax > 0.f ? amax / 448.f : 1.f;
    const float inv = 1.f / scale;
    unsigned char* d = dst + r * ldd;
    for (int c = lane * 8; c < cols; c += 256) {
      const uint4 raw = ld_v4(s + c);
      const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&raw);
      uint2 out;
      unsigned char* ob = reinterpret_cast<unsigned char*>(&out);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        ob[q] = (unsigned char)__nv_cvt_float_to_fp8(__bfloat162float(v[q]) * inv, __NV_SATFINITE,
                                                      __NV_E4M3);
      *reinterpret_cast<uint2*>(d + c) = out;
    }
    if (lane == 0) *reinterpret_cast<float*>(d + cols) = scale;
  }
}

int quant_rows_e4m3(const void* src, long long lds, void* dst, long long ldd, long long rows,
                    const int32_t* rows_dev, int cols, cudaStream_t s) {
  if (cols % 256 != 0 && cols % 8 != 0) { set_error("quant: cols %% 8 != 0"); return MX_ERR_UNSUPPORTED; }
  long long blocks = (rows + 7) / 8;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pdl_launch(k_quant_rows, (int)blocks, 256, 0, s, static_cast<const __nv_bfloat16*>(src), lds,
                                            static_cast<unsigned char*>(dst), ldd, rows, rows_dev,
                                            cols);
  MX_LAUNCH_CHECK();
  return MX_OK;
}

}  // namespace mx

using namespace mx;

extern "C" {

int mx_quant_rows_e4m3(const void* src, long long lds, void* dst, long long ldd, long long rows,
                       int cols, void* stream) {
  return quant_rows_e4m3(src, lds, dst, ldd, rows, nullptr, cols, static_cast<cudaStream_t>(stream));
}

int mx_grouped_gemm_fp8(const void* A, long long lda, const void* B, const float* b_scales,
                        void* D, const int32_t* offs, const int32_t* cnts, int G, long long M_total,
                        int N, int K, int swiglu, void* stream) {
  return grouped_gemm_fp8(A, lda, B, b_scales, D, offs, cnts, nullptr, G, M_total, M_total, N, K,
                          swiglu, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
