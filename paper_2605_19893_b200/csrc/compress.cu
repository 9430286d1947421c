// compress.cu -- compressed-cache append on sm_100a.
//
// Replaces nsa::extend_compressed_layer / pool_block (src/nsa_cache.cpp:14-66).
// Block i pools rows [i*d, i*d + l) of one KV head: keys get the per-offset
// position embedding, values are plain means.  Accumulation is fp64 in the
// reference's order (per offset o: += k, += pe, then += v), scaled by 1/l and
// rounded to fp32, so ck is bit-identical to the reference on the same bf16
// rows.  ck16 / cv are the bf16 (RNE) copies the attention kernel streams.
// When the cache carries digit planes (ckd / ckexp), each (block, head) row of
// ck is also written as a 31-bit fixed-point integer on the row's own
// power-of-two grid (X = round(ck 2^(30 - e)), max |ck| < 2^e), split into
// four signed base-256 digits: the routing kernel (route3.cu) feeds them to
// the integer tensor pipe without converting anything per call.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attend.h"
#include "sm100.cuh"

namespace specsv_b200 {
namespace {

// max |v| over the (block, head) row held by this CTA (blockDim threads)
__device__ float row_absmax(float v, float* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  float m = 0.f;
  for (int i = 0; i < nw; ++i) m = fmaxf(m, red[i]);
  return m;
}

// four signed base-256 digits of round(x 2^(30 - e)) (|result| <= 2^30):
// byte s is the digit of weight 256^s, in [-128, 127]
__device__ __forceinline__ uint32_t digits4(float x, int e) {
  const int X = __float2int_rn(ldexpf(x, 30 - e));
  return (static_cast<uint32_t>(X) + 0x80808080u) ^ 0x80808080u;
}

// the digit planes of one (block, head) row: fk[r] is element threadIdx.x + r blockDim.
// ckexp packs the row exponent e (low 16 bits, signed) and, in bits 16..23, how many
// elements the 31-bit grid rounds (the others it represents exactly: the routing
// kernel's error bound counts only the rounded ones)
template <int kPer>
__device__ void write_digit_row(const float (&fk)[kPer], int dh, int8_t* ckd, int32_t* ckexp,
                                int64_t row) {
  __shared__ float red[32];
  __shared__ int inexact;
  float a = 0.f;
#pragma unroll
  for (int r = 0; r < kPer; ++r)
    if (threadIdx.x + r * blockDim.x < dh) a = fmaxf(a, fabsf(fk[r]));
  if (threadIdx.x == 0) inexact = 0;
  const float mx = row_absmax(a, red);  // (its barriers order the reset)
  int e = 0;
  if (mx > 0.f) frexpf(mx, &e);  // mx < 2^e
  int8_t* dst = ckd + row * 4 * dh;
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < kPer; ++r) {
    const int x = threadIdx.x + r * blockDim.x;
    if (x >= dh) break;
    const float sx = ldexpf(fk[r], 30 - e);
    cnt += (float)__float2int_rn(sx) != sx ? 1 : 0;
    const uint32_t w = digits4(fk[r], e);
#pragma unroll
    for (int s = 0; s < 4; ++s) dst[s * dh + x] = static_cast<int8_t>((w >> (8 * s)) & 0xFFu);
  }
  if (cnt) atomicAdd(&inexact, cnt);
  __syncthreads();
  if (threadIdx.x == 0) ckexp[row] = (e & 0xFFFF) | (min(inexact, 255) << 16);
}

// fp64 sums of one compressed block's l rows (key + positional embedding,
// value) for element x, in the reference's order (nsa_cache.cpp); the loads of
// eight rows go out together ahead of their (ordered) adds
__device__ __forceinline__ void pool_rows(const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v,
                                          const float* __restrict__ pe, int64_t b, int h, int x, int hkv,
                                          int dh, int l, int d, double& acc_k, double& acc_v) {
  for (int o0 = 0; o0 < l; o0 += 8) {
    float kk[8], vv[8], pp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int o = o0 + u;
      kk[u] = vv[u] = pp[u] = 0.f;
      if (o < l) {
        const int64_t off = ((b * d + o) * hkv + h) * dh + x;
        kk[u] = __bfloat162float(k[off]);
        vv[u] = __bfloat162float(v[off]);
        if (pe != nullptr) pp[u] = pe[o * dh + x];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (o0 + u < l) {
        acc_k = __dadd_rn(acc_k, (double)kk[u]);
        if (pe != nullptr) acc_k = __dadd_rn(acc_k, (double)pp[u]);
        acc_v = __dadd_rn(acc_v, (double)vv[u]);
      }
    }
  }
}

__global__ void compress_kernel(const __nv_bfloat16* __restrict__ k,
                                const __nv_bfloat16* __restrict__ v, const float* __restrict__ pe,
                                float* __restrict__ ck, __nv_bfloat16* __restrict__ ck16,
                                __nv_bfloat16* __restrict__ cv, int8_t* __restrict__ ckd,
                                int32_t* __restrict__ ckexp, int64_t first, int hkv, int dh, int l,
                                int d) {
  const int64_t b = first + blockIdx.x;
  const int h = blockIdx.y;
  const double inv_l = 1.0 / (double)l;
  float fkr[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int x = threadIdx.x + r * blockDim.x;
    fkr[r] = 0.f;
    if (x >= dh) continue;
    double acc_k = 0.0, acc_v = 0.0;
    pool_rows(k, v, pe, b, h, x, hkv, dh, l, d, acc_k, acc_v);
    const float fk = (float)__dmul_rn(acc_k, inv_l);
    const float fv = (float)__dmul_rn(acc_v, inv_l);
    const int64_t o = (b * hkv + h) * dh + x;
    ck[o] = fk;
    ck16[o] = __float2bfloat16_rn(fk);
    cv[o] = __float2bfloat16_rn(fv);
    fkr[r] = fk;
  }
  if (ckd != nullptr) write_digit_row(fkr, dh, ckd, ckexp, b * hkv + h);
}

// the blocks a commit completed, in every layer at once: grid (block, head,
// layer); the same pooling as compress_kernel
__global__ void compress_layers_kernel(const __grid_constant__ CompressLayers c) {
  sm100::griddep_wait();  // (programmatic dependent launch) the committed rows are in
  const int j = blockIdx.z;
  if ((int64_t)blockIdx.x >= c.count[j]) return;
  const int64_t b = c.first[j] + blockIdx.x;
  const int h = blockIdx.y;
  const int hkv = c.hkv, dh = c.dh, l = c.l, d = c.d;
  const __nv_bfloat16* k = static_cast<const __nv_bfloat16*>(c.k[j]);
  const __nv_bfloat16* v = static_cast<const __nv_bfloat16*>(c.v[j]);
  const float* pe = c.pe[j];
  const double inv_l = 1.0 / (double)l;
  float fkr[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int x = threadIdx.x + r * blockDim.x;
    fkr[r] = 0.f;
    if (x >= dh) continue;
    double acc_k = 0.0, acc_v = 0.0;
    pool_rows(k, v, pe, b, h, x, hkv, dh, l, d, acc_k, acc_v);
    const float fk = (float)__dmul_rn(acc_k, inv_l);
    const float fv = (float)__dmul_rn(acc_v, inv_l);
    const int64_t o = (b * hkv + h) * dh + x;
    c.ck[j][o] = fk;
    static_cast<__nv_bfloat16*>(c.ck16[j])[o] = __float2bfloat16_rn(fk);
    static_cast<__nv_bfloat16*>(c.cv[j])[o] = __float2bfloat16_rn(fv);
    fkr[r] = fk;
  }
  if (c.ckd[j] != nullptr) write_digit_row(fkr, dh, static_cast<int8_t*>(c.ckd[j]), c.ckexp[j], b * hkv + h);
}

}  // namespace

cudaError_t launch_compress_layers(const CompressLayers& c, int n_layers, int64_t max_count,
                                   cudaStream_t stream) {
  if (n_layers <= 0 || max_count <= 0) return cudaSuccess;
  if (max_count > 65535) return cudaErrorInvalidValue;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)max_count, c.hkv, n_layers);
  lc.blockDim = dim3(c.dh < 256 ? c.dh : 256);
  lc.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&lc, compress_layers_kernel, c);
  return cudaGetLastError();
}

cudaError_t launch_compress(const void* k, const void* v, const float* pe, float* ck, void* ck16,
                            void* cv, void* ckd, int32_t* ckexp, int64_t first, int64_t last, int hkv,
                            int dh, int l, int d, cudaStream_t stream) {
  if (last <= first) return cudaSuccess;
  const int64_t nb = last - first;
  for (int64_t done = 0; done < nb; done += 65535) {
    const int64_t chunk = nb - done < 65535 ? nb - done : 65535;
    compress_kernel<<<dim3((unsigned)chunk, hkv), dh < 256 ? dh : 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), pe, ck,
        static_cast<__nv_bfloat16*>(ck16), static_cast<__nv_bfloat16*>(cv), static_cast<int8_t*>(ckd),
        ckexp, first + done, hkv, dh, l, d);
  }
  return cudaGetLastError();
}

}  // namespace specsv_b200
