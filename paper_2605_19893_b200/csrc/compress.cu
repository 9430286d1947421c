// compress.cu -- compressed-cache append on sm_100a.
//
// Replaces nsa::extend_compressed_layer / pool_block (src/nsa_cache.cpp:14-66).
// Block i pools rows [i*d, i*d + l) of one KV head: keys get the per-offset
// position embedding, values are plain means.  Accumulation is fp64 in the
// reference's order (per offset o: += k, += pe, then += v), scaled by 1/l and
// rounded to fp32, so ck is bit-identical to the reference on the same bf16
// rows.  ck16 / cv are the bf16 (RNE) copies the attention kernel streams.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attend.h"

namespace specsv_b200 {
namespace {

__global__ void compress_kernel(const __nv_bfloat16* __restrict__ k,
                                const __nv_bfloat16* __restrict__ v, const float* __restrict__ pe,
                                float* __restrict__ ck, __nv_bfloat16* __restrict__ ck16,
                                __nv_bfloat16* __restrict__ cv, int64_t first, int hkv, int dh,
                                int l, int d) {
  const int64_t b = first + blockIdx.x;
  const int h = blockIdx.y;
  const double inv_l = 1.0 / (double)l;
  for (int x = threadIdx.x; x < dh; x += blockDim.x) {
    double acc_k = 0.0, acc_v = 0.0;
    for (int o = 0; o < l; ++o) {
      const int64_t off = ((b * d + o) * hkv + h) * dh + x;
      acc_k = __dadd_rn(acc_k, (double)__bfloat162float(k[off]));
      if (pe != nullptr) acc_k = __dadd_rn(acc_k, (double)pe[o * dh + x]);
      acc_v = __dadd_rn(acc_v, (double)__bfloat162float(v[off]));
    }
    const float fk = (float)__dmul_rn(acc_k, inv_l);
    const float fv = (float)__dmul_rn(acc_v, inv_l);
    const int64_t o = (b * hkv + h) * dh + x;
    ck[o] = fk;
    ck16[o] = __float2bfloat16_rn(fk);
    cv[o] = __float2bfloat16_rn(fv);
  }
}

// the blocks a commit completed, in every layer at once: grid (block, head,
// layer); the same pooling as compress_kernel
__global__ void compress_layers_kernel(const __grid_constant__ CompressLayers c) {
  const int j = blockIdx.z;
  if ((int64_t)blockIdx.x >= c.count[j]) return;
  const int64_t b = c.first[j] + blockIdx.x;
  const int h = blockIdx.y;
  const int hkv = c.hkv, dh = c.dh, l = c.l, d = c.d;
  const __nv_bfloat16* k = static_cast<const __nv_bfloat16*>(c.k[j]);
  const __nv_bfloat16* v = static_cast<const __nv_bfloat16*>(c.v[j]);
  const float* pe = c.pe[j];
  const double inv_l = 1.0 / (double)l;
  for (int x = threadIdx.x; x < dh; x += blockDim.x) {
    double acc_k = 0.0, acc_v = 0.0;
    for (int o = 0; o < l; ++o) {
      const int64_t off = ((b * d + o) * hkv + h) * dh + x;
      acc_k = __dadd_rn(acc_k, (double)__bfloat162float(k[off]));
      if (pe != nullptr) acc_k = __dadd_rn(acc_k, (double)pe[o * dh + x]);
      acc_v = __dadd_rn(acc_v, (double)__bfloat162float(v[off]));
    }
    const float fk = (float)__dmul_rn(acc_k, inv_l);
    const float fv = (float)__dmul_rn(acc_v, inv_l);
    const int64_t o = (b * hkv + h) * dh + x;
    c.ck[j][o] = fk;
    static_cast<__nv_bfloat16*>(c.ck16[j])[o] = __float2bfloat16_rn(fk);
    static_cast<__nv_bfloat16*>(c.cv[j])[o] = __float2bfloat16_rn(fv);
  }
}

}  // namespace

cudaError_t launch_compress_layers(const CompressLayers& c, int n_layers, int64_t max_count,
                                   cudaStream_t stream) {
  if (n_layers <= 0 || max_count <= 0) return cudaSuccess;
  if (max_count > 65535) return cudaErrorInvalidValue;
  compress_layers_kernel<<<dim3((unsigned)max_count, c.hkv, n_layers), c.dh < 256 ? c.dh : 256, 0,
                           stream>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_compress(const void* k, const void* v, const float* pe, float* ck, void* ck16,
                            void* cv, int64_t first, int64_t last, int hkv, int dh, int l, int d,
                            cudaStream_t stream) {
  if (last <= first) return cudaSuccess;
  const int64_t nb = last - first;
  for (int64_t done = 0; done < nb; done += 65535) {
    const int64_t chunk = nb - done < 65535 ? nb - done : 65535;
    compress_kernel<<<dim3((unsigned)chunk, hkv), dh < 256 ? dh : 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(k), static_cast<const __nv_bfloat16*>(v), pe, ck,
        static_cast<__nv_bfloat16*>(ck16), static_cast<__nv_bfloat16*>(cv), first + done, hkv, dh,
        l, d);
  }
  return cudaGetLastError();
}

}  // namespace specsv_b200
