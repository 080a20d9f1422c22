// Shared device-side declarations for the fedsim B200 kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fedsim_b200.h"

namespace fs {

constexpr int kNumSMs = 148;

// Flat parameter layout of the MLP (numpy_backend.py:3-14, unpack_layers
// numpy_backend.py:23-35): per layer W (fan_in x fan_out, row-major), then b.
struct MlpLayout {
  int L;                          // weight layers (hidden + head)
  int f[FS_MAX_LAYERS + 1];       // f[0]=input dim ... f[L]=1
  int64_t woff[FS_MAX_LAYERS];    // offset of W_l
  int64_t boff[FS_MAX_LAYERS];    // offset of b_l
  int64_t M;                      // total parameter count
  int sum_hidden;                 // sum of hidden widths (mask bits per row)
  int max_hidden;                 // widest hidden layer
};

inline int make_layout(const int32_t* dims, int32_t n_dims, MlpLayout* out) {
  if (n_dims < 3 || n_dims > FS_MAX_LAYERS + 1) return FS_EINVAL;
  MlpLayout m{};
  m.L = n_dims - 1;
  int64_t off = 0;
  for (int i = 0; i < n_dims; ++i) {
    if (dims[i] < 1) return FS_EINVAL;
    m.f[i] = dims[i];
  }
  if (m.f[m.L] != 1) return FS_EINVAL;
  for (int l = 0; l < m.L; ++l) {
    m.woff[l] = off;
    off += (int64_t)m.f[l] * m.f[l + 1];
    m.boff[l] = off;
    off += m.f[l + 1];
  }
  m.M = off;
  m.sum_hidden = 0;
  m.max_hidden = 0;
  for (int l = 1; l < m.L; ++l) {
    m.sum_hidden += m.f[l];
    if (m.f[l] > m.max_hidden) m.max_hidden = m.f[l];
  }
  *out = m;
  return FS_OK;
}

void set_error(const char* fmt, ...);
int check_launch(const char* what);
// Force-load the kernels that publish flags a trainer spins on (the flagged
// K3 and fs_publish_flag). Under CUDA lazy loading the first launch of a
// kernel may synchronise the context; if a consumer is already spinning on
// its flags, that first launch would never return.
void preload_mask_producer();
void preload_flag_publisher();

// wide-layer bf16 trainer (fs_train_wide.cu), reached through fs_train_bf16
size_t wide_workspace_bytes(const fs_train_desc* d);
int wide_train(const fs_train_desc* d, const void* features_bf16, const float* labels, cudaStream_t st);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size:
// the attribute call costs microseconds of host time, paid per launch before.
void ensure_smem_impl(const void* fn, int bytes);
template <class K>
inline void ensure_smem(K* kern, int bytes) {
  ensure_smem_impl(reinterpret_cast<const void*>(kern), bytes);
}

}  // namespace fs
