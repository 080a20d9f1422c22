#include <mutex>
#include <unordered_map>
// C-ABI plumbing: thread-local error messages and launch checks.
#include <cstdarg>
#include <cstdio>

#include "fs_common.cuh"

namespace fs {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FS_ECUDA;
  }
  return FS_OK;
}

}  // namespace fs

extern "C" const char* fs_last_error(void) { return fs::g_err; }

extern "C" int32_t fs_struct_sizes(size_t* out, int32_t n) {
  const size_t sz[6] = {sizeof(fs_train_desc),  sizeof(fs_client_done),   sizeof(fs_async_world),
                        sizeof(fs_async_yield), sizeof(fs_async_logview), sizeof(fs_async_device)};
  for (int32_t i = 0; out && i < n && i < 6; ++i) out[i] = sz[i];
  return 6;
}

extern "C" int fs_abi_version(void) { return FS_ABI_VERSION; }

namespace fs {
void ensure_smem_impl(const void* fn, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> set_to;
  std::lock_guard<std::mutex> lock(mu);
  auto it = set_to.find(fn);
  if (it != set_to.end() && it->second >= bytes) return;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  set_to[fn] = bytes;
}
}  // namespace fs

namespace {
__global__ void fill_u64_kernel(uint64_t* dst, uint64_t v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = v;
}
}  // namespace

// dst[0..n) = value (8-byte words; a double's bits or a device pointer): the
// per-request launch arguments that are one value for a whole round
extern "C" int fs_fill_u64(uint64_t* dst, uint64_t value, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && !dst)) {
    fs::set_error("fs_fill_u64: invalid arguments");
    return FS_EINVAL;
  }
  if (n == 0) return FS_OK;
  const int blocks = (int)((n + 255) / 256 < 64 ? (n + 255) / 256 : 64);
  fill_u64_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(dst, value, n);
  return fs::check_launch("fill_u64_kernel");
}

namespace {
__global__ void publish_flag_kernel(int32_t* flag, int32_t v) {
  __threadfence();
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
}  // namespace

void fs::preload_flag_publisher() {
  static const bool done = [] {
    cudaFuncAttributes at;
    return cudaFuncGetAttributes(&at, publish_flag_kernel) == cudaSuccess;
  }();
  (void)done;
}

extern "C" int fs_publish_flag(int32_t* flag, int32_t value, void* stream) {
  if (!flag) {
    fs::set_error("fs_publish_flag: null flag");
    return FS_EINVAL;
  }
  publish_flag_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  return fs::check_launch("publish_flag_kernel");
}

extern "C" int fs_upload_chunks(void* dst_a, const void* src_a, int64_t a_row_bytes, void* dst_b,
                                const void* src_b, int64_t b_row_bytes, const int64_t* bounds, int32_t n_chunks,
                                int32_t* flags, int32_t tag, void* stream) {
  if (n_chunks < 0 || a_row_bytes < 0 || b_row_bytes < 0 || (n_chunks > 0 && (!bounds || !flags))) {
    fs::set_error("fs_upload_chunks: invalid arguments");
    return FS_EINVAL;
  }
  const cudaStream_t st = (cudaStream_t)stream;
  for (int32_t c = 0; c < n_chunks; ++c) {
    const int64_t r0 = bounds[2 * c], r1 = bounds[2 * c + 1];
    if (r1 < r0 || r0 < 0) {
      fs::set_error("fs_upload_chunks: chunk %d has rows [%lld, %lld)", c, (long long)r0, (long long)r1);
      return FS_EINVAL;
    }
    if (r1 > r0 && a_row_bytes > 0 &&
        cudaMemcpyAsync(static_cast<char*>(dst_a) + r0 * a_row_bytes, static_cast<const char*>(src_a) + r0 * a_row_bytes,
                        (size_t)((r1 - r0) * a_row_bytes), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return fs::check_launch("fs_upload_chunks");
    if (r1 > r0 && b_row_bytes > 0 &&
        cudaMemcpyAsync(static_cast<char*>(dst_b) + r0 * b_row_bytes, static_cast<const char*>(src_b) + r0 * b_row_bytes,
                        (size_t)((r1 - r0) * b_row_bytes), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return fs::check_launch("fs_upload_chunks");
    publish_flag_kernel<<<1, 1, 0, st>>>(flags + c, tag);
  }
  return fs::check_launch("fs_upload_chunks");
}

extern "C" int fs_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return FS_OK;
  if (!dst || !src) {
    fs::set_error("fs_memcpy_d2d: null pointer");
    return FS_EINVAL;
  }
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
    return fs::check_launch("fs_memcpy_d2d");
  return FS_OK;
}
