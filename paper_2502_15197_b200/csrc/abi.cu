// Library-wide C-ABI entry points: error string, version, workspace sizing/initialisation.
#include "abi_util.h"
#include "launch.h"

#include <mutex>
#include <set>

namespace tetris {
namespace abi {
char* err_buf() {
  static thread_local char buf[512] = {0};
  return buf;
}
}  // namespace abi
}  // namespace tetris

extern "C" const char* tetris_last_error(void) { return tetris::abi::err_buf(); }

extern "C" int tetris_abi_version(void) { return 1; }

extern "C" size_t tetris_workspace_bytes(int op, int32_t B, int32_t k, int32_t V) {
  if (B < 0 || k < 0 || V < 0) return 0;
  return tetris::abi::region_offset(op, B, k, V, tetris::abi::WS_END);
}

extern "C" int tetris_workspace_init(void* ws, size_t ws_bytes, tetris_stream_t stream) {
  if (!ws && ws_bytes) return tetris::abi::fail(TETRIS_INVALID_ARGUMENT, "null workspace");
  if (!ws_bytes) return TETRIS_OK;
  cudaError_t e = cudaMemsetAsync(ws, 0, ws_bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return tetris::abi::cuda_fail(e);
  return TETRIS_OK;
}

// host ranges this library registered itself (tetris_unmap_host releases only those; caller-pinned memory is the
// caller's)
static std::mutex g_reg_mu;
static std::set<void*> g_registered;

extern "C" int tetris_map_host(void* host_ptr, size_t bytes, void** dev_ptr) {
  if (!host_ptr || !dev_ptr) return tetris::abi::fail(TETRIS_INVALID_ARGUMENT, "null pointer");
  cudaError_t e = cudaHostGetDevicePointer(dev_ptr, host_ptr, 0);
  if (e == cudaSuccess) return TETRIS_OK;
  cudaGetLastError();  // not pinned yet: register it
  e = cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) return tetris::abi::cuda_fail(e);
  {
    std::lock_guard<std::mutex> lock(g_reg_mu);
    g_registered.insert(host_ptr);
  }
  e = cudaHostGetDevicePointer(dev_ptr, host_ptr, 0);
  if (e != cudaSuccess) return tetris::abi::cuda_fail(e);
  return TETRIS_OK;
}

extern "C" int tetris_unmap_host(void* host_ptr) {
  if (!host_ptr) return TETRIS_OK;
  {
    std::lock_guard<std::mutex> lock(g_reg_mu);
    auto it = g_registered.find(host_ptr);
    if (it == g_registered.end()) return TETRIS_OK;  // pinned by the caller, or never mapped: nothing to release
    g_registered.erase(it);
  }
  cudaError_t e = cudaHostUnregister(host_ptr);
  if (e != cudaSuccess) return tetris::abi::cuda_fail(e);
  return TETRIS_OK;
}

extern "C" int tetris_spec_max_requests(void) { return tetris::spec_max_requests(); }

extern "C" int tetris_debug_timestamps(void* dev_buf) {
  tetris::set_debug_buffer((long long*)dev_buf);
  return TETRIS_OK;
}
