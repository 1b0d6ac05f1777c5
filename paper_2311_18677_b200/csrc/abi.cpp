// Status / error plumbing of the extern "C" surface (include/swb200.h).
// Mirrors the reference's exception hierarchy (errors.py:4-31) as int codes;
// the message of the last failure is kept per host thread.
#include <cstdarg>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/swb200.h"

static thread_local char g_err[1024] = "";

int swb_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int swb_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "%s launch failed: %s", what,
                         cudaGetErrorString(e));
  return SWB_OK;
}

extern "C" int swb_abi_version(void) { return SWB_ABI_VERSION; }

extern "C" const char* swb_last_error(void) { return g_err; }

extern "C" int swb_sync_stream(uintptr_t stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "stream sync: %s", cudaGetErrorString(e));
  return SWB_OK;
}

extern "C" int swb_enable_peer(int peer_device) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (peer_device == dev) return SWB_OK;
  int can = 0;
  cudaDeviceCanAccessPeer(&can, dev, peer_device);
  if (!can)
    return swb_set_error(SWB_ERR_CONFIG, "device %d cannot access peer %d", dev,
                         peer_device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return SWB_OK;
  }
  if (e != cudaSuccess)
    return swb_set_error(SWB_ERR_CUDA, "enable peer %d: %s", peer_device,
                         cudaGetErrorString(e));
  return SWB_OK;
}
