// devattr.cu -- per-device launch attributes.
//
// cudaFuncSetAttribute (the dynamic shared-memory opt-in) and the SM count are
// properties of a (device, kernel) pair, not of the process: one process may
// drive several GPUs through several hivf_ctx (the in-process shard group of
// hivf_group_create).  Every launcher therefore goes through these helpers,
// keyed by the calling thread's current device (the C-ABI entry points set it
// to the context's device before launching).
#include <cstdlib>
#include <mutex>
#include <map>
#include <utility>

#include "kernels.h"

namespace hivf {

namespace {
std::mutex g_mu;
std::map<std::pair<int, const void*>, int> g_optin;  // bytes opted in per (device, kernel)
int g_sms[kMaxDevices] = {};
}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HIVF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int device_sm_count() {
  const int d = current_device();
  if (d < 0 || d >= kMaxDevices) return 148;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_sms[d]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
    g_sms[d] = v;
  }
  return g_sms[d];
}

cudaError_t smem_optin(const void* kernel, int bytes) {
  const int d = current_device();
  std::lock_guard<std::mutex> lk(g_mu);
  int& have = g_optin[{d, kernel}];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

}  // namespace hivf
