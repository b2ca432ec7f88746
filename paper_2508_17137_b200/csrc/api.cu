// Error reporting, version and device checks for the C ABI (include/moeb.h).
#include <cstdarg>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "common.cuh"

namespace moeb {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return fail(MOEB_ECUDA, "%s: %s", what, cudaGetErrorString(err));
  return MOEB_OK;
}

static int device_attr(cudaDeviceAttr attr) {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, attr, dev);
  return v;
}

int max_smem_per_block() { return device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin); }
int max_smem_per_sm() { return device_attr(cudaDevAttrMaxSharedMemoryPerMultiprocessor); }
int num_sms() { return device_attr(cudaDevAttrMultiProcessorCount); }

// cudaFuncSetAttribute costs tens of microseconds of host time per call;
// remember the largest dynamic shared memory already granted per (device,
// kernel) and only call it to raise the limit.
bool smem_attr_needed(const void* f, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> granted;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  int& g = granted[{dev, f}];
  if (bytes <= g) return false;
  g = bytes;
  return true;
}

}  // namespace moeb

__global__ void moeb_probe_kernel(int* out) { *out = 0x100a; }

extern "C" {

const char* moeb_last_error(void) { return moeb::g_last_error.c_str(); }

int moeb_version(void) { return 100; }

int moeb_device_check(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return moeb::fail(MOEB_EDEVICE, "no CUDA device");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
    return moeb::fail(MOEB_EDEVICE, "cudaGetDeviceProperties failed");
  if (prop.major != 10 || prop.minor != 0)
    return moeb::fail(MOEB_EDEVICE, "libmoeb is built for sm_100a (B200); device %s is sm_%d%d",
                      prop.name, prop.major, prop.minor);
  cudaFuncAttributes attr;
  if (cudaFuncGetAttributes(&attr, moeb_probe_kernel) != cudaSuccess)
    return moeb::fail(MOEB_EDEVICE, "kernels not loadable on %s", prop.name);
  return MOEB_OK;
}

}  // extern "C"
