// Shared helpers for the libmoeb kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "moeb.h"

namespace moeb {

// Thread-local last-error message (moeb_last_error); set by every failing
// entry point, never thrown across the C ABI.
void set_error(const char* fmt, ...);
void clear_error();
int fail(int code, const char* fmt, ...);
// Returns MOEB_ECUDA (and records the message) if the last launch failed.
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline int words_for(int E) { return (E + 63) / 64; }

// Largest dynamic shared memory one block may use, and per SM.
int max_smem_per_block();
int max_smem_per_sm();
int num_sms();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when it raises the
// kernel's limit on this device (the call itself costs host time per launch)
bool smem_attr_needed(const void* f, int bytes);
template <class F>
inline void set_smem(F* f, int bytes) {
  if (smem_attr_needed(reinterpret_cast<const void*>(f), bytes)) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    // these kernels size their grids for full shared-memory residency
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
  }
}

}  // namespace moeb

#define MOEB_REQUIRE(cond, ...)                       \
  do {                                                \
    if (!(cond)) return ::moeb::fail(MOEB_EINVAL, __VA_ARGS__); \
  } while (0)

// Iterate the set bits of a W-word mask in ascending expert order.
#define MOEB_FOR_EACH_BIT(W_, words_, ex_, body_)     \
  _Pragma("unroll") for (int w_ = 0; w_ < (W_); ++w_) { \
    uint64_t m_ = (words_)[w_];                       \
    while (m_) {                                      \
      const int ex_ = w_ * 64 + __ffsll((long long)m_) - 1; \
      m_ &= m_ - 1;                                   \
      body_                                           \
    }                                                 \
  }

__device__ __forceinline__ int popc_words1(uint64_t x) { return __popcll(x); }
