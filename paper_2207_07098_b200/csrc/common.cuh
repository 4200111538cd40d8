// Shared helpers for the semflow-b200 CUDA library (sm_100a, FP64 throughout).
//
// Arithmetic modes.  Every kernel that mirrors a reference loop is templated on
// EX ("exact"): with EX=true additions and multiplications are issued with the
// _rn intrinsics so ptxas cannot contract them into FMAs, which makes the result
// bit-identical to the reference numba lane (`_numba.py`, fastmath=False, no
// contraction) whenever the loop order is the same.  EX=false lets the compiler
// use DFMA (the production path; agrees with the reference to ~1e-16 relative).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Device-side bounds checks of the checked build (libsemflow_b200_checked.so,
// nvcc -DSF_CHECKS; SEMFLOW_B200_CHECKED=1 loads it): an index out of range traps
// the kernel with the failing condition printed -- this pool closes
// compute-sanitizer, so the GPU tests run against this build instead.
#ifdef SF_CHECKS
#include <cstdio>
#define SF_CHECK(cond)                                                                           \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("SF_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                  \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define SF_CHECK(cond) \
  do {              \
  } while (0)
#endif

namespace sf {

template <bool EX>
__device__ __forceinline__ double mul(double a, double b) {
  if constexpr (EX) return __dmul_rn(a, b); else return a * b;
}
template <bool EX>
__device__ __forceinline__ double add(double a, double b) {
  if constexpr (EX) return __dadd_rn(a, b); else return a + b;
}
template <bool EX>
__device__ __forceinline__ double sub(double a, double b) {
  if constexpr (EX) return __dsub_rn(a, b); else return a - b;
}
// acc + a*b : two roundings in EX mode, one DFMA otherwise.
template <bool EX>
__device__ __forceinline__ double mac(double acc, double a, double b) {
  if constexpr (EX) return __dadd_rn(acc, __dmul_rn(a, b)); else return fma(a, b, acc);
}

// Status codes of the C ABI (also in include/semflow_b200.h).
enum Status : int {
  SF_OK = 0,
  SF_ERR_ARG = 1,
  SF_ERR_CUDA = 2,
  SF_ERR_UNSUPPORTED = 3,
};

void set_error(const char* fmt, ...);
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Reduction geometry shared by every deterministic dot-product kernel: a fixed
// grid of RED_BLOCKS blocks x RED_THREADS threads; each thread folds its grid-
// stride slice sequentially, warps and blocks combine by fixed trees and the last
// block to finish combines the per-block partials in block order.  The result is
// a pure function of the inputs and P (never of scheduling).
constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 148 * 8;

}  // namespace sf
