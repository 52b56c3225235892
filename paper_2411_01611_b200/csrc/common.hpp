// Shared host-side plumbing for libembcomm_gpu: error model, CUDA checks.
//
// Internally the library throws ec::Error; every extern "C" entry point wraps
// its body in ec::guard(), which maps the error to the ABI status code and
// stores the message for ec_last_error() (no exception crosses the ABI —
// the reference's ValidationError / InvariantError split,
// core/include/embcomm/error.hpp:10-19, becomes EC_EINVAL / EC_EINVARIANT).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "embcomm_gpu.h"

namespace ec {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void invalid(const std::string& m) { throw Error(EC_EINVAL, m); }
[[noreturn]] inline void invariant(const std::string& m) { throw Error(EC_EINVARIANT, m); }

void set_last_error(const std::string& m);

template <class F>
int guard(F&& f) noexcept {
  try {
    f();
    return EC_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return EC_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return EC_EINVARIANT;
  }
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? EC_ENOMEM : EC_ECUDA;
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                          std::to_string(line) + ")");
  }
}

#define EC_CUDA(x) ::ec::cuda_check((x), #x, __FILE__, __LINE__)
#define EC_LAUNCH() ::ec::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Number of SMs of the current device (148 on B200), cached per device.
int sm_count(int device);

// Make `device` current and fail loudly when there is no usable GPU.
void use_device(int device);

// Device buffer owned by RAII.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    free();
    n = count;
    if (count) EC_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  size_t bytes() const { return n * sizeof(T); }
};

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// SplitMix64 output mix (core/include/embcomm/rng.hpp:18-20).
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// substream_seed (rng.hpp:33-38).
__host__ __device__ inline uint64_t substream(uint64_t master, uint64_t index) {
  return mix64(master + (index + 1) * kGolden);
}

}  // namespace ec
