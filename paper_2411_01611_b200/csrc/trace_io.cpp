// Binary trace ingest.  The reference reads traces in
// a text format only (`d=<int> E=<int>` then one sample per line,
// core/src/trace.cpp:51-101), which is desk-scale; Criteo-shaped replays need
// billions of ids.  This is the same Trace (core/include/embcomm/trace.hpp:
// 18-30: num_features d, vocab_size E, row-major Q x d uint32 ids) in a binary
// container that is mapped, not parsed:
//
//   offset  0  char[8]  magic "ECTRACE1"
//           8  uint32   version (1)
//          12  uint32   reserved (0)
//          16  int64    d  (>= 1)
//          24  uint64   E  (1 .. 2^32 - 1)
//          32  uint64   Q  (>= 1 samples)
//          40  uint32   ids[Q * d], little-endian, sample-major
//
// Validation mirrors parse_trace: d >= 1, 1 <= E <= UINT32_MAX, a non-empty
// body of exactly Q*d ids, every id < E (the error names the offending
// sample and its "line" = sample + 2, as the text format would).
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"

namespace ec {

namespace {

constexpr char kMagic[8] = {'E', 'C', 'T', 'R', 'A', 'C', 'E', '1'};

struct Header {
  char magic[8];
  uint32_t version;
  uint32_t reserved;
  int64_t d;
  uint64_t vocab;
  uint64_t samples;
};
static_assert(sizeof(Header) == 40, "trace header layout");

struct TraceFile {
  int fd = -1;
  void* map = nullptr;
  size_t map_len = 0;
  Header h{};
  const uint32_t* ids = nullptr;
  ~TraceFile() {
    if (map && map != MAP_FAILED) munmap(map, map_len);
    if (fd >= 0) close(fd);
  }
};

// First id >= vocab, scanned with a few threads (traces can be GBs).
uint64_t first_out_of_range(const uint32_t* ids, uint64_t n, uint64_t vocab) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const uint64_t parts = n < (1u << 20) ? 1 : hw;
  std::vector<uint64_t> bad(parts, n);
  std::vector<std::thread> th;
  for (uint64_t k = 0; k < parts; ++k) {
    th.emplace_back([&, k] {
      const uint64_t lo = n * k / parts, hi = n * (k + 1) / parts;
      for (uint64_t i = lo; i < hi; ++i)
        if (ids[i] >= vocab) {
          bad[k] = i;
          return;
        }
    });
  }
  for (auto& t : th) t.join();
  return *std::min_element(bad.begin(), bad.end());
}

void check_header(const Header& h) {
  if (std::memcmp(h.magic, kMagic, sizeof(kMagic)) != 0) invalid("not a binary trace (bad magic)");
  if (h.version != 1) invalid("unsupported binary trace version " + std::to_string(h.version));
  if (h.d < 1) invalid("lookups per sample must be >= 1");
  if (h.vocab < 1) invalid("vocabulary size must be >= 1");
  if (h.vocab > 0xFFFFFFFFull) invalid("vocabulary too large for 32-bit ids");
  if (h.samples < 1) invalid("empty trace");
}

void check_ids(const Header& h, const uint32_t* ids) {
  const uint64_t n = h.samples * static_cast<uint64_t>(h.d);
  const uint64_t i = first_out_of_range(ids, n, h.vocab);
  if (i < n) {
    const uint64_t sample = i / static_cast<uint64_t>(h.d);
    invalid("line " + std::to_string(sample + 2) + ": id " + std::to_string(ids[i]) + " out of range [0, " +
            std::to_string(h.vocab) + ")");
  }
}

}  // namespace
}  // namespace ec

using namespace ec;

struct ec_trace_s {
  TraceFile f;
};

namespace ec {
namespace {

// Pinned host -> device by SM loads of the mapped source, from a few CTAs.
// The host link is shared with the cold tier's random 64 B row reads; a
// copy-engine burst of the next batch's ids starves those (measured with
// tools/hostlink_bench: 7187 rows 35 -> 63 us beside a 1.7 MB
// cudaMemcpyAsync) while an 8-CTA pull leaves them at 46 us and lands in
// ~66 us, within a step.  Kaggle e2e step (bench.py, interleaved runs on one
// box): copy engine 0.132 ms, 4 CTAs 0.130-0.146, 8 CTAs 0.101-0.107,
// 16 CTAs 0.125-0.133.  With HBM-resident rows nothing else uses the link
// and the copy engine is the faster choice (the pull then bounds the step).
__global__ void k_h2d_pull(const int4* __restrict__ src, int4* __restrict__ dst, uint64_t n16,
                           const uint8_t* __restrict__ src_tail, uint8_t* __restrict__ dst_tail, int tail) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16; i += stride)
    dst[i] = src[i];
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
}

// Device address of a pinned, mapped host buffer, else nullptr.
const void* mapped_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool is_device(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice;
}

}  // namespace
}  // namespace ec

extern "C" {

// Stream-ordered copy between any two UVA addresses (pinned host <-> device):
// the input-pipeline primitive of a training loop, with one call's host cost.
int ec_copy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
  return guard([&] {
    if (!bytes) return;
    if (!dst || !src) invalid("null argument");
    EC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  });
}

// The same for pinned (mapped) host -> device, pulled by `ctas` CTAs' loads
// (k_h2d_pull) instead of the copy engine: for inputs that share the host
// link with the pinned-host cold tier.  Other address kinds, misaligned
// (16-byte) ends or ctas <= 0 fall back to ec_copy_async.
int ec_copy_async_pull(void* dst, const void* src, uint64_t bytes, int ctas, void* stream) {
  return guard([&] {
    if (!bytes) return;
    if (!dst || !src) invalid("null argument");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const void* msrc = ctas > 0 ? mapped_host(src) : nullptr;
    if (msrc && is_device(dst) && (reinterpret_cast<uintptr_t>(msrc) % 16) == 0 &&
        (reinterpret_cast<uintptr_t>(dst) % 16) == 0) {
      const uint64_t n16 = bytes / 16;
      const int tail = static_cast<int>(bytes % 16);
      k_h2d_pull<<<ctas, 512, 0, st>>>(static_cast<const int4*>(msrc), static_cast<int4*>(dst), n16,
                                       static_cast<const uint8_t*>(msrc) + n16 * 16,
                                       static_cast<uint8_t*>(dst) + n16 * 16, tail);
      EC_CUDA(cudaGetLastError());
      return;
    }
    EC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  });
}

int ec_trace_save_binary(const char* path, const uint32_t* ids_host, uint64_t num_samples, int64_t num_features,
                         uint64_t vocab) {
  return guard([&] {
    if (!path || (!ids_host && num_samples)) invalid("null argument");
    Header h{};
    std::memcpy(h.magic, kMagic, sizeof(kMagic));
    h.version = 1;
    h.d = num_features;
    h.vocab = vocab;
    h.samples = num_samples;
    check_header(h);
    check_ids(h, ids_host);
    FILE* f = std::fopen(path, "wb");
    if (!f) invalid(std::string("cannot write trace file ") + path);
    const uint64_t n = num_samples * static_cast<uint64_t>(num_features);
    const bool ok = std::fwrite(&h, sizeof(h), 1, f) == 1 && std::fwrite(ids_host, sizeof(uint32_t), n, f) == n;
    const bool closed = std::fclose(f) == 0;
    if (!ok || !closed) invalid(std::string("short write to trace file ") + path);
  });
}

int ec_trace_open_binary(const char* path, ec_trace* out) {
  return guard([&] {
    if (!path || !out) invalid("null argument");
    *out = nullptr;
    auto t = std::make_unique<ec_trace_s>();
    TraceFile& f = t->f;
    f.fd = open(path, O_RDONLY);
    if (f.fd < 0) invalid(std::string("cannot open trace file ") + path);
    struct stat st {};
    if (fstat(f.fd, &st) != 0) invalid(std::string("cannot stat trace file ") + path);
    const uint64_t size = static_cast<uint64_t>(st.st_size);
    if (size < sizeof(Header)) invalid("truncated binary trace (no header)");
    f.map_len = size;
    f.map = mmap(nullptr, size, PROT_READ, MAP_PRIVATE, f.fd, 0);
    if (f.map == MAP_FAILED) invalid(std::string("cannot map trace file ") + path);
    madvise(f.map, size, MADV_SEQUENTIAL);
    std::memcpy(&f.h, f.map, sizeof(Header));
    check_header(f.h);
    // samples * d * 4 must not wrap: bound samples by the file's id capacity first
    if (f.h.d <= 0 || f.h.samples > (size - sizeof(Header)) / sizeof(uint32_t) / static_cast<uint64_t>(f.h.d))
      invalid("binary trace size " + std::to_string(size) + " is too small for the header's " +
              std::to_string(f.h.samples) + " samples of " + std::to_string(f.h.d) + " ids");
    const uint64_t n = f.h.samples * static_cast<uint64_t>(f.h.d);
    if (size != sizeof(Header) + n * sizeof(uint32_t))
      invalid("binary trace size " + std::to_string(size) + " != header + " + std::to_string(n) + " ids");
    f.ids = reinterpret_cast<const uint32_t*>(static_cast<const char*>(f.map) + sizeof(Header));
    check_ids(f.h, f.ids);
    *out = t.release();
  });
}

void ec_trace_destroy(ec_trace t) { delete t; }

int ec_trace_info(ec_trace t, uint64_t* num_samples, int64_t* num_features, uint64_t* vocab) {
  return guard([&] {
    if (!t) invalid("null trace");
    if (num_samples) *num_samples = t->f.h.samples;
    if (num_features) *num_features = t->f.h.d;
    if (vocab) *vocab = t->f.h.vocab;
  });
}

int ec_trace_ids(ec_trace t, const uint32_t** ids_host) {
  return guard([&] {
    if (!t || !ids_host) invalid("null argument");
    *ids_host = t->f.ids;
  });
}

// Samples [first, first + count) of the trace into device memory (sample-
// major, count * d ids), through a pinned double-buffered staging area so a
// multi-GB trace streams at the host link's copy bandwidth.
int ec_trace_upload(ec_trace t, uint64_t first, uint64_t count, uint32_t* ids_dev, void* stream) {
  return guard([&] {
    if (!t || (!ids_dev && count)) invalid("null argument");
    const TraceFile& f = t->f;
    if (first > f.h.samples || count > f.h.samples - first) invalid("sample range out of the trace");
    const uint64_t d = static_cast<uint64_t>(f.h.d);
    const uint32_t* src = f.ids + first * d;
    uint64_t n = count * d;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    constexpr uint64_t kChunk = 8ull << 20;  // ids per staging buffer (32 MiB)
    uint32_t* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    try {
      for (int k = 0; k < 2; ++k) {
        EC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&stage[k]), std::min(n, kChunk) * sizeof(uint32_t) + 4,
                              cudaHostAllocDefault));
        EC_CUDA(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
      }
      for (uint64_t off = 0, k = 0; off < n; off += kChunk, k ^= 1) {
        const uint64_t m = std::min(kChunk, n - off);
        EC_CUDA(cudaEventSynchronize(done[k]));  // this staging buffer's last copy is done
        std::memcpy(stage[k], src + off, m * sizeof(uint32_t));
        EC_CUDA(cudaMemcpyAsync(ids_dev + off, stage[k], m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        EC_CUDA(cudaEventRecord(done[k], st));
      }
      for (int k = 0; k < 2; ++k) EC_CUDA(cudaEventSynchronize(done[k]));
    } catch (...) {
      for (int k = 0; k < 2; ++k) {
        if (done[k]) cudaEventDestroy(done[k]);
        if (stage[k]) cudaFreeHost(stage[k]);
      }
      throw;
    }
    for (int k = 0; k < 2; ++k) {
      cudaEventDestroy(done[k]);
      cudaFreeHost(stage[k]);
    }
  });
}

}  // extern "C"
