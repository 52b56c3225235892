// K4: unique-only exchange between row shards.
//
// Rows are sharded owner(id) = id % world; the hot-row cache is replicated,
// so only misses owned by another rank cross NVLink — exactly the E\C term of
// the reference's cost model (core/src/cost_model.cpp:88-111), minus rows the
// requester owns itself.
//
// forward, per rank:
//   ex_route   misses owned by others, grouped by owner: (owner-local row
//              index, unique slot); plus the list of cache hits (for the hot
//              gradient sync); counts vector [world requests..., hits]
//   counts     all-gathered -> every rank knows the full request matrix
//   ids        all-to-all-v of 4-byte owner-local row indices
//   ex_serve   owner gathers the requested rows (HBM or pinned host shard)
//   rows       all-to-all-v of rows back to the requesters
//   ex_unpack  rows land in the requester's compact unique-row buffer
// backward:
//   ex_pack    row gradients of remote misses (request order) and of cache hits
//   grads      all-to-all-v of miss gradients to owners; hit lists to every rank
//   ex_apply   owners apply remote gradients source rank by source rank; every
//              rank applies every rank's hit gradients to its cache replica in
//              rank order 0..world-1, so replicas stay bit-identical
//
// Transports: NCCL (one process per GPU; ec_tables_attach_comm) or an
// in-process loopback group (ec_group_*: several ranks on one device,
// cudaMemcpyAsync between their buffers) that drives the same phases in lock
// step — the data path is shared, only the byte movement differs.
#include <nccl.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <numeric>
#include <vector>

#include "device_util.cuh"
#include "engine.hpp"

namespace ec {

#define EC_NCCL(x)                                                                                  \
  do {                                                                                              \
    const ncclResult_t r_ = (x);                                                                    \
    if (r_ != ncclSuccess) throw Error(EC_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

struct Exchange {
  ncclComm_t comm = nullptr;
  int W = 1;
  DevBuf<int64_t> shard_off;   // [W*(T+1)]: row offset of table t in rank r's shard
  DevBuf<int> cnt;             // [W+2]: requests per owner, hit count, scratch
  DevBuf<int> cursor;          // [W]
  DevBuf<int64_t> off;         // [W]: start of each owner's request segment
  DevBuf<int> allcnt;          // [W*(W+1)] gathered counts
  int* allcnt_host = nullptr;  // pinned
  DevBuf<uint32_t> send_idx, send_slot, recv_idx, hot_g, hot_slot, hot_slot_all;
  DevBuf<float> send_rows, recv_rows, grad_send, grad_recv, hot_grad, hot_grad_all;
  // plan of the current batch (host)
  std::vector<int64_t> scnt, soff, rcnt, roff, hcnt, hoff;
  int64_t nsend = 0, nrecv = 0, nhot_all = 0;

  // peer-memory (P2P) exchange: every rank's shard and hot list visible here
  bool p2p = false;
  unsigned epoch = 0;               // steps started (barrier generations)
  bool step_open = false;           // a forward whose step was not applied yet
  DevBuf<PeerView> peers;           // [W]
  std::vector<PeerView> peers_host;
  // hot rows this rank owns (cache slot % W == rank): sources' gradients in,
  // the updated rows out (PeerView::hin_* / upd_*)
  DevBuf<uint32_t> hin_slot;        // [W * hcap]
  DevBuf<float> hin_grad;           // [W * hcap * D]
  DevBuf<int> hin_cnt;              // [W]
  int64_t hcap = 0;
  DevBuf<float> hacc;               // [ceil(K / W) * D] gradient sums of owned slots (zero between steps)
  DevBuf<unsigned> hmark;           // [ceil(K / W)] owned slot touched this step
  DevBuf<uint32_t> upd_slot;        // [min(W * hcap, K / W)] owned slots updated this step
  DevBuf<float> upd_rows;           //   and their new values
  DevBuf<int> upd_cnt;              // [1]
  DevBuf<unsigned> flags;           // [2W] barrier words peers write into
  DevBuf<unsigned> done;            // arrival counter of a kernel that signals a barrier
  std::vector<void*> ipc_opened;    // peer allocations mapped by cudaIpcOpenMemHandle
  // pinned-host shards: miss gradients sent to this rank as owner
  DevBuf<uint32_t> inbox_idx;       // [W * cap]
  DevBuf<float> inbox_grad;         // [W * cap * D]
  DevBuf<int> inbox_cnt;            // [W]
  DevBuf<uint32_t> ver;             // [shard rows]: step generation of each row's last inbox update
  int64_t inbox_cap = 0;
  std::vector<std::pair<void*, size_t>> host_maps;  // peers' host shards mapped here

  ~Exchange() {
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (auto& m : host_maps) {
      cudaHostUnregister(m.first);
      munmap(m.first, m.second);
    }
    if (comm) ncclCommDestroy(comm);
    if (allcnt_host) cudaFreeHost(allcnt_host);
  }
};

template <class T>
static void grow(DevBuf<T>& b, size_t n) {
  if (b.n < n) b.alloc(std::max<size_t>(n, b.n + b.n / 2));
}

// ------------------------------------------------------------ kernels
// Remote misses counted per owner (pass 1) and written grouped by owner
// (pass 2, after offsets); cache hits listed with their unique slot.
__global__ void k_route(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                        const uint32_t* __restrict__ missq, const uint32_t* __restrict__ uniq,
                        const uint16_t* __restrict__ utab, const int64_t* __restrict__ shard_off, int rank, int world,
                        int* __restrict__ cnt, int* __restrict__ cursor, const int64_t* __restrict__ off,
                        uint32_t* __restrict__ send_idx, uint32_t* __restrict__ send_slot, int fill) {
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  for (int base = blockIdx.x * blockDim.x; base < nm; base += gridDim.x * blockDim.x) {
    const int q = base + threadIdx.x;
    int owner = -1;
    uint32_t g = 0, id = 0;
    if (q < nm) {
      g = missq[q];
      id = uniq[g];
      owner = static_cast<int>(id % world);
      if (owner == rank) owner = -1;  // served locally by k_gather / k_gather_host
    }
    if (!fill) {
      const unsigned peers = __match_any_sync(kFull, owner);
      if (owner >= 0 && (__ffs(peers) - 1) == lane_id()) atomicAdd(cnt + owner, __popc(peers));
    } else if (owner >= 0) {
      const int t = utab[g];
      const int64_t pos = off[owner] + atomicAdd(cursor + owner, 1);
      send_idx[pos] = static_cast<uint32_t>(shard_off[static_cast<int64_t>(owner) * (T + 1) + t] + id / world);
      send_slot[pos] = g;
    }
  }
}

__global__ void k_hot_list(const int* __restrict__ ctr, int T, const int32_t* __restrict__ usrc,
                           int* __restrict__ hot_cnt, uint32_t* __restrict__ hot_g, uint32_t* __restrict__ hot_slot) {
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  for (int base = blockIdx.x * blockDim.x; base < U; base += gridDim.x * blockDim.x) {
    const int g = base + threadIdx.x;
    const bool hit = g < U && usrc[g] >= 0;
    const unsigned hb = __ballot_sync(kFull, hit);
    int b0 = 0;
    if (hb && lane_id() == __ffs(hb) - 1) b0 = atomicAdd(hot_cnt, __popc(hb));
    b0 = __shfl_sync(kFull, b0, __ffs(hb ? hb : 1u) - 1);
    if (hit) {
      const int pos = b0 + __popc(hb & ((1u << lane_id()) - 1));
      hot_g[pos] = static_cast<uint32_t>(g);
      hot_slot[pos] = static_cast<uint32_t>(usrc[g]);
    }
  }
}

__global__ void k_offsets(const int* __restrict__ cnt, int world, int64_t* __restrict__ off, int* __restrict__ cursor) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t run = 0;
    for (int o = 0; o < world; ++o) {
      off[o] = run;
      run += cnt[o];
      cursor[o] = 0;
    }
  }
}

// dst[k] = src row idx[k] (float4 granularity; vec4 = D/4)
__global__ void k_rows_gather(const float* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n, int vec4,
                              float* __restrict__ dst) {
  const int64_t total = n * vec4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / vec4;
    const int c = static_cast<int>(i - k * vec4);
    reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[static_cast<int64_t>(idx[k]) * vec4 + c];
  }
}

// dst row idx[k] = src[k]
__global__ void k_rows_scatter(const float* __restrict__ src, const uint32_t* __restrict__ idx, int64_t n, int vec4,
                               float* __restrict__ dst) {
  const int64_t total = n * vec4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / vec4;
    const int c = static_cast<int>(i - k * vec4);
    reinterpret_cast<float4*>(dst)[static_cast<int64_t>(idx[k]) * vec4 + c] = reinterpret_cast<const float4*>(src)[i];
  }
}

// row idx[k] -= lr * g[k]; one launch per source rank keeps the order fixed.
__global__ void k_rows_sgd(float* __restrict__ rows, const uint32_t* __restrict__ idx, const float* __restrict__ g,
                           int64_t n, int vec4, float lr) {
  const int64_t total = n * vec4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / vec4;
    const int c = static_cast<int>(i - k * vec4);
    float4* w = reinterpret_cast<float4*>(rows) + static_cast<int64_t>(idx[k]) * vec4 + c;
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 v = *w;
    v.x -= lr * gv.x;
    v.y -= lr * gv.y;
    v.z -= lr * gv.z;
    v.w -= lr * gv.w;
    *w = v;
  }
}

// ---- P2P exchange kernels
// Backward, after the gradient reduction: cache hits go to this rank's
// published hot list (applied by every rank in rank order); misses update
// their owner's shard row in place with -lr*g (float atomics: the owner's row
// may receive several ranks' updates in one step; it is not replicated).
// Device barrier pieces folded into the exchange kernels: a kernel may wait
// for barrier `wait_b` in its prologue (every block, threads < world spin on
// this rank's flag words) and signal barrier `sig_b` from its last block to
// finish (a grid-wide arrival counter), saving the separate barrier launches.
// The driver folds the signals only: a spinning prologue in every block would
// hold the SMs a prefetch on another stream could use while a peer is late.
constexpr uint64_t kP2PTimeoutNs = 60ull * 1000 * 1000 * 1000;
struct P2PSync {
  const unsigned* flags = nullptr;  // this rank's words (waits)
  const PeerView* peers = nullptr;  // every rank's words (signals)
  unsigned* done = nullptr;         // arrival counter of the signalling kernel (0 between launches)
  int world = 0, rank = 0;
  int wait_b = -1, sig_b = -1;
  unsigned epoch = 0;
};

__device__ void p2p_spin(const unsigned* flags, int world, int b, unsigned epoch) {
  const unsigned* f = flags + b * world + threadIdx.x;
  unsigned v;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (unsigned k = 1;; ++k) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (static_cast<int>(v - epoch) >= 0) break;
    if ((k & 1023) == 0) {  // a peer that never arrives (died, or called fwd/bwd fewer times)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > kP2PTimeoutNs) {
        printf("embcomm p2p: barrier %d generation %u: rank %d never arrived\n", b, epoch, threadIdx.x);
        __trap();  // fail the step loudly instead of hanging the GPU
      }
    }
  }
  __threadfence_system();
}

__device__ __forceinline__ void p2p_post(const PeerView* peers, int world, int rank, int b, unsigned epoch) {
  unsigned* f = peers[threadIdx.x].flags + b * world + rank;
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
}

__device__ __forceinline__ void p2p_prologue(const P2PSync& s) {
  if (s.wait_b < 0) return;
  if (static_cast<int>(threadIdx.x) < s.world) p2p_spin(s.flags, s.world, s.wait_b, s.epoch);
  __syncthreads();
}

__device__ __forceinline__ void p2p_epilogue(const P2PSync& s) {
  if (s.sig_b < 0) return;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this block's writes (local and over NVLink) before its arrival
    s_last = atomicAdd(s.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  if (threadIdx.x == 0) *s.done = 0;
  __threadfence_system();
  if (static_cast<int>(threadIdx.x) < s.world) p2p_post(s.peers, s.world, s.rank, s.sig_b, s.epoch);
}

template <int VEC>
__global__ void k_p2p_apply(const TableDev* __restrict__ td, int T, const int* __restrict__ ctr,
                            const uint32_t* __restrict__ uniq, const uint16_t* __restrict__ utab,
                            const int32_t* __restrict__ usrc, const float* __restrict__ ugrad, float lr,
                            const PeerView* __restrict__ peers, const int64_t* __restrict__ shard_off, int rank,
                            int world, int64_t hcap, int64_t inbox_cap, int part, P2PSync sync) {
  constexpr int D = VEC * 4;
  p2p_prologue(sync);
  const int U = counters(const_cast<int*>(ctr), T).ubase[T];
  const int sub = lane_id() / VEC, c = lane_id() % VEC;
  constexpr int RPW = 32 / VEC;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int g0 = warp * RPW; g0 < U; g0 += nwarps * RPW) {  // warp-uniform trip count (ballots inside)
    const int g = g0 + sub;
    const bool live = g < U;
    const int32_t s = live ? usrc[g] : -1;
    const float4 gv = live ? ldg4(ugrad + static_cast<int64_t>(g) * D + c * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
    // part & 1 -- hits: the gradient goes to the slot's owner (slot % world),
    // appended to this rank's segment of the owner's hot inbox; lane c == 0 of
    // a row's group claims the position, one atomic per (warp, owner)
    const bool hit = (part & 1) && live && s >= 0;
    const int ho = hit ? s % world : -1;
    const unsigned same = __match_any_sync(kFull, hit && c == 0 ? ho : -1);
    int pos = 0;
    if (hit && c == 0 && __ffs(same) - 1 == lane_id())
      pos = atomicAdd(peers[ho].hin_cnt + rank, __popc(same));
    pos = __shfl_sync(kFull, pos, hit && c == 0 ? __ffs(same) - 1 : 0) + __popc(same & ((1u << lane_id()) - 1));
    pos = __shfl_sync(kFull, pos, sub * VEC);  // (lane c == 0 of this row's group)
    const int sent = __popc(__ballot_sync(kFull, hit && c == 0 && ho != rank));
    if (sent && lane_id() == 0) atomicAdd(counters(const_cast<int*>(ctr), T).hot_out, sent);
    if (hit) {
      const int64_t k = static_cast<int64_t>(rank) * hcap + pos;
      if (c == 0) peers[ho].hin_slot[k] = static_cast<uint32_t>(s);
      st4(peers[ho].hin_grad + k * D + c * 4, gv);
    }
    // part & 2 -- misses: the owner's row (index in its shard)
    const bool miss = (part & 2) && live && s < 0;
    const uint32_t id = miss ? uniq[g] : 0;
    const int o = static_cast<int>(id % world);
    const int64_t row = miss ? shard_off[static_cast<int64_t>(o) * (T + 1) + utab[g]] + id / world : 0;
    if (inbox_cap) {
      // pinned-host shards (no float atomics over PCIe): append to the
      // owner's inbox segment for this source rank; the owner applies the
      // segments in rank order
      int ip = 0;
      if (miss && c == 0) ip = atomicAdd(peers[o].inbox_cnt + rank, 1);
      ip = __shfl_sync(kFull, ip, sub * VEC);
      if (miss) {
        const int64_t k = static_cast<int64_t>(rank) * inbox_cap + ip;
        if (c == 0) peers[o].inbox_idx[k] = static_cast<uint32_t>(row);
        st4(peers[o].inbox_grad + k * D + c * 4, gv);
      }
    } else if (miss) {  // HBM shards: straight into the owner's row
      float* w = peers[o].store + row * D + c * 4;
      atomicAdd(w + 0, -lr * gv.x);
      atomicAdd(w + 1, -lr * gv.y);
      atomicAdd(w + 2, -lr * gv.z);
      atomicAdd(w + 3, -lr * gv.w);
    }
  }
  p2p_epilogue(sync);
}

// Owner side, pinned-host shards: source rank p's miss gradients into this
// rank's shard (launched for p = 0..world-1; rows are unique within one
// source's segment, so each launch is a plain read-modify-write).
template <int VEC>
__global__ void k_p2p_inbox_apply(const uint32_t* __restrict__ idx, const float* __restrict__ grad,
                                  const int* __restrict__ cnt, float* __restrict__ store, float lr,
                                  uint32_t* __restrict__ ver, unsigned epoch, P2PSync sync) {
  constexpr int D = VEC * 4;
  p2p_prologue(sync);
  const int64_t total = static_cast<int64_t>(*cnt) * VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / VEC;
    const int c = static_cast<int>(i - k * VEC);
    float* w = store + static_cast<int64_t>(idx[k]) * D + c * 4;
    const float4 gv = ldg4(grad + k * D + c * 4);
    float4 v = *reinterpret_cast<const float4*>(w);
    v = make_float4(v.x - lr * gv.x, v.y - lr * gv.y, v.z - lr * gv.z, v.w - lr * gv.w);
    st4(w, v);
    if (c == 0) ver[idx[k]] = epoch;  // read by peers' prefetch patch after barrier 1
  }
  p2p_epilogue(sync);
}

// A prefetched batch's host rows were read while the step before ran; rows
// that step updated (stamped with its generation by their owner) are read
// again once every rank passed barrier 1.
template <int VEC>
__global__ void k_p2p_patch(const int* __restrict__ ctr, int T, const uint32_t* __restrict__ missq,
                            const uint32_t* __restrict__ uniq, const uint16_t* __restrict__ utab,
                            float* __restrict__ urows, const PeerView* __restrict__ peers,
                            const int64_t* __restrict__ shard_off, int world, unsigned epoch) {
  constexpr int D = VEC * 4;
  const int nm = *counters(const_cast<int*>(ctr), T).miss_total;
  const int64_t total = static_cast<int64_t>(nm) * VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = static_cast<int>(i / VEC);
    const int c = static_cast<int>(i - static_cast<int64_t>(q) * VEC);
    const uint32_t g = missq[q];
    const uint32_t id = uniq[g];
    const int o = static_cast<int>(id % world);
    const int64_t row = shard_off[static_cast<int64_t>(o) * (T + 1) + utab[g]] + id / world;
    const PeerView pv = peers[o];
    if (*reinterpret_cast<const volatile uint32_t*>(pv.ver + row) != epoch) continue;
    st4(urows + static_cast<int64_t>(g) * D + c * 4, *reinterpret_cast<const float4*>(pv.store + row * D + c * 4));
  }
}


// Hot rows (the replicated cache), owner-partitioned: slot s is owned by rank
// s % world.  After barrier 0 every owner sums the gradients its inbox holds
// for its slots (every source rank's segment; fp32 REDs, at most `world` per
// slot) and marks each touched slot once; then it applies w - lr * sum to its
// replica, publishes (slot, new row), and signals barrier 1; then every rank
// copies every owner's updated rows into its own replica.  Replicas stay
// bit-identical (all copy the owner's value), and a rank moves ~H rows out
// and |union of hits| rows in per step instead of reading W-1 peers' full
// hot lists and applying them in W rank-ordered passes.
template <int VEC>
__global__ void k_p2p_hot_reduce(const uint32_t* __restrict__ hin_slot, const float* __restrict__ hin_grad,
                                 const int* __restrict__ hin_cnt, int64_t hcap, int world, float* __restrict__ hacc,
                                 unsigned* __restrict__ hmark, uint32_t* __restrict__ upd_slot, int* __restrict__ upd_cnt) {
  constexpr int D = VEC * 4;
  for (int p = 0; p < world; ++p) {
    const int n = hin_cnt[p];
    const int64_t total = static_cast<int64_t>(n) * VEC;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t k = i / VEC;
      const int c = static_cast<int>(i - k * VEC);
      const int64_t e = static_cast<int64_t>(p) * hcap + k;
      const uint32_t slot = hin_slot[e];
      const uint32_t j = slot / static_cast<uint32_t>(world);
      atomicAdd(reinterpret_cast<float4*>(hacc + static_cast<int64_t>(j) * D + c * 4), ldg4(hin_grad + e * D + c * 4));
      if (c == 0 && atomicExch(hmark + j, 1u) == 0u) upd_slot[atomicAdd(upd_cnt, 1)] = slot;
    }
  }
}

template <int VEC>
__global__ void k_p2p_hot_update(const uint32_t* __restrict__ upd_slot, const int* __restrict__ upd_cnt, int world,
                                 float* __restrict__ cache, float* __restrict__ hacc, unsigned* __restrict__ hmark,
                                 float* __restrict__ upd_rows, int* __restrict__ hin_cnt, float lr, P2PSync sync) {
  constexpr int D = VEC * 4;
  const int64_t total = static_cast<int64_t>(*upd_cnt) * VEC;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / VEC;
    const int c = static_cast<int>(i - k * VEC);
    const uint32_t slot = upd_slot[k];
    const uint32_t j = slot / static_cast<uint32_t>(world);
    float* a = hacc + static_cast<int64_t>(j) * D + c * 4;
    const float4 g = *reinterpret_cast<const float4*>(a);
    float* w = cache + static_cast<int64_t>(slot) * D + c * 4;
    float4 v = *reinterpret_cast<const float4*>(w);
    v = make_float4(v.x - lr * g.x, v.y - lr * g.y, v.z - lr * g.z, v.w - lr * g.w);
    st4(w, v);
    st4(upd_rows + k * D + c * 4, v);
    st4(a, make_float4(0.f, 0.f, 0.f, 0.f));
    if (c == 0) hmark[j] = 0u;
  }
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < world) hin_cnt[threadIdx.x] = 0;  // (read by the reduce)
  p2p_epilogue(sync);
}

// Every other owner's updated hot rows into this rank's replica (one launch).
template <int VEC>
__global__ void k_p2p_hot_copy(const PeerView* __restrict__ peers, int world, int rank, float* __restrict__ cache,
                               int* __restrict__ ctr, int T) {
  constexpr int D = VEC * 4;
  for (int o = 0; o < world; ++o) {
    if (o == rank) continue;
    const PeerView pv = peers[o];
    const int n = *reinterpret_cast<const volatile int*>(pv.upd_cnt);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(counters(ctr, T).hot_in, n);
    const int64_t total = static_cast<int64_t>(n) * VEC;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t k = i / VEC;
      const int c = static_cast<int>(i - k * VEC);
      st4(cache + static_cast<int64_t>(pv.upd_slot[k]) * D + c * 4,
          *reinterpret_cast<const float4*>(pv.upd_rows + k * D + c * 4));
    }
  }
}

// Device barrier over peer memory, split in two so a loopback group can
// enqueue every rank's signal before any rank's wait on one stream.
// Barrier b (0: hot lists published -- every rank is past its forward reads;
// 1: step applied) of generation `epoch`.
__global__ void k_p2p_signal(const PeerView* __restrict__ peers, int world, int rank, int b, unsigned epoch) {
  if (static_cast<int>(threadIdx.x) >= world) return;
  __threadfence_system();  // this rank's writes of the step before the word
  p2p_post(peers, world, rank, b, epoch);
}
__global__ void k_p2p_wait(const unsigned* __restrict__ flags, int world, int b, unsigned epoch) {
  if (static_cast<int>(threadIdx.x) < world) p2p_spin(flags, world, b, epoch);
}

static P2PSync p2p_sync(const Exchange& x, int rank, int wait_b, int sig_b) {
  P2PSync s;
  s.flags = x.flags.p;
  s.peers = x.peers.p;
  s.done = x.done.p;
  s.world = x.W;
  s.rank = rank;
  s.wait_b = wait_b;
  s.sig_b = sig_b;
  s.epoch = x.epoch;
  return s;
}

static int grid_rows(int64_t n, int vec4, int device) {
  const int64_t want = (n * vec4 + 255) / 256;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, sm_count(device) * 8)));
}

// ------------------------------------------------------------ phases
void Engine::ex_init(int W_) {
  if (!ex) ex = new Exchange;
  ex->W = W_;
  std::vector<int64_t> so(static_cast<size_t>(W_) * (T + 1), 0);
  for (int r = 0; r < W_; ++r)
    for (uint32_t t = 0; t < T; ++t) {
      const uint64_t lr = rows[t] > static_cast<uint64_t>(r) ? (rows[t] - r + W_ - 1) / W_ : 0;
      so[static_cast<size_t>(r) * (T + 1) + t + 1] = so[static_cast<size_t>(r) * (T + 1) + t] + lr;
    }
  for (int r = 0; r < W_; ++r)
    if (so[static_cast<size_t>(r) * (T + 1) + T] > 0xFFFFFFFFll) invalid("a shard holds at most 2^32 rows");
  ex->shard_off.alloc(so.size());
  EC_CUDA(cudaMemcpy(ex->shard_off.p, so.data(), so.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
  ex->cnt.alloc(W_ + 2);
  ex->cursor.alloc(W_);
  ex->off.alloc(W_);
  ex->allcnt.alloc(static_cast<size_t>(W_) * (W_ + 1));
  if (!ex->allcnt_host)
    EC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ex->allcnt_host), static_cast<size_t>(W_) * (W_ + 1) * sizeof(int),
                          cudaHostAllocDefault));
  const size_t N = max_n * T;
  grow(ex->send_idx, N);
  grow(ex->send_slot, N);
  grow(ex->hot_g, N);
  grow(ex->hot_slot, N);
  grow(ex->send_rows, N * D);  // reused as the served-rows buffer on the owner side (grown per plan)
  grow(ex->recv_rows, N * D);
  grow(ex->grad_send, N * D);
  grow(ex->hot_grad, N * D);
}

// Route misses by owner, list hits; counts for the plan land in ex->cnt
// ([0, W): requests per owner, [W]: hits).
void Engine::ex_route(cudaStream_t st) {
  Exchange& x = *ex;
  EC_CUDA(cudaMemsetAsync(x.cnt.p, 0, (x.W + 2) * sizeof(int), st));
  const int grid = sm_count(device) * 2;
  k_route<<<grid, 256, 0, st>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p, x.shard_off.p, rank, world, x.cnt.p,
                                x.cursor.p, x.off.p, x.send_idx.p, x.send_slot.p, 0);
  launched();
  k_offsets<<<1, 32, 0, st>>>(x.cnt.p, x.W, x.off.p, x.cursor.p);
  launched();
  k_route<<<grid, 256, 0, st>>>(tdev.p, T, ctr.p, missq.p, uniq.p, utab.p, x.shard_off.p, rank, world, x.cnt.p,
                                x.cursor.p, x.off.p, x.send_idx.p, x.send_slot.p, 1);
  launched();
  k_hot_list<<<grid, 256, 0, st>>>(ctr.p, T, usrc.p, x.cnt.p + x.W, x.hot_g.p, x.hot_slot.p);
  launched();
}

// Exchange plan of `rank` from the gathered count matrix m[r*(W+1) + o]
// (row r: requests rank r sends to each owner o, then r's hit count).
void exchange_plan(const int* m, int W, int rank, int64_t* scnt, int64_t* soff, int64_t* rcnt, int64_t* roff,
                   int64_t* hcnt, int64_t* hoff) {
  int64_t s = 0, r = 0, h = 0;
  for (int p = 0; p < W; ++p) {
    if (m[rank * (W + 1) + p] < 0 || m[p * (W + 1) + rank] < 0 || m[p * (W + 1) + W] < 0)
      invalid("negative count in the exchange matrix");
    if (p == rank && m[rank * (W + 1) + rank] != 0) invalid("a rank never requests rows from itself");
    scnt[p] = m[rank * (W + 1) + p];
    soff[p] = s;
    s += scnt[p];
    rcnt[p] = m[p * (W + 1) + rank];
    roff[p] = r;
    r += rcnt[p];
    hcnt[p] = m[p * (W + 1) + W];
    hoff[p] = h;
    h += hcnt[p];
  }
}

void Engine::ex_plan() {
  Exchange& x = *ex;
  const int W = x.W;
  x.scnt.assign(W, 0);
  x.soff.assign(W, 0);
  x.rcnt.assign(W, 0);
  x.roff.assign(W, 0);
  x.hcnt.assign(W, 0);
  x.hoff.assign(W, 0);
  exchange_plan(x.allcnt_host, W, rank, x.scnt.data(), x.soff.data(), x.rcnt.data(), x.roff.data(), x.hcnt.data(),
                x.hoff.data());
  const int64_t s = std::accumulate(x.scnt.begin(), x.scnt.end(), int64_t{0});
  const int64_t r = std::accumulate(x.rcnt.begin(), x.rcnt.end(), int64_t{0});
  const int64_t h = std::accumulate(x.hcnt.begin(), x.hcnt.end(), int64_t{0});
  x.nsend = s;
  x.nrecv = r;
  x.nhot_all = h;
  grow(x.recv_idx, static_cast<size_t>(r) + 1);
  grow(x.send_rows, static_cast<size_t>(std::max(r, s)) * D + 1);
  grow(x.grad_recv, static_cast<size_t>(r) * D + 1);
  grow(x.hot_slot_all, static_cast<size_t>(h) + 1);
  grow(x.hot_grad_all, static_cast<size_t>(h) * D + 1);
  last_wire_rows = static_cast<uint64_t>(s);
  const uint64_t rowb = static_cast<uint64_t>(D) * sizeof(float);
  // forward ids + rows, backward miss grads, hot lists (slot + grad) out and in
  last_wire_bytes = static_cast<uint64_t>(s) * (4 + rowb) + static_cast<uint64_t>(r) * (4 + rowb) +
                    static_cast<uint64_t>(s) * rowb + static_cast<uint64_t>(r) * rowb +
                    static_cast<uint64_t>(x.hcnt[rank]) * (4 + rowb) * (W - 1) +
                    static_cast<uint64_t>(h - x.hcnt[rank]) * (4 + rowb);
}

// Owner side: gather the rows other ranks requested from the local shard.
void Engine::ex_serve(cudaStream_t st) {
  Exchange& x = *ex;
  if (!x.nrecv) return;
  k_rows_gather<<<grid_rows(x.nrecv, D / 4, device), 256, 0, st>>>(store_base, x.recv_idx.p, x.nrecv, D / 4,
                                                                   x.send_rows.p);
  launched();
}

void Engine::ex_unpack(cudaStream_t st) {
  Exchange& x = *ex;
  if (!x.nsend) return;
  k_rows_scatter<<<grid_rows(x.nsend, D / 4, device), 256, 0, st>>>(x.recv_rows.p, x.send_slot.p, x.nsend, D / 4,
                                                                     urows.p);
  launched();
}

void Engine::ex_pack_bwd(cudaStream_t st) {
  Exchange& x = *ex;
  if (x.nsend) {
    k_rows_gather<<<grid_rows(x.nsend, D / 4, device), 256, 0, st>>>(ugrad.p, x.send_slot.p, x.nsend, D / 4,
                                                                     x.grad_send.p);
    launched();
  }
  const int64_t nh = x.hcnt[rank];
  if (nh) {
    k_rows_gather<<<grid_rows(nh, D / 4, device), 256, 0, st>>>(ugrad.p, x.hot_g.p, nh, D / 4, x.hot_grad.p);
    launched();
  }
  // own hit list into the rank-ordered all-ranks buffer
  if (nh) {
    EC_CUDA(cudaMemcpyAsync(x.hot_slot_all.p + x.hoff[rank], x.hot_slot.p, nh * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, st));
    EC_CUDA(cudaMemcpyAsync(x.hot_grad_all.p + x.hoff[rank] * D, x.hot_grad.p, nh * D * sizeof(float),
                            cudaMemcpyDeviceToDevice, st));
  }
}

// Owner: remote miss gradients by source rank; all ranks: hot gradients in
// rank order into the cache replica.
void Engine::ex_apply_bwd(float lr, cudaStream_t st) {
  Exchange& x = *ex;
  for (int p = 0; p < x.W; ++p) {
    if (p == rank || !x.rcnt[p]) continue;
    k_rows_sgd<<<grid_rows(x.rcnt[p], D / 4, device), 256, 0, st>>>(store_base, x.recv_idx.p + x.roff[p],
                                                                     x.grad_recv.p + x.roff[p] * D, x.rcnt[p], D / 4, lr);
    launched();
  }
  for (int p = 0; p < x.W; ++p) {
    if (!x.hcnt[p]) continue;
    k_rows_sgd<<<grid_rows(x.hcnt[p], D / 4, device), 256, 0, st>>>(cache.p, x.hot_slot_all.p + x.hoff[p],
                                                                     x.hot_grad_all.p + x.hoff[p] * D, x.hcnt[p], D / 4,
                                                                     lr);
    launched();
  }
}

// ------------------------------------------------------------ P2P driver
// Per step (generation e = ++epoch): forward waits barrier 1 of e-1 (every
// rank applied the previous step) and pulls remote rows in k_gather; backward
// publishes its hot list (and, for pinned-host shards, its miss gradients into
// the owners' inboxes), signals barrier 0 and waits for it -- every rank is
// then past its forward, so no one still reads the rows about to change --
// updates owners' rows (HBM: atomics over NVLink; host: each owner applies
// its inbox), applies every rank's hot list in rank order, signals barrier 1.
// Two device barriers, no host synchronisation, no NCCL call.
bool Engine::p2p_on() const { return ex != nullptr && ex->p2p; }
bool Engine::p2p_step_open() const { return p2p_on() && ex->step_open; }
const PeerView* Engine::p2p_peers() const { return p2p_on() ? ex->peers.p : nullptr; }
const int64_t* Engine::p2p_shard_off() const { return p2p_on() ? ex->shard_off.p : nullptr; }

void Engine::p2p_alloc() {
  if (storage == EC_STORAGE_HOST && store_host_fd < 0) invalid("host shard is not shareable (world must be > 1)");
  if (!ex) ex_init(world);
  Exchange& x = *ex;
  const size_t N = max_n * T;
  if (storage == EC_STORAGE_HOST && x.inbox_cap < static_cast<int64_t>(N)) {
    x.inbox_cap = static_cast<int64_t>(N);
    x.inbox_idx.alloc(x.W * N);
    x.inbox_grad.alloc(x.W * N * D);
    x.inbox_cnt.alloc(x.W);
    EC_CUDA(cudaMemset(x.inbox_cnt.p, 0, x.inbox_cnt.bytes()));
    x.ver.alloc(std::max<uint64_t>(store_off[T], 1));
    EC_CUDA(cudaMemset(x.ver.p, 0, x.ver.bytes()));  // generation 0 is never a step
  }
  if (x.hcap < static_cast<int64_t>(N)) {  // a source sends at most its batch's N unique rows
    x.hcap = static_cast<int64_t>(N);
    x.hin_slot.alloc(x.W * N);
    x.hin_grad.alloc(x.W * N * D);
    x.hin_cnt.alloc(x.W);
    EC_CUDA(cudaMemset(x.hin_cnt.p, 0, x.hin_cnt.bytes()));
    x.upd_slot.alloc(x.W * N);
    x.upd_rows.alloc(x.W * N * D);
  }
  if (!x.upd_cnt.n) {
    x.upd_cnt.alloc(1);
    EC_CUDA(cudaMemset(x.upd_cnt.p, 0, sizeof(int)));
  }
  p2p_hot_alloc();
  if (!x.done.n) {
    x.done.alloc(1);
    EC_CUDA(cudaMemset(x.done.p, 0, sizeof(unsigned)));
  }
  if (x.flags.n < static_cast<size_t>(kP2PBarriers * x.W)) {
    x.flags.alloc(kP2PBarriers * x.W);
    EC_CUDA(cudaMemset(x.flags.p, 0, x.flags.bytes()));
  }
}

// owner-side accumulators for the slots this rank owns (re-sized with the cache)
void Engine::p2p_hot_alloc() {
  if (!ex) return;
  Exchange& x = *ex;
  const size_t own = (cache_k_total + x.W - 1) / x.W;
  if (x.hmark.n >= std::max<size_t>(own, 1)) return;
  x.hacc.alloc(std::max<size_t>(own, 1) * D);
  x.hmark.alloc(std::max<size_t>(own, 1));
  EC_CUDA(cudaMemset(x.hacc.p, 0, x.hacc.bytes()));
  EC_CUDA(cudaMemset(x.hmark.p, 0, x.hmark.bytes()));
}

PeerView Engine::p2p_self() const {
  const Exchange& x = *ex;
  return PeerView{store_base,  x.upd_slot.p,  x.upd_rows.p,  x.upd_cnt.p,  x.hin_slot.p, x.hin_grad.p,
                  x.hin_cnt.p, x.flags.p,     x.inbox_idx.p, x.inbox_grad.p, x.inbox_cnt.p, x.ver.p};
}

void Engine::p2p_set_peers(const std::vector<PeerView>& v) {
  Exchange& x = *ex;
  if (static_cast<int>(v.size()) != x.W) invalid("peer table needs one entry per rank");
  x.peers_host = v;
  x.peers.alloc(v.size());
  EC_CUDA(cudaMemcpy(x.peers.p, v.data(), v.size() * sizeof(PeerView), cudaMemcpyHostToDevice));
  // flags were zeroed at allocation and only ever grow (generation numbers):
  // re-importing keeps the epoch, so a peer's early signal is never wiped
  x.p2p = true;
  clear_graphs();
}

void Engine::p2p_signal(int b, cudaStream_t st) {
  k_p2p_signal<<<1, 32, 0, st>>>(ex->peers.p, ex->W, rank, b, ex->epoch);
  launched();
}
void Engine::p2p_wait(int b, unsigned epoch, cudaStream_t st) {
  k_p2p_wait<<<1, 32, 0, st>>>(ex->flags.p, ex->W, b, epoch);
  launched();
}

// A forward with no backward after it (evaluation) still has to release the
// peers waiting for its step to be applied: nothing was, so barrier 1 only.
void Engine::p2p_close_open(cudaStream_t st) {
  if (!ex->step_open) return;
  p2p_signal(1, st);
  ex->step_open = false;
}

void Engine::p2p_fwd_begin(cudaStream_t st) {
  Exchange& x = *ex;
  p2p_close_open(st);
  ++x.epoch;
  x.step_open = true;
  p2p_wait(1, x.epoch - 1, st);
  EC_CUDA(cudaEventRecord(ev_b1, st));  // a host-row prefetch may start reading from here
  last_wire_rows = 0;  // (counted on the device: Counters::wire)
  last_wire_bytes = 0;
}

template <int VEC>
void Engine::p2p_publish(float lr, cudaStream_t st, int part, int wait_b, int sig_b) {
  Exchange& x = *ex;
  k_p2p_apply<VEC><<<row_grid(), 256, 0, st>>>(tdev.p, static_cast<int>(T), ctr.p, uniq.p, utab.p, usrc.p,
                                                   ugrad.p, lr, x.peers.p, x.shard_off.p, rank, world, x.hcap,
                                                   storage == EC_STORAGE_HOST ? x.inbox_cap : 0, part,
                                                   p2p_sync(x, rank, wait_b, sig_b));
  launched();
}
void Engine::p2p_bwd_publish(float lr, cudaStream_t st) {
  if (!ex->step_open) invalid("the peer-memory exchange takes one backward per forward");
  PhaseScope ph(prof, kPhaseExchange, st);
  // hits; pinned-host shards also their misses (inbox appends change no row);
  // the last block signals barrier 0
  EC_DISPATCH_VEC(p2p_publish, lr, st, storage == EC_STORAGE_HOST ? 3 : 1, -1, 0);
}

template <int VEC>
void Engine::p2p_hot(float lr, cudaStream_t st) {
  Exchange& x = *ex;
  // (after the barrier-0 wait kernel: a one-block spin leaves the SMs to a
  // prefetch on another stream, a spinning prologue in every block would not);
  // the last kernel signals barrier 1 from its last block
  const bool host = storage == EC_STORAGE_HOST;
  if (!host) p2p_publish<VEC>(lr, st, 2, -1, -1);  // misses: atomics into the owners' rows
  if (host) {  // owner: every source's miss gradients, rank order (inbox allocated by p2p_alloc)
    for (int p = 0; p < x.W; ++p) {
      k_p2p_inbox_apply<VEC><<<host_grid(), 256, 0, st>>>(x.inbox_idx.p + p * x.inbox_cap,
                                                          x.inbox_grad.p + p * x.inbox_cap * D, x.inbox_cnt.p + p,
                                                          store_base, lr, x.ver.p, x.epoch, p2p_sync(x, rank, -1, -1));
      launched();
    }
    EC_CUDA(cudaMemsetAsync(x.inbox_cnt.p, 0, x.inbox_cnt.bytes(), st));  // sources append after barrier 1
  }
  // owner: every source's hit gradients for this rank's slots, then the
  // update (its last block signals barrier 1); upd_cnt is free to reset:
  // every replica finished copying the last step's rows before barrier 0
  p2p_hot_alloc();
  EC_CUDA(cudaMemsetAsync(x.upd_cnt.p, 0, sizeof(int), st));
  const int hg = sm_count(device) * 2;
  k_p2p_hot_reduce<VEC><<<hg, 256, 0, st>>>(x.hin_slot.p, x.hin_grad.p, x.hin_cnt.p, x.hcap, x.W, x.hacc.p, x.hmark.p,
                                            x.upd_slot.p, x.upd_cnt.p);
  launched();
  k_p2p_hot_update<VEC><<<hg, 256, 0, st>>>(x.upd_slot.p, x.upd_cnt.p, x.W, cache.p, x.hacc.p, x.hmark.p,
                                            x.upd_rows.p, x.hin_cnt.p, lr, p2p_sync(x, rank, -1, 1));
  launched();
}

template <int VEC>
void Engine::p2p_hot_copy(cudaStream_t st) {
  k_p2p_hot_copy<VEC><<<sm_count(device) * 2, 256, 0, st>>>(ex->peers.p, ex->W, rank, cache.p, ctr.p,
                                                            static_cast<int>(T));
  launched();
}

template <int VEC>
void Engine::p2p_patch(cudaStream_t st) {
  k_p2p_patch<VEC><<<host_grid(), 256, 0, st>>>(ctr.p, static_cast<int>(T), missq.p, uniq.p, utab.p, urows.p,
                                                ex->peers.p, ex->shard_off.p, world, ex->epoch - 1);
  launched();
}
void Engine::p2p_patch_prefetched(cudaStream_t st) { EC_DISPATCH_VEC(p2p_patch, st); }

void Engine::p2p_bwd_owner(float lr, cudaStream_t st) {
  PhaseScope ph(prof, kPhaseExchange, st);
  p2p_wait(0, ex->epoch, st);
  EC_DISPATCH_VEC(p2p_hot, lr, st);  // its last kernel signals barrier 1
}
void Engine::p2p_bwd_replica(cudaStream_t st) {
  PhaseScope ph(prof, kPhaseExchange, st);
  p2p_wait(1, ex->epoch, st);  // every owner applied its rows
  EC_DISPATCH_VEC(p2p_hot_copy, st);
  ex->step_open = false;
}
void Engine::p2p_bwd_finish(float lr, cudaStream_t st) {
  p2p_bwd_owner(lr, st);
  p2p_bwd_replica(st);
}

// ------------------------------------------------------------ NCCL driver
bool Engine::comm_ready() const { return ex != nullptr && (ex->comm != nullptr || in_group || ex->p2p); }

// Tables, dims, per-table rows, batch capacity and storage tier: a peer's
// shard offsets and inbox segments are computed from the local copy of these,
// so ranks that disagree would index each other's memory wrongly.
uint64_t Engine::geometry_digest() const {
  uint64_t h = mix64(0x65634765ull ^ world);
  auto add = [&](uint64_t v) { h = mix64(h ^ (v + kGolden)); };
  add(T);
  add(D);
  add(max_n);
  add(static_cast<uint64_t>(storage));
  for (uint64_t r : rows) add(r);
  return h;
}

void Engine::attach_comm(const uint8_t* id128) {
  use_device(device);
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(&id, id128, sizeof(id));
  ex_init(world);
  if (ex->comm) {
    ncclCommDestroy(ex->comm);
    ex->comm = nullptr;
  }
  EC_NCCL(ncclCommInitRank(&ex->comm, world, id, rank));
  // every rank's geometry digest, compared before any step moves rows
  DevBuf<uint64_t> dg(static_cast<size_t>(world) + 1);
  const uint64_t mine = geometry_digest();
  EC_CUDA(cudaMemcpy(dg.p, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  cudaStream_t s;
  EC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const ncclResult_t r = ncclAllGather(dg.p, dg.p + 1, 1, ncclUint64, ex->comm, s);
  const cudaError_t ce = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  std::vector<uint64_t> all(world);
  if (r == ncclSuccess && ce == cudaSuccess)
    EC_CUDA(cudaMemcpy(all.data(), dg.p + 1, world * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (r != ncclSuccess || ce != cudaSuccess) {
    ncclCommDestroy(ex->comm);
    ex->comm = nullptr;
    EC_NCCL(r);
    EC_CUDA(ce);
  }
  for (int p = 0; p < world; ++p)
    if (all[p] != mine) {
      ncclCommDestroy(ex->comm);
      ex->comm = nullptr;
      invalid("rank " + std::to_string(p) + " has a different table geometry (tables, dim, rows, batch "
              "capacity or storage tier) than rank " + std::to_string(rank));
    }
}

void Engine::destroy_comm() {
  delete ex;
  ex = nullptr;
}

uint64_t Engine::exch_bytes() const {
  if (!ex) return 0;
  return ex->send_idx.bytes() + ex->send_slot.bytes() + ex->recv_idx.bytes() + ex->hot_g.bytes() +
         ex->hot_slot.bytes() + ex->hot_slot_all.bytes() + ex->send_rows.bytes() + ex->recv_rows.bytes() +
         ex->grad_send.bytes() + ex->grad_recv.bytes() + ex->hot_grad.bytes() + ex->hot_grad_all.bytes();
}

static void nccl_alltoallv(ncclComm_t comm, int W, int rank, const void* send, const std::vector<int64_t>& scnt,
                           const std::vector<int64_t>& soff, void* recv, const std::vector<int64_t>& rcnt,
                           const std::vector<int64_t>& roff, size_t elem, cudaStream_t st) {
  EC_NCCL(ncclGroupStart());
  for (int p = 0; p < W; ++p) {
    if (p == rank) continue;
    if (scnt[p])
      EC_NCCL(ncclSend(static_cast<const char*>(send) + soff[p] * elem, scnt[p] * elem, ncclUint8, p, comm, st));
    if (rcnt[p]) EC_NCCL(ncclRecv(static_cast<char*>(recv) + roff[p] * elem, rcnt[p] * elem, ncclUint8, p, comm, st));
  }
  EC_NCCL(ncclGroupEnd());
}

// Host wait for the counts all-gather (the one host synchronisation of the
// NCCL transport: ncclSend/ncclRecv sizes are host arguments).  Polls the
// stream and ncclCommGetAsyncError instead of blocking in
// cudaStreamSynchronize, so a peer that died or a broken link fails the step
// with EC_ENCCL (communicator aborted) instead of hanging it; same for a wait
// longer than EC_NCCL_TIMEOUT_S seconds (default 60).
static void nccl_wait(ncclComm_t& comm, cudaStream_t st) {
  static const double limit = [] {
    const char* v = std::getenv("EC_NCCL_TIMEOUT_S");
    return v && *v ? std::atof(v) : 60.0;
  }();
  cudaEvent_t ev;
  EC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  EC_CUDA(cudaEventRecord(ev, st));
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned k = 0;; ++k) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) {
      cudaEventDestroy(ev);
      EC_CUDA(q);
    }
    ncclResult_t ar = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError(comm, &ar);
    const bool late = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit;
    if (r != ncclSuccess || (ar != ncclSuccess && ar != ncclInProgress) || late) {
      cudaEventDestroy(ev);
      ncclCommAbort(comm);  // unblocks the kernels still waiting on the dead peer
      comm = nullptr;
      throw Error(EC_ENCCL, late ? "NCCL exchange: counts all-gather exceeded EC_NCCL_TIMEOUT_S; communicator aborted"
                                 : std::string("NCCL exchange: asynchronous error: ") +
                                       ncclGetErrorString(r != ncclSuccess ? r : ar) + "; communicator aborted");
    }
    if (k > 64) std::this_thread::yield();
  }
  cudaEventDestroy(ev);
}

void Engine::exchange_fwd(cudaStream_t st) {
  Exchange& x = *ex;
  PhaseScope ph(prof, kPhaseExchange, st);
  ex_route(st);
  EC_NCCL(ncclAllGather(x.cnt.p, x.allcnt.p, x.W + 1, ncclInt32, x.comm, st));
  EC_CUDA(cudaMemcpyAsync(x.allcnt_host, x.allcnt.p, static_cast<size_t>(x.W) * (x.W + 1) * sizeof(int),
                          cudaMemcpyDeviceToHost, st));
  nccl_wait(x.comm, st);  // request sizes are needed on the host
  ex_plan();
  nccl_alltoallv(x.comm, x.W, rank, x.send_idx.p, x.scnt, x.soff, x.recv_idx.p, x.rcnt, x.roff, sizeof(uint32_t), st);
  ex_serve(st);
  const size_t rowb = static_cast<size_t>(D) * sizeof(float);
  nccl_alltoallv(x.comm, x.W, rank, x.send_rows.p, x.rcnt, x.roff, x.recv_rows.p, x.scnt, x.soff, rowb, st);
  ex_unpack(st);
}

void Engine::exchange_bwd(float lr, cudaStream_t st) {
  Exchange& x = *ex;
  PhaseScope ph(prof, kPhaseExchange, st);
  ex_pack_bwd(st);
  const size_t rowb = static_cast<size_t>(D) * sizeof(float);
  nccl_alltoallv(x.comm, x.W, rank, x.grad_send.p, x.scnt, x.soff, x.grad_recv.p, x.rcnt, x.roff, rowb, st);
  // hit lists: this rank's list to every peer, every peer's list into its rank slot
  EC_NCCL(ncclGroupStart());
  for (int p = 0; p < x.W; ++p) {
    if (p == rank) continue;
    const int64_t mine = x.hcnt[rank];
    if (mine) {
      EC_NCCL(ncclSend(x.hot_slot.p, mine * sizeof(uint32_t), ncclUint8, p, x.comm, st));
      EC_NCCL(ncclSend(x.hot_grad.p, mine * rowb, ncclUint8, p, x.comm, st));
    }
    if (x.hcnt[p]) {
      EC_NCCL(ncclRecv(x.hot_slot_all.p + x.hoff[p], x.hcnt[p] * sizeof(uint32_t), ncclUint8, p, x.comm, st));
      EC_NCCL(ncclRecv(x.hot_grad_all.p + x.hoff[p] * D, x.hcnt[p] * rowb, ncclUint8, p, x.comm, st));
    }
  }
  EC_NCCL(ncclGroupEnd());
  ex_apply_bwd(lr, st);
}

}  // namespace ec

// ===================================================================== ABI
using namespace ec;

struct ec_group_s {
  std::vector<ec_tables> members;
};

extern "C" {

int ec_shard_rows(const uint64_t* rows, uint32_t num_tables, int world, int rank, uint64_t* local_rows) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) invalid("rank/world out of range");
    for (uint32_t t = 0; t < num_tables; ++t)
      local_rows[t] = rows[t] > static_cast<uint64_t>(rank) ? (rows[t] - rank + world - 1) / world : 0;
  });
}

int ec_exchange_plan(const int* counts, int world, int rank, int64_t* scnt, int64_t* soff, int64_t* rcnt,
                     int64_t* roff, int64_t* hcnt, int64_t* hoff) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) invalid("rank/world out of range");
    exchange_plan(counts, world, rank, scnt, soff, rcnt, roff, hcnt, hoff);
  });
}

int ec_comm_unique_id(uint8_t* id128) {
  return guard([&] {
    ncclUniqueId id;
    EC_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
  });
}

int ec_tables_attach_comm(ec_tables t, const uint8_t* id128) {
  return guard([&] {
    if (!t) invalid("null tables handle");
    if (t->e.world < 2) invalid("attach_comm needs world > 1");
    t->e.attach_comm(id128);
  });
}

int ec_group_create(ec_tables* members, int n, ec_group* out) {
  return guard([&] {
    if (n < 2) invalid("a loopback group needs at least two ranks");
    auto* g = new ec_group_s;
    for (int r = 0; r < n; ++r) {
      Engine& e = members[r]->e;
      if (e.world != n || e.rank != r) {
        delete g;
        invalid("group member " + std::to_string(r) + " must be rank " + std::to_string(r) + " of world " +
                std::to_string(n));
      }
      if (e.device != members[0]->e.device || e.D != members[0]->e.D || e.T != members[0]->e.T) {
        delete g;
        invalid("group members must share device, dim and table count");
      }
      e.ex_init(n);
      e.in_group = true;
      g->members.push_back(members[r]);
    }
    *out = g;
  });
}

void ec_group_destroy(ec_group g) {
  if (!g) return;
  for (auto m : g->members) m->e.in_group = false;
  delete g;
}

// Lock-step forward of every rank of a loopback group on one device/stream.
int ec_group_lookup_fwd(ec_group g, const ec_batch* batches, float* const* outs, void* stream) {
  return guard([&] {
    if (!g) invalid("null group");
    cudaStream_t st = as_stream(stream);
    const int W = static_cast<int>(g->members.size());
    if (g->members[0]->e.p2p_on()) {  // peer-memory exchange: the same kernels as across GPUs
      for (int r = 0; r < W; ++r) g->members[r]->e.p2p_close_open(st);  // every signal before any wait
      for (int r = 0; r < W; ++r) {
        Engine& e = g->members[r]->e;
        e.forward_prologue(batches[r], outs[r], st);
        e.p2p_fwd_begin(st);
        e.enqueue_dedup_partition(batches[r].indices_dev, st);
        e.gather_local(st);
        e.pool(st);
        e.have_fwd = true;
      }
      return;
    }
    for (int r = 0; r < W; ++r) {
      Engine& e = g->members[r]->e;
      e.forward_prologue(batches[r], outs[r], st);
      e.enqueue_dedup_partition(batches[r].indices_dev, st);
      e.gather_local(st);
      e.ex_route(st);
    }
    // counts: every rank's vector into every rank's matrix
    std::vector<int> cnts(static_cast<size_t>(W) * (W + 1));
    for (int r = 0; r < W; ++r)
      EC_CUDA(cudaMemcpyAsync(cnts.data() + static_cast<size_t>(r) * (W + 1), g->members[r]->e.ex->cnt.p,
                              (W + 1) * sizeof(int), cudaMemcpyDeviceToHost, st));
    EC_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < W; ++r) {
      Engine& e = g->members[r]->e;
      std::memcpy(e.ex->allcnt_host, cnts.data(), cnts.size() * sizeof(int));
      e.ex_plan();
    }
    // ids: requester r's segment for owner o -> owner o's segment for requester r
    for (int r = 0; r < W; ++r)
      for (int o = 0; o < W; ++o) {
        Exchange& a = *g->members[r]->e.ex;
        Exchange& b = *g->members[o]->e.ex;
        if (r == o || !a.scnt[o]) continue;
        EC_CUDA(cudaMemcpyAsync(b.recv_idx.p + b.roff[r], a.send_idx.p + a.soff[o], a.scnt[o] * sizeof(uint32_t),
                                cudaMemcpyDeviceToDevice, st));
      }
    for (int r = 0; r < W; ++r) g->members[r]->e.ex_serve(st);
    const size_t D = g->members[0]->e.D;
    for (int r = 0; r < W; ++r)
      for (int o = 0; o < W; ++o) {
        Exchange& a = *g->members[r]->e.ex;
        Exchange& b = *g->members[o]->e.ex;
        if (r == o || !a.scnt[o]) continue;
        EC_CUDA(cudaMemcpyAsync(a.recv_rows.p + a.soff[o] * D, b.send_rows.p + b.roff[r] * D,
                                a.scnt[o] * D * sizeof(float), cudaMemcpyDeviceToDevice, st));
      }
    for (int r = 0; r < W; ++r) {
      Engine& e = g->members[r]->e;
      e.ex_unpack(st);
      e.pool(st);
      e.have_fwd = true;
    }
  });
}

int ec_group_lookup_bwd(ec_group g, const float* const* grads, float lr, void* stream) {
  return guard([&] {
    if (!g) invalid("null group");
    cudaStream_t st = as_stream(stream);
    const int W = static_cast<int>(g->members.size());
    const size_t D = g->members[0]->e.D;
    for (int r = 0; r < W; ++r) g->members[r]->e.rows_trained = true;
    if (g->members[0]->e.p2p_on()) {
      for (int r = 0; r < W; ++r) {  // validate before enqueuing anything
        Engine& e = g->members[r]->e;
        if (!e.have_fwd) invalid("ec_group_lookup_bwd needs a preceding forward");
        if (!e.p2p_step_open()) invalid("the peer-memory exchange takes one backward per forward");
        if (!grads[r]) invalid("null gradient");
      }
      // every rank's signal of barrier 0 precedes every rank's wait on one stream
      for (int r = 0; r < W; ++r) {
        Engine& e = g->members[r]->e;
        e.scatter_grads(grads[r], st);
        e.p2p_bwd_publish(lr, st);  // (its last block signals barrier 0)
      }
      // every owner's barrier-1 signal precedes every replica's wait on one stream
      for (int r = 0; r < W; ++r) g->members[r]->e.p2p_bwd_owner(lr, st);
      for (int r = 0; r < W; ++r) g->members[r]->e.p2p_bwd_replica(st);
      return;
    }
    for (int r = 0; r < W; ++r) {
      Engine& e = g->members[r]->e;
      if (!e.have_fwd) invalid("ec_group_lookup_bwd needs a preceding forward");
      e.scatter_and_apply_local(grads[r], lr, st);
      e.ex_pack_bwd(st);
    }
    for (int r = 0; r < W; ++r)
      for (int o = 0; o < W; ++o) {
        Exchange& a = *g->members[r]->e.ex;  // requester
        Exchange& b = *g->members[o]->e.ex;  // owner
        if (r == o) continue;
        if (a.scnt[o])
          EC_CUDA(cudaMemcpyAsync(b.grad_recv.p + b.roff[r] * D, a.grad_send.p + a.soff[o] * D,
                                  a.scnt[o] * D * sizeof(float), cudaMemcpyDeviceToDevice, st));
        const int64_t nh = a.hcnt[r];
        if (nh) {
          EC_CUDA(cudaMemcpyAsync(b.hot_slot_all.p + b.hoff[r], a.hot_slot.p, nh * sizeof(uint32_t),
                                  cudaMemcpyDeviceToDevice, st));
          EC_CUDA(cudaMemcpyAsync(b.hot_grad_all.p + b.hoff[r] * D, a.hot_grad.p, nh * D * sizeof(float),
                                  cudaMemcpyDeviceToDevice, st));
        }
      }
    for (int r = 0; r < W; ++r) g->members[r]->e.ex_apply_bwd(lr, st);
  });
}

// Loopback group on the peer-memory exchange: every member sees the others'
// shards and hot lists directly (same device), through the kernels a
// multi-process job uses over NVLink (ec_tables_p2p_export/import).
int ec_group_set_p2p(ec_group g, int enable) {
  return guard([&] {
    if (!g) invalid("null group");
    if (!enable) {
      for (auto m : g->members)
        if (m->e.ex) m->e.ex->p2p = false;
      return;
    }
    std::vector<PeerView> views;
    for (auto m : g->members) {
      use_device(m->e.device);
      m->e.p2p_alloc();
      views.push_back(m->e.p2p_self());
    }
    for (auto m : g->members) m->e.p2p_set_peers(views);
  });
}

// Multi-process: this rank's peer-visible allocations, to be all-gathered
// and passed to every rank's ec_tables_p2p_import.  Blob: CUDA IPC handles of
// {shard (HBM), updated hot slots, their rows, their count, hot inbox slots,
// gradients, counts, barrier words, miss inbox indices, gradients, counts,
// row generations} (unused ones zero), then the host
// shard's memfd as {pid, fd, bytes} (pinned-host tier; zeros for HBM).
namespace {
constexpr int kP2PHandles = 12;
struct HostSeg {
  int64_t pid, fd;
  uint64_t bytes;
  int64_t present;
  uint64_t geometry;  // Engine::geometry_digest of the exporting rank
  int64_t rank;
};
constexpr uint64_t kP2PBlob = kP2PHandles * sizeof(cudaIpcMemHandle_t) + sizeof(HostSeg);
}  // namespace

int ec_tables_p2p_export(ec_tables t, uint8_t* blob, uint64_t cap, uint64_t* len) {
  return guard([&] {
    if (!t || !len) invalid("null argument");
    Engine& e = t->e;
    use_device(e.device);
    e.p2p_alloc();
    *len = kP2PBlob;
    if (!blob) return;
    if (cap < kP2PBlob) invalid("p2p export blob needs " + std::to_string(kP2PBlob) + " bytes");
    std::memset(blob, 0, kP2PBlob);
    const Exchange& x = *e.ex;
    void* ptrs[kP2PHandles] = {e.store_dev.p,  x.upd_slot.p,  x.upd_rows.p,   x.upd_cnt.p,
                               x.hin_slot.p,   x.hin_grad.p,  x.hin_cnt.p,    x.flags.p,
                               x.inbox_idx.p,  x.inbox_grad.p, x.inbox_cnt.p, x.ver.p};
    for (int k = 0; k < kP2PHandles; ++k) {
      if (!ptrs[k]) continue;
      cudaIpcMemHandle_t h;
      EC_CUDA(cudaIpcGetMemHandle(&h, ptrs[k]));
      std::memcpy(blob + k * sizeof(h), &h, sizeof(h));
    }
    HostSeg hs{0, 0, 0, 0, e.geometry_digest(), e.rank};
    if (e.storage == EC_STORAGE_HOST) {
      hs.pid = static_cast<int64_t>(getpid());
      hs.fd = e.store_host_fd;
      hs.bytes = e.store_host_bytes;
      hs.present = 1;
    }
    std::memcpy(blob + kP2PHandles * sizeof(cudaIpcMemHandle_t), &hs, sizeof(hs));
  });
}

int ec_tables_p2p_disable(ec_tables t) {
  return guard([&] {
    if (!t) invalid("null tables handle");
    if (t->e.ex) t->e.ex->p2p = false;
  });
}

int ec_tables_p2p_import(ec_tables t, const uint8_t* blobs, uint64_t blob_len) {
  return guard([&] {
    if (!t || !blobs) invalid("null argument");
    Engine& e = t->e;
    if (e.world < 2) invalid("the peer-memory exchange needs world > 1");
    if (blob_len != kP2PBlob) invalid("unexpected p2p blob size");
    use_device(e.device);
    e.p2p_alloc();
    Exchange& x = *e.ex;
    for (int p = 0; p < e.world; ++p) {  // validate every blob before opening any handle
      HostSeg hs;
      std::memcpy(&hs, blobs + p * blob_len + kP2PHandles * sizeof(cudaIpcMemHandle_t), sizeof(hs));
      if (hs.present != (e.storage == EC_STORAGE_HOST ? 1 : 0)) invalid("ranks disagree on the storage tier");
      if (hs.rank != p) invalid("p2p blob " + std::to_string(p) + " was exported by rank " + std::to_string(hs.rank));
      if (hs.geometry != e.geometry_digest())
        invalid("rank " + std::to_string(p) + " has a different table geometry (tables, dim, rows, batch capacity "
                "or storage tier) than rank " + std::to_string(e.rank));
    }
    std::vector<PeerView> views(e.world);
    for (int p = 0; p < e.world; ++p) {
      if (p == e.rank) {
        views[p] = e.p2p_self();
        continue;
      }
      const uint8_t* b = blobs + p * blob_len;
      void* ptrs[kP2PHandles] = {};
      const cudaIpcMemHandle_t zero{};
      for (int k = 0; k < kP2PHandles; ++k) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, b + k * sizeof(h), sizeof(h));
        if (std::memcmp(&h, &zero, sizeof(h)) == 0) continue;
        EC_CUDA(cudaIpcOpenMemHandle(&ptrs[k], h, cudaIpcMemLazyEnablePeerAccess));
        x.ipc_opened.push_back(ptrs[k]);
      }
      HostSeg hs;
      std::memcpy(&hs, b + kP2PHandles * sizeof(cudaIpcMemHandle_t), sizeof(hs));
      if (hs.present) {  // the peer's shard, mapped here and read over this GPU's own link
        const std::string path = "/proc/" + std::to_string(hs.pid) + "/fd/" + std::to_string(hs.fd);
        const int fd = open(path.c_str(), O_RDWR);
        if (fd < 0) invalid("cannot open peer host shard " + path + " (peers must share a node)");
        const uint64_t huge = 2ull << 20;
        const size_t maplen = (hs.bytes + huge - 1) / huge * huge;
        void* m = mmap(nullptr, maplen, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) invalid("cannot map peer host shard " + path);
        if (cudaHostRegister(m, maplen, cudaHostRegisterMapped | cudaHostRegisterPortable) != cudaSuccess) {
          cudaGetLastError();
          munmap(m, maplen);
          invalid("cannot register peer host shard " + path);
        }
        x.host_maps.emplace_back(m, maplen);
        EC_CUDA(cudaHostGetDevicePointer(&ptrs[0], m, 0));
      }
      views[p] = PeerView{static_cast<float*>(ptrs[0]),       static_cast<const uint32_t*>(ptrs[1]),
                          static_cast<const float*>(ptrs[2]), static_cast<const int*>(ptrs[3]),
                          static_cast<uint32_t*>(ptrs[4]),    static_cast<float*>(ptrs[5]),
                          static_cast<int*>(ptrs[6]),         static_cast<unsigned*>(ptrs[7]),
                          static_cast<uint32_t*>(ptrs[8]),    static_cast<float*>(ptrs[9]),
                          static_cast<int*>(ptrs[10]),        static_cast<uint32_t*>(ptrs[11])};
    }
    e.p2p_set_peers(views);
  });
}

}  // extern "C"
