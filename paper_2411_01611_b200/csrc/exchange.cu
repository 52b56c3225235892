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

#include <algorithm>
#include <cstring>
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

  ~Exchange() {
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

// ------------------------------------------------------------ NCCL driver
bool Engine::comm_ready() const { return ex != nullptr && (ex->comm != nullptr || in_group); }

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

void Engine::exchange_fwd(cudaStream_t st) {
  Exchange& x = *ex;
  PhaseScope ph(prof, kPhaseExchange, st);
  ex_route(st);
  EC_NCCL(ncclAllGather(x.cnt.p, x.allcnt.p, x.W + 1, ncclInt32, x.comm, st));
  EC_CUDA(cudaMemcpyAsync(x.allcnt_host, x.allcnt.p, static_cast<size_t>(x.W) * (x.W + 1) * sizeof(int),
                          cudaMemcpyDeviceToHost, st));
  EC_CUDA(cudaStreamSynchronize(st));  // request sizes are needed on the host
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

}  // extern "C"
