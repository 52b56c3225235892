"""EmbeddingTables: the lookup engine (K1..K6) behind a torch-friendly API.

Thin wrapper over ``ec_tables_*`` / ``ec_lookup_*`` (include/embcomm_gpu.h).
Torch provides device buffers and the current stream; every computation is
one of the library's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from ._native import ValidationError, check

STORAGE = {"hbm": 0, "host": 1}


def _stream_ptr(torch, device):
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # an int, without a Stream object
    if raw is not None:
        return raw(device)
    return torch.cuda.current_stream(device).cuda_stream


def _offsets_array(cache, table_offsets):
    """int64 ndarray of a table-offsets sequence, memoised by value (the
    per-step host cost of a lookup is a few microseconds of Python)."""
    if isinstance(table_offsets, np.ndarray) and table_offsets.dtype == np.int64 and table_offsets.flags.c_contiguous:
        return table_offsets
    key = tuple(table_offsets)
    a = cache.get(key)
    if a is None:
        if len(cache) > 64:
            cache.clear()
        a = cache[key] = np.ascontiguousarray(key, dtype=np.int64)
    return a


class EmbeddingTables:
    """Row-wise sharded fp32 embedding tables with a replicated HBM hot-row cache.

    rows: E_t per table; dim: D (4, 8, 16, 32, 64 or 128); storage: cold tier
    "hbm" or "host" (pinned, read by the GPU over the host link); rank/world:
    owner(id) = id % world.
    """

    def __init__(self, rows: Sequence[int], dim: int, *, storage: str = "hbm", rank: int = 0, world: int = 1,
                 max_lookups_per_table: int, max_batch_size: int, device: int = 0):
        import torch
        self.torch = torch
        self._offs_cache = {}
        self._batch_cache = {}  # (indices ptr, offsets, bag offsets, B, P) -> ctypes Batch (per-step host cost)
        self._stats_bufs = None
        self.rows = [int(r) for r in rows]
        self.T = len(self.rows)
        self.D = int(dim)
        self.device = device
        self.world = world
        self.rank = rank
        self._rows_c = (C.c_uint64 * self.T)(*self.rows)
        cfg = N.TablesConfig(self.T, self.D, C.cast(self._rows_c, C.POINTER(C.c_uint64)), STORAGE[storage], rank,
                             world, max_lookups_per_table, max_batch_size, device)
        h = C.c_void_p()
        check(N.lib().ec_tables_create(C.byref(cfg), C.byref(h)))
        self._h = h
        self._offsets = None
        self._out = None

    def close(self):
        if getattr(self, "_h", None):
            N.lib().ec_tables_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- contents
    def memory(self):
        d, h = C.c_uint64(), C.c_uint64()
        check(N.lib().ec_tables_memory(self._h, C.byref(d), C.byref(h)))
        return {"device_bytes": d.value, "host_bytes": h.value}

    PHASES = ("k_insert", "k_compact", "k_inverse_partition", "k_gather", "k_gather_host", "exchange", "k_pool",
              "k_scatter", "k_apply", "k_apply_host", "k_dedup_cluster", "k_clear_miss_sums")

    def use_graphs(self, enable: bool = True):
        """CUDA-graph replay of forward/backward (needs a non-default stream)."""
        check(N.lib().ec_tables_use_graphs(self._h, 1 if enable else 0))

    def dedup_mode(self, mode: str = "auto"):
        """"auto" (cluster per table when the tables fill the GPU), "tiles", "cluster", or "table"
        (one CTA per table, batches of <= 16384 lookups per table)."""
        check(N.lib().ec_tables_dedup_mode(self._h, {"auto": 0, "tiles": 1, "cluster": 2, "table": 3}[mode]))

    def scatter_mode(self, mode: str = "auto"):
        """Backward gradient reduction: "auto", "atomic" or "transpose"."""
        check(N.lib().ec_tables_scatter_mode(self._h, {"auto": 0, "atomic": 1, "transpose": 2}[mode]))

    def profile(self, enable: bool = True):
        """Per-phase CUDA-event timing of forward/backward (see ec_tables_profile)."""
        check(N.lib().ec_tables_profile(self._h, 1 if enable else 0))

    def profile_timeline(self, cap: int = 1 << 16):
        """[(phase name, start ms, end ms)] of the profiled kernels since the last call."""
        buf = np.zeros(3 * cap, np.float64)
        n = C.c_uint64()
        check(N.lib().ec_tables_profile_timeline(self._h, buf.ctypes.data, cap, C.byref(n)))
        k = min(cap, n.value)
        return [(self.PHASES[int(buf[3 * i])], float(buf[3 * i + 1]), float(buf[3 * i + 2])) for i in range(k)]

    def profile_read(self, reset: bool = True):
        ms = np.zeros(len(self.PHASES), np.float64)
        calls = np.zeros(len(self.PHASES), np.uint64)
        launches = C.c_uint64()
        check(N.lib().ec_tables_profile_read(self._h, ms.ctypes.data, calls.ctypes.data, C.byref(launches),
                                             1 if reset else 0))
        return {"ms": dict(zip(self.PHASES, ms.tolist())), "calls": dict(zip(self.PHASES, calls.tolist())),
                "launches": int(launches.value)}

    def init_synthetic(self, seed: int, scale: float = 0.05):
        check(N.lib().ec_tables_init_synthetic(self._h, seed, scale, _stream_ptr(self.torch, self.device)))

    def place_cache(self, cached_ids: Sequence):
        """cached_ids[t]: ids of table t held in the HBM cache (e.g. dist.top_ids(k_t))."""
        arrs = [np.ascontiguousarray(c if c is not None else [], dtype=np.uint32) for c in cached_ids]
        if len(arrs) != self.T:
            raise ValidationError("need one cache id list per table")
        ptrs = (C.c_void_p * self.T)(*[a.ctypes.data if a.size else None for a in arrs])
        ks = np.array([a.size for a in arrs], dtype=np.uint64)
        self.torch.cuda.current_stream(self.device).synchronize()
        check(N.lib().ec_tables_place_cache(self._h, ptrs, ks.ctypes.data))

    def read_rows(self, table: int, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        out = np.empty((ids.size, self.D), np.float32)
        self.torch.cuda.current_stream(self.device).synchronize()
        check(N.lib().ec_tables_read_rows(self._h, table, ids.ctypes.data, ids.size, out.ctypes.data))
        return out

    def write_rows(self, table: int, ids, rows):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        rows = np.ascontiguousarray(rows, dtype=np.float32).reshape(ids.size, self.D)
        self.torch.cuda.current_stream(self.device).synchronize()
        check(N.lib().ec_tables_write_rows(self._h, table, ids.ctypes.data, ids.size, rows.ctypes.data))

    # -------------------------------------------------------------- batch
    def forward(self, indices, table_offsets: Sequence[int], batch_size: int, pooling: int = 0,
                bag_offsets=None, out=None):
        """Pooled lookup.  indices: int32/uint32 CUDA tensor of all tables'
        lookups concatenated; table_offsets: T+1 host ints; fixed pooling
        (bag_offsets None) or CSR bag_offsets (int64 CUDA, T*B+1, table-major).
        Returns [batch_size, T*D] fp32."""
        torch = self.torch
        if indices.dtype not in (torch.int32, torch.uint32) or not indices.is_cuda or not indices.is_contiguous():
            raise ValidationError("indices must be a contiguous int32/uint32 CUDA tensor")
        offs = _offsets_array(self._offs_cache, table_offsets)
        if offs.size != self.T + 1:
            raise ValidationError("table_offsets needs num_tables+1 entries")
        self._offsets = offs
        if out is None:
            out = torch.empty((batch_size, self.T * self.D), dtype=torch.float32, device=indices.device)
        elif (out.dtype != torch.float32 or not out.is_contiguous() or out.device != indices.device
              or out.numel() != batch_size * self.T * self.D):
            raise ValidationError(f"out must be a contiguous float32 tensor of {batch_size * self.T * self.D} "
                                  "elements on the indices' device")
        bo = 0
        if bag_offsets is not None:
            if (bag_offsets.dtype != torch.int64 or not bag_offsets.is_cuda or not bag_offsets.is_contiguous()
                    or bag_offsets.numel() != self.T * batch_size + 1):
                raise ValidationError("bag_offsets must be a contiguous int64 CUDA tensor of num_tables * "
                                      "batch_size + 1 entries")
            bo = bag_offsets.data_ptr()
        b = self._batch(indices.data_ptr(), offs, bo or None, batch_size, pooling)
        check(N.lib().ec_lookup_fwd(self._h, b, out.data_ptr(), _stream_ptr(torch, self.device)))
        self._out = out
        return out

    def prefetch(self, indices, table_offsets: Sequence[int], batch_size: int, pooling: int = 0, bag_offsets=None,
                 stream=None):
        """Start the next batch (dedup, hit/miss, host-miss gather) while the
        current one finishes; the next forward() with the same `indices`
        tensor consumes it.  Same geometry as the last forward.  `stream`: the
        torch stream that produced `indices` (default: the current stream);
        the prefetch starts after the work enqueued there."""
        offs = _offsets_array(self._offs_cache, table_offsets)
        bo = bag_offsets.data_ptr() if bag_offsets is not None else None
        self._pf_offs = offs  # keep alive for the call
        b = self._batch(indices.data_ptr(), offs, bo, batch_size, pooling)
        sp = stream.cuda_stream if stream is not None else _stream_ptr(self.torch, self.device)
        check(N.lib().ec_lookup_prefetch(self._h, b, sp))

    def _batch(self, ptr, offs, bo, batch_size, pooling):
        """ctypes ec_batch by reference, memoised (the offsets array is kept
        alive by the offsets cache)."""
        key = (ptr, id(offs), bo, batch_size, pooling)
        b = self._batch_cache.get(key)
        if b is None:
            if len(self._batch_cache) > 64:
                self._batch_cache.clear()
            st = N.Batch(ptr, offs.ctypes.data_as(C.POINTER(C.c_int64)), bo, batch_size, pooling)
            b = self._batch_cache[key] = (C.byref(st), st, offs)
        return b[0]

    def schedule(self, sample_ids):
        """Hot/normal order of a dataset (sample-major [q, T] int32/uint32 CUDA
        tensor): returns (order tensor, number of hot samples).  A sample is hot
        iff all its ids are cached (classify_samples, trace.cpp:185-204)."""
        torch = self.torch
        q = sample_ids.numel() // self.T
        order = torch.empty(q, dtype=torch.int32, device=sample_ids.device)
        nh = C.c_uint64()
        check(N.lib().ec_tables_schedule(self._h, sample_ids.data_ptr(), q, order.data_ptr(), C.byref(nh),
                                         _stream_ptr(torch, self.device)))
        return order, int(nh.value)

    def gather_batch(self, sample_ids, order, first: int, count: int, out=None):
        """Samples order[first:first+count] as a table-major pooling-1 batch."""
        torch = self.torch
        if out is None:
            out = torch.empty(count * self.T, dtype=torch.int32, device=sample_ids.device)
        check(N.lib().ec_tables_gather_batch(self._h, sample_ids.data_ptr(), order.data_ptr(), first, count,
                                             out.data_ptr(), _stream_ptr(torch, self.device)))
        return out

    def prefetch_drop(self):
        """Discard pending prefetched batches."""
        check(N.lib().ec_lookup_prefetch_drop(self._h, _stream_ptr(self.torch, self.device)))

    def prefetch_wait(self):
        """Make the current stream wait for a pending prefetch and the last
        backward's deferred host-tier write-back."""
        check(N.lib().ec_lookup_prefetch_wait(self._h, _stream_ptr(self.torch, self.device)))

    def backward(self, grad, lr: float):
        torch = self.torch
        if grad.dtype != torch.float32 or not grad.is_cuda or not grad.is_contiguous():
            raise ValidationError("grad must be a contiguous fp32 CUDA tensor")
        check(N.lib().ec_lookup_bwd(self._h, grad.data_ptr(), lr, _stream_ptr(torch, self.device)))

    def stats(self, per_table: bool = False):
        s = N.BatchStats()
        u = np.zeros(self.T, np.int64)
        m = np.zeros(self.T, np.int64)
        check(N.lib().ec_lookup_stats(self._h, _stream_ptr(self.torch, self.device), C.byref(s), u.ctypes.data,
                                      m.ctypes.data))
        d = s.as_dict()
        if per_table:
            d["unique_per_table"] = u
            d["miss_per_table"] = m
        return d

    def stats_enqueue(self, slot: int) -> None:
        """Queue a copy of the last forward's counters into pinned ring slot
        `slot` on the current stream (no synchronisation)."""
        check(N.lib().ec_lookup_stats_enqueue(self._h, _stream_ptr(self.torch, self.device), slot))

    def stats_collect(self, slot: int, per_table: bool = False):
        """Wait for slot `slot`'s copy and decode it like stats()."""
        s = N.BatchStats()
        u = np.empty(self.T, np.int64)
        m = np.empty(self.T, np.int64)
        check(N.lib().ec_lookup_stats_collect(self._h, slot, C.byref(s), u.ctypes.data, m.ctypes.data))
        d = s.as_dict()
        if per_table:
            d["unique_per_table"] = u
            d["miss_per_table"] = m
        return d

    # ------------------------------------------------------ parity exports
    def export_unique(self, table: int) -> np.ndarray:
        n = C.c_uint64()
        check(N.lib().ec_export_unique(self._h, table, None, 0, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        check(N.lib().ec_export_unique(self._h, table, out.ctypes.data, out.size, C.byref(n)))
        return out

    def export_inverse(self, table: int) -> np.ndarray:
        n = int(self._offsets[table + 1] - self._offsets[table])
        out = np.empty(n, np.uint32)
        check(N.lib().ec_export_inverse(self._h, table, out.ctypes.data))
        return out

    def export_hit(self, table: int) -> np.ndarray:
        U = self.export_unique(table).size
        out = np.empty(U, np.uint8)
        check(N.lib().ec_export_hit(self._h, table, out.ctypes.data))
        return out

    def export_rows(self, table: int) -> np.ndarray:
        U = self.export_unique(table).size
        out = np.empty((U, self.D), np.float32)
        check(N.lib().ec_export_rows(self._h, table, out.ctypes.data))
        return out

    # ---------------------------------------------------------- multi-GPU
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(N.lib().ec_comm_unique_id(buf))
        return bytes(buf)

    def attach_comm(self, uid: bytes):
        buf = (C.c_uint8 * 128)(*uid)
        check(N.lib().ec_tables_attach_comm(self._h, buf))

    def p2p_export(self) -> bytes:
        """This rank's peer-visible allocations as CUDA IPC handles (one
        process per GPU); all-gather them and pass the list to p2p_import."""
        n = C.c_uint64()
        check(N.lib().ec_tables_p2p_export(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint8 * n.value)()
        check(N.lib().ec_tables_p2p_export(self._h, buf, n.value, C.byref(n)))
        return bytes(buf)

    def p2p_import(self, blobs: Sequence[bytes]):
        """Switch to the peer-memory exchange with every rank's export blob
        (rank order).  Each step then ends at a device-side barrier."""
        if len(blobs) != self.world or len({len(b) for b in blobs}) != 1:
            raise ValueError("p2p_import needs one equal-sized blob per rank")
        raw = b"".join(blobs)
        buf = (C.c_uint8 * len(raw)).from_buffer_copy(raw)
        check(N.lib().ec_tables_p2p_import(self._h, buf, len(blobs[0])))

    def p2p_disable(self):
        """Leave the peer-memory exchange (every rank must, e.g. after some
        rank's import failed); attach_comm then selects NCCL."""
        check(N.lib().ec_tables_p2p_disable(self._h))



def shard_rows(rows: Sequence[int], world: int, rank: int) -> list[int]:
    """Rows of each table owned by `rank` under owner(id) = id % world."""
    r = (C.c_uint64 * len(rows))(*rows)
    out = np.zeros(len(rows), np.uint64)
    check(N.lib().ec_shard_rows(r, len(rows), world, rank, out.ctypes.data))
    return [int(x) for x in out]


def exchange_plan(counts, world: int, rank: int) -> dict:
    """Per-batch exchange plan of `rank` from the all-gathered count matrix
    (world x (world+1): requests to each owner, then the hit count)."""
    m = np.ascontiguousarray(counts, dtype=np.int32).reshape(world, world + 1)
    outs = [np.zeros(world, np.int64) for _ in range(6)]
    check(N.lib().ec_exchange_plan(m.ctypes.data, world, rank, *[o.ctypes.data for o in outs]))
    return dict(zip(("send_cnt", "send_off", "recv_cnt", "recv_off", "hot_cnt", "hot_off"), outs))


class EmbeddingGroup:
    """In-process loopback group: ranks 0..n-1 of row-sharded tables on one
    device, driven in lock step (same routing / serve / gradient return /
    rank-ordered replica update as the NCCL path, device copies as transport)."""

    def __init__(self, members: Sequence[EmbeddingTables], p2p: bool = False):
        self.members = list(members)
        arr = (C.c_void_p * len(self.members))(*[m._h.value for m in self.members])
        h = C.c_void_p()
        check(N.lib().ec_group_create(arr, len(self.members), C.byref(h)))
        self._h = h
        if p2p:  # peer-memory exchange (the multi-process NVLink kernels, loopback)
            check(N.lib().ec_group_set_p2p(self._h, 1))

    def close(self):
        if getattr(self, "_h", None):
            N.lib().ec_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, indices, table_offsets, batch_size: int, pooling: int):
        """indices[r]: rank r's int32 CUDA ids; same geometry on every rank."""
        torch = self.members[0].torch
        n = len(self.members)
        offs = np.ascontiguousarray(table_offsets, dtype=np.int64)
        batches = (N.Batch * n)(*[N.Batch(indices[r].data_ptr(), offs.ctypes.data_as(C.POINTER(C.c_int64)), None,
                                          batch_size, pooling) for r in range(n)])
        outs = [torch.empty((batch_size, m.T * m.D), dtype=torch.float32, device=indices[0].device)
                for m in self.members]
        optr = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
        for m in self.members:
            m._offsets = offs
        check(N.lib().ec_group_lookup_fwd(self._h, batches, optr, _stream_ptr(torch, self.members[0].device)))
        return outs

    def backward(self, grads, lr: float):
        torch = self.members[0].torch
        gptr = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        check(N.lib().ec_group_lookup_bwd(self._h, gptr, lr, _stream_ptr(torch, self.members[0].device)))
