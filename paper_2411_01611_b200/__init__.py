"""embcomm-b200: B200-native embedding-lookup hot path of arXiv 2411.01611.

Python mirror of the reference library's core/ API (namespace ``embcomm``,
/root/reference/proj/core/include/embcomm/*.hpp) over the C-ABI of
``libembcomm_gpu.so`` (include/embcomm_gpu.h).  Same names, argument meaning
and error behaviour: ``ValidationError`` where the reference throws
ValidationError, ``InvariantError`` where it throws InvariantError.

* Cost model / planner / distributions run on the host in the reference's
  arithmetic order (bit-identical results).
* Sampling, the Monte Carlo simulator, trace classification and the whole
  lookup engine (dedup, hit/miss, gather, pool, backward, exchange) run as
  sm_100a kernels.  There is no CPU fallback: every call fails loudly without
  a GPU or without the built library.

Torch is used only for device memory and streams in ``EmbeddingTables``.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from ._native import (CudaError, EmbcommError, InvariantError, NcclError,  # noqa: F401
                      OutOfMemoryError, ValidationError, check)

__all__ = [
    "ValidationError", "InvariantError", "CudaError", "EmbcommError",
    "EmbeddingDistribution", "DistributionKind", "DistributionSpec", "materialize", "materialize_extended",
    "scale", "default_shape", "WorkloadSpec", "CostBreakdown", "kCostUnitsNote", "batch_presence_prob",
    "expected_unique_per_batch", "expected_unique_from_rank", "coalesced_batch_cost", "baseline_epoch_cost",
    "coalesced_epoch_cost", "cached_epoch_cost", "DeviceModel", "max_batch_size", "MarginalReport",
    "delta_comm", "CachePlan", "optimal_cache_size_scan", "optimal_cache_size_search", "memory_io_proxy",
    "place_topk_global", "expected_unique_many", "cost_curve", "SplitMix64", "substream_seed", "DiscreteSampler", "sample_batch", "Stat",
    "SimResult", "measure_unique", "simulate_epoch", "Trace", "BinaryTrace", "copy_async", "classify_samples", "build_schedule",
    "SampleClasses", "BatchSchedule", "SkewTable", "build_skew_table", "estimate_distribution", "EmbeddingTables", "EmbeddingGroup", "shard_rows", "exchange_plan",
]

kCostUnitsNote = "one unit = one embedding vector = one transmitted index"
kRngAlgorithm = "splitmix64"


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


# ------------------------------------------------------------- distribution
class EmbeddingDistribution:
    """EmbeddingDistribution (core/include/embcomm/distribution.hpp:19-49)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._sampler = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and N is not None and N._lib is not None:
            for s in self._sampler.values():
                N._lib.ec_sampler_destroy(s)
            N._lib.ec_dist_destroy(h)
            self._h = None

    @classmethod
    def from_probabilities(cls, probs) -> "EmbeddingDistribution":
        p = np.ascontiguousarray(probs, dtype=np.float64)
        h = C.c_void_p()
        check(N.lib().ec_dist_from_probabilities(p.ctypes.data, p.size, C.byref(h)))
        return cls(h.value)

    @classmethod
    def uniform(cls, size: int) -> "EmbeddingDistribution":
        h = C.c_void_p()
        check(N.lib().ec_dist_uniform(size, C.byref(h)))
        return cls(h.value)

    def size(self) -> int:
        return int(N.lib().ec_dist_size(self._h))

    def __len__(self):
        return self.size()

    def prob(self, id_: int) -> float:
        out = C.c_double()
        check(N.lib().ec_dist_prob(self._h, id_, C.byref(out)))
        return out.value

    def prob_at_rank(self, rank: int) -> float:
        out = C.c_double()
        check(N.lib().ec_dist_prob_at_rank(self._h, rank, C.byref(out)))
        return out.value

    def id_at_rank(self, rank: int) -> int:
        out = C.c_uint32()
        check(N.lib().ec_dist_id_at_rank(self._h, rank, C.byref(out)))
        return out.value

    def rank_of(self, id_: int) -> int:
        out = C.c_uint64()
        check(N.lib().ec_dist_rank_of(self._h, id_, C.byref(out)))
        return out.value

    def ranked_probs(self) -> np.ndarray:
        out = np.empty(self.size(), np.float64)
        check(N.lib().ec_dist_export(self._h, out.ctypes.data, None))
        return out

    def rank_to_id(self) -> np.ndarray:
        out = np.empty(self.size(), np.uint32)
        check(N.lib().ec_dist_export(self._h, None, out.ctypes.data))
        return out

    def top_ids(self, k: int) -> np.ndarray:
        if k < 0:
            raise ValidationError(f"cannot take top {k}")
        out = np.empty(k, np.uint32)
        check(N.lib().ec_dist_top_ids(self._h, k, out.ctypes.data))
        return out

    def mass_of(self, ids) -> float:
        a = _u32(ids)
        out = C.c_double()
        check(N.lib().ec_dist_mass_of(self._h, a.ctypes.data, a.size, C.byref(out)))
        return out.value

    def sampler(self, device: int = 0) -> "DiscreteSampler":
        return DiscreteSampler(self, device)


class DistributionKind(enum.IntEnum):
    """DistributionKind (core/include/embcomm/distribution_spec.hpp:14)."""
    zipf = 0
    exponential = 1
    half_normal = 2
    empirical = 3


def default_shape(kind: DistributionKind) -> float:
    out = C.c_double()
    check(N.lib().ec_default_shape(int(kind), C.byref(out)))
    return out.value


@dataclass
class DistributionSpec:
    """DistributionSpec (core/include/embcomm/distribution_spec.hpp:36-53)."""
    kind: DistributionKind = DistributionKind.zipf
    size: int = 0
    shape: float = 0.0
    probs: list = field(default_factory=list)

    @staticmethod
    def parametric(kind: DistributionKind, size: int, shape: float) -> "DistributionSpec":
        if kind == DistributionKind.empirical:
            raise ValidationError("use DistributionSpec::empirical for explicit probabilities")
        if size == 0:
            raise ValidationError("distribution size must be >= 1")
        if not (shape > 0.0) or not np.isfinite(shape):
            raise ValidationError("shape parameter must be positive and finite")
        return DistributionSpec(DistributionKind(kind), int(size), float(shape))

    @staticmethod
    def empirical(probs) -> "DistributionSpec":
        probs = list(probs)
        if not probs:
            raise ValidationError("distribution size must be >= 1")
        return DistributionSpec(DistributionKind.empirical, len(probs), 0.0, probs)


def materialize(spec: DistributionSpec) -> EmbeddingDistribution:
    """materialize (core/src/distribution_spec.cpp:195-203)."""
    if spec.size == 0:
        raise ValidationError("distribution size must be >= 1")
    if spec.kind == DistributionKind.empirical:
        return EmbeddingDistribution.from_probabilities(spec.probs)
    h = C.c_void_p()
    check(N.lib().ec_dist_materialize(int(spec.kind), spec.size, spec.shape, C.byref(h)))
    return EmbeddingDistribution(h.value)


def materialize_extended(spec: DistributionSpec, factor: int) -> EmbeddingDistribution:
    """materialize_extended (core/src/distribution_spec.cpp:215-226)."""
    h = C.c_void_p()
    check(N.lib().ec_dist_materialize_extended(int(spec.kind), spec.size, spec.shape, factor, C.byref(h)))
    return EmbeddingDistribution(h.value)


def scale(spec: DistributionSpec, factor: int) -> DistributionSpec:
    """scale (core/src/distribution_spec.cpp:205-213)."""
    if spec.kind == DistributionKind.empirical:
        raise ValidationError("scale requires a parametric distribution")
    if factor < 1:
        raise ValidationError("scale factor must be >= 1")
    return DistributionSpec.parametric(spec.kind, spec.size * factor, spec.shape)


# --------------------------------------------------------------- cost model
@dataclass(frozen=True)
class WorkloadSpec:
    """WorkloadSpec (cost_model.hpp:17-25); validates Q >= b >= 1, d >= 1."""
    num_samples: int
    batch_size: int
    lookups_per_sample: int

    def __post_init__(self):
        check(N.lib().ec_workload_validate(C.byref(self._c())))

    def _c(self):
        return N.Workload(self.num_samples, self.batch_size, self.lookups_per_sample)


@dataclass
class CostBreakdown:
    """CostBreakdown (cost_model.hpp:27-32)."""
    index_cost: float = 0.0
    embedding_cost: float = 0.0
    total: float = 0.0
    units_note: str = kCostUnitsNote

    @classmethod
    def _from(cls, c: N.Cost):
        return cls(c.index_cost, c.embedding_cost, c.total)


def batch_presence_prob(p: float, b: int) -> float:
    out = C.c_double()
    check(N.lib().ec_batch_presence_prob(p, b, C.byref(out)))
    return out.value


def expected_unique_per_batch(dist: EmbeddingDistribution, b: int) -> float:
    out = C.c_double()
    check(N.lib().ec_expected_unique_per_batch(dist._h, b, C.byref(out)))
    return out.value


def expected_unique_from_rank(dist: EmbeddingDistribution, b: int, first_rank: int) -> float:
    out = C.c_double()
    check(N.lib().ec_expected_unique_from_rank(dist._h, b, first_rank, C.byref(out)))
    return out.value


def coalesced_batch_cost(dist: EmbeddingDistribution, b: int) -> CostBreakdown:
    out = N.Cost()
    check(N.lib().ec_coalesced_batch_cost(dist._h, b, C.byref(out)))
    return CostBreakdown._from(out)


def baseline_epoch_cost(spec: WorkloadSpec) -> float:
    out = C.c_double()
    check(N.lib().ec_baseline_epoch_cost(C.byref(spec._c()), C.byref(out)))
    return out.value


def coalesced_epoch_cost(dist: EmbeddingDistribution, spec: WorkloadSpec) -> CostBreakdown:
    out = N.Cost()
    check(N.lib().ec_coalesced_epoch_cost(dist._h, C.byref(spec._c()), C.byref(out)))
    return CostBreakdown._from(out)


def cached_epoch_cost(dist: EmbeddingDistribution, spec: WorkloadSpec, cache_ids) -> CostBreakdown:
    c = _u32(cache_ids)
    out = N.Cost()
    check(N.lib().ec_cached_epoch_cost(dist._h, C.byref(spec._c()), c.ctypes.data, c.size, C.byref(out)))
    return CostBreakdown._from(out)


# ------------------------------------------------------------------ planner
@dataclass(frozen=True)
class DeviceModel:
    """DeviceModel (cache_planner.hpp:16-24), parameter-count units."""
    total_params: int
    activation_params_per_sample: int
    embedding_params: int
    memory_efficiency: float = 1.0

    def __post_init__(self):
        check(N.lib().ec_device_model_validate(C.byref(self._c())))

    def _c(self):
        return N.DeviceModelC(self.total_params, self.activation_params_per_sample, self.embedding_params,
                              self.memory_efficiency)


def max_batch_size(device: DeviceModel, cache_size: int) -> Optional[int]:
    out = C.c_int64()
    check(N.lib().ec_max_batch_size(C.byref(device._c()), cache_size, C.byref(out)))
    return None if out.value < 0 else out.value


@dataclass
class MarginalReport:
    candidate_id: int = 0
    presence_gain: float = 0.0
    threshold: float = 0.0
    delta_comm: float = 0.0
    recommend: bool = False


def delta_comm(dist: EmbeddingDistribution, device: DeviceModel, num_samples: int,
               current_cache_size: int) -> MarginalReport:
    out = N.Marginal()
    check(N.lib().ec_delta_comm(dist._h, C.byref(device._c()), num_samples, current_cache_size, C.byref(out)))
    return MarginalReport(out.candidate_id, out.presence_gain, out.threshold, out.delta_comm, bool(out.recommend))


@dataclass
class CachePlan:
    cache_size: int = 0
    cached_ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    batch_size: int = 0
    expected_epoch_cost: CostBreakdown = field(default_factory=CostBreakdown)
    feasible: bool = False
    used_scan_fallback: bool = False


def _plan(fn, dist, device, spec):
    out = N.CachePlanC()
    ids = np.empty(dist.size(), np.uint32)
    check(fn(dist._h, C.byref(device._c()), C.byref(spec._c()), C.byref(out), ids.ctypes.data))
    k = int(out.cache_size) if out.feasible else 0
    return CachePlan(k, ids[:k].copy(), int(out.batch_size), CostBreakdown._from(out.expected_epoch_cost),
                     bool(out.feasible), bool(out.used_scan_fallback))


def optimal_cache_size_scan(dist, device: DeviceModel, spec: WorkloadSpec) -> CachePlan:
    return _plan(N.lib().ec_optimal_cache_size_scan, dist, device, spec)


def optimal_cache_size_search(dist, device: DeviceModel, spec: WorkloadSpec) -> CachePlan:
    return _plan(N.lib().ec_optimal_cache_size_search, dist, device, spec)


def memory_io_proxy(dist, spec: WorkloadSpec, cache_ids) -> float:
    c = _u32(cache_ids)
    out = C.c_double()
    check(N.lib().ec_memory_io_proxy(dist._h, C.byref(spec._c()), c.ctypes.data, c.size, C.byref(out)))
    return out.value


def expected_unique_many(dist: EmbeddingDistribution, batch_sizes, first_ranks=None, device: int = 0) -> np.ndarray:
    """Many expected_unique_from_rank evaluations at once on the GPU (fp64
    terms, device reduction: ~1e-12 relative to the bit-exact host sum)."""
    b = np.ascontiguousarray(batch_sizes, dtype=np.int64)
    f = None if first_ranks is None else np.ascontiguousarray(first_ranks, dtype=np.uint64)
    out = np.empty(b.size, np.float64)
    check(N.lib().ec_expected_unique_many(dist._h, b.ctypes.data, None if f is None else f.ctypes.data, b.size,
                                          device, out.ctypes.data))
    return out


def cost_curve(dist: EmbeddingDistribution, device_model: DeviceModel, num_samples: int, lookups_per_sample: int,
               cache_sizes, device: int = 0):
    """Planner cost of caching each top-k prefix at its Eq. 7 batch size
    (cache_planner.cpp:24-53), all k on the GPU.  Returns (list of
    CostBreakdown, batch sizes; -1 where no batch fits)."""
    ks = np.ascontiguousarray(cache_sizes, dtype=np.int64)
    out = (N.Cost * ks.size)()
    bs = np.empty(ks.size, np.int64)
    w = N.Workload(num_samples, 1, lookups_per_sample)
    check(N.lib().ec_cost_curve(dist._h, C.byref(device_model._c()), C.byref(w), ks.ctypes.data, ks.size, device,
                                out, bs.ctypes.data))
    return [CostBreakdown._from(c) for c in out], bs


def place_topk_global(dists: Sequence[EmbeddingDistribution], budget_rows: int) -> list[int]:
    """Per-table cache sizes for the global top-`budget_rows` rows by probability."""
    arr = (C.c_void_p * len(dists))(*[d._h.value for d in dists])
    k = np.zeros(len(dists), np.uint64)
    check(N.lib().ec_place_topk_global(arr, len(dists), budget_rows, k.ctypes.data))
    return [int(x) for x in k]


# -------------------------------------------------------------- RNG/sampler
MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


class SplitMix64:
    """Generator state holder (core/include/embcomm/rng.hpp:12-27); draws are
    produced on the GPU by sample_batch, which advances ``state``."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


def substream_seed(master: int, index: int) -> int:
    return int(N.lib().ec_substream_seed(master & MASK64, index & MASK64))


class DiscreteSampler:
    """DiscreteSampler (core/include/embcomm/simulator.hpp:18-27) on the GPU."""

    def __init__(self, dist: EmbeddingDistribution, device: int = 0):
        self.dist = dist
        self.device = device
        if device not in dist._sampler:
            h = C.c_void_p()
            check(N.lib().ec_sampler_create(dist._h, device, C.byref(h)))
            dist._sampler[device] = h
        self._h = dist._sampler[device]

    def sample_into(self, ids_dev_ptr: int, seed: int, start: int, count: int, stream: int = 0):
        """Device ids[i] = draw #(start+i) of SplitMix64(seed)."""
        check(N.lib().ec_sample_stream(self._h, seed & MASK64, start, count, ids_dev_ptr, stream))


def sample_batch(dist: EmbeddingDistribution, batch_size: int, lookups_per_sample: int,
                 rng: SplitMix64, device: int = 0) -> np.ndarray:
    """sample_batch (core/src/simulator.cpp:132-143)."""
    if batch_size < 1:
        raise ValidationError("batch size must be >= 1")
    if lookups_per_sample < 1:
        raise ValidationError("lookups per sample must be >= 1")
    s = DiscreteSampler(dist, device)
    out = np.empty(batch_size * lookups_per_sample, np.uint32)
    st = C.c_uint64(rng.state)
    check(N.lib().ec_sample_batch(s._h, batch_size, lookups_per_sample, C.byref(st), out.ctypes.data))
    rng.state = st.value
    return out


# ---------------------------------------------------------------- simulator
@dataclass
class Stat:
    mean: float = 0.0
    std_error: float = 0.0


@dataclass
class SimResult:
    """SimResult (core/include/embcomm/simulator.hpp:34-48)."""
    unique_per_batch: Stat = field(default_factory=Stat)
    non_cached_unique: Stat = field(default_factory=Stat)
    measured_epoch_cost: CostBreakdown = field(default_factory=CostBreakdown)
    hot_batch_fraction: float = 0.0
    portion_usage: list = field(default_factory=list)

    @classmethod
    def _from(cls, r: N.SimResultC):
        return cls(Stat(r.unique_mean, r.unique_std_error), Stat(r.non_cached_mean, r.non_cached_std_error),
                   CostBreakdown._from(r.measured_epoch_cost), r.hot_batch_fraction)


def measure_unique(dist: EmbeddingDistribution, batch_size: int, trials: int, seed: int,
                   device: int = 0) -> SimResult:
    """measure_unique (core/src/simulator.cpp:145-167), counted on the GPU."""
    s = DiscreteSampler(dist, device)
    out = N.SimResultC()
    check(N.lib().ec_measure_unique(s._h, batch_size, trials, seed & MASK64, C.byref(out)))
    return SimResult._from(out)


@dataclass
class Trace:
    """Trace (core/include/embcomm/trace.hpp:18-30): row-major Q x d ids."""
    num_features: int = 0
    vocab_size: int = 0
    ids: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def num_samples(self) -> int:
        return len(self.ids) // self.num_features if self.num_features > 0 else 0

    def sample(self, i: int) -> np.ndarray:
        d = self.num_features
        return np.asarray(self.ids)[i * d:(i + 1) * d]

    def save_binary(self, path) -> None:
        """Write the binary trace container (ec_trace_save_binary; SURVEY §8f
        row 4): the reference's Trace without text parsing."""
        ids = _u32(self.ids)
        check(N.lib().ec_trace_save_binary(os.fsencode(path), ids.ctypes.data, self.num_samples(),
                                           self.num_features, self.vocab_size))

    @staticmethod
    def load_binary(path) -> "BinaryTrace":
        """Map a binary trace (validated like parse_trace); .trace() views it
        as a Trace without copying."""
        return BinaryTrace(path)


def copy_async(dst, src, stream=None, pull_ctas: int = 0) -> None:
    """dst.copy_(src, non_blocking=True) for contiguous same-size tensors (pinned
    host <-> device) through one ec_copy_async call: an input pipeline's copy
    without the framework dispatch cost.  pull_ctas > 0: pinned host -> device
    pulled by that many CTAs (ec_copy_async_pull) -- for inputs sharing the
    host link with a pinned-host cold tier."""
    import torch
    nbytes = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() != nbytes or not (dst.is_contiguous() and src.is_contiguous()):
        raise ValidationError("copy_async needs contiguous tensors of equal byte size")
    s = stream if stream is not None else torch.cuda.current_stream()
    if pull_ctas > 0:
        check(N.lib().ec_copy_async_pull(dst.data_ptr(), src.data_ptr(), nbytes, int(pull_ctas), s.cuda_stream))
    else:
        check(N.lib().ec_copy_async(dst.data_ptr(), src.data_ptr(), nbytes, s.cuda_stream))


class BinaryTrace:
    """A mapped binary trace file (ec_trace_open_binary)."""

    def __init__(self, path):
        h = C.c_void_p()
        check(N.lib().ec_trace_open_binary(os.fsencode(path), C.byref(h)))
        self._h = h
        q, d, e = C.c_uint64(), C.c_int64(), C.c_uint64()
        check(N.lib().ec_trace_info(self._h, C.byref(q), C.byref(d), C.byref(e)))
        self.num_samples, self.num_features, self.vocab_size = int(q.value), int(d.value), int(e.value)
        p = C.c_void_p()
        check(N.lib().ec_trace_ids(self._h, C.byref(p)))
        n = self.num_samples * self.num_features
        buf = (C.c_uint32 * n).from_address(p.value)
        buf._owner = self  # views of the mapping keep the mapping alive
        self._ids = np.frombuffer(buf, dtype=np.uint32)
        self._ids.flags.writeable = False

    def trace(self) -> Trace:
        """Zero-copy read-only view of the mapped ids (the view keeps the
        mapping alive)."""
        return Trace(self.num_features, self.vocab_size, self._ids)

    def upload(self, out, first: int = 0, count: Optional[int] = None) -> None:
        """Samples [first, first+count) into a CUDA int32/uint32 tensor
        (count*d ids, sample-major) via pinned double-buffered staging."""
        import torch
        count = self.num_samples - first if count is None else count
        check(N.lib().ec_trace_upload(self._h, first, count, out.data_ptr(),
                                      torch.cuda.current_stream(out.device).cuda_stream))

    def close(self) -> None:
        """Unmap now; only safe when no view from trace() is still in use."""
        if self._h:
            self._ids = None
            N.lib().ec_trace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def simulate_epoch(source, *args, device: int = 0) -> SimResult:
    """simulate_epoch — both reference overloads (core/src/simulator.cpp:169-273):

    * ``simulate_epoch(dist, spec, cache_ids, epochs, seed)``
    * ``simulate_epoch(trace, batch_size, cache_ids)``
    """
    out = N.SimResultC()
    if isinstance(source, Trace):
        batch_size, cache_ids = args
        ids = _u32(source.ids)
        c = _u32(cache_ids)
        check(N.lib().ec_simulate_trace(ids.ctypes.data, source.num_samples(), source.num_features,
                                        source.vocab_size, batch_size, c.ctypes.data, c.size, device, C.byref(out)))
        return SimResult._from(out)
    spec, cache_ids, epochs, seed = args
    s = DiscreteSampler(source, device)
    c = _u32(cache_ids)
    check(N.lib().ec_simulate_epoch(s._h, C.byref(spec._c()), c.ctypes.data, c.size, epochs, seed & MASK64,
                                    C.byref(out)))
    return SimResult._from(out)


@dataclass
class SampleClasses:
    hot: list
    normal: list


@dataclass
class BatchSchedule:
    hot_batches: list
    normal_batches: list
    batch_size: int


def classify_samples(trace: Trace, cache_ids, device: int = 0) -> SampleClasses:
    """classify_samples (core/src/trace.cpp:185-204) on the GPU."""
    ids = _u32(trace.ids)
    c = _u32(cache_ids)
    q = trace.num_samples()
    hot = np.zeros(q, np.uint8)
    check(N.lib().ec_classify_samples(ids.ctypes.data, q, trace.num_features, trace.vocab_size, c.ctypes.data,
                                      c.size, device, hot.ctypes.data))
    idx = np.arange(q, dtype=np.uint32)
    return SampleClasses(idx[hot == 1].tolist(), idx[hot == 0].tolist())


def build_schedule(trace: Trace, cache_ids, batch_size: int, shuffle_seed: Optional[int] = None,
                   device: int = 0) -> BatchSchedule:
    """build_schedule (core/src/trace.cpp:206-240): stable hot/normal partition
    on the GPU, each class optionally shuffled by the reference's seeded
    Fisher-Yates (trace.cpp:211-222), packed into batches of batch_size."""
    if batch_size < 1:
        raise ValidationError("batch size must be >= 1")
    ids = _u32(trace.ids)
    c = _u32(cache_ids)
    q = trace.num_samples()
    order = np.zeros(q, np.uint32)
    nh = C.c_uint64()
    check(N.lib().ec_build_schedule(ids.ctypes.data, q, trace.num_features, trace.vocab_size, c.ctypes.data,
                                    c.size, device, 0 if shuffle_seed is None else 1,
                                    C.c_uint64(0 if shuffle_seed is None else shuffle_seed),
                                    order.ctypes.data, C.byref(nh)))
    h = int(nh.value)

    def pack(v):
        return [v[i:i + batch_size].tolist() for i in range(0, len(v), batch_size)]
    return BatchSchedule(pack(order[:h]), pack(order[h:]), batch_size)


@dataclass
class SkewTable:
    """SkewTable (core/include/embcomm/trace.hpp:39-51): observed ids ranked by
    (count desc, id asc) with the running share of all accesses."""
    ids: np.ndarray
    counts: np.ndarray
    cum_fraction: np.ndarray
    total_accesses: int

    @property
    def entries(self):
        return list(zip(self.ids.tolist(), self.counts.tolist(), self.cum_fraction.tolist()))


def build_skew_table(trace: Trace, device: int = 0) -> SkewTable:
    """build_skew_table (core/src/trace.cpp:128-150); histogram on the GPU."""
    ids = _u32(trace.ids)
    cap = max(1, min(ids.size, trace.vocab_size))
    oid = np.empty(cap, np.uint32)
    cnt = np.empty(cap, np.uint64)
    cum = np.empty(cap, np.float64)
    n = C.c_uint64()
    check(N.lib().ec_build_skew_table(ids.ctypes.data, ids.size, trace.vocab_size, device, oid.ctypes.data,
                                      cnt.ctypes.data, cum.ctypes.data, C.byref(n)))
    k = n.value
    return SkewTable(oid[:k].copy(), cnt[:k].copy(), cum[:k].copy(), int(ids.size))


def estimate_distribution(table: SkewTable, vocab_size: int, smoothing: float = 0.0) -> EmbeddingDistribution:
    """estimate_distribution (core/src/trace.cpp:161-183)."""
    ids = _u32(table.ids)
    cnt = np.ascontiguousarray(table.counts, dtype=np.uint64)
    h = C.c_void_p()
    check(N.lib().ec_estimate_distribution(ids.ctypes.data, cnt.ctypes.data, ids.size, table.total_accesses,
                                           vocab_size, smoothing, C.byref(h)))
    return EmbeddingDistribution(h.value)


from .tables import EmbeddingGroup, EmbeddingTables, exchange_plan, shard_rows  # noqa: E402
