"""ctypes binding of libembcomm_gpu.so (include/embcomm_gpu.h).

Loading fails loudly when the library is missing: there is no Python or CPU
fallback for any entry point.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("EC_LIB_NAME", "libembcomm_gpu.so"))  # (A/B builds)

EC_OK, EC_EINVAL, EC_EINVARIANT, EC_ECUDA, EC_ENCCL, EC_ENOMEM = 0, 2, 3, 4, 5, 6


class EmbcommError(RuntimeError):
    code = -1


class ValidationError(EmbcommError, ValueError):
    """embcomm::ValidationError (core/include/embcomm/error.hpp:10-13)."""
    code = EC_EINVAL


class InvariantError(EmbcommError):
    """embcomm::InvariantError (core/include/embcomm/error.hpp:16-19)."""
    code = EC_EINVARIANT


class CudaError(EmbcommError):
    code = EC_ECUDA


class NcclError(EmbcommError):
    code = EC_ENCCL


class OutOfMemoryError(EmbcommError, MemoryError):
    code = EC_ENOMEM


_ERR = {EC_EINVAL: ValidationError, EC_EINVARIANT: InvariantError, EC_ECUDA: CudaError,
        EC_ENCCL: NcclError, EC_ENOMEM: OutOfMemoryError}


class Workload(C.Structure):
    _fields_ = [("num_samples", C.c_int64), ("batch_size", C.c_int64), ("lookups_per_sample", C.c_int64)]


class Cost(C.Structure):
    _fields_ = [("index_cost", C.c_double), ("embedding_cost", C.c_double), ("total", C.c_double)]


class DeviceModelC(C.Structure):
    _fields_ = [("total_params", C.c_int64), ("activation_params_per_sample", C.c_int64),
                ("embedding_params", C.c_int64), ("memory_efficiency", C.c_double)]


class Marginal(C.Structure):
    _fields_ = [("candidate_id", C.c_uint32), ("presence_gain", C.c_double), ("threshold", C.c_double),
                ("delta_comm", C.c_double), ("recommend", C.c_int32)]


class CachePlanC(C.Structure):
    _fields_ = [("cache_size", C.c_uint64), ("batch_size", C.c_int64), ("expected_epoch_cost", Cost),
                ("feasible", C.c_int32), ("used_scan_fallback", C.c_int32)]


class SimResultC(C.Structure):
    _fields_ = [("unique_mean", C.c_double), ("unique_std_error", C.c_double),
                ("non_cached_mean", C.c_double), ("non_cached_std_error", C.c_double),
                ("measured_epoch_cost", Cost), ("hot_batch_fraction", C.c_double)]


class TablesConfig(C.Structure):
    _fields_ = [("num_tables", C.c_uint32), ("dim", C.c_uint32), ("rows_host", C.POINTER(C.c_uint64)),
                ("storage", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32),
                ("max_lookups_per_table", C.c_uint64), ("max_batch_size", C.c_uint32), ("device", C.c_int32)]


class Batch(C.Structure):
    _fields_ = [("indices_dev", C.c_void_p), ("table_offsets_host", C.POINTER(C.c_int64)),
                ("bag_offsets_dev", C.c_void_p), ("batch_size", C.c_uint32), ("pooling", C.c_uint32)]


class BatchStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("lookups", "unique_rows", "hit_rows", "miss_rows", "index_units",
                                          "model_bytes", "wire_rows", "wire_bytes", "hot_tables",
                                          "hot_sync_rows", "hot_sync_bytes")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


vp, u64, i64, u32, i32, f64, f32 = (C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32, C.c_int32,
                                    C.c_double, C.c_float)
P = C.POINTER

# name -> argtypes (every function returns int status unless listed in _RESTYPE)
_SIGS = {
    "ec_last_error": [], "ec_version": [], "ec_cost_units_note": [], "ec_rng_algorithm": [],
    "ec_substream_seed": [u64, u64],
    "ec_dist_from_probabilities": [vp, u64, P(vp)],
    "ec_dist_uniform": [u64, P(vp)],
    "ec_dist_materialize": [C.c_int, u64, f64, P(vp)],
    "ec_dist_materialize_extended": [C.c_int, u64, f64, i64, P(vp)],
    "ec_default_shape": [C.c_int, P(f64)],
    "ec_dist_destroy": [vp],
    "ec_dist_size": [vp],
    "ec_dist_prob": [vp, u32, P(f64)],
    "ec_dist_prob_at_rank": [vp, u64, P(f64)],
    "ec_dist_id_at_rank": [vp, u64, P(u32)],
    "ec_dist_rank_of": [vp, u32, P(u64)],
    "ec_dist_top_ids": [vp, u64, vp],
    "ec_dist_mass_of": [vp, vp, u64, P(f64)],
    "ec_dist_export": [vp, vp, vp],
    "ec_workload_validate": [P(Workload)],
    "ec_batch_presence_prob": [f64, i64, P(f64)],
    "ec_expected_unique_per_batch": [vp, i64, P(f64)],
    "ec_expected_unique_from_rank": [vp, i64, u64, P(f64)],
    "ec_coalesced_batch_cost": [vp, i64, P(Cost)],
    "ec_baseline_epoch_cost": [P(Workload), P(f64)],
    "ec_coalesced_epoch_cost": [vp, P(Workload), P(Cost)],
    "ec_cached_epoch_cost": [vp, P(Workload), vp, u64, P(Cost)],
    "ec_device_model_validate": [P(DeviceModelC)],
    "ec_max_batch_size": [P(DeviceModelC), i64, P(i64)],
    "ec_delta_comm": [vp, P(DeviceModelC), i64, i64, P(Marginal)],
    "ec_optimal_cache_size_scan": [vp, P(DeviceModelC), P(Workload), P(CachePlanC), vp],
    "ec_optimal_cache_size_search": [vp, P(DeviceModelC), P(Workload), P(CachePlanC), vp],
    "ec_memory_io_proxy": [vp, P(Workload), vp, u64, P(f64)],
    "ec_place_topk_global": [vp, u32, u64, vp],
    "ec_expected_unique_many": [vp, vp, vp, u64, C.c_int, vp],
    "ec_cost_curve": [vp, P(DeviceModelC), P(Workload), vp, u64, C.c_int, vp, vp],
    "ec_sampler_create": [vp, C.c_int, P(vp)],
    "ec_sampler_destroy": [vp],
    "ec_sample_stream": [vp, u64, u64, u64, vp, vp],
    "ec_sample_batch": [vp, i64, i64, P(u64), vp],
    "ec_measure_unique": [vp, i64, i64, u64, P(SimResultC)],
    "ec_simulate_epoch": [vp, P(Workload), vp, u64, i64, u64, P(SimResultC)],
    "ec_simulate_trace": [vp, u64, i64, u64, i64, vp, u64, C.c_int, P(SimResultC)],
    "ec_classify_samples": [vp, u64, i64, u64, vp, u64, C.c_int, vp],
    "ec_schedule_order": [vp, u64, i64, u64, vp, u64, C.c_int, vp, P(u64)],
    "ec_build_schedule": [vp, u64, i64, u64, vp, u64, C.c_int, C.c_int, u64, vp, P(u64)],
    "ec_build_skew_table": [vp, u64, u64, C.c_int, vp, vp, vp, P(u64)],
    "ec_estimate_distribution": [vp, vp, u64, u64, u64, f64, P(vp)],
    "ec_tables_create": [P(TablesConfig), P(vp)],
    "ec_tables_destroy": [vp],
    "ec_tables_memory": [vp, P(u64), P(u64)],
    "ec_tables_profile": [vp, C.c_int],
    "ec_tables_use_graphs": [vp, C.c_int],
    "ec_tables_dedup_mode": [vp, C.c_int],
    "ec_tables_scatter_mode": [vp, C.c_int],
    "ec_tables_profile_read": [vp, vp, vp, P(u64), C.c_int],
    "ec_tables_profile_timeline": [vp, vp, u64, P(u64)],
    "ec_tables_init_synthetic": [vp, u64, f32, vp],
    "ec_tables_place_cache": [vp, vp, vp],
    "ec_tables_read_rows": [vp, u32, vp, u64, vp],
    "ec_tables_write_rows": [vp, u32, vp, u64, vp],
    "ec_lookup_fwd": [vp, P(Batch), vp, vp],
    "ec_lookup_bwd": [vp, vp, f32, vp],
    "ec_lookup_prefetch": [vp, P(Batch), vp],
    "ec_lookup_prefetch_wait": [vp, vp],
    "ec_lookup_prefetch_drop": [vp, vp],
    "ec_trace_save_binary": [C.c_char_p, vp, u64, i64, u64],
    "ec_trace_open_binary": [C.c_char_p, P(vp)],
    "ec_trace_destroy": [vp],
    "ec_trace_info": [vp, P(u64), P(i64), P(u64)],
    "ec_trace_ids": [vp, P(vp)],
    "ec_trace_upload": [vp, u64, u64, vp, vp],
    "ec_copy_async": [vp, vp, u64, vp],
    "ec_copy_async_pull": [vp, vp, u64, C.c_int, vp],
    "ec_tables_schedule": [vp, vp, u64, vp, P(u64), vp],
    "ec_tables_gather_batch": [vp, vp, vp, u64, u32, vp, vp],
    "ec_lookup_stats": [vp, vp, P(BatchStats), vp, vp],
    "ec_lookup_stats_enqueue": [vp, vp, i32],
    "ec_lookup_stats_collect": [vp, i32, P(BatchStats), vp, vp],
    "ec_export_unique": [vp, u32, vp, u64, P(u64)],
    "ec_export_inverse": [vp, u32, vp],
    "ec_export_hit": [vp, u32, vp],
    "ec_export_rows": [vp, u32, vp],
    "ec_comm_unique_id": [vp],
    "ec_tables_attach_comm": [vp, vp],
    "ec_shard_rows": [vp, u32, C.c_int, C.c_int, vp],
    "ec_exchange_plan": [vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp],
    "ec_group_create": [vp, C.c_int, P(vp)],
    "ec_group_destroy": [vp],
    "ec_group_lookup_fwd": [vp, P(Batch), vp, vp],
    "ec_group_lookup_bwd": [vp, vp, f32, vp],
    "ec_group_set_p2p": [vp, C.c_int],
    "ec_tables_p2p_export": [vp, vp, u64, P(u64)],
    "ec_tables_p2p_import": [vp, vp, u64],
    "ec_tables_p2p_disable": [vp],
}
_RESTYPE = {
    "ec_last_error": C.c_char_p, "ec_version": C.c_char_p, "ec_cost_units_note": C.c_char_p,
    "ec_rng_algorithm": C.c_char_p, "ec_substream_seed": u64, "ec_dist_size": u64,
    "ec_dist_destroy": None, "ec_sampler_destroy": None, "ec_tables_destroy": None, "ec_group_destroy": None,
    "ec_trace_destroy": None,
}

_lib = None


def lib():
    """The loaded library; raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "or `make -C paper_2411_01611_b200/csrc`")
        L = C.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, C.c_int)
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(rc: int) -> None:
    if rc != EC_OK:
        msg = lib().ec_last_error().decode(errors="replace")
        raise _ERR.get(rc, EmbcommError)(msg)
