"""ctypes binding of libpqg.so (include/pqg.h).

Loading fails loudly: there is no CPU fallback anywhere in the package.  The
library is built in-tree (``paper_2604_21645_b200/libpqg.so``) by
``__graft_entry__.build()`` / ``make -C paper_2604_21645_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpqg.so")

PQG_OK = 0
PQG_EINVAL = -1
PQG_ERANGE = -2
PQG_ECUDA = -3
PQG_ENOMEM = -4
PQG_EUNSUPPORTED = -5
PQG_ECHUNK = -6  # a pipeline chunk task failed (std::runtime_error)
PQG_EIO = -7  # file / format error (std::runtime_error, the reference's message)

_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_i32 = C.c_int
_f64 = C.c_double

# name -> (restype, argtypes); every data pointer is a void* (host or device)
_SIGS = {
    "pqg_ctx_create": (_i32, [_i32, C.POINTER(_vp)]),
    "pqg_ctx_destroy": (None, [_vp]),
    "pqg_ctx_set_stream": (_i32, [_vp, _vp]),
    "pqg_ctx_sync": (_i32, [_vp]),
    "pqg_ctx_stream": (_vp, [_vp]),
    "pqg_ctx_check_errors": (_i32, [_vp]),
    "pqg_last_error": (C.c_char_p, []),
    "pqg_ctx_launches": (_u64, [_vp]),
    "pqg_profile_enable": (_i32, [_vp, _i32]),
    "pqg_profile_read": (_i32, [_vp, C.c_char_p, C.POINTER(_u64), C.POINTER(_f64)]),
    "pqg_version": (C.c_char_p, []),
    "pqg_fp32_probe": (_i32, [_vp, C.POINTER(_f64)]),
    "pqg_nearest_batch": (_i32, [_vp, _vp, _u64, _u64, _vp, _u64, _vp, _vp]),
    "pqg_kmeans_fit": (_i32, [_vp, _vp, _u64, _u64, _u64, _u32, _u64, _f64, _vp, _vp,
                              C.POINTER(_f64), C.POINTER(_u32), _vp]),
    "pqg_pq_fit": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _u64, _vp, _vp, _vp]),
    "pqg_pq_fit_ex": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _u64, _vp, _vp, _vp, _vp]),
    "pqg_pq_encode": (_i32, [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp]),
    "pqg_pq_decode": (_i32, [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp]),
    "pqg_sq_error": (_i32, [_vp, _vp, _vp, _u64, _vp]),
    "pqg_pq_recon_sse": (_i32, [_vp, _vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp]),
    "pqg_pq_encode_sse": (_i32, [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp, _vp]),
    "pqg_adc_tables": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _u64, _vp]),
    "pqg_adc_lookup": (_i32, [_vp, _vp, _u32, _u32, _vp, _u64, _vp]),
    "pqg_ivf_assign": (_i32, [_vp, _vp, _u64, _u32, _u32, _u32, _vp, _vp, _u64, _vp]),
    "pqg_ivf_build_with_centroids": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _vp, _u64, _vp,
                                            _u64, C.POINTER(_vp)]),
    "pqg_ivf_build": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _vp, _u64, _u64, _u64, _u32,
                             C.POINTER(_vp)]),
    "pqg_index_create": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _u64, _vp, _vp, _vp,
                                C.POINTER(_vp)]),
    "pqg_index_destroy": (None, [_vp]),
    "pqg_index_info": (_i32, [_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32),
                              C.POINTER(_u32), C.POINTER(_u32)]),
    "pqg_index_export": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pqg_index_add": (_i32, [_vp, _vp, _vp, _vp, _u64]),
    "pqg_index_merge": (_i32, [_vp, _vp, _vp, C.POINTER(_vp)]),
    "pqg_index_search": (_i32, [_vp, _vp, _vp, _u64, _u64, _u64, _i32, _f64, _vp, _vp, _vp]),
    "pqg_index_search_ex": (_i32, [_vp, _vp, _vp, _u64, _u64, _u64, _i32, _f64, _vp, _vp, _vp, _vp]),
    "pqg_index_probe": (_i32, [_vp, _vp, _vp, _u64, _u64, _vp]),
    "pqg_index_search_subset": (_i32, [_vp, _vp, _vp, _u64, _u64, _vp, _u64, _u64, _i32, _f64, _vp,
                                       _vp, _vp]),
    "pqg_flat_scan": (_i32, [_vp, _vp, _u32, _u32, _u32, _vp, _vp, _u64, _vp, _u64, _u64, _i32,
                             _f64, _vp, _vp, _vp]),
    "pqg_topk_merge": (_i32, [_vp, _vp, _vp, _vp, _u32, _u64, _u64, _vp, _vp, _vp]),
    "pqg_index_serialize": (_i32, [_vp, _vp, _vp, _u64, C.POINTER(_u64)]),
    "pqg_index_deserialize": (_i32, [_vp, _vp, _u64, C.c_char_p, C.POINTER(_vp)]),
    "pqg_index_save": (_i32, [_vp, _vp, C.c_char_p]),
    "pqg_index_load": (_i32, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "pqg_codes_save": (_i32, [_vp, _vp, _u64, _u32, _u32, C.c_char_p]),
    "pqg_codes_file_info": (_i32, [C.c_char_p, C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_u32)]),
    "pqg_codes_load": (_i32, [_vp, C.c_char_p, _vp, _u64]),
    "pqg_codebook_save": (_i32, [_vp, _vp, _u32, _u32, _u32, C.c_char_p]),
    "pqg_codebook_file_info": (_i32, [C.c_char_p, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32)]),
    "pqg_codebook_load": (_i32, [_vp, C.c_char_p, _vp, _u64]),
    "pqg_assign_pass": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _vp, _u64, _vp, _vp]),
    "pqg_update_pass": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _vp, _u64, _vp, _vp, _vp]),
    "pqg_rows_sum_f64": (_i32, [_vp, _vp, _u64, _u32, _vp]),
    "pqg_kmeans_init_rows": (_i32, [_u64, _u64, _u64, _vp]),
    "pqg_kmshard_create": (_i32, [_vp, _vp, _u64, _u64, _u32, _u32, _u32, _u64, _u32, _f64, C.POINTER(_vp)]),
    "pqg_kmshard_destroy": (None, [_vp]),
    "pqg_kmshard_sizes": (_i32, [_vp, C.POINTER(_u64), C.POINTER(_u64)]),
    "pqg_kmshard_init_table": (_i32, [_vp, _vp, _vp, _u64, _vp]),
    "pqg_kmshard_partials": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "pqg_kmshard_apply": (_i32, [_vp, _vp, _vp, _vp, _vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32),
                                 C.POINTER(_i32)]),
    "pqg_kmshard_pack": (_i32, [_vp, _vp, _vp, _u64, _vp]),
    "pqg_kmshard_replay": (_i32, [_vp, _vp, _vp, _vp, _vp, _u64, _vp, _u32]),
    "pqg_nccl_get_unique_id": (_i32, [_vp]),
    "pqg_nccl_comm_init": (_i32, [C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "pqg_nccl_comm_init_all": (_i32, [C.c_int, _vp, _vp]),
    "pqg_nccl_comm_destroy": (None, [_vp]),
    "pqg_kmeans_fit_sharded": (_i32, [_vp, _vp, _vp, _u64, _u64, _u32, _u32, _u32, _u64, _u32, _vp, _f64, _vp, _vp,
                                      _vp, _vp, _vp, _vp]),
    "pqg_kmshard_replay_step": (_i32, [_vp, _vp, _vp]),
    "pqg_kmshard_replay_finish": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "pqg_kmshard_reseed_candidates": (_i32, [_vp, _vp, _u64, _u32, _vp, _vp, _vp]),
    "pqg_kmshard_reseed_apply": (_i32, [_vp, _vp, _vp, _vp, _u32, _u32, _vp, _vp, _vp]),
    "pqg_kmshard_result": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pqg_train_chunks": (_i32, [_vp, _vp, _u64, _u64, _u64, _u32, _u32, _u32, _u64, _vp, _vp,
                                _vp]),
    "pqg_pipeline_run": (_i32, [_vp, _vp, _u64, _u64, _u64, _u32, _u32, _u64, _u32, _u64, _i32,
                                _vp, C.POINTER(_f64), _vp, _vp, C.POINTER(_u64), C.POINTER(_vp),
                                _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


class PQGError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load libpqg.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (the package has no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Raise the Python analogue of the reference's exception for a status."""
    if rc == PQG_OK:
        return
    msg = load().pqg_last_error().decode(errors="replace")
    if rc == PQG_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == PQG_ERANGE:
        raise IndexError(msg)          # std::out_of_range
    if rc == PQG_EIO:
        raise PQGError(msg)            # the reference's runtime_error (file / format)
    if rc == PQG_ECHUNK:
        raise PQGError(msg)            # run_chunk_tasks' runtime_error("chunk <id>: ...")
    raise PQGError(f"{what}: {msg} (status {rc})")
