"""ctypes binding of the C ABI in include/sgc_b200.h (libsgc_b200.so, built in-tree).

The product path has no fallback: if the shared library is missing or no sm_100 device is
present, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGC_LIB", os.path.join(HERE, "libsgc_b200.so"))

SGC_OK, SGC_DOMAIN, SGC_CAPACITY, SGC_INTEGRITY, SGC_PARSE, SGC_LOGIC, SGC_CUDA = range(7)
VOCAB = 260


class Error(RuntimeError):
    """subgcache::Error (errors.hpp:9-12)."""


class DomainError(Error, ValueError):
    """errors.hpp:25-27."""


class CapacityError(Error):
    """errors.hpp:30-32."""


class IntegrityError(Error):
    """errors.hpp:20-22."""


class ParseError(Error):
    """errors.hpp:15-18."""


class LogicError(Error):
    """std::logic_error (lm_core.cpp:95, cache_engine.cpp:211)."""


class CudaError(Error):
    """device or runtime failure."""


_EXC = {SGC_DOMAIN: DomainError, SGC_CAPACITY: CapacityError, SGC_INTEGRITY: IntegrityError,
        SGC_PARSE: ParseError, SGC_LOGIC: LogicError, SGC_CUDA: CudaError}


class LmConfig(C.Structure):
    _fields_ = [("layers", C.c_uint32), ("heads", C.c_uint32), ("model_dim", C.c_uint32),
                ("ffn_hidden", C.c_uint32), ("max_seq_len", C.c_uint32),
                ("max_new_tokens", C.c_uint32), ("seed", C.c_uint64)]


class GnnConfig(C.Structure):
    _fields_ = [("layers", C.c_uint32), ("heads", C.c_uint32), ("dim", C.c_uint32),
                ("seed", C.c_uint64), ("text_seed", C.c_uint64), ("text_salt", C.c_uint64)]


class Subgraphs(C.Structure):
    _fields_ = [("count", C.c_uint32), ("node_off", C.POINTER(C.c_uint64)),
                ("nodes", C.POINTER(C.c_uint32)), ("edge_off", C.POINTER(C.c_uint64)),
                ("edges", C.POINTER(C.c_uint32))]


class TokenLists(C.Structure):
    _fields_ = [("count", C.c_uint32), ("off", C.POINTER(C.c_uint64)),
                ("tokens", C.POINTER(C.c_int32))]


class RetrievalConfig(C.Structure):
    _fields_ = [("strategy", C.c_int), ("k", C.c_uint32), ("edge_cost", C.c_double),
                ("ego_hops", C.c_uint32), ("ego_entity_cap", C.c_uint32), ("dim", C.c_uint32),
                ("text_seed", C.c_uint64), ("hash_salt", C.c_uint64)]


class Batch(C.Structure):
    _fields_ = [("retrieved", Subgraphs), ("questions", TokenLists), ("answers", TokenLists),
                ("own_prefix", TokenLists), ("clusters", C.c_uint32), ("linkage", C.c_int),
                ("question_budget", C.c_uint32), ("soft_prefix", C.c_int),
                ("pointer_bonus", C.c_float), ("gnn", GnnConfig),
                ("precomputed_embeddings", C.POINTER(C.c_float)),
                ("cluster_owner", C.POINTER(C.c_uint32)), ("rank", C.c_int),
                ("world_size", C.c_int), ("waves", C.c_uint32), ("max_new_tokens", C.c_uint32),
                ("split_clusters", C.c_int), ("transfer_prefix", C.c_int),
                ("verify_prefix", C.c_int)]


class BatchOut(C.Structure):
    _fields_ = [("embeddings", C.POINTER(C.c_float)), ("labels", C.POINTER(C.c_uint32)),
                ("merge_left", C.POINTER(C.c_uint32)), ("merge_right", C.POINTER(C.c_uint32)),
                ("merge_dist", C.POINTER(C.c_double)), ("prefix_len", C.POINTER(C.c_uint64)),
                ("logits", C.POINTER(C.c_float)), ("first_token", C.POINTER(C.c_int32)),
                ("fallback", C.POINTER(C.c_uint8)), ("owner", C.POINTER(C.c_uint32)),
                ("ttft_ms", C.POINTER(C.c_float)), ("waves", C.c_uint32),
                ("stage_ms", C.c_double * 8),
                ("prefill_rows", C.c_uint64), ("extend_rows", C.c_uint64),
                ("tokens", C.POINTER(C.c_int32)), ("n_tokens", C.POINTER(C.c_uint32)),
                ("rt_ms", C.POINTER(C.c_float)), ("decode_rows", C.c_uint64),
                ("seal_ms", C.POINTER(C.c_float)), ("pftt_ms", C.POINTER(C.c_float)),
                ("query_rank", C.POINTER(C.c_uint32)), ("prefilled", C.POINTER(C.c_uint8)),
                ("prefix_bytes_sent", C.c_uint64), ("prefix_bytes_received", C.c_uint64),
                ("prefix_digest", C.POINTER(C.c_uint64)), ("kv_pages_peak", C.c_uint64),
                ("kv_page_bytes", C.c_uint64), ("ttft_dequeue_ms", C.POINTER(C.c_float))]


# sgc_host_transport callbacks (include/sgc_b200.h)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                          C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                          C.POINTER(C.c_int))


class HostTransport(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allgather", ALLGATHER_FN), ("exchange", EXCHANGE_FN)]


def make_host_transport(t):
    """sgc_host_transport whose callbacks call t.allgather / t.exchange (see host.Context);
    returns (struct, callbacks) -- keep both alive while the context uses them."""

    def _allgather(user, send, recv, nbytes):
        try:
            out = t.allgather(C.string_at(send, nbytes), nbytes)
            C.memmove(recv, out, len(out))
            return 0
        except Exception as e:  # noqa: BLE001 -- reported as a status to the C side
            print("host transport allgather failed:", e)
            return 1

    def _exchange(user, ns, sbuf, sbytes, speer, nr, rbuf, rbytes, rpeer):
        try:
            sends = [(C.string_at(sbuf[i], sbytes[i]), speer[i]) for i in range(ns)]
            recvs = [(rbytes[i], rpeer[i]) for i in range(nr)]
            got = t.exchange(sends, recvs)
            for i in range(nr):
                C.memmove(rbuf[i], got[i], rbytes[i])
            return 0
        except Exception as e:  # noqa: BLE001
            print("host transport exchange failed:", e)
            return 1

    cbs = (ALLGATHER_FN(_allgather), EXCHANGE_FN(_exchange))
    return HostTransport(None, cbs[0], cbs[1]), cbs


# every symbol include/sgc_b200.h declares (checked by tests/test_boundary.py)
EXPORTS = [
    "sgc_last_error", "sgc_version", "sgc_ctx_create", "sgc_ctx_destroy", "sgc_ctx_set_stream",
    "sgc_ctx_launch_count", "sgc_model_create", "sgc_model_destroy", "sgc_model_weight",
    "sgc_graph_upload", "sgc_graph_destroy", "sgc_encode_subgraphs", "sgc_text_features",
    "sgc_pairwise_distances", "sgc_agglomerate", "sgc_build_representatives", "sgc_prefill",
    "sgc_kv_release", "sgc_kv_count", "sgc_kv_tokens", "sgc_kv_digest", "sgc_kv_resident_bytes",
    "sgc_kv_read", "sgc_extend", "sgc_run_subgcache", "sgc_gemm_bf16", "sgc_set_timing",
    "sgc_get_timing", "sgc_lpt_assign", "sgc_set_option", "sgc_attention_bf16", "sgc_extend_generate", "sgc_retrieve", "sgc_balance_members",
    "sgc_kv_pages", "sgc_probe_fp64_tflops", "sgc_gnn_stats", "sgc_kv_fork", "sgc_fork_fork", "sgc_fork_extend", "sgc_fork_tokens",
    "sgc_fork_prefix_tokens", "sgc_fork_last_logits", "sgc_fork_truncate", "sgc_fork_release_suffix",
    "sgc_fork_destroy", "sgc_comm_unique_id", "sgc_comm_init_nccl", "sgc_comm_init_host", "sgc_comm_destroy", "sgc_comm_info",
]

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    P, vp = C.POINTER, C.c_void_p
    L.sgc_last_error.restype = C.c_char_p
    L.sgc_version.restype = C.c_char_p
    L.sgc_ctx_create.argtypes = [C.c_int, P(vp)]
    L.sgc_ctx_destroy.argtypes = [vp]
    L.sgc_ctx_set_stream.argtypes = [vp, vp]
    L.sgc_ctx_launch_count.argtypes = [vp]
    L.sgc_ctx_launch_count.restype = C.c_uint64
    L.sgc_model_create.argtypes = [vp, P(LmConfig), P(vp)]
    L.sgc_model_destroy.argtypes = [vp]
    L.sgc_model_weight.argtypes = [vp, C.c_int, C.c_uint32, C.c_int, P(C.c_float), C.c_size_t]
    L.sgc_graph_upload.argtypes = [vp, C.c_uint32, P(C.c_uint32), C.c_char_p, P(C.c_uint64),
                                   C.c_uint32, P(C.c_uint32), P(C.c_uint32), C.c_char_p,
                                   P(C.c_uint64), P(vp)]
    L.sgc_graph_destroy.argtypes = [vp]
    L.sgc_encode_subgraphs.argtypes = [vp, vp, P(GnnConfig), P(Subgraphs), P(C.c_float)]
    L.sgc_text_features.argtypes = [vp, vp, C.c_uint32, C.c_uint64, C.c_uint64, P(C.c_float)]
    L.sgc_pairwise_distances.argtypes = [vp, P(C.c_float), C.c_uint32, C.c_uint32, P(C.c_double)]
    L.sgc_agglomerate.argtypes = [vp, P(C.c_float), C.c_uint32, C.c_uint32, C.c_int, C.c_uint32,
                                  P(C.c_uint32), P(C.c_uint32), P(C.c_uint32), P(C.c_double),
                                  P(C.c_uint64)]
    L.sgc_build_representatives.argtypes = [vp, vp, P(Subgraphs), P(C.c_uint32), C.c_uint32,
                                            C.c_uint32, P(C.c_uint64), P(C.c_uint32), C.c_uint64,
                                            P(C.c_uint64), P(C.c_uint32), C.c_uint64,
                                            P(C.c_uint64), P(C.c_int32), C.c_uint64,
                                            P(C.c_uint32)]
    L.sgc_prefill.argtypes = [vp, vp, P(TokenLists), P(C.c_float), P(C.c_uint8), P(vp),
                              P(C.c_float)]
    L.sgc_kv_release.argtypes = [vp]
    L.sgc_kv_count.argtypes = [vp]
    L.sgc_kv_count.restype = C.c_uint32
    L.sgc_kv_tokens.argtypes = [vp, C.c_uint32]
    L.sgc_kv_tokens.restype = C.c_uint64
    L.sgc_kv_digest.argtypes = [vp, C.c_uint32]
    L.sgc_kv_digest.restype = C.c_uint64
    L.sgc_kv_resident_bytes.argtypes = [vp]
    L.sgc_kv_resident_bytes.restype = C.c_uint64
    L.sgc_kv_read.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_int, P(C.c_float)]
    L.sgc_kv_pages.argtypes = [vp, C.c_uint32, P(C.c_int32)]
    L.sgc_kv_pages.restype = C.c_uint32
    L.sgc_kv_fork.argtypes = [vp, C.c_uint32, P(vp)]
    L.sgc_probe_fp64_tflops.argtypes = [vp, P(C.c_double)]
    L.sgc_gnn_stats.argtypes = [vp, P(C.c_uint64), P(C.c_uint64)]
    L.sgc_fork_fork.argtypes = [vp, P(vp)]
    L.sgc_fork_extend.argtypes = [vp, vp, P(vp), C.c_uint32, P(TokenLists), P(C.c_float)]
    L.sgc_fork_tokens.argtypes = [vp]
    L.sgc_fork_tokens.restype = C.c_uint64
    L.sgc_fork_prefix_tokens.argtypes = [vp]
    L.sgc_fork_prefix_tokens.restype = C.c_uint64
    L.sgc_fork_last_logits.argtypes = [vp, P(C.c_float)]
    L.sgc_fork_truncate.argtypes = [vp, C.c_uint64]
    L.sgc_fork_release_suffix.argtypes = [vp]
    L.sgc_fork_destroy.argtypes = [vp]
    L.sgc_extend.argtypes = [vp, vp, vp, P(C.c_uint32), P(TokenLists), P(TokenLists), C.c_float,
                             P(C.c_float), P(C.c_int32)]
    L.sgc_run_subgcache.argtypes = [vp, vp, vp, P(Batch), P(BatchOut)]
    L.sgc_gemm_bf16.argtypes = [vp, vp, vp, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
    L.sgc_set_timing.argtypes = [vp, C.c_int]
    L.sgc_retrieve.argtypes = [vp, vp, P(RetrievalConfig), C.c_uint32, C.c_char_p, P(C.c_uint64),
                               P(C.c_uint64), P(C.c_uint32), C.c_uint64, P(C.c_uint64), P(C.c_uint32),
                               C.c_uint64]
    L.sgc_extend_generate.argtypes = [vp, vp, vp, P(C.c_uint32), P(TokenLists), P(TokenLists), C.c_float,
                                      C.c_uint32, P(C.c_float), P(C.c_int32), P(C.c_int32), P(C.c_uint32)]
    L.sgc_attention_bf16.argtypes = [vp, vp, vp, vp, C.c_uint32, vp, vp, vp, P(C.c_int32), C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.c_uint32, vp]
    L.sgc_get_timing.argtypes = [vp, C.c_char_p, P(C.c_double), P(C.c_uint64)]
    L.sgc_set_option.argtypes = [vp, C.c_char_p, C.c_int64]
    L.sgc_lpt_assign.argtypes = [P(C.c_double), C.c_uint32, C.c_int, P(C.c_uint32)]
    L.sgc_balance_members.argtypes = [P(C.c_double), C.c_uint32, P(C.c_uint32), P(C.c_double), C.c_uint32,
                                      C.c_int, P(C.c_uint32), P(C.c_uint32)]
    L.sgc_comm_unique_id.argtypes = [P(C.c_uint8)]
    L.sgc_comm_init_nccl.argtypes = [vp, P(C.c_uint8), C.c_int, C.c_int]
    L.sgc_comm_init_host.argtypes = [vp, P(HostTransport), C.c_int, C.c_int]
    L.sgc_comm_destroy.argtypes = [vp]
    L.sgc_comm_info.argtypes = [vp, P(C.c_int), P(C.c_int), P(C.c_int)]
    _lib = L
    return L


def check(status: int) -> None:
    if status != SGC_OK:
        msg = load().sgc_last_error().decode(errors="replace")
        raise _EXC.get(status, Error)(msg)
