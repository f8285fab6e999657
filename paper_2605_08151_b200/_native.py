"""ctypes binding of libspectre.so — the C ABI declared in include/spectre.h.

Loading is strict: if the library is missing the import of any product path
fails with an ImportError naming the build command.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "libspectre.so"
_lib = None


class SpectreError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


class OracleConfig(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("n_requests", C.c_int32),
        ("max_concurrency", C.c_int32),
        ("gamma", C.c_int32),
        ("output_len", C.c_int32),
        ("variant", C.c_int32),
        ("fairness_period", C.c_int32),
        ("has_fixed_l", C.c_int32),
        ("max_rounds", C.c_int32),
        ("alpha", C.c_double),
        ("t_target", C.c_double),
        ("t_draft", C.c_double),
        ("delay", C.c_double),
        ("t_target_slope", C.c_double),
        ("ema_decay", C.c_double),
        ("fixed_threshold_l", C.c_double),
        ("t_draft_slope", C.c_double),
        ("t_draft_init", C.c_double),
        ("t_draft_free_batch", C.c_int32),
        ("reply_timeout", C.c_double),
    ]


_P = C.c_void_p
ORACLE_OUTPUT_FIELDS = (
    "committed", "committed_pos", "admitted_at", "finished_at",
    "round_mode", "round_participants", "round_delta", "round_n_roll",
    "round_content_sum", "round_content_n", "round_queries", "round_draft_tokens",
    "round_n_padded", "round_started", "round_dispatch", "round_commit",
    "round_draft_start", "round_draft_done", "round_r_hat_ema",
    "round_accepted_len_ema", "round_r_star", "scalars",
)


class OracleOutputs(C.Structure):
    _fields_ = [(name, _P) for name in ORACLE_OUTPUT_FIELDS]


def _sig(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


def lib():
    """Load libspectre.so once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("SPECTRE_LIB", _LIB_PATH))
    if not path.exists():
        raise ImportError(
            f"libspectre.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(str(path))
    i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
    _sig(L, "spectre_version", C.c_char_p, [])
    _sig(L, "spectre_last_error", C.c_char_p, [])
    _sig(L, "spectre_oracle_stream", C.c_int, [u64, i32, _P, _P, _P, i64, _P])
    _sig(L, "spectre_oracle_propose", C.c_int,
         [u64, dbl, _P, _P, _P, _P, _P, _P, i32, i64, _P])
    _sig(L, "spectre_oracle_verify", C.c_int, [u64, _P, _P, _P, _P, i32, _P, _P, i64, _P])
    _sig(L, "spectre_mt19937_init_by_array", C.c_int, [_P, i32, _P])
    _sig(L, "spectre_mt19937_uniforms", C.c_int, [_P, _P, i64, _P])
    _sig(L, "spectre_oracle_workspace_bytes", C.c_size_t, [C.POINTER(OracleConfig)])
    _sig(L, "spectre_oracle_run", C.c_int,
         [C.POINTER(OracleConfig), _P, _P, i64, _P, C.POINTER(OracleOutputs), _P])
    _bind_model(L)
    _lib = L
    return L


class ModelDims(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_q_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("rms_eps", C.c_float), ("rope_theta", C.c_double)]


class ModelWeights(C.Structure):
    _fields_ = [(n, _P) for n in ("embed", "attn_norm", "wqkv", "wo", "mlp_norm", "wgu", "wd",
                                  "final_norm", "lm_head", "k_cache", "v_cache")]


class DecodeConfig(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_req", C.c_int32), ("gamma", C.c_int32),
                ("output_len", C.c_int32), ("prompt_len", C.c_int32), ("variant", C.c_int32),
                ("controller", C.c_int32), ("r_kind", C.c_int32), ("max_rounds", C.c_int32),
                ("ctx_cap", C.c_int32), ("has_fixed_l", C.c_int32), ("alpha", C.c_double),
                ("t_target", C.c_double), ("t_draft", C.c_double), ("ema_decay", C.c_double),
                ("fixed_threshold_l", C.c_double), ("temperature", C.c_double),
                ("role", C.c_int32), ("breaker_threshold", C.c_int32),
                ("breaker_cooldown", C.c_int32), ("draft_prompt_keep", C.c_int32),
                ("background_requests", C.c_int32), ("background_output_len", C.c_int32),
                ("fairness_period", C.c_int32), ("draft_capacity", C.c_int32),
                ("reply_timeout_rounds", C.c_int32), ("alpha_switch_pos", C.c_int32),
                ("alpha_late", C.c_double)]


TRACE_FIELDS = ("mode", "participants", "delta", "n_roll", "content_sum", "content_n",
                "n_padded", "t_round_ns", "t_verify_ns", "t_draft_ns", "r_hat_ema",
                "accepted_len_ema", "r_star", "n_stale", "n_regular", "n_forced",
                "fair_counter", "timeout")


class RoundTraceBufs(C.Structure):
    _fields_ = [(n, _P) for n in TRACE_FIELDS]


def _bind_model(L) -> None:
    i32, i64 = C.c_int32, C.c_int64
    _sig(L, "spectre_gemm_bf16", C.c_int,
         [_P, _P, _P, i32, i32, i32, i32, i32, i32, _P, _P, _P, _P, i32, i32, _P])
    _sig(L, "spectre_gemm_argmax_blocks", i32, [i32, i32])
    _sig(L, "spectre_engine_step", C.c_int, [_P, i32, i32, _P])
    _sig(L, "spectre_engine_exchange", C.c_int, [_P, _P, i32, i32, i32, i32, _P])
    _sig(L, "spectre_enable_peer_access", C.c_int, [i32, i32])
    _sig(L, "spectre_ipc_export", C.c_int, [_P, _P, C.POINTER(C.c_uint64)])
    _sig(L, "spectre_ipc_open", C.c_int, [_P, C.c_uint64, C.POINTER(_P), C.POINTER(_P)])
    _sig(L, "spectre_ipc_close", C.c_int, [_P])
    _sig(L, "spectre_engine_attach", _P, [_P, _P, _P, _P, C.c_size_t])
    _sig(L, "spectre_engine_workspace_bytes", C.c_size_t,
         [C.POINTER(ModelDims), C.POINTER(ModelDims), C.POINTER(DecodeConfig)])
    _sig(L, "spectre_engine_create", C.c_void_p,
         [C.POINTER(ModelDims), C.POINTER(ModelWeights), C.POINTER(ModelDims),
          C.POINTER(ModelWeights), C.POINTER(DecodeConfig), _P, C.c_size_t])
    _sig(L, "spectre_engine_destroy", C.c_int, [_P])
    _sig(L, "spectre_engine_prefill", C.c_int, [_P, _P, _P])
    _sig(L, "spectre_engine_run", C.c_int, [_P, i32, i32, C.POINTER(i32), _P])
    _sig(L, "spectre_engine_graph_status", C.c_int, [_P])
    _sig(L, "spectre_engine_read", C.c_int,
         [_P, _P, _P, C.POINTER(RoundTraceBufs), C.POINTER(i32), _P])
    _sig(L, "spectre_engine_read_committed", C.c_int, [_P, _P, _P])
    _sig(L, "spectre_engine_read_background", C.c_int, [_P, _P, _P, C.POINTER(i32), _P])
    _sig(L, "spectre_engine_launch_chains", C.c_int, [_P, i32, C.POINTER(i64), _P])
    _sig(L, "spectre_engine_forward", C.c_int,
         [_P, i32, _P, _P, _P, i32, _P, _P, _P, _P, _P, _P])


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().spectre_last_error().decode(errors="replace")
        raise SpectreError(f"{what} failed ({status}): {msg}")


def version() -> str:
    return lib().spectre_version().decode()


def require_cuda():
    """The product path runs on a CUDA device only (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the SPECTRE B200 decode loop requires a CUDA device; "
                           "no CPU fallback exists (use oracle/ for CPU checks)")
    return torch


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
