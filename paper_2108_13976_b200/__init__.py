"""paper_2108_13976_b200 — B200-native WarpDrive Tag env-step hot path.

Python host mirror of the reference's C++ API for this path, bound through the
C ABI in ``include/wdg_b200.h`` (``lib/libwdg_b200.so``, hand-written sm_100a
kernels). Names, argument meaning and error behaviour follow the reference:

=====================================  =========================================
reference (proj/include/warp/…)        here
=====================================  =========================================
``DataStore`` data_store.hpp:54-113    :class:`DataStore` (device-resident;
                                       host views become :meth:`pull`/:meth:`push`)
``TagConfig`` tag_env.hpp:29-66        :class:`TagConfig`
``register_tag_arrays`` :112           :func:`register_tag_arrays`
``build_tag_plan`` :116                :func:`build_tag_plan`
``StepEngine::run_step`` step_engine   :meth:`StepEngine.run_step`
``sample_actions`` sampler.hpp:35      :func:`sample_actions` (device logits)
``ResetManager`` reset_manager.hpp     :class:`ResetManager`
``RolloutDriver`` harness.cpp:428-505  :class:`RolloutDriver` (fused kernel)
``warp::Error`` / ``Errc``             :class:`WarpError` (``.code`` = wd_status)
=====================================  =========================================

There is no CPU fallback: without the built library or a CUDA device every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libwdg_b200.so")
if os.environ.get("WDG_LIB_VARIANT"):  # tuning builds (tools/), never set by product/tests/bench
    LIB_PATH = os.path.join(_HERE, "lib", "variants", os.environ["WDG_LIB_VARIANT"], "libwdg_b200.so")

# wd_status numbering (proj/include/warp/warp_c.h:22-38) + WDG_ERR_CUDA.
STATUS_NAMES = ["WD_OK", "WD_ERR_INVALID_ARGUMENT", "WD_ERR_DUPLICATE_NAME", "WD_ERR_SHAPE_MISMATCH",
                "WD_ERR_STORE_LOCKED", "WD_ERR_MISSING_PLACEHOLDER", "WD_ERR_UNKNOWN_NAME",
                "WD_ERR_INDEX_OUT_OF_RANGE", "WD_ERR_INVALID_CONFIG", "WD_ERR_STEP_FAILURE",
                "WD_ERR_NON_FINITE", "WD_ERR_PARSE", "WD_ERR_IO", "WD_ERR_STATE", "WD_ERR_UNKNOWN",
                "WDG_ERR_CUDA"]
(OK, INVALID_ARGUMENT, DUPLICATE_NAME, SHAPE_MISMATCH, STORE_LOCKED, MISSING_PLACEHOLDER,
 UNKNOWN_NAME, INDEX_OUT_OF_RANGE, INVALID_CONFIG, STEP_FAILURE, NON_FINITE, PARSE, IO, STATE,
 UNKNOWN, CUDA_ERROR) = range(16)

REAL32, INT32, BOOL8 = 0, 1, 2
DISCRETE, CONTINUOUS = 0, 1
FULL, PARTIAL = 0, 1
_NP = {REAL32: np.float32, INT32: np.int32, BOOL8: np.uint8}

# WDG_STAT_* (episode statistics vector)
STAT_EPISODES, STAT_TAGGER_RETURN, STAT_RUNNER_RETURN, STAT_TAG_EVENTS, STAT_ENV_STEPS = range(5)
STAT_COUNT = 8

EXPORTED_SYMBOLS = [
    "wdg_version", "wdg_status_name", "wdg_last_error", "wdg_device_count", "wdg_set_device",
    "wdg_set_fault_tag_radius_bias", "wdg_store_create", "wdg_store_destroy",
    "wdg_store_set_env_offset", "wdg_store_set_stream", "wdg_store_register_array",
    "wdg_store_lock", "wdg_store_locked", "wdg_store_num_envs", "wdg_store_num_agents",
    "wdg_store_handle", "wdg_store_num_arrays", "wdg_store_info", "wdg_store_push",
    "wdg_store_pull", "wdg_store_device_ptr", "wdg_store_restore_snapshot", "wdg_store_synchronize",
    "wdg_tag_config_init", "wdg_tag_config_validate", "wdg_tag_obs_dim", "wdg_register_tag_arrays",
    "wdg_tag_zero_on_reset", "wdg_build_tag_plan", "wdg_tag_plan_destroy", "wdg_run_step",
    "wdg_tag_plan_geometry", "wdg_sample_actions", "wdg_reset_manager_create",
    "wdg_reset_manager_destroy", "wdg_detect_done", "wdg_auto_reset", "wdg_auto_reset_on_done",
    "wdg_episodes_started", "wdg_rollout_create", "wdg_rollout_destroy", "wdg_rollout_set_logits",
    "wdg_rollout_set_fused", "wdg_rollout_set_graphs", "wdg_rollout_step", "wdg_rollout_run",
    "wdg_rollout_next_step", "wdg_rollout_check", "wdg_rollout_stats", "wdg_rollout_reset_stats",
    "wdg_rollout_stats_device_ptr", "wdg_rollout_step_host", "wdg_rollout_step_host_obs",
    "wdg_rollout_set_host_chunks", "wdg_rollout_reduce_stats_into", "wdg_rollout_set_overlap",
    "wdg_set_tuning", "wdg_build_tag_reference", "wdg_nccl_version", "wdg_comm_unique_id", "wdg_comm_init", "wdg_comm_wrap",
    "wdg_comm_destroy", "wdg_comm_info", "wdg_stats_allreduce",
    "wdg_policy_create", "wdg_policy_destroy", "wdg_policy_init", "wdg_policy_param_count",
    "wdg_policy_set_params", "wdg_policy_get_params", "wdg_policy_forward", "wdg_rollout_set_policies",
    "wdg_rollout_policy_outputs", "wdg_copy_to_host", "wdg_rollout_set_keep_policy_outputs",
    "wdg_batch_create", "wdg_batch_destroy", "wdg_batch_get_view", "wdg_rollout_collect", "wdg_compute_returns",
    "wdg_session_open", "wdg_session_open_file", "wdg_session_close", "wdg_session_set_seed",
    "wdg_session_set_workers", "wdg_session_set_output_dir", "wdg_session_config_json",
    "wdg_session_config_hash", "wdg_session_run_check", "wdg_session_run_bench_envs",
    "wdg_session_run_bench_agents", "wdg_session_run_training", "wdg_session_report_json",
    "wdg_session_summary", "wdg_session_dump_array", "wdg_rollout_launches",
]

POLICY_F64, POLICY_BF16 = 0, 1


class WarpError(RuntimeError):
    """warp::Error (proj/include/warp/common.hpp:30-37); ``code`` is the
    wd_status value, ``status`` its name."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.status = STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else str(code)
        super().__init__(f"{self.status}: {message}")


class _TagConfigC(C.Structure):
    _fields_ = [("variant", C.c_int32), ("obs_mode", C.c_int32), ("grid_size", C.c_int64),
                ("world_length", C.c_double), ("num_taggers", C.c_int64), ("num_runners", C.c_int64),
                ("episode_length", C.c_int64), ("tag_radius", C.c_double), ("k_nearest", C.c_int64),
                ("tag_reward", C.c_double), ("tagged_penalty", C.c_double),
                ("max_speed_tagger", C.c_double), ("max_speed_runner", C.c_double),
                ("accel_delta", C.c_double), ("turn_delta", C.c_double), ("seed", C.c_uint64)]


class _BatchViewC(C.Structure):
    _fields_ = [("horizon", C.c_int64), ("num_envs", C.c_int64), ("num_agents", C.c_int64),
                ("obs_dim", C.c_int64), ("num_categories", C.c_int64), ("obs", C.c_void_p),
                ("actions", C.c_void_p), ("rewards", C.c_void_p), ("done", C.c_void_p),
                ("active", C.c_void_p), ("values", C.c_void_p), ("logp", C.c_void_p),
                ("bootstrap", C.c_void_p)]


class _ArrayInfoC(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("kind", C.c_int32), ("ndim", C.c_int32),
                ("shape", C.c_int64 * 8), ("total_elems", C.c_int64), ("env_stride", C.c_int64),
                ("agent_stride", C.c_int64), ("has_agent_axis", C.c_int32),
                ("snapshot_on_reset", C.c_int32)]


_lib = None


def library_path() -> str:
    return LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built (run __graft_entry__.build()); "
                          "the B200 Tag path has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, U64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    sig = {
        "wdg_version": (C.c_char_p, []),
        "wdg_status_name": (C.c_char_p, [I32]),
        "wdg_last_error": (C.c_char_p, []),
        "wdg_device_count": (I32, [C.POINTER(I32)]),
        "wdg_set_device": (I32, [I32]),
        "wdg_set_fault_tag_radius_bias": (None, [C.c_float]),
        "wdg_store_create": (I32, [I64, I64, C.POINTER(P)]),
        "wdg_store_destroy": (None, [P]),
        "wdg_store_set_env_offset": (I32, [P, I64]),
        "wdg_store_set_stream": (I32, [P, P]),
        "wdg_store_register_array": (I32, [P, C.c_char_p, C.POINTER(I64), I32, I32, I32, P, I64,
                                           C.POINTER(I32)]),
        "wdg_store_lock": (I32, [P]),
        "wdg_store_locked": (I32, [P, C.POINTER(I32)]),
        "wdg_store_num_envs": (I32, [P, C.POINTER(I64)]),
        "wdg_store_num_agents": (I32, [P, C.POINTER(I64)]),
        "wdg_store_handle": (I32, [P, C.c_char_p, C.POINTER(I32)]),
        "wdg_store_num_arrays": (I32, [P, C.POINTER(I32)]),
        "wdg_store_info": (I32, [P, I32, C.POINTER(_ArrayInfoC)]),
        "wdg_store_push": (I32, [P, I32, I64, I64, P, I64]),
        "wdg_store_pull": (I32, [P, I32, I64, I64, P, I64]),
        "wdg_store_device_ptr": (I32, [P, I32, C.POINTER(P)]),
        "wdg_store_restore_snapshot": (I32, [P, C.POINTER(I64), I64]),
        "wdg_store_synchronize": (I32, [P]),
        "wdg_tag_config_init": (I32, [C.POINTER(_TagConfigC)]),
        "wdg_tag_config_validate": (I32, [C.POINTER(_TagConfigC)]),
        "wdg_tag_obs_dim": (I64, [C.POINTER(_TagConfigC)]),
        "wdg_register_tag_arrays": (I32, [P, C.POINTER(_TagConfigC)]),
        "wdg_tag_zero_on_reset": (I32, [C.POINTER(C.c_char_p), I32, C.POINTER(I32)]),
        "wdg_build_tag_plan": (I32, [P, C.POINTER(_TagConfigC), C.POINTER(P)]),
        "wdg_tag_plan_destroy": (None, [P]),
        "wdg_run_step": (I32, [P, I64]),
        "wdg_tag_plan_geometry": (I32, [P] + [C.POINTER(I32)] * 5),
        "wdg_sample_actions": (I32, [P, P, I64, I64, I64, I64, U64]),
        "wdg_reset_manager_create": (I32, [P, I32, C.POINTER(C.c_char_p), I32, P, C.POINTER(P)]),
        "wdg_reset_manager_destroy": (None, [P]),
        "wdg_detect_done": (I32, [P, C.POINTER(I64), I64, C.POINTER(I64)]),
        "wdg_auto_reset": (I32, [P, C.POINTER(I64), I64]),
        "wdg_auto_reset_on_done": (I32, [P]),
        "wdg_episodes_started": (I32, [P, I64, C.POINTER(I64)]),
        "wdg_rollout_create": (I32, [P, P, P, U64, C.POINTER(P)]),
        "wdg_rollout_destroy": (None, [P]),
        "wdg_rollout_set_logits": (I32, [P, P, I64]),
        "wdg_rollout_set_fused": (I32, [P, I32]),
        "wdg_rollout_set_graphs": (I32, [P, I32]),
        "wdg_rollout_step": (I32, [P]),
        "wdg_rollout_run": (I32, [P, I64]),
        "wdg_rollout_next_step": (I32, [P, C.POINTER(I64)]),
        "wdg_rollout_check": (I32, [P]),
        "wdg_rollout_stats": (I32, [P, C.POINTER(D), I32]),
        "wdg_rollout_reset_stats": (I32, [P]),
        "wdg_rollout_stats_device_ptr": (I32, [P, C.POINTER(C.POINTER(D))]),
        "wdg_rollout_step_host": (I32, [P, P, I64, P, P]),
        "wdg_rollout_step_host_obs": (I32, [P, P, I64, P, P, P, I64]),
        "wdg_rollout_set_host_chunks": (I32, [P, I32]),
        "wdg_rollout_set_overlap": (I32, [P, I32]),
        "wdg_set_tuning": (I32, [C.c_char_p, I64]),
        "wdg_build_tag_reference": (I32, [P, P, C.POINTER(P)]),
        "wdg_nccl_version": (I32, [C.POINTER(I32)]),
        "wdg_comm_unique_id": (I32, [P, I64]),
        "wdg_comm_init": (I32, [I32, I32, P, I64, C.POINTER(P)]),
        "wdg_comm_wrap": (I32, [P, C.POINTER(P)]),
        "wdg_comm_destroy": (None, [P]),
        "wdg_comm_info": (I32, [P, C.POINTER(I32), C.POINTER(I32)]),
        "wdg_stats_allreduce": (I32, [P, P, P]),
        "wdg_rollout_reduce_stats_into": (I32, [P, P]),
        "wdg_policy_create": (I32, [I64, C.POINTER(I64), I32, I64, I64, C.POINTER(P)]),
        "wdg_policy_destroy": (None, [P]),
        "wdg_policy_init": (I32, [P, U64]),
        "wdg_policy_param_count": (I32, [P, C.POINTER(I64)]),
        "wdg_policy_set_params": (I32, [P, P, I64]),
        "wdg_policy_get_params": (I32, [P, P, I64]),
        "wdg_policy_forward": (I32, [P, P, I64, I64, I64, I64, P, P, I32, P]),
        "wdg_rollout_set_policies": (I32, [P, P, P, I32]),
        "wdg_rollout_policy_outputs": (I32, [P, C.POINTER(P), C.POINTER(P)]),
        "wdg_copy_to_host": (I32, [P, P, I64]),
        "wdg_rollout_set_keep_policy_outputs": (I32, [P, I32]),
        "wdg_batch_create": (I32, [P, I64, C.POINTER(P)]),
        "wdg_batch_destroy": (None, [P]),
        "wdg_batch_get_view": (I32, [P, C.POINTER(_BatchViewC)]),
        "wdg_rollout_collect": (I32, [P, P]),
        "wdg_compute_returns": (I32, [P, D, P, P]),
        "wdg_session_open": (I32, [C.c_char_p, C.POINTER(P)]),
        "wdg_session_open_file": (I32, [C.c_char_p, C.POINTER(P)]),
        "wdg_session_close": (None, [P]),
        "wdg_session_set_seed": (I32, [P, U64]),
        "wdg_session_set_workers": (I32, [P, I32]),
        "wdg_session_set_output_dir": (I32, [P, C.c_char_p]),
        "wdg_session_config_json": (C.c_char_p, [P]),
        "wdg_session_config_hash": (C.c_char_p, [P]),
        "wdg_session_run_check": (I32, [P]),
        "wdg_session_run_bench_envs": (I32, [P]),
        "wdg_session_run_bench_agents": (I32, [P]),
        "wdg_session_run_training": (I32, [P]),
        "wdg_session_report_json": (C.c_char_p, [P]),
        "wdg_session_summary": (C.c_char_p, [P]),
        "wdg_session_dump_array": (I32, [P, C.c_char_p, C.c_char_p]),
        "wdg_rollout_launches": (I32, [P, C.POINTER(I64)]),
    }
    for name, (res, args) in sig.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if os.environ.get("WDG_LIB_VARIANT"):  # older tuning builds lack newer entry points
                continue
            raise
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return _load()


def _check(status: int):
    if status != OK:
        msg = _load().wdg_last_error().decode(errors="replace")
        raise WarpError(status, msg)


def copy_to_host(device_ptr, out: np.ndarray) -> np.ndarray:
    """Synchronous device -> host copy into the contiguous numpy array `out`."""
    _check(_load().wdg_copy_to_host(C.c_void_p(_ptr(device_ptr)), out.ctypes.data, out.nbytes))
    return out


def version() -> str:
    return _load().wdg_version().decode()


def device_count() -> int:
    n = C.c_int32()
    _check(_load().wdg_device_count(C.byref(n)))
    return n.value


def set_fault_tag_radius_bias(bias: float):
    """detail::fault_hooks().tag_radius_bias (tag_env.hpp:155-158): test-only
    mutation of the device kernels' tag radius."""
    _load().wdg_set_fault_tag_radius_bias(float(bias))


def set_tuning(key: str, value: int = -1):
    """Plan tuning override (wdg_set_tuning): how a plan maps the step onto
    the GPU, never what it computes; value < 0 or key "reset" restores the
    plan's own choice."""
    _check(_load().wdg_set_tuning(key.encode(), value))


def _ptr(x) -> int:
    """Device address from an int or an object exposing data_ptr() (torch)."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"expected a device pointer or tensor, got {type(x)}")


# ---------------------------------------------------------------------------
@dataclass
class TagConfig:
    """TagConfig (proj/include/warp/tag_env.hpp:29-45), same defaults."""
    variant: int = DISCRETE
    grid_size: int = 20
    world_length: float = 20.0
    num_taggers: int = 2
    num_runners: int = 10
    episode_length: int = 500
    tag_radius: float = 1.0
    obs_mode: int = FULL
    k_nearest: int = 5
    tag_reward: float = 1.0
    tagged_penalty: float = -1.0
    max_speed_tagger: float = 1.0
    max_speed_runner: float = 1.0
    accel_delta: float = 0.1
    turn_delta: float = 0.5235987755982988
    seed: int = 0

    def num_agents(self) -> int:
        return self.num_taggers + self.num_runners

    def action_categories(self) -> int:
        return 2 if self.variant == CONTINUOUS else 1

    def action_choices(self) -> int:
        return 3 if self.variant == CONTINUOUS else 5

    def obs_dim(self) -> int:
        return int(_load().wdg_tag_obs_dim(C.byref(self._c())))

    def validate(self):
        _check(_load().wdg_tag_config_validate(C.byref(self._c())))

    def _c(self) -> _TagConfigC:
        return _TagConfigC(variant=self.variant, obs_mode=self.obs_mode, grid_size=self.grid_size,
                           world_length=self.world_length, num_taggers=self.num_taggers,
                           num_runners=self.num_runners, episode_length=self.episode_length,
                           tag_radius=self.tag_radius, k_nearest=self.k_nearest,
                           tag_reward=self.tag_reward, tagged_penalty=self.tagged_penalty,
                           max_speed_tagger=self.max_speed_tagger,
                           max_speed_runner=self.max_speed_runner, accel_delta=self.accel_delta,
                           turn_delta=self.turn_delta, seed=self.seed)


@dataclass
class ArraySpec:
    """ArraySpec (data_store.hpp:31-36)."""
    name: str
    shape: Sequence[int]
    kind: int = REAL32
    snapshot_on_reset: bool = False


@dataclass
class ArrayInfo:
    """ArrayInfo (data_store.hpp:42-48)."""
    spec: ArraySpec
    total_elems: int
    env_stride: int
    agent_stride: int
    has_agent_axis: bool


class DataStore:
    """Device-resident named-array store (data_store.hpp:54-113)."""

    def __init__(self, num_envs: int, num_agents: int):
        self._lib = _load()
        h = C.c_void_p()
        _check(self._lib.wdg_store_create(num_envs, num_agents, C.byref(h)))
        self._h = h
        self._num_envs = num_envs
        self._num_agents = num_agents
        self._deps = []  # plans/resets/rollouts that must die first

    def __del__(self):
        self.close()

    def close(self):
        for d in reversed(getattr(self, "_deps", [])):
            d.close()
        self._deps = []
        if getattr(self, "_h", None):
            self._lib.wdg_store_destroy(self._h)
            self._h = None

    @property
    def handle_ptr(self):
        return self._h

    def num_envs(self) -> int:
        return self._num_envs

    def num_agents(self) -> int:
        return self._num_agents

    def set_env_offset(self, offset: int):
        _check(self._lib.wdg_store_set_env_offset(self._h, offset))

    def set_stream(self, stream):
        """cudaStream_t (int) or an object with .cuda_stream (torch.cuda.Stream)."""
        s = getattr(stream, "cuda_stream", stream)
        _check(self._lib.wdg_store_set_stream(self._h, C.c_void_p(int(s or 0))))

    def register_array(self, spec: ArraySpec, initial=None) -> int:
        shape = (C.c_int64 * len(spec.shape))(*[int(d) for d in spec.shape])
        data, count = None, 0
        if initial is not None:
            arr = np.ascontiguousarray(np.asarray(initial, dtype=_NP[spec.kind]))
            data, count = arr.ctypes.data, arr.size
        out = C.c_int32()
        _check(self._lib.wdg_store_register_array(self._h, spec.name.encode(), shape, len(spec.shape),
                                                  spec.kind, 1 if spec.snapshot_on_reset else 0,
                                                  data, count, C.byref(out)))
        return out.value

    def lock(self):
        _check(self._lib.wdg_store_lock(self._h))

    def locked(self) -> bool:
        v = C.c_int32()
        _check(self._lib.wdg_store_locked(self._h, C.byref(v)))
        return bool(v.value)

    def has_array(self, name: str) -> bool:
        try:
            self.handle(name)
            return True
        except WarpError:
            return False

    def handle(self, name: str) -> int:
        v = C.c_int32()
        _check(self._lib.wdg_store_handle(self._h, name.encode(), C.byref(v)))
        return v.value

    def _h_of(self, name_or_handle) -> int:
        return self.handle(name_or_handle) if isinstance(name_or_handle, str) else int(name_or_handle)

    def info(self, name_or_handle) -> ArrayInfo:
        ci = _ArrayInfoC()
        _check(self._lib.wdg_store_info(self._h, self._h_of(name_or_handle), C.byref(ci)))
        spec = ArraySpec(ci.name.decode(), [ci.shape[i] for i in range(ci.ndim)], ci.kind,
                         bool(ci.snapshot_on_reset))
        return ArrayInfo(spec, ci.total_elems, ci.env_stride, ci.agent_stride, bool(ci.has_agent_axis))

    def array_names(self):
        n = C.c_int32()
        _check(self._lib.wdg_store_num_arrays(self._h, C.byref(n)))
        return [self.info(i).spec.name for i in range(n.value)]

    def pull(self, name_or_handle, env_begin: int = 0, env_count: Optional[int] = None) -> np.ndarray:
        """Copy of env rows [env_begin, env_begin+env_count) in the reference
        layout (replaces the aliasing f32/i32/u8 views, data_store.hpp:78-89)."""
        h = self._h_of(name_or_handle)
        inf = self.info(h)
        if env_count is None:
            env_count = self._num_envs - env_begin
        out = np.empty([env_count] + list(inf.spec.shape[1:]), dtype=_NP[inf.spec.kind])
        _check(self._lib.wdg_store_pull(self._h, h, env_begin, env_count, out.ctypes.data, out.nbytes))
        return out

    def push(self, name_or_handle, values, env_begin: int = 0):
        h = self._h_of(name_or_handle)
        inf = self.info(h)
        arr = np.ascontiguousarray(np.asarray(values, dtype=_NP[inf.spec.kind]))
        row = inf.env_stride
        if arr.size % row:
            raise WarpError(SHAPE_MISMATCH, "push: value count is not a whole number of env rows")
        _check(self._lib.wdg_store_push(self._h, h, env_begin, arr.size // row, arr.ctypes.data, arr.nbytes))

    def device_ptr(self, name_or_handle) -> int:
        p = C.c_void_p()
        _check(self._lib.wdg_store_device_ptr(self._h, self._h_of(name_or_handle), C.byref(p)))
        return int(p.value or 0)

    def restore_snapshot(self, env_ids: Iterable[int]):
        ids = np.ascontiguousarray(np.asarray(list(env_ids), dtype=np.int64))
        _check(self._lib.wdg_store_restore_snapshot(self._h, ids.ctypes.data_as(C.POINTER(C.c_int64)), ids.size))

    def synchronize(self):
        _check(self._lib.wdg_store_synchronize(self._h))


def register_tag_arrays(store: DataStore, cfg: TagConfig):
    """register_tag_arrays (tag_env.hpp:112): same arrays, episode-0 state
    computed on device."""
    _check(_load().wdg_register_tag_arrays(store._h, C.byref(cfg._c())))


def tag_zero_on_reset():
    names = (C.c_char_p * 16)()
    n = C.c_int32()
    _check(_load().wdg_tag_zero_on_reset(names, 16, C.byref(n)))
    return [names[i].decode() for i in range(n.value)]


class TagPlan:
    """TagPlan (tag_env.hpp:104-107); must not outlive its store."""

    def __init__(self, store: DataStore, cfg: TagConfig, reference: bool = False):
        """reference=True: the device TagReference twin (tag_env.cpp:505-595),
        the consistency check's independent brute-force implementation."""
        self._lib = _load()
        h = C.c_void_p()
        build = self._lib.wdg_build_tag_reference if reference else self._lib.wdg_build_tag_plan
        _check(build(store._h, C.byref(cfg._c()), C.byref(h)))
        self.reference = reference
        self._h = h
        self.store = store
        self.cfg = cfg
        store._deps.append(self)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_tag_plan_destroy(self._h)
            self._h = None

    def geometry(self) -> dict:
        v = [C.c_int32() for _ in range(5)]
        _check(self._lib.wdg_tag_plan_geometry(self._h, *[C.byref(x) for x in v]))
        keys = ["threads_per_cta", "envs_per_cta", "grid_ctas", "uses_grid", "smem_bytes"]
        return {k: x.value for k, x in zip(keys, v)}


def build_tag_plan(store: DataStore, cfg: TagConfig) -> TagPlan:
    """build_tag_plan (tag_env.hpp:116, tag_env.cpp:363-480)."""
    return TagPlan(store, cfg)


@dataclass
class EngineConfig:
    """EngineConfig (step_engine.hpp:52-57). worker_count/deterministic are
    accepted for API parity; the device engine is one CTA per env."""
    num_envs: int = 1
    num_agents: int = 1
    worker_count: int = 1
    deterministic: bool = True


class StepEngine:
    """StepEngine (step_engine.hpp:90-107): run_step launches the Tag step
    kernel (phases = in-CTA barriers)."""

    def __init__(self, cfg: EngineConfig = EngineConfig()):
        if not cfg.deterministic:
            raise WarpError(INVALID_ARGUMENT, "EngineConfig: only deterministic execution exists in v1")
        self.cfg = cfg

    def run_step(self, plan: TagPlan, store: DataStore, step_index: int):
        if plan.store is not store:
            raise WarpError(INVALID_ARGUMENT, "run_step: plan belongs to another store")
        if not store.locked():
            raise WarpError(STATE, "run_step: store is not locked")
        _check(_load().wdg_run_step(plan._h, step_index))


def sample_actions(store: DataStore, logits, logits_count: int, num_categories: int,
                   num_choices: int, step: int, seed: int):
    """sample_actions (sampler.hpp:35-36) over DEVICE f64 logits [E,A,C,V]
    (a device address or a CUDA tensor)."""
    _check(_load().wdg_sample_actions(store._h, C.c_void_p(_ptr(logits)), logits_count,
                                      num_categories, num_choices, step, seed))


def make_tag_reinit(plan: TagPlan):
    """make_tag_reinit (tag_env.hpp:124-125): the reinit for ResetPolicy."""
    return plan


@dataclass
class ResetPolicy:
    """ResetPolicy (reset_manager.hpp:11-19); reinitialize = make_tag_reinit(plan) or None."""
    auto_reset: bool = True
    zero_on_reset: list = field(default_factory=list)
    reinitialize: Optional[TagPlan] = None


class ResetManager:
    """ResetManager (reset_manager.hpp:21-43) with a device episode counter."""

    def __init__(self, store: DataStore, policy: ResetPolicy):
        self._lib = _load()
        names = (C.c_char_p * max(1, len(policy.zero_on_reset)))(*[n.encode() for n in policy.zero_on_reset])
        h = C.c_void_p()
        plan_h = policy.reinitialize._h if policy.reinitialize is not None else None
        _check(self._lib.wdg_reset_manager_create(store._h, 1 if policy.auto_reset else 0, names,
                                                  len(policy.zero_on_reset), plan_h, C.byref(h)))
        self._h = h
        self.store = store
        self.policy = policy
        store._deps.append(self)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_reset_manager_destroy(self._h)
            self._h = None

    def auto_enabled(self) -> bool:
        return self.policy.auto_reset

    def detect_done(self, store: Optional[DataStore] = None):
        n = self.store.num_envs()
        ids = (C.c_int64 * n)()
        cnt = C.c_int64()
        _check(self._lib.wdg_detect_done(self._h, ids, n, C.byref(cnt)))
        return [ids[i] for i in range(cnt.value)]

    def auto_reset(self, store_or_ids, env_ids=None):
        ids = store_or_ids if env_ids is None else env_ids
        arr = np.ascontiguousarray(np.asarray(list(ids), dtype=np.int64))
        _check(self._lib.wdg_auto_reset(self._h, arr.ctypes.data_as(C.POINTER(C.c_int64)), arr.size))

    def auto_reset_on_done(self):
        _check(self._lib.wdg_auto_reset_on_done(self._h))

    def episodes_started(self, env_id: int) -> int:
        v = C.c_int64()
        _check(self._lib.wdg_episodes_started(self._h, env_id, C.byref(v)))
        return v.value


class RolloutDriver:
    """RolloutDriver (harness.cpp:428-505): each step is sample(t) -> run_step(t)
    -> [episode stats] -> reset-on-done, fused into ONE kernel launch."""

    def __init__(self, store: DataStore, plan: TagPlan, resets: Optional[ResetManager],
                 sample_seed: int):
        self._lib = _load()
        h = C.c_void_p()
        _check(self._lib.wdg_rollout_create(store._h, plan._h, resets._h if resets else None,
                                            sample_seed, C.byref(h)))
        self._h = h
        self.store = store
        store._deps.append(self)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_rollout_destroy(self._h)
            self._h = None

    def set_logits(self, logits=None, count: int = 0):
        _check(self._lib.wdg_rollout_set_logits(self._h, C.c_void_p(_ptr(logits)), count))

    def set_policies(self, tagger: Optional[Policy], runner: Optional[Policy] = None,
                     precision: int = POLICY_F64):
        """forward_policies (harness.cpp:445-476) on device before every step;
        runner=None -> one shared policy; tagger=None -> uniform policy."""
        if tagger is not None and runner is None:
            runner = tagger
        self._policies = (tagger, runner)  # keep alive while in use
        _check(self._lib.wdg_rollout_set_policies(self._h, tagger._h if tagger else None,
                                                  runner._h if runner else None, precision))

    def set_keep_policy_outputs(self, keep: bool):
        _check(self._lib.wdg_rollout_set_keep_policy_outputs(self._h, 1 if keep else 0))

    def policy_outputs(self):
        """(logits, values) device addresses of the last policy forward."""
        lg, vl = C.c_void_p(), C.c_void_p()
        _check(self._lib.wdg_rollout_policy_outputs(self._h, C.byref(lg), C.byref(vl)))
        return lg.value or 0, vl.value or 0

    def collect(self, batch: "RolloutBatch"):
        """Trainer::collect (trainer.cpp:315-403): horizon captured policy steps."""
        _check(self._lib.wdg_rollout_collect(self._h, batch._h))

    def set_fused(self, fused: bool):
        _check(self._lib.wdg_rollout_set_fused(self._h, 1 if fused else 0))

    def set_graphs(self, enabled: bool):
        _check(self._lib.wdg_rollout_set_graphs(self._h, 1 if enabled else 0))

    def set_overlap(self, enabled: bool):
        """Overlapped consecutive launches (default on); off = serial launches."""
        _check(self._lib.wdg_rollout_set_overlap(self._h, 1 if enabled else 0))

    def step(self):
        _check(self._lib.wdg_rollout_step(self._h))

    def step_host(self, host_logits, count: int, host_rewards=None, host_done=None,
                  host_obs=None, obs_count: int = 0):
        """One step from HOST buffers (addresses or pinned CPU tensors /
        numpy arrays): rewards and done as they were before reset-on-done
        (trainer.cpp:382-394), observations after it; results valid after
        store.synchronize()."""
        def hp(x):
            if x is None:
                return None
            if isinstance(x, np.ndarray):
                return x.ctypes.data
            return _ptr(x)
        if host_obs is None:
            _check(self._lib.wdg_rollout_step_host(self._h, C.c_void_p(hp(host_logits)), count,
                                                   C.c_void_p(hp(host_rewards)),
                                                   C.c_void_p(hp(host_done))))
        else:
            _check(self._lib.wdg_rollout_step_host_obs(self._h, C.c_void_p(hp(host_logits)), count,
                                                       C.c_void_p(hp(host_rewards)),
                                                       C.c_void_p(hp(host_done)),
                                                       C.c_void_p(hp(host_obs)), obs_count))

    def set_host_chunks(self, chunks: int):
        """Env chunks of the pipelined step_host (0 = automatic)."""
        _check(self._lib.wdg_rollout_set_host_chunks(self._h, chunks))

    def reduce_stats_into(self, device_out):
        _check(self._lib.wdg_rollout_reduce_stats_into(self._h, C.c_void_p(_ptr(device_out))))

    def run(self, steps: int):
        _check(self._lib.wdg_rollout_run(self._h, steps))

    def launches(self) -> int:
        v = C.c_int64()
        _check(self._lib.wdg_rollout_launches(self._h, C.byref(v)))
        return v.value

    def next_step(self) -> int:
        v = C.c_int64()
        _check(self._lib.wdg_rollout_next_step(self._h, C.byref(v)))
        return v.value

    def check(self):
        _check(self._lib.wdg_rollout_check(self._h))

    def stats(self) -> np.ndarray:
        out = (C.c_double * STAT_COUNT)()
        _check(self._lib.wdg_rollout_stats(self._h, out, STAT_COUNT))
        return np.array(out[:], dtype=np.float64)

    def reset_stats(self):
        _check(self._lib.wdg_rollout_reset_stats(self._h))

    def stats_device_ptr(self) -> int:
        p = C.POINTER(C.c_double)()
        _check(self._lib.wdg_rollout_stats_device_ptr(self._h, C.byref(p)))
        return C.cast(p, C.c_void_p).value or 0


def nccl_version() -> int:
    v = C.c_int32()
    _check(_load().wdg_nccl_version(C.byref(v)))
    return v.value


def comm_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0 creates it, every rank passes it to Comm)."""
    buf = (C.c_uint8 * 128)()
    _check(_load().wdg_comm_unique_id(buf, 128))
    return bytes(buf)


class Comm:
    """NCCL communicator of the statistics all-reduce (wdg_comm_*): created
    from a unique id (ncclCommInitRank over `world` ranks, one GPU each), or
    wrapping an existing ncclComm_t address (e.g. ProcessGroupNCCL._comm_ptr())."""

    def __init__(self, world: int = 1, rank: int = 0, unique_id: Optional[bytes] = None,
                 wrap: Optional[int] = None):
        self._lib = _load()
        h = C.c_void_p()
        if wrap is not None:
            _check(self._lib.wdg_comm_wrap(C.c_void_p(wrap), C.byref(h)))
        else:
            if unique_id is None or len(unique_id) != 128:
                raise ValueError("Comm needs the 128-byte unique id from comm_unique_id()")
            buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
            _check(self._lib.wdg_comm_init(world, rank, buf, 128, C.byref(h)))
        self._h = h
        w, r = C.c_int32(), C.c_int32()
        _check(self._lib.wdg_comm_info(h, C.byref(w), C.byref(r)))
        self.world, self.rank = w.value, r.value

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def stats_allreduce(self, rollout: "RolloutDriver", device_out):
        """This shard's tracker sums reduced on device, then ncclAllReduce(sum)
        into device_out (device double[8]) on the store's stream."""
        _check(self._lib.wdg_stats_allreduce(rollout._h, self._h, C.c_void_p(_ptr(device_out))))


class Policy:
    """PolicyParams + forward (proj/include/warp/policy_model.hpp) with the
    parameters on device: the reference MLP (tanh hidden layers, per-category
    logit heads, a value head)."""

    def __init__(self, obs_dim: int, hidden=(64, 64), num_categories: int = 1, num_choices: int = 1,
                 seed: Optional[int] = None):
        self._lib = _load()
        hs = (C.c_int64 * len(hidden))(*[int(h) for h in hidden])
        h = C.c_void_p()
        _check(self._lib.wdg_policy_create(int(obs_dim), hs, len(hidden), int(num_categories),
                                           int(num_choices), C.byref(h)))
        self._h = h
        self.obs_dim, self.hidden = int(obs_dim), [int(x) for x in hidden]
        self.num_categories, self.num_choices = int(num_categories), int(num_choices)
        if seed is not None:
            self.init(seed)

    @classmethod
    def for_tag(cls, cfg: "TagConfig", hidden=(64, 64), seed: Optional[int] = None) -> "Policy":
        return cls(cfg.obs_dim(), hidden, cfg.action_categories(), cfg.action_choices(), seed)

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_policy_destroy(self._h)
            self._h = None

    def init(self, seed: int):
        """init_policy(seed, dims) (policy_model.cpp:107-144)."""
        _check(self._lib.wdg_policy_init(self._h, int(seed)))

    def param_count(self) -> int:
        v = C.c_int64()
        _check(self._lib.wdg_policy_param_count(self._h, C.byref(v)))
        return v.value

    def get_params(self) -> np.ndarray:
        out = np.zeros(self.param_count(), dtype=np.float64)
        _check(self._lib.wdg_policy_get_params(self._h, out.ctypes.data, out.size))
        return out

    def set_params(self, params):
        arr = np.ascontiguousarray(params, dtype=np.float64)
        _check(self._lib.wdg_policy_set_params(self._h, arr.ctypes.data, arr.size))

    def forward(self, obs, num_envs: int, num_agents: int, logits, values=None, agent_begin: int = 0,
                agent_end: Optional[int] = None, precision: int = POLICY_F64, stream=None):
        """forward over agents [agent_begin, agent_end) of DEVICE f32 obs
        [E, A, obs_dim] into DEVICE f64 logits [E, A, C*V] / values [E, A]."""
        end = num_agents if agent_end is None else agent_end
        st = None if stream is None else C.c_void_p(getattr(stream, "cuda_stream", stream))
        _check(self._lib.wdg_policy_forward(self._h, C.c_void_p(_ptr(obs)), num_envs, num_agents, agent_begin,
                                            end, C.c_void_p(_ptr(logits)), C.c_void_p(_ptr(values)),
                                            precision, st))


class RolloutBatch:
    """RolloutBatch (trainer.hpp:36-49) in HBM, filled by RolloutDriver.collect."""

    FIELDS = {"obs": np.float32, "actions": np.int32, "rewards": np.float32, "done": np.uint8,
              "active": np.uint8, "values": np.float64, "logp": np.float64, "bootstrap": np.float64}

    def __init__(self, store: DataStore, horizon: int):
        self._lib = _load()
        h = C.c_void_p()
        _check(self._lib.wdg_batch_create(store._h, int(horizon), C.byref(h)))
        self._h = h
        v = _BatchViewC()
        _check(self._lib.wdg_batch_get_view(self._h, C.byref(v)))
        self.view = v
        T, E, A, D, Cc = v.horizon, v.num_envs, v.num_agents, v.obs_dim, v.num_categories
        self.shapes = {"obs": (T, E, A, D), "actions": (T, E, A, Cc), "rewards": (T, E, A), "done": (T, E),
                       "active": (T, E, A), "values": (T, E, A), "logp": (T, E, A), "bootstrap": (E, A)}
        store._deps.append(self)

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_batch_destroy(self._h)
            self._h = None

    def device_ptr(self, name: str) -> int:
        return getattr(self.view, name)

    def pull(self, name: str) -> np.ndarray:
        out = np.zeros(self.shapes[name], dtype=self.FIELDS[name])
        return copy_to_host(self.device_ptr(name), out)

    def compute_returns(self, gamma: float, out=None, stream=None):
        """compute_returns (trainer.cpp:73-88) into a device f64 [T,E,A] buffer
        (a torch tensor or address); returns it."""
        st = None if stream is None else C.c_void_p(getattr(stream, "cuda_stream", stream))
        _check(self._lib.wdg_compute_returns(self._h, float(gamma), C.c_void_p(_ptr(out)), st))
        return out


class Session:
    """wd_session (proj/include/warp/warp_c.h:51-86) on the device path."""

    def __init__(self, config_json: str = "{}", path: Optional[str] = None):
        self._lib = _load()
        h = C.c_void_p()
        if path is not None:
            _check(self._lib.wdg_session_open_file(path.encode(), C.byref(h)))
        else:
            _check(self._lib.wdg_session_open(config_json.encode(), C.byref(h)))
        self._h = h

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wdg_session_close(self._h)
            self._h = None

    def set_seed(self, seed: int):
        _check(self._lib.wdg_session_set_seed(self._h, int(seed)))

    def set_workers(self, workers: int):
        _check(self._lib.wdg_session_set_workers(self._h, int(workers)))

    def set_output_dir(self, d: str):
        _check(self._lib.wdg_session_set_output_dir(self._h, d.encode()))

    def config_json(self) -> str:
        return self._lib.wdg_session_config_json(self._h).decode()

    def config_hash(self) -> str:
        return self._lib.wdg_session_config_hash(self._h).decode()

    def run_check(self):
        _check(self._lib.wdg_session_run_check(self._h))

    def run_bench_envs(self):
        _check(self._lib.wdg_session_run_bench_envs(self._h))

    def run_bench_agents(self):
        _check(self._lib.wdg_session_run_bench_agents(self._h))

    def run_training(self):
        _check(self._lib.wdg_session_run_training(self._h))

    def report_json(self) -> Optional[str]:
        r = self._lib.wdg_session_report_json(self._h)
        return r.decode() if r else None

    def summary(self) -> Optional[str]:
        r = self._lib.wdg_session_summary(self._h)
        return r.decode() if r else None

    def dump_array(self, name: str, csv_path: str):
        _check(self._lib.wdg_session_dump_array(self._h, name.encode(), csv_path.encode()))


class Workspace:
    """build_workspace (harness.cpp:402-423): store + plan + engine + resets."""

    def __init__(self, cfg: TagConfig, num_envs: int, env_offset: int = 0, stream=None,
                 reference: bool = False):
        """reference=True builds the device TagReference twin as the plan
        (the check's second store, harness.cpp:572-584)."""
        cfg.validate()
        self.cfg = cfg
        self.store = DataStore(num_envs, cfg.num_agents())
        if stream is not None:
            self.store.set_stream(stream)
        if env_offset:
            self.store.set_env_offset(env_offset)
        register_tag_arrays(self.store, cfg)
        self.store.lock()
        self.plan = TagPlan(self.store, cfg, reference=reference)
        self.engine = StepEngine(EngineConfig(num_envs, cfg.num_agents()))
        self.resets = ResetManager(self.store, ResetPolicy(True, tag_zero_on_reset(),
                                                           make_tag_reinit(self.plan)))

    def close(self):
        self.store.close()
