"""oracle — TEST INFRASTRUCTURE ONLY.

ctypes bindings for the two CPU checkers of the Tag hot path:

* :class:`OracleWorld` — our plain-C restatement (``oracle/tag_oracle.c``),
  every function citing the reference lines it restates;
* :class:`RefWorld` — the reference itself, compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libwarpref.so`` by
  ``oracle/Makefile`` (driven through ``oracle/ref_driver.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwarpref.so")

DISCRETE, CONTINUOUS = 0, 1
FULL, PARTIAL = 0, 1


class TagConfigC(C.Structure):
    """Mirror of ``wdg_tag_config`` (include/wdg_b200.h) = TagConfig
    (proj/include/warp/tag_env.hpp:29-45)."""

    _fields_ = [
        ("variant", C.c_int32),
        ("obs_mode", C.c_int32),
        ("grid_size", C.c_int64),
        ("world_length", C.c_double),
        ("num_taggers", C.c_int64),
        ("num_runners", C.c_int64),
        ("episode_length", C.c_int64),
        ("tag_radius", C.c_double),
        ("k_nearest", C.c_int64),
        ("tag_reward", C.c_double),
        ("tagged_penalty", C.c_double),
        ("max_speed_tagger", C.c_double),
        ("max_speed_runner", C.c_double),
        ("accel_delta", C.c_double),
        ("turn_delta", C.c_double),
        ("seed", C.c_uint64),
    ]


DEFAULTS = dict(variant=DISCRETE, obs_mode=FULL, grid_size=20, world_length=20.0, num_taggers=2,
                num_runners=10, episode_length=500, tag_radius=1.0, k_nearest=5, tag_reward=1.0,
                tagged_penalty=-1.0, max_speed_tagger=1.0, max_speed_runner=1.0, accel_delta=0.1,
                turn_delta=0.5235987755982988, seed=0)


def make_config(**kw) -> TagConfigC:
    d = dict(DEFAULTS)
    d.update(kw)
    return TagConfigC(**d)


def obs_dim(cfg) -> int:
    a = cfg.num_taggers + cfg.num_runners
    vis = cfg.k_nearest if cfg.obs_mode == PARTIAL else a - 1
    cont = cfg.variant == CONTINUOUS
    return vis * (7 if cont else 4) + (5 if cont else 2) + 1


# name -> (dtype, per-agent? , trailing dims fn)
def array_layout(cfg, num_envs):
    a = cfg.num_taggers + cfg.num_runners
    c = 2 if cfg.variant == CONTINUOUS else 1
    lay = {
        "loc_x": (np.float32, (num_envs, a)),
        "loc_y": (np.float32, (num_envs, a)),
        "is_tagger": (np.uint8, (num_envs, a)),
        "active": (np.uint8, (num_envs, a)),
        "step_count": (np.int32, (num_envs,)),
        "observations": (np.float32, (num_envs, a, obs_dim(cfg))),
        "sampled_actions": (np.int32, (num_envs, a, c)),
        "rewards": (np.float32, (num_envs, a)),
        "done": (np.uint8, (num_envs,)),
        "tag_credits": (np.int32, (num_envs, a)),
        "was_tagged": (np.uint8, (num_envs, a)),
    }
    if cfg.variant == CONTINUOUS:
        lay["speed"] = (np.float32, (num_envs, a))
        lay["direction"] = (np.float32, (num_envs, a))
    return lay


# compare_stores order (proj/src/harness.cpp:536) then the remaining state.
COMPARE_ORDER = ["sampled_actions", "rewards", "done", "observations", "loc_x", "loc_y", "active",
                 "tag_credits", "was_tagged", "step_count", "is_tagger", "speed", "direction"]

_oracle_lib = None
_ref_lib = None


def _dbl_p(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def oracle_lib():
    global _oracle_lib
    if _oracle_lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle library missing: {ORACLE_SO} (run make -C oracle)")
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_mix64.restype = C.c_uint64
        lib.oracle_mix64.argtypes = [C.c_uint64]
        lib.oracle_key_bits.restype = C.c_uint64
        lib.oracle_key_bits.argtypes = [C.c_uint64] + [C.c_int64] * 5
        lib.oracle_uniform.restype = C.c_double
        lib.oracle_uniform.argtypes = [C.c_uint64] + [C.c_int64] * 5
        lib.oracle_substream.restype = C.c_uint64
        lib.oracle_substream.argtypes = [C.c_uint64, C.c_uint64]
        lib.oracle_sample_from_logits.restype = C.c_int32
        lib.oracle_sample_from_logits.argtypes = [C.POINTER(C.c_double), C.c_int64, C.c_double]
        lib.oracle_create.restype = C.c_int
        lib.oracle_create.argtypes = [C.POINTER(TagConfigC), C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]
        lib.oracle_destroy.argtypes = [C.c_void_p]
        lib.oracle_sample.restype = C.c_int
        lib.oracle_sample.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_uint64]
        lib.oracle_step.restype = C.c_int
        lib.oracle_step.argtypes = [C.c_void_p, C.c_int64]
        lib.oracle_track.argtypes = [C.c_void_p]
        lib.oracle_reset_done.restype = C.c_int64
        lib.oracle_reset_done.argtypes = [C.c_void_p]
        lib.oracle_reset_ids.restype = C.c_int
        lib.oracle_reset_ids.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64]
        lib.oracle_rollout.restype = C.c_int
        lib.oracle_rollout.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64]
        lib.oracle_array.restype = C.c_void_p
        lib.oracle_array.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_int64)]
        lib.oracle_episodes.restype = C.c_int64
        lib.oracle_episodes.argtypes = [C.c_void_p, C.c_int64]
        lib.oracle_stats.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int32]
        I64P = C.POINTER(C.c_int64)
        lib.oracle_policy_param_count.restype = C.c_int64
        lib.oracle_policy_param_count.argtypes = [C.c_int64, I64P, C.c_int32, C.c_int64, C.c_int64]
        lib.oracle_policy_init.restype = C.c_int
        lib.oracle_policy_init.argtypes = [C.c_uint64, C.c_int64, I64P, C.c_int32, C.c_int64, C.c_int64,
                                           C.POINTER(C.c_double), C.c_int64]
        lib.oracle_policy_forward.restype = C.c_int
        lib.oracle_policy_forward.argtypes = [C.POINTER(C.c_double), C.c_int64, I64P, C.c_int32, C.c_int64,
                                              C.c_int64, C.POINTER(C.c_float), C.c_int64,
                                              C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.oracle_sinf_replica.restype = C.c_float
        lib.oracle_sinf_replica.argtypes = [C.c_float]
        lib.oracle_cosf_replica.restype = C.c_float
        lib.oracle_cosf_replica.argtypes = [C.c_float]
        lib.oracle_trig_mismatches.restype = C.c_int64
        lib.oracle_trig_mismatches.argtypes = [C.c_float, C.c_float, C.c_uint32]
        lib.oracle_logp.restype = None
        lib.oracle_compute_returns.restype = None
        lib.oracle_logp.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_int64, C.c_int64, C.c_int64,
                                    C.POINTER(C.c_double)]
        lib.oracle_compute_returns.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                               C.c_int64, C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_double)]
        _oracle_lib = lib
    return _oracle_lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference build missing: {REF_SO} (run make -C oracle ref)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_set_fault_bias.argtypes = [C.c_float]
        lib.ref_world_create.restype = C.c_int
        lib.ref_world_create.argtypes = [C.POINTER(TagConfigC), C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]
        lib.ref_world_destroy.argtypes = [C.c_void_p]
        lib.ref_world_sample.restype = C.c_int
        lib.ref_world_sample.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_uint64]
        lib.ref_world_step.restype = C.c_int
        lib.ref_world_step.argtypes = [C.c_void_p, C.c_int64]
        lib.ref_world_reset.restype = C.c_int
        lib.ref_world_reset.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        lib.ref_world_reset_ids.restype = C.c_int
        lib.ref_world_reset_ids.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_int64]
        lib.ref_world_rollout.restype = C.c_int
        lib.ref_world_rollout.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.c_int64, C.c_uint64]
        lib.ref_world_pull.restype = C.c_int
        lib.ref_world_pull.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
        lib.ref_world_push.restype = C.c_int
        lib.ref_world_push.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int64]
        lib.ref_world_episodes.restype = C.c_int64
        lib.ref_world_episodes.argtypes = [C.c_void_p, C.c_int64]
        lib.ref_hw_threads.restype = C.c_int
        lib.ref_bench_sharded.restype = C.c_int
        lib.ref_bench_sharded.argtypes = [C.POINTER(TagConfigC), C.c_int64, C.c_int, C.c_int64, C.c_int64,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        for fn in ("ref_bench_sharded_total", "ref_bench_engine"):
            f = getattr(lib, fn)
            f.restype = C.c_int
            f.argtypes = [C.POINTER(TagConfigC), C.c_int64, C.c_int, C.c_int64, C.c_int64,
                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        if hasattr(lib, "ref_config_canonical"):
            lib.ref_config_canonical.restype = C.c_int64
            lib.ref_config_canonical.argtypes = [C.c_char_p, C.c_int32, C.c_char_p, C.c_int64]
        I64P = C.POINTER(C.c_int64)
        lib.ref_policy_init.restype = C.c_int
        lib.ref_policy_init.argtypes = [C.c_uint64, C.c_int64, I64P, C.c_int32, C.c_int64, C.c_int64,
                                        C.POINTER(C.c_double), C.c_int64]
        lib.ref_policy_forward.restype = C.c_int
        lib.ref_policy_forward.argtypes = [C.POINTER(C.c_double), C.c_int64, I64P, C.c_int32, C.c_int64,
                                           C.c_int64, C.POINTER(C.c_float), C.c_int64,
                                           C.POINTER(C.c_double), C.POINTER(C.c_double)]
        lib.ref_compute_returns.restype = C.c_int
        lib.ref_compute_returns.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_uint8), C.POINTER(C.c_double),
                                            C.c_int64, C.c_int64, C.c_int64, C.c_double, C.POINTER(C.c_double)]
        _ref_lib = lib
    return _ref_lib


class OracleWorld:
    """The C restatement: a store of ``num_envs`` Tag envs after
    register_tag_arrays (tag_env.cpp:280-341)."""

    def __init__(self, cfg: TagConfigC, num_envs: int, env_offset: int = 0):
        self.lib = oracle_lib()
        self.cfg = cfg
        self.num_envs = num_envs
        self.layout = array_layout(cfg, num_envs)
        h = C.c_void_p()
        st = self.lib.oracle_create(C.byref(cfg), num_envs, env_offset, C.byref(h))
        if st != 0:
            raise ValueError(f"oracle_create failed with status {st}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.oracle_destroy(self.h)
            self.h = None

    def view(self, name):
        """Live numpy view aliasing the oracle's buffer."""
        nb = C.c_int64()
        p = self.lib.oracle_array(self.h, name.encode(), C.byref(nb))
        if not p:
            raise KeyError(name)
        dt, shape = self.layout[name]
        buf = (C.c_char * nb.value).from_address(p)
        return np.frombuffer(buf, dtype=dt).reshape(shape)

    def pull(self, name):
        return self.view(name).copy()

    def push(self, name, arr):
        v = self.view(name)
        v[...] = np.asarray(arr, dtype=v.dtype).reshape(v.shape)

    def sample(self, step, seed, logits=None):
        if logits is not None:
            logits = np.ascontiguousarray(logits, dtype=np.float64)
        return self.lib.oracle_sample(self.h, _dbl_p(logits), step, seed)

    def step(self, step):
        return self.lib.oracle_step(self.h, step)

    def track(self):
        self.lib.oracle_track(self.h)

    def reset_done(self):
        return self.lib.oracle_reset_done(self.h)

    def reset_ids(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        return self.lib.oracle_reset_ids(self.h, ids.ctypes.data_as(C.POINTER(C.c_int64)), len(ids))

    def rollout(self, first_step, n, seed, logits=None):
        if logits is not None:
            logits = np.ascontiguousarray(logits, dtype=np.float64)
        st = self.lib.oracle_rollout(self.h, _dbl_p(logits), first_step, n, seed)
        if st != 0:
            raise ValueError(f"oracle_rollout status {st}")

    def episodes(self, env):
        return self.lib.oracle_episodes(self.h, env)

    def stats(self):
        out = (C.c_double * 8)()
        self.lib.oracle_stats(self.h, out, 8)
        return np.array(out[:], dtype=np.float64)

    def snapshot(self):
        return {n: self.pull(n) for n in self.layout}


class RefWorld:
    """The reference itself (oracle/_ref): build_workspace-equivalent world
    with the StepEngine at worker_count=1, or the sequential TagReference."""

    def __init__(self, cfg: TagConfigC, num_envs: int, sequential: bool = False):
        self.lib = ref_lib()
        self.cfg = cfg
        self.num_envs = num_envs
        self.layout = array_layout(cfg, num_envs)
        h = C.c_void_p()
        st = self.lib.ref_world_create(C.byref(cfg), num_envs, 1 if sequential else 0, C.byref(h))
        if st != 0:
            raise ValueError(f"ref_world_create: {st} {self.lib.ref_last_error().decode()}")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_world_destroy(self.h)
            self.h = None

    def _check(self, st):
        if st != 0:
            raise RuntimeError(f"reference error {st}: {self.lib.ref_last_error().decode()}")

    def pull(self, name):
        dt, shape = self.layout[name]
        out = np.empty(shape, dtype=dt)
        self._check(self.lib.ref_world_pull(self.h, name.encode(), out.ctypes.data, out.nbytes))
        return out

    def push(self, name, arr):
        dt, shape = self.layout[name]
        a = np.ascontiguousarray(np.asarray(arr, dtype=dt).reshape(shape))
        self._check(self.lib.ref_world_push(self.h, name.encode(), a.ctypes.data, a.nbytes))

    def sample(self, step, seed, logits=None):
        if logits is not None:
            logits = np.ascontiguousarray(logits, dtype=np.float64)
        return self.lib.ref_world_sample(self.h, _dbl_p(logits), step, seed)

    def step(self, step):
        self._check(self.lib.ref_world_step(self.h, step))

    def reset_done(self):
        n = C.c_int64()
        self._check(self.lib.ref_world_reset(self.h, C.byref(n)))
        return n.value

    def reset_ids(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        self._check(self.lib.ref_world_reset_ids(self.h, ids.ctypes.data_as(C.POINTER(C.c_int64)), len(ids)))

    def rollout(self, first_step, n, seed, logits=None):
        if logits is not None:
            logits = np.ascontiguousarray(logits, dtype=np.float64)
        self._check(self.lib.ref_world_rollout(self.h, _dbl_p(logits), first_step, n, seed))

    def episodes(self, env):
        return self.lib.ref_world_episodes(self.h, env)

    def snapshot(self):
        return {n: self.pull(n) for n in self.layout}


def ref_set_fault_bias(bias: float):
    ref_lib().ref_set_fault_bias(bias)


def bench_reference_sharded(cfg: TagConfigC, envs_per_thread: int, threads: int, warmup: int, steps: int):
    """Times the reference RolloutDriver loop on `threads` independent
    single-worker worlds. Returns (env_steps_per_s, setup_s, run_s)."""
    lib = ref_lib()
    sps, setup, run = C.c_double(), C.c_double(), C.c_double()
    st = lib.ref_bench_sharded(C.byref(cfg), envs_per_thread, threads, warmup, steps,
                               C.byref(sps), C.byref(setup), C.byref(run))
    if st != 0:
        raise RuntimeError(f"ref_bench_sharded: {st} {lib.ref_last_error().decode()}")
    return sps.value, setup.value, run.value


def bench_reference_total(cfg: TagConfigC, total_envs: int, threads: int, warmup: int, steps: int):
    """The reference RolloutDriver loop over `total_envs` envs split across
    `threads` independent single-worker worlds. (env_steps_per_s, setup_s, run_s)."""
    lib = ref_lib()
    sps, setup, run = C.c_double(), C.c_double(), C.c_double()
    st = lib.ref_bench_sharded_total(C.byref(cfg), total_envs, threads, warmup, steps,
                                     C.byref(sps), C.byref(setup), C.byref(run))
    if st != 0:
        raise RuntimeError(f"ref_bench_sharded_total: {st} {lib.ref_last_error().decode()}")
    return sps.value, setup.value, run.value


def bench_reference_engine(cfg: TagConfigC, num_envs: int, workers: int, warmup: int, steps: int):
    """ONE reference world whose StepEngine runs `workers` threads (may hang at
    workers > 1: run it in a child process). (env_steps_per_s, setup_s, run_s)."""
    lib = ref_lib()
    sps, setup, run = C.c_double(), C.c_double(), C.c_double()
    st = lib.ref_bench_engine(C.byref(cfg), num_envs, workers, warmup, steps,
                              C.byref(sps), C.byref(setup), C.byref(run))
    if st != 0:
        raise RuntimeError(f"ref_bench_engine: {st} {lib.ref_last_error().decode()}")
    return sps.value, setup.value, run.value


def first_divergence(a: dict, b: dict, order=COMPARE_ORDER):
    """compare_stores (proj/src/harness.cpp:533-559): first differing
    (array, env, flat index) in causal order, bitwise."""
    for name in order:
        if name not in a or name not in b:
            continue
        x, y = a[name], b[name]
        xb = x.reshape(x.shape[0], -1).view(np.uint8) if x.ndim > 1 else x.reshape(-1, 1).view(np.uint8)
        yb = y.reshape(y.shape[0], -1).view(np.uint8) if y.ndim > 1 else y.reshape(-1, 1).view(np.uint8)
        if xb.shape != yb.shape:
            return (name, -1, -1)
        diff = np.nonzero((xb != yb).any(axis=1))[0]
        if len(diff):
            e = int(diff[0])
            flat = int(np.nonzero(xb[e] != yb[e])[0][0]) // x.dtype.itemsize
            return (name, e, flat)
    return None


# ---- policy network (proj/src/policy_model.cpp) ------------------------------
class PolicyDims:
    """PolicyDims (policy_model.hpp:20-28)."""

    def __init__(self, obs_dim, hidden=(64, 64), num_categories=1, num_choices=1):
        self.obs_dim = int(obs_dim)
        self.hidden = [int(h) for h in hidden]
        self.num_categories = int(num_categories)
        self.num_choices = int(num_choices)

    def _h(self):
        return (C.c_int64 * len(self.hidden))(*self.hidden)

    def args(self):
        return (self.obs_dim, self._h(), len(self.hidden), self.num_categories, self.num_choices)

    def logits_width(self):
        return self.num_categories * self.num_choices


def policy_param_count(dims: PolicyDims) -> int:
    return int(oracle_lib().oracle_policy_param_count(*dims.args()))


def policy_init(seed: int, dims: PolicyDims, ref: bool = False) -> np.ndarray:
    """init_policy flattened in for_each_param order: the C restatement, or
    the reference itself (ref=True)."""
    n = policy_param_count(dims)
    out = np.zeros(n, dtype=np.float64)
    fn = ref_lib().ref_policy_init if ref else oracle_lib().oracle_policy_init
    st = fn(seed, *dims.args(), _dbl_p(out), n)
    if st != 0:
        raise ValueError(f"policy init failed with status {st}")
    return out


def policy_forward(params: np.ndarray, dims: PolicyDims, obs: np.ndarray, ref: bool = False):
    """forward over f32 rows [rows, obs_dim] -> (logits [rows, C*V], values [rows])."""
    obs = np.ascontiguousarray(obs, dtype=np.float32).reshape(-1, dims.obs_dim)
    params = np.ascontiguousarray(params, dtype=np.float64)
    rows = obs.shape[0]
    logits = np.zeros((rows, dims.logits_width()), dtype=np.float64)
    values = np.zeros(rows, dtype=np.float64)
    fn = ref_lib().ref_policy_forward if ref else oracle_lib().oracle_policy_forward
    st = fn(_dbl_p(params), *dims.args(), obs.ctypes.data_as(C.POINTER(C.c_float)), rows,
            _dbl_p(logits), _dbl_p(values))
    if st != 0:
        raise ValueError(f"policy forward failed with status {st}")
    return logits, values


def tag_policy_logits(world, cfg, params_tagger, params_runner, dims: PolicyDims, ref: bool = False):
    """RolloutDriver::forward_policies (harness.cpp:445-476) on a world's
    current observations: taggers [0, T) use params_tagger, runners the other."""
    E = world.num_envs
    A = cfg.num_taggers + cfg.num_runners
    T = cfg.num_taggers
    obs = world.pull("observations").reshape(E, A, dims.obs_dim)
    W = dims.logits_width()
    logits = np.zeros((E, A, W), dtype=np.float64)
    if params_runner is None or params_runner is params_tagger:
        lg, _ = policy_forward(params_tagger, dims, obs.reshape(-1, dims.obs_dim), ref)
        logits[:] = lg.reshape(E, A, W)
    else:
        lt, _ = policy_forward(params_tagger, dims, obs[:, :T].reshape(-1, dims.obs_dim), ref)
        lr, _ = policy_forward(params_runner, dims, obs[:, T:].reshape(-1, dims.obs_dim), ref)
        logits[:, :T] = lt.reshape(E, T, W)
        logits[:, T:] = lr.reshape(E, A - T, W)
    return logits.reshape(-1)


def tag_policy_forward(world, cfg, params_tagger, params_runner, dims: PolicyDims, ref: bool = False):
    """(logits [E*A*C*V], values [E*A]) of forward_policies on a world's obs."""
    E = world.num_envs
    A = cfg.num_taggers + cfg.num_runners
    T = cfg.num_taggers
    obs = world.pull("observations").reshape(E, A, dims.obs_dim)
    W = dims.logits_width()
    logits = np.zeros((E, A, W), dtype=np.float64)
    values = np.zeros((E, A), dtype=np.float64)
    if params_runner is None or params_runner is params_tagger:
        lg, v = policy_forward(params_tagger, dims, obs.reshape(-1, dims.obs_dim), ref)
        logits[:], values[:] = lg.reshape(E, A, W), v.reshape(E, A)
    else:
        lt, vt = policy_forward(params_tagger, dims, obs[:, :T].reshape(-1, dims.obs_dim), ref)
        lr, vr = policy_forward(params_runner, dims, obs[:, T:].reshape(-1, dims.obs_dim), ref)
        logits[:, :T], values[:, :T] = lt.reshape(E, T, W), vt.reshape(E, T)
        logits[:, T:], values[:, T:] = lr.reshape(E, A - T, W), vr.reshape(E, A - T)
    return logits.reshape(-1), values.reshape(-1)


def logp_of(logits: np.ndarray, actions: np.ndarray, C: int, V: int) -> np.ndarray:
    """category_stats(...).logp summed over categories (trainer.cpp:386-392)."""
    rows = actions.size // C
    lg = np.ascontiguousarray(logits, dtype=np.float64)
    ac = np.ascontiguousarray(actions, dtype=np.int32)
    out = np.zeros(rows, dtype=np.float64)
    oracle_lib().oracle_logp(_dbl_p(lg), ac.ctypes.data_as(C_i32p()), rows, C, V, _dbl_p(out))
    return out


def C_i32p():
    return C.POINTER(C.c_int32)


def compute_returns(rewards, done, bootstrap, gamma: float, ref: bool = False) -> np.ndarray:
    """compute_returns (trainer.cpp:73-88); rewards [T,E,A], done [T,E], bootstrap [E,A]."""
    r = np.ascontiguousarray(rewards, dtype=np.float32)
    d = np.ascontiguousarray(done, dtype=np.uint8)
    b = np.ascontiguousarray(bootstrap, dtype=np.float64)
    T, E, A = r.shape
    out = np.zeros((T, E, A), dtype=np.float64)
    fn = ref_lib().ref_compute_returns if ref else oracle_lib().oracle_compute_returns
    st = fn(r.ctypes.data_as(C.POINTER(C.c_float)), d.ctypes.data_as(C.POINTER(C.c_uint8)), _dbl_p(b),
            T, E, A, float(gamma), _dbl_p(out))
    if ref and st:
        raise ValueError(f"compute_returns failed with status {st}")
    return out


def collect(world, cfg, params_tagger, params_runner, dims: PolicyDims, horizon: int, first_step: int,
            seed: int):
    """Trainer::collect (trainer.cpp:315-403) on the oracle world: per step
    the pre-step obs and values, the sampled actions / active flags / logp at
    sample time, rewards and done before reset; then the bootstrap values."""
    E = world.num_envs
    A = cfg.num_taggers + cfg.num_runners
    Cc, V = dims.num_categories, dims.num_choices
    out = {k: [] for k in ("obs", "actions", "rewards", "done", "active", "values", "logp")}
    for t in range(horizon):
        out["obs"].append(world.pull("observations").copy())
        logits, values = tag_policy_forward(world, cfg, params_tagger, params_runner, dims)
        out["values"].append(values.reshape(E, A))
        world.sample(first_step + t, seed, logits)
        acts = world.pull("sampled_actions").copy()
        out["actions"].append(acts)
        out["active"].append(world.pull("active").copy())
        out["logp"].append(logp_of(logits, acts, Cc, V).reshape(E, A))
        world.step(first_step + t)
        world.track()
        out["rewards"].append(world.pull("rewards").copy())
        out["done"].append(world.pull("done").copy())
        world.reset_done()
    res = {k: np.stack(v) for k, v in out.items()}
    res["bootstrap"] = tag_policy_forward(world, cfg, params_tagger, params_runner, dims)[1].reshape(E, A)
    return res


_LIBM_REPLICA = None


def libm_matches_replica(stride: int = 997) -> bool:
    """True when this host's libm sinf/cosf are the glibc FMA variant that the
    device replica follows (checked on every `stride`-th float in [-2pi, 2pi])."""
    global _LIBM_REPLICA
    if _LIBM_REPLICA is None:
        _LIBM_REPLICA = oracle_lib().oracle_trig_mismatches(0.0, 6.2831855, stride) == 0
    return _LIBM_REPLICA


def ref_config_canonical(text: str, hash: bool = False):
    """The reference's RunConfig::from_string(text).to_json_string() /
    config_hash() (harness.cpp:279-322); (status, string)."""
    lib = ref_lib()
    if not hasattr(lib, "ref_config_canonical"):
        return None, None
    buf = C.create_string_buffer(1 << 16)
    n = lib.ref_config_canonical(text.encode(), 1 if hash else 0, buf, len(buf))
    return (0, buf.value.decode()) if n >= 0 else (int(-n), None)
