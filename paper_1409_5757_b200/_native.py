"""ctypes binding of the C ABI in include/efft_b200.h (libefft_b200.so).

The library is built in-tree by ``__graft_entry__.build()`` (csrc/Makefile).
There is no CPU fallback: if the library is missing every transform raises
``NativeLibraryMissing``.
"""

import ctypes
import os

from . import errors

# EFFT_LIB: another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("EFFT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libefft_b200.so")

EFFT_OK = 0
EFFT_C64 = 1
EFFT_C128 = 2
EFFT_R32 = 3
EFFT_FORWARD = -1
EFFT_INVERSE = 1
EFFT_FLAG_CHECK_FINITE = 0x1
EFFT_FLAG_SCALE_INVERSE = 0x2

# status code -> exception class (include/efft_b200.h, reference errors.py)
_STATUS = {
    1: ValueError,
    2: errors.SplitsTooLarge,
    3: errors.SizeConstraintViolation,
    4: errors.BinsizeNotPowerOfTwo,
    5: errors.AllocationFailure,
    6: errors.SizeMismatch,
    7: ValueError,
    8: errors.DeviceError,
    9: errors.DeviceError,
}

# every symbol the header declares
EXPORTED = (
    "efft_plan_create",
    "efft_plan_describe",
    "efft_plan_workspace_bytes",
    "efft_plan_launches",
    "efft_execute",
    "efft_execute_host",
    "efft_release_host_buffers",
    "efft_execute_host_batch",
    "efft_execute_outofcore",
    "efft_outofcore_blocks",
    "efft_nonfinite_seen",
    "efft_plan_destroy",
    "efft_plan_enable_timing",
    "efft_plan_create_columns",
    "efft_permute_swap01",
    "efft_permute_swap12",
    "efft_plan_launch_times",
    "efft_plan_create_sharded",
    "efft_execute_sharded",
    "efft_sharded_split",
    "efft_plan_create_shard_rank",
    "efft_execute_shard_pass",
    "efft_last_error",
    "efft_version",
)

_lib = None


def load():
    """Load libefft_b200.so once (no GPU needed to load)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise errors.NativeLibraryMissing(
            f"{LIB_PATH} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise errors.NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
    vp, i32, i64, u32, sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32,
                             ctypes.c_size_t)
    lib.efft_plan_create.argtypes = [ctypes.POINTER(vp), i64, i32, i32, i32, u32]
    lib.efft_plan_describe.argtypes = [vp, ctypes.c_char_p, sz]
    lib.efft_plan_workspace_bytes.argtypes = [vp, ctypes.POINTER(sz)]
    lib.efft_plan_launches.argtypes = [vp, ctypes.POINTER(i32)]
    lib.efft_execute.argtypes = [vp, vp, vp, vp]
    lib.efft_execute_host.argtypes = [vp, vp, vp, vp]
    lib.efft_release_host_buffers.argtypes = [i32]
    lib.efft_execute_host_batch.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), i32, vp]
    lib.efft_execute_outofcore.argtypes = [i64, i32, i32, i32, u32, vp, vp, ctypes.c_size_t]
    lib.efft_outofcore_blocks.argtypes = [i64, i32, ctypes.c_size_t, ctypes.POINTER(i64)]
    lib.efft_nonfinite_seen.argtypes = [vp, ctypes.POINTER(i32), vp]
    lib.efft_plan_destroy.argtypes = [vp]
    lib.efft_plan_enable_timing.argtypes = [vp, i32]
    lib.efft_plan_create_columns.argtypes = [ctypes.POINTER(vp), i64, i64, i32, i32, i32, i64, i64, u32]
    lib.efft_permute_swap01.argtypes = [vp, vp, i64, i64, i64, i32, vp]
    lib.efft_permute_swap12.argtypes = [vp, vp, i64, i64, i64, i32, vp]
    lib.efft_plan_launch_times.argtypes = [vp, ctypes.POINTER(ctypes.c_float), i32]
    lib.efft_plan_create_sharded.argtypes = [ctypes.POINTER(vp), i64, i32, i32, i32, ctypes.POINTER(i32), u32]
    lib.efft_execute_sharded.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]
    lib.efft_sharded_split.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.efft_plan_create_shard_rank.argtypes = [ctypes.POINTER(vp), i64, i32, i32, i32, i32, i32, u32]
    lib.efft_execute_shard_pass.argtypes = [vp, i32, vp, vp, vp]
    lib.efft_last_error.restype = ctypes.c_char_p
    lib.efft_last_error.argtypes = []
    lib.efft_version.argtypes = []
    for name in EXPORTED:
        if name not in ("efft_last_error",):
            getattr(lib, name).restype = i32
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == EFFT_OK:
        return
    msg = load().efft_last_error().decode(errors="replace")
    exc = _STATUS.get(rc, errors.DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def release_host_buffers(device: int = 0) -> None:
    check(load().efft_release_host_buffers(device), "efft_release_host_buffers")


def outofcore_blocks(n: int, dtype: int, device_bytes: int):
    """(N1, N2, columns per step-1 block, rows per step-2 block) -- host only."""
    b = (ctypes.c_int64 * 4)()
    check(load().efft_outofcore_blocks(n, dtype, device_bytes, b), "efft_outofcore_blocks")
    return tuple(int(v) for v in b)


def execute_outofcore(n: int, dtype: int, direction: int, device: int, flags: int, h_in: int, h_out: int,
                      device_bytes: int) -> None:
    check(load().efft_execute_outofcore(n, dtype, direction, device, flags, h_in, h_out, device_bytes),
          "efft_execute_outofcore")


def permute_swap01(d_in: int, d_out: int, n0: int, n1: int, n2: int, elem: int, stream: int) -> None:
    check(load().efft_permute_swap01(d_in, d_out, n0, n1, n2, elem, stream), "efft_permute_swap01")


def permute_swap12(d_in: int, d_out: int, n0: int, n1: int, n2: int, elem: int, stream: int) -> None:
    check(load().efft_permute_swap12(d_in, d_out, n0, n1, n2, elem, stream), "efft_permute_swap12")


class NativePlan:
    """Owns one efft_plan_t."""

    def __init__(self, n: int, dtype: int, direction: int, device: int, flags: int = 0, *,
                 columns=None):
        lib = load()
        h = ctypes.c_void_p()
        if columns is None:
            check(lib.efft_plan_create(ctypes.byref(h), n, dtype, direction, device, flags),
                  "efft_plan_create")
        else:
            cols, tw_mod, tw_offset = columns
            check(lib.efft_plan_create_columns(ctypes.byref(h), n, cols, dtype, direction, device,
                                               tw_mod, tw_offset, flags),
                  "efft_plan_create_columns")
        self._h = h
        self.n, self.dtype, self.direction, self.device = n, dtype, direction, device

    @property
    def handle(self):
        return self._h

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(4096)
        check(load().efft_plan_describe(self._h, buf, 4096))
        return buf.value.decode()

    def workspace_bytes(self) -> int:
        v = ctypes.c_size_t()
        check(load().efft_plan_workspace_bytes(self._h, ctypes.byref(v)))
        return v.value

    def launches(self) -> int:
        v = ctypes.c_int()
        check(load().efft_plan_launches(self._h, ctypes.byref(v)))
        return v.value

    def execute(self, d_in: int, d_out: int, stream: int) -> None:
        check(load().efft_execute(self._h, d_in, d_out, stream), "efft_execute")

    def execute_host(self, h_in: int, h_out: int, stream: int) -> None:
        check(load().efft_execute_host(self._h, h_in, h_out, stream), "efft_execute_host")

    def execute_host_batch(self, h_in: list, h_out: list, stream: int) -> None:
        """Pipelined end-to-end transforms h_in[k] -> h_out[k] (host pointers)."""
        k = len(h_in)
        arr_in = (ctypes.c_void_p * k)(*h_in)
        arr_out = (ctypes.c_void_p * k)(*h_out)
        check(load().efft_execute_host_batch(self._h, arr_in, arr_out, k, stream), "efft_execute_host_batch")

    def nonfinite_seen(self, stream: int) -> bool:
        v = ctypes.c_int()
        check(load().efft_nonfinite_seen(self._h, ctypes.byref(v), stream))
        return bool(v.value)

    def enable_timing(self, on=True) -> None:
        """on: False/0 off, True = the last execution, int K = average over the last K."""
        check(load().efft_plan_enable_timing(self._h, int(on)))

    def launch_times_ms(self) -> list:
        n = self.launches()
        arr = (ctypes.c_float * n)()
        check(load().efft_plan_launch_times(self._h, arr, n))
        return list(arr)

    def close(self) -> None:
        if self._h:
            load().efft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedPlan:
    """One efft_plan_create_sharded plan: the six-step over G devices of this
    process (device ids may repeat: emulated ranks on one GPU)."""

    def __init__(self, n: int, dtype: int, direction: int, devices, flags: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        devs = (ctypes.c_int * len(devices))(*devices)
        check(lib.efft_plan_create_sharded(ctypes.byref(h), n, dtype, direction, len(devices), devs, flags),
              "efft_plan_create_sharded")
        self._h = h
        self.n, self.dtype, self.direction, self.devices = n, dtype, direction, list(devices)

    def split(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(load().efft_sharded_split(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def workspace_bytes(self) -> int:
        v = ctypes.c_size_t()
        check(load().efft_plan_workspace_bytes(self._h, ctypes.byref(v)))
        return v.value

    def execute(self, d_in: list, d_out: list, streams: list) -> None:
        g = len(self.devices)
        if not (len(d_in) == len(d_out) == len(streams) == g):
            raise ValueError(f"need {g} input, output and stream pointers")
        arr = lambda v: (ctypes.c_void_p * g)(*v)  # noqa: E731
        check(load().efft_execute_sharded(self._h, arr(d_in), arr(d_out), arr(streams)), "efft_execute_sharded")

    def close(self) -> None:
        if self._h:
            load().efft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardRankPlan:
    """One rank's local passes of the sharded six-step (efft_plan_create_shard_rank)."""

    def __init__(self, n: int, dtype: int, direction: int, world: int, rank: int, device: int, flags: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        check(lib.efft_plan_create_shard_rank(ctypes.byref(h), n, dtype, direction, world, rank, device, flags),
              "efft_plan_create_shard_rank")
        self._h = h

    def split(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(load().efft_sharded_split(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def execute_pass(self, which: int, d_in: int, d_out: int, stream: int) -> None:
        check(load().efft_execute_shard_pass(self._h, which, d_in, d_out, stream), "efft_execute_shard_pass")

    def close(self) -> None:
        if self._h:
            load().efft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

