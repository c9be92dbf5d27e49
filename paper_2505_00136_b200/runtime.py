"""Runtime lifecycle, name-for-name with the reference (taskgp runtime.py:369-403).

The reference's runtime is a work-stealing pool of W Python threads
(runtime.py:144-362).  On B200 the work is scheduled as grouped kernel
launches on CUDA streams inside ``libgpb200``, so "starting the runtime"
means binding a CUDA device (``gpb_init``: device selection, kernel
attributes, streams) and "stopping" it means synchronising and releasing
it (``gpb_finalize``).  The observable contract is kept: one runtime per
process (``AlreadyRunning``), model calls require a live runtime
(``NotRunning``), and ``RuntimeConfig`` validates like the reference.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Callable, TypeVar

from . import _lib
from .errors import InvalidConfig, NotRunning

T = TypeVar("T")

WORKERS_ENV_VAR = "TASKGP_WORKERS"  # runtime.py:36 (accepted for parity)
DEVICE_ENV_VAR = "GPB_DEVICE"


@dataclass(frozen=True)
class RuntimeConfig:
    """Runtime configuration (runtime.py:50-78).

    ``worker_count`` is validated exactly like the reference (None -> the
    ``TASKGP_WORKERS`` variable -> cpu count; must be >= 1) but host threads
    do no math here.  ``device`` selects the CUDA device (default: the
    ``GPB_DEVICE`` variable, else ``LOCAL_RANK``, else 0).
    """

    worker_count: int | None = None
    extra_args: tuple[str, ...] = ()
    device: int | None = None

    def resolved_worker_count(self) -> int:
        count = self.worker_count
        if count is None:
            env = os.environ.get(WORKERS_ENV_VAR)
            if env is not None:
                try:
                    count = int(env)
                except ValueError as exc:
                    raise InvalidConfig(f"{WORKERS_ENV_VAR}={env!r} is not an integer") from exc
            else:
                count = os.cpu_count() or 1
        if count < 1:
            raise InvalidConfig(f"worker_count must be >= 1, got {count}")
        return count

    def resolved_device(self) -> int:
        if self.device is not None:
            return int(self.device)
        for var in (DEVICE_ENV_VAR, "LOCAL_RANK"):
            if os.environ.get(var) is not None:
                return int(os.environ[var])
        return 0


class Runtime:
    """A started device runtime (the handle ``start_runtime`` returns)."""

    def __init__(self, config: RuntimeConfig):
        config.resolved_worker_count()
        self.config = config
        self.device = config.resolved_device()
        lib = _lib.load()
        handle = ctypes.c_void_p()
        _lib.check(lib.gpb_init(self.device, ctypes.byref(handle)))
        self._handle = handle

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._handle

    def is_live(self) -> bool:
        cur = _lib.load().gpb_current()
        return bool(cur) and cur == self._handle.value

    def stop(self) -> None:
        global _current
        if not self.is_live():
            raise NotRunning("runtime is not running")
        _lib.check(_lib.load().gpb_finalize(self._handle))
        if _current is self:
            _current = None


_current: Runtime | None = None


def start_runtime(config: RuntimeConfig | None = None) -> Runtime:
    """Start the process-wide runtime; ``AlreadyRunning`` if one is live."""
    global _current
    rt = Runtime(config or RuntimeConfig())
    _current = rt
    return rt


def stop_runtime() -> None:
    """Stop the live runtime; ``NotRunning`` if there is none."""
    if _current is None or not _current.is_live():
        raise NotRunning("no runtime is running")
    _current.stop()


def current_runtime() -> Runtime | None:
    if _current is not None and _current.is_live():
        return _current
    return None


def require_runtime() -> Runtime:
    rt = current_runtime()
    if rt is None:
        raise NotRunning("this call needs a running runtime (start_runtime())")
    return rt


def run_as_root(fn: Callable[[], T]) -> T:
    """Run ``fn`` under the live runtime (runtime.py:401-403 contract)."""
    require_runtime()
    return fn()
