"""GPU energy per token (the paper's second headline metric) through the host
library's C ABI (include/msw_host.h, include/modeswitch/energy.hpp): an NVML
power sampler recording the reference's "timestamp_ms,power_w" trace format
and the reference's trapezoid energy_from_power_trace (sim.cpp:10-78)."""
from __future__ import annotations

import ctypes as C

from ._capi import check_host, host_lib


def energy_from_trace(csv_path: str, tokens: int) -> float:
    """Joules per token of a power-trace CSV (reference semantics; DataError -> MswError code 3)."""
    j = C.c_double()
    check_host(host_lib().msw_energy_from_trace(csv_path.encode(), int(tokens), C.byref(j)))
    return j.value


class PowerSampler:
    """with PowerSampler(device) as ps: ...work...; then ps.finish(tokens) -> J/token.
    Polls NVML every period_ms on a host thread (no effect on the GPU stream)."""

    def __init__(self, device: int = 0, period_ms: float = 10.0, csv_path: str | None = None):
        self.device, self.period_ms, self.csv_path = device, period_ms, csv_path
        self._h = None
        self.joules_per_token = None
        self.counter_joules_per_token = None
        self.samples = 0

    def __enter__(self):
        h = C.c_void_p()
        check_host(host_lib().msw_power_start(self.device, self.period_ms, C.byref(h)))
        self._h = h
        return self

    def finish(self, tokens: int) -> float:
        """J/token by the reference's trapezoid rule over the recorded trace.
        `counter_joules_per_token` is the same window from the driver's
        total-energy counter (None where unsupported)."""
        j, n, cj = C.c_double(), C.c_int32(), C.c_double()
        h, self._h = self._h, None
        check_host(host_lib().msw_power_stop(h, self.csv_path.encode() if self.csv_path else None,
                                             int(tokens), C.byref(j), C.byref(n), C.byref(cj)))
        self.joules_per_token, self.samples = j.value, n.value
        self.counter_joules_per_token = cj.value / tokens if cj.value >= 0 else None
        return j.value

    def __exit__(self, *exc):
        if self._h is not None:  # not finished explicitly: stop and discard (1 token)
            try:
                self.finish(1)
            except Exception:
                pass
        return False
