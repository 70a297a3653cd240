"""Per-call latency of the drop-in's small calls on the GPU (one system):
derivative, energy, rk4_step and a 1000-step integrate, given the reference's
own objects -- what a reference caller stepping one system sees (the
reference's derivative-timing window, harness.py:718-726, allows 1e-5 s per
component).  Prints one JSON line."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import oscbench  # noqa: E402

from paper_1702_02207_b200 import oscillator as gpu  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        for _ in range(n // 5):
            fn()
        ts.append((time.perf_counter() - t) / (n // 5))
    return statistics.median(ts)


system = oscbench.build_chain([0.002, 0.002], [20250.0, 20250.0])
state = oscbench.PhaseState((2.0, -3.0), (0.0, 0.0))
out = {
    "derivative_us": per_call(lambda: gpu.derivative(system, state)) * 1e6,
    "energy_us": per_call(lambda: gpu.energy(system, state)) * 1e6,
    "rk4_step_us": per_call(lambda: gpu.rk4_step(system, state, 1e-6)) * 1e6,
    "integrate_1000_steps_us": per_call(lambda: gpu.integrate(system, state, 1e-6, 1000, 1000),
                                        n=500) * 1e6,
    "reference_derivative_us": per_call(lambda: oscbench.derivative(system, state)) * 1e6,
}
out["derivative_us_per_component"] = out["derivative_us"] / 4
print(json.dumps(out))
