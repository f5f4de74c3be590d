"""The CPU oracle (oracle/, test infrastructure) timed on the host cores: BASELINE config 3
(N = 128^3, M = 1e6) median of 3 runs and config 4 (N = 256^3, M = 1e7) once, the full transform
each time (O2 spread by plane ownership on all cores, scipy FFT with all workers, deconvolve/crop).
Prints one line per run plus the host facts (profiles/r2_cpu_oracle.txt)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

cores, model = bench._host_cpu()
print(f"host: {cores} usable cores, CPU model {model!r}")
for cfg_name, reps in (("3", 3), ("4", 1)):
    cfg = bench.CONFIGS[cfg_name]
    runs = [bench._oracle_run(cfg, "uniform", cfg["M"]) for _ in range(reps)]
    for t, ts, tf in runs:
        print(f"config {cfg_name}: total {t:.3f} s (spread {ts:.3f} s, FFT + deconvolve {tf:.3f} s) = "
              f"{cfg['M'] / t:.4g} points/s")
    med = statistics.median(r[0] for r in runs)
    print(f"config {cfg_name}: median of {reps}: {med:.3f} s = {cfg['M'] / med:.4g} points/s on {cores} threads")
