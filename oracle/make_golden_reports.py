"""Reference run reports for the report / CLI parity tests (run in the container where
/root/reference exists; the outputs are committed under tests/golden/reports/).

Writes a small KNRM matrix with the REFERENCE's save_matrix and runs the reference's
own CLI (`python -m numakmeans.cli train ...`) on it, keeping its report text."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "reports")
REF = "/root/reference/pkg/src"

CASES = {
    # name: (rows, d, k, extra CLI args)
    "kpp_prune": (3000, 6, 9, ["--init", "kmeanspp", "--seed", "4"]),
    "forgy_dense": (2500, 4, 7, ["--init", "forgy", "--seed", "2", "--no-prune"]),
    "rp_prune_tol": (2000, 3, 5, ["--init", "random-partition", "--seed", "1", "--tolerance", "3"]),
    # semi-external runs (outofcore.py): the report carries the I/O counters
    "sem_cache": (3000, 6, 9, ["--mode", "sem", "--seed", "4", "-T", "2", "--refresh-start", "2",
                               "--cache-capacity", "48000"]),
    "sem_nocache_pages": (2000, 5, 6, ["--mode", "sem", "--no-cache", "--page-size", "1000",
                                       "--task-size", "300", "-T", "3", "--seed", "3"]),
    "sem_plain": (2500, 4, 7, ["--mode", "sem", "--no-prune", "--seed", "2", "--refresh-start", "1",
                               "--cache-capacity", "20000"]),
}


def main() -> None:
    sys.path.insert(0, REF)
    from numakmeans.matrix import save_matrix  # reference writer: the format under test
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:] or list(CASES)
    for name in names:
        n, d, k, extra = CASES[name]
        rng = np.random.default_rng(100 + n)
        centers = rng.uniform(-6, 6, (k, d))
        x = centers[rng.integers(0, k, n)] + rng.standard_normal((n, d))
        data = os.path.join(OUT, f"{name}.knrm")
        save_matrix(x, data)
        cmd = [sys.executable, "-m", "numakmeans.cli", "train", "--data", f"tests/golden/reports/{name}.knrm",
               "--k", str(k), "--max-iters", "40", *extra]
        env = dict(os.environ, PYTHONPATH=REF)
        rep = subprocess.run(cmd, capture_output=True, text=True, check=True, env=env,
                             cwd=os.path.join(HERE, "..")).stdout
        with open(os.path.join(OUT, f"{name}.report"), "w") as fh:
            fh.write(rep)
        with open(os.path.join(OUT, f"{name}.args"), "w") as fh:
            fh.write(" ".join(["--k", str(k), "--max-iters", "40", *extra]) + "\n")
        print(name, len(rep.splitlines()), "lines")


if __name__ == "__main__":
    main()
