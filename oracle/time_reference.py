"""TEST / MEASUREMENT INFRASTRUCTURE: time the reference's own CPU path.

Runs skiff's ``oracle_execute`` (/root/reference/pkg/src/skiff/runtime/
oracle.py:28-32, single-threaded by design) on the fixture programs of
oracle/gen_golden.py at the sizes it can finish (SURVEY.md §8(d) "CPU
baseline" item 1: matmul at small cubes, reported per inner iteration with
the 1024^3 figure extrapolated; BFS at n <= 10^3; one SRAD iteration and the
gaussian stage at toy sizes).  It needs /root/reference, so it runs in the
build container, not on the GPU box; the output is committed as
profiles/r01_reference_interpreter.json.

    PYTHONDONTWRITEBYTECODE=1 python oracle/time_reference.py
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import gen_golden as G  # noqa: E402  (imports skiff from /root/reference)


def timed(src, entry, dcs, args, reps=1):
    mod, _ = G.lower(G.parse(src))
    t = time.perf_counter()
    for _ in range(reps):
        G.oracle_execute(mod, entry, list(dcs), list(args), max_steps=2_000_000_000)
    return (time.perf_counter() - t) / reps


def main():
    out = {"what": "skiff oracle_execute (the reference's CPU path), 1 thread, build container CPU",
           "cpu": os.uname().machine, "host_threads": os.cpu_count()}
    rng = np.random.default_rng(0)
    mm = {}
    for n in (8, 16, 24):
        a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
        s = timed(G.MATMUL, "matmul", [n, n, n], [a, b])
        mm[f"{n}^3"] = {"s": round(s, 4), "us_per_inner_iter": round(s / n ** 3 * 1e6, 2)}
    per = mm["24^3"]["us_per_inner_iter"]
    mm["1024^3_extrapolated_s"] = round(per * 1024 ** 3 / 1e6, 1)
    mm["note"] = ("writes copy the whole result array (oracle.py:167-196), so the per-iteration cost "
                  "grows with n; the 1024^3 figure extrapolates the 24^3 rate and is a lower bound")
    out["matmul"] = mm
    bfs = {}
    for n in (200, 1000):
        g = np.load(os.path.join(G.OUT, f"bfs_{n}.npz"))
        m = int(g["edges"].shape[0])
        s = timed(G.BFS, "bfs", [n, m], [g["starting"].astype(np.uint64), g["no_of_edges"].astype(np.uint64),
                                          g["edges"].astype(np.uint64), np.uint64(int(g["source"]))])
        bfs[f"n={n}"] = {"m": m, "s": round(s, 4), "teps": round(m / s, 1)}
    out["bfs"] = bfs
    print(json.dumps(out, indent=1))
    return out


if __name__ == "__main__":
    res = main()
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "r01_reference_interpreter.json")
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
