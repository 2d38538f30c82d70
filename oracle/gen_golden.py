"""Generate tests/golden/*.npz by running the REFERENCE interpreter.

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

TEST INFRASTRUCTURE.  Imports skiff from /root/reference/pkg/src (read-only;
only present in the build container, never on the GPU box), parses and
lowers small Juno fixture programs written in the reference's own language
(frontend.py / lower.py), and executes them with
``skiff.runtime.oracle.oracle_execute`` (runtime/oracle.py:28-32).  Inputs
and outputs are stored as .npz fixtures; tests/test_oracle_golden.py then
checks the C restatement (oracle/juno_oracle.c) against them bit-for-bit,
which is what pins the oracle.

Fixture shapes avoid the interpreter's known defects:
accumulators live in output arrays, clamped stencil indices come from index
arrays, and `if v > acc { acc = v }` expresses the Python-builtin max fold.
sqrt/exp/log are not expressible in the reference frontend;
those stages are pinned up to the transcendental only.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _skiff():
    sys.path.insert(0, REF)
    from skiff.frontend import parse
    from skiff.lower import lower
    from skiff.runtime.oracle import oracle_execute
    return parse, lower, oracle_execute


parse, lower, oracle_execute = _skiff()


def run(src: str, entry: str, dcs, args):
    mod, _ = lower(parse(src))
    return oracle_execute(mod, entry, list(dcs), list(args), max_steps=500_000_000)


# ---------------------------------------------------------------- programs
MATMUL = """
#[entry]
fn matmul<n, m, l: usize>(a: f32[n, m], b: f32[m, l]) -> f32[n, l] {
  let res : f32[n, l];
  @outer for i in 0..n {
    @middle for j in 0..l {
      @inner for k in 0..m {
        res[i, j] += a[i, k] * b[k, j];
      }
    }
  }
  return res;
}
"""

GAUSS = """
#[entry]
fn gaussian_smoothing<n, m, gs: usize>(input: f32[n, m], filter: f32[gs, gs],
                                       ri: u64[n, gs], ci: u64[m, gs]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n {
    for c in 0..m {
      for i in 0..gs {
        for j in 0..gs {
          res[r, c] += input[ri[r, i], ci[c, j]] * filter[i, j];
        }
      }
    }
  }
  return res;
}
"""

# dilate (pad 0, acc 0) and erode (pad 1, acc 1) with explicit in-frame masks;
# for in-frame taps v = x*1*1*st == x*st exactly, out of frame v = 0*st / 1*st.
MORPH = """
#[entry]
fn dilate<n, m, sz: usize>(input: f32[n, m], st: f32[sz, sz], ri: u64[n, sz], ci: u64[m, sz],
                           rv: f32[n, sz], cv: f32[m, sz]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n {
    for c in 0..m {
      for i in 0..sz {
        for j in 0..sz {
          let v : f32 = input[ri[r, i], ci[c, j]] * rv[r, i] * cv[c, j] * st[i, j];
          if v > res[r, c] { res[r, c] = v; }
        }
      }
    }
  }
  return res;
}

#[entry]
fn erode<n, m, sz: usize>(input: f32[n, m], st: f32[sz, sz], ri: u64[n, sz], ci: u64[m, sz],
                          rv: f32[n, sz], cv: f32[m, sz]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n { for c in 0..m { res[r, c] = 1.0; } }
  for r in 0..n {
    for c in 0..m {
      for i in 0..sz {
        for j in 0..sz {
          let w : f32 = rv[r, i] * cv[c, j];
          let v : f32 = (input[ri[r, i], ci[c, j]] * w + (1.0 - w)) * st[i, j];
          if v < res[r, c] { res[r, c] = v; }
        }
      }
    }
  }
  return res;
}

#[entry]
fn combine_laplacian<n, m: usize>(d: f32[n, m], e: f32[n, m], x: f32[n, m]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n { for c in 0..m { res[r, c] = d[r, c] + e[r, c] - 2.0 * x[r, c]; } }
  return res;
}

#[entry]
fn sign_image<n, m: usize>(x: f32[n, m]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n { for c in 0..m { if x[r, c] > 0.0 { res[r, c] = 1.0; } } }
  return res;
}

#[entry]
fn difference<n, m: usize>(d: f32[n, m], e: f32[n, m]) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n { for c in 0..m { res[r, c] = d[r, c] - e[r, c]; } }
  return res;
}
"""

GRAD2 = """
#[entry]
fn gradient_sq<n, m, sb: usize>(input: f32[n, m], sx: f32[sb, sb], sy: f32[sb, sb],
                                ri: u64[n, sb], ci: u64[m, sb]) -> f32[n, m] {
  let gx : f32[n, m];
  let gy : f32[n, m];
  for r in 0..n {
    for c in 0..m {
      for i in 0..sb {
        for j in 0..sb {
          gx[r, c] += input[ri[r, i], ci[c, j]] * sx[i, j];
          gy[r, c] += input[ri[r, i], ci[c, j]] * sy[i, j];
        }
      }
    }
  }
  let res : f32[n, m];
  for r in 0..n { for c in 0..m { res[r, c] = gx[r, c] * gx[r, c] + gy[r, c] * gy[r, c]; } }
  return res;
}
"""

MAXG = """
#[entry]
fn max_gradient<n, m: usize>(g: f32[n, m]) -> f32 {
  let mx : f32 = g[0, 0];
  for i in 0..n {
    for j in 0..m {
      if g[i, j] > mx { mx = g[i, j]; }
    }
  }
  return mx;
}
"""

REJECT = """
#[entry]
fn reject_zero_crossings<n, m: usize>(zc: f32[n, m], g: f32[n, m], mx: f32, theta: f32) -> f32[n, m] {
  let res : f32[n, m];
  for r in 0..n {
    for c in 0..m {
      if zc[r, c] > 0.0 && g[r, c] > theta * mx { res[r, c] = 1.0; }
    }
  }
  return res;
}
"""

BFS = """
#[entry]
fn bfs<n, m: usize>(starting: u64[n], nedges: u64[n], edges: u64[m], source: u64) -> i32[n] {
  let cost : i32[n];
  let mask : bool[n];
  let visited : bool[n];
  for i in 0..n { cost[i] = -1; }
  cost[source] = 0;
  mask[source] = true;
  visited[source] = true;
  let again : bool = true;
  while again {
    again = false;
    let updating : bool[n];
    for u in 0..n {
      if mask[u] {
        mask[u] = false;
        let k : u64 = starting[u];
        while k < starting[u] + nedges[u] {
          let v : u64 = edges[k];
          if !visited[v] {
            cost[v] = cost[u] + 1;
            updating[v] = true;
          }
          k = k + 1;
        }
      }
    }
    for v in 0..n {
      if updating[v] {
        mask[v] = true;
        visited[v] = true;
        again = true;
      }
    }
  }
  return cost;
}
"""

# one SRAD iteration's coefficient + update given J and q0sqr (the exp/log
# extract/compress and the statistics are outside the fixture)
SRAD_ITER = """
#[entry]
fn srad_iter<rows, cols: usize>(J: f32[rows, cols], q0sqr: f32, lambda: f32,
                                iN: u64[rows], iS: u64[rows], jW: u64[cols], jE: u64[cols]) -> f32[rows, cols] {
  let dN : f32[rows, cols];
  let dS : f32[rows, cols];
  let dW : f32[rows, cols];
  let dE : f32[rows, cols];
  let c : f32[rows, cols];
  for i in 0..rows {
    for j in 0..cols {
      let Jc : f32 = J[i, j];
      dN[i, j] = J[iN[i], j] - Jc;
      dS[i, j] = J[iS[i], j] - Jc;
      dW[i, j] = J[i, jW[j]] - Jc;
      dE[i, j] = J[i, jE[j]] - Jc;
      let G2 : f32 = (dN[i, j] * dN[i, j] + dS[i, j] * dS[i, j] + dW[i, j] * dW[i, j] + dE[i, j] * dE[i, j]) / (Jc * Jc);
      let L : f32 = (dN[i, j] + dS[i, j] + dW[i, j] + dE[i, j]) / Jc;
      let num : f32 = (0.5 * G2) - (0.0625 * (L * L));
      let den : f32 = 1.0 + (0.25 * L);
      let qsqr : f32 = num / (den * den);
      let den2 : f32 = (qsqr - q0sqr) / (q0sqr * (1.0 + q0sqr));
      c[i, j] = 1.0 / (1.0 + den2);
      if c[i, j] < 0.0 { c[i, j] = 0.0; }
      if c[i, j] > 1.0 { c[i, j] = 1.0; }
    }
  }
  let res : f32[rows, cols];
  for i in 0..rows {
    for j in 0..cols {
      let D : f32 = c[i, j] * dN[i, j] + c[iS[i], j] * dS[i, j] + c[i, j] * dW[i, j] + c[i, jE[j]] * dE[i, j];
      res[i, j] = J[i, j] + 0.25 * lambda * D;
    }
  }
  return res;
}
"""

BP_ADJUST = """
#[entry]
fn adjust_weights<ndelta, nly: usize>(delta: f32[ndelta], ly: f32[nly], w: f32[nly, ndelta],
                                      oldw: f32[nly, ndelta]) -> f32[nly, ndelta] {
  let res : f32[nly, ndelta];
  for k in 0..nly {
    for j in 0..ndelta {
      if j > 0 {
        let new_dw : f32 = 0.3 * delta[j] * ly[k] + 0.3 * oldw[k, j];
        res[k, j] = w[k, j] + new_dw;
      }
    }
  }
  return res;
}

#[entry]
fn layer_sum<n1, n2: usize>(l1: f32[n1], conn: f32[n1, n2]) -> f32[n2] {
  let s : f32[n2];
  for j in 0..n2 {
    for k in 0..n1 {
      s[j] += conn[k, j] * l1[k];
    }
  }
  return s;
}
"""

CAVA_SCALE = """
#[entry]
fn scale<r, c: usize>(input: u8[3, r, c]) -> f32[3, r, c] {
  let res : f32[3, r, c];
  for ch in 0..3 {
    for y in 0..r {
      for x in 0..c {
        res[ch, y, x] = f32(input[ch, y, x]) * 1.0 / 255.0;
      }
    }
  }
  return res;
}

#[entry]
fn transform<r, c: usize>(input: f32[3, r, c], tstw: f32[3, 3]) -> f32[3, r, c] {
  let res : f32[3, r, c];
  for y in 0..r {
    for x in 0..c {
      for ch in 0..3 {
        for q in 0..3 {
          res[ch, y, x] += tstw[ch, q] * input[q, y, x];
        }
      }
    }
  }
  return res;
}
"""


def clamp_idx(n, k):
    h = k // 2
    return np.array([[min(max(r + i - h, 0), n - 1) for i in range(k)] for r in range(n)], np.uint64)


def inframe(n, k):
    h = k // 2
    return np.array([[1.0 if 0 <= r + i - h < n else 0.0 for i in range(k)] for r in range(n)], np.float32)


def gen_matmul(rng):
    out = {}
    for tag, (n, m, l) in {"8x8x8": (8, 8, 8), "5x13x7": (5, 13, 7), "16x16x16": (16, 16, 16)}.items():
        a = rng.uniform(-1, 1, (n, m)).astype(np.float32)
        b = rng.uniform(-1, 1, (m, l)).astype(np.float32)
        out[f"{tag}_a"], out[f"{tag}_b"] = a, b
        out[f"{tag}_res"] = run(MATMUL, "matmul", [n, m, l], [a, b])
    # matmul(I2, A) = A
    a = rng.uniform(-1, 1, (2, 2)).astype(np.float32)
    out["eye_a"] = a
    out["eye_res"] = run(MATMUL, "matmul", [2, 2, 2], [np.eye(2, dtype=np.float32), a])
    return out


def gen_edge(rng, n, m, gs, theta=0.1):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2503_10855_b200.workloads import edge_filters, edge_frame
    g, st, sx, sy, _ = edge_filters(gs=gs)
    img = edge_frame(n, m, seed=int(rng.integers(1 << 30)), blobs=4)
    sm = run(GAUSS, "gaussian_smoothing", [n, m, gs], [img, g, clamp_idx(n, gs), clamp_idx(m, gs)])
    ri, ci, rv, cv = clamp_idx(n, 3), clamp_idx(m, 3), inframe(n, 3), inframe(m, 3)
    d = run(MORPH, "dilate", [n, m, 3], [sm, st, ri, ci, rv, cv])
    e = run(MORPH, "erode", [n, m, 3], [sm, st, ri, ci, rv, cv])
    lap = run(MORPH, "combine_laplacian", [n, m], [d, e, sm])
    sgn = run(MORPH, "sign_image", [n, m], [lap])
    zd = run(MORPH, "dilate", [n, m, 3], [sgn, st, ri, ci, rv, cv])
    ze = run(MORPH, "erode", [n, m, 3], [sgn, st, ri, ci, rv, cv])
    zc = run(MORPH, "difference", [n, m], [zd, ze])
    g2 = run(GRAD2, "gradient_sq", [n, m, 3], [sm, sx, sy, ri, ci])
    grad = np.sqrt(g2)  # IEEE f32 sqrt (not expressible in the reference frontend)
    mx = run(MAXG, "max_gradient", [n, m], [grad])
    out = run(REJECT, "reject_zero_crossings", [n, m], [zc, grad, mx, np.float32(theta)])
    return dict(input=img, gaussian=g, structure=st, sx=sx, sy=sy, theta=np.float32(theta), smoothed=sm,
                laplacian=lap, zero_crossings=zc, gradient_sq=g2, gradient=grad, max_gradient=np.float32(mx),
                out=out)


def gen_bfs(rng, n):
    deg = rng.integers(1, 5, n).astype(np.uint64)
    starting = np.zeros(n, np.uint64)
    starting[1:] = np.cumsum(deg[:-1])
    m = int(deg.sum())
    edges = rng.integers(0, n, max(m, 1)).astype(np.uint64)[:m]
    src = int(rng.integers(n))
    cost = run(BFS, "bfs", [n, m], [starting, deg, edges if m else np.zeros(0, np.uint64), np.uint64(src)])
    return dict(starting=starting.astype(np.uint32), no_of_edges=deg.astype(np.uint32),
                edges=edges.astype(np.uint32), source=np.uint32(src), cost=cost)


def gen_srad(rng, rows, cols):
    J = np.exp(rng.uniform(0, 1, (rows, cols))).astype(np.float32)
    q0 = np.float32(rng.uniform(0.05, 0.3))
    iN = np.array([max(i - 1, 0) for i in range(rows)], np.uint64)
    iS = np.array([min(i + 1, rows - 1) for i in range(rows)], np.uint64)
    jW = np.array([max(j - 1, 0) for j in range(cols)], np.uint64)
    jE = np.array([min(j + 1, cols - 1) for j in range(cols)], np.uint64)
    lam = np.float32(0.5)
    res = run(SRAD_ITER, "srad_iter", [rows, cols], [J, q0, lam, iN, iS, jW, jE])
    return dict(J=J, q0sqr=q0, lam=lam, out=res)


def gen_bp(rng, n1, n2):
    delta = rng.uniform(-0.1, 0.1, n2).astype(np.float32)
    ly = rng.random(n1, dtype=np.float32)
    ly[0] = 1.0
    w = rng.random((n1, n2), dtype=np.float32)
    oldw = rng.uniform(-0.05, 0.05, (n1, n2)).astype(np.float32)
    adj = run(BP_ADJUST, "adjust_weights", [n2, n1], [delta, ly, w, oldw])
    s = run(BP_ADJUST, "layer_sum", [n1, n2], [ly, w])
    return dict(delta=delta, ly=ly, w=w, oldw=oldw, adjusted=adj, layer_sum=s)


def gen_cava(rng, r, c):
    raw = rng.integers(0, 256, (3, r, c), dtype=np.uint8)
    sc = run(CAVA_SCALE, "scale", [r, c], [raw])
    tstw = (np.eye(3) + 0.05 * rng.standard_normal((3, 3))).astype(np.float32)
    tr = run(CAVA_SCALE, "transform", [r, c], [sc, tstw])
    return dict(raw=raw, scaled=sc, tstw=tstw, transformed=tr)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(20250314)
    jobs = {
        "matmul": lambda: gen_matmul(rng),
        "edge_12x16_g7": lambda: gen_edge(rng, 12, 16, 7),
        "edge_9x11_g3": lambda: gen_edge(rng, 9, 11, 3),
        "bfs_200": lambda: gen_bfs(rng, 200),
        "bfs_60": lambda: gen_bfs(rng, 60),
        "bfs_1000": lambda: gen_bfs(rng, 1000),
        "srad_iter_10x13": lambda: gen_srad(rng, 10, 13),
        "bp_33x5": lambda: gen_bp(rng, 33, 5),
        "cava_stages_6x8": lambda: gen_cava(rng, 6, 8),
    }
    manifest = []
    for name, fn in jobs.items():
        t = time.time()
        data = fn()
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in data.items()})
        h = hashlib.sha256(open(path, "rb").read()).hexdigest()[:16]
        manifest.append(f"{name}.npz {h}")
        print(f"{name}: {time.time() - t:.1f}s -> {path}")
    with open(os.path.join(OUT, "MANIFEST"), "w") as f:
        f.write("# generated by oracle/gen_golden.py from skiff oracle_execute "
                "(/root/reference/pkg/src/skiff/runtime/oracle.py:28-32)\n")
        f.write("\n".join(manifest) + "\n")


if __name__ == "__main__":
    main()
