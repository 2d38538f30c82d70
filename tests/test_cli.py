"""CLI + tensor JSON interchange (paper_2503_10855_b200/cli.py, tensor_io.py).

The tensor format must be byte-identical to the reference's
(skiff/runtime/values.py:135-168): checked against the reference's own
dump_tensor when skiff is importable here."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2503_10855_b200 import cli, tensor_io

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_SKIFF_PATHS = [p for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref"))
                if os.path.isdir(os.path.join(p, "skiff"))]


def _ref_values():
    for p in _SKIFF_PATHS:
        if p not in sys.path:
            sys.path.append(p)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    try:
        from skiff.runtime import values
    except ImportError:
        pytest.skip("reference skiff package not importable")
    return values


SAMPLES = [
    np.array([[1.5, -0.1, 3e-39], [np.inf, -0.0, 1 / 3]], np.float32),
    np.arange(-3, 3, dtype=np.int32).reshape(2, 3),
    np.array([0, 255, 7], np.uint8),
    np.array([2 ** 63 - 1, -5], np.int64),
    np.array([2 ** 64 - 1], np.uint64),
    np.array([0.1, 1e300], np.float64),
    np.array([True, False]),
    np.float32(0.1),
    np.int64(-7),
]


@pytest.mark.parametrize("i", range(len(SAMPLES)))
def test_tensor_roundtrip_bit_exact(tmp_path, i):
    v = SAMPLES[i]
    p = tmp_path / "t.json"
    tensor_io.dump_tensor(v, str(p))
    back = tensor_io.load_tensor(str(p))
    want = np.asarray(v).astype(np.uint8) if np.asarray(v).dtype == np.bool_ else np.asarray(v)
    assert np.asarray(back).shape == want.shape
    assert np.asarray(back).tobytes() == want.tobytes()


@pytest.mark.parametrize("i", range(len(SAMPLES)))
def test_tensor_files_byte_identical_to_reference(tmp_path, i):
    values = _ref_values()
    v = SAMPLES[i]
    ours, ref = tmp_path / "ours.json", tmp_path / "ref.json"
    tensor_io.dump_tensor(v, str(ours))
    values.dump_tensor(v, str(ref))
    assert ours.read_bytes() == ref.read_bytes()
    a, b = tensor_io.load_tensor(str(ref)), values.load_tensor(str(ours))
    assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    assert type(a) is type(b) or isinstance(a, np.ndarray)


def test_unknown_dtype_rejected(tmp_path):
    p = tmp_path / "bad.json"
    p.write_text(json.dumps({"dtype": "f16", "shape": [1], "data": [1.0]}))
    with pytest.raises(tensor_io.TensorFormatError):
        tensor_io.load_tensor(str(p))


def test_dc_parsing():
    assert cli._parse_dcs(["m=2", "n=1", "l=3"], ("n", "m", "l")) == [1, 2, 3]
    assert cli._parse_dcs(["4", "5"], ("a", "b")) == [4, 5]
    with pytest.raises(ValueError):
        cli._parse_dcs(["n=1"], ("n", "m"))
    with pytest.raises(ValueError):
        cli._parse_dcs(["q=1"], ("n",))


def test_usage_errors_exit_2(tmp_path, capsys):
    assert cli.main(["run", "nope"]) == 2
    assert cli.main(["run", "matmul", "--input", str(tmp_path / "missing.json")]) == 2
    a = tmp_path / "a.json"
    tensor_io.dump_tensor(np.eye(2, dtype=np.float32), str(a))
    assert cli.main(["run", "matmul", "--dc", "n=2", "--input", str(a), "--input", str(a)]) == 2
    assert cli.main(["entries"]) == 0
    assert "matmul<n, m, l>" in capsys.readouterr().out


@pytest.mark.gpu
def test_cli_runs_matmul_identity(tmp_path):
    # SPEC.md:585 run example "matmul 4x4 identity"
    rng = np.random.default_rng(3)
    a = rng.uniform(-1, 1, (4, 4)).astype(np.float32)
    tensor_io.dump_tensor(np.eye(4, dtype=np.float32), str(tmp_path / "i.json"))
    tensor_io.dump_tensor(a, str(tmp_path / "a.json"))
    out = tmp_path / "c.json"
    r = subprocess.run([sys.executable, "-m", "paper_2503_10855_b200", "run", "matmul", "--dc", "n=4", "--dc", "m=4",
                        "--dc", "l=4", "--input", str(tmp_path / "i.json"), "--input", str(tmp_path / "a.json"),
                        "-o", str(out)], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    metrics = json.loads(r.stdout.strip().splitlines()[-1])
    assert metrics["kernel"] == "matmul" and metrics["gpu_launches"] >= 1
    assert metrics["h2d_bytes"] == 128 and metrics["d2h_bytes"] == 64
    # 3xTF32 keeps the fp32 bound of SURVEY §8(d), not bit-exactness:
    # (2*gamma_4 + 8u) * |I||A| = ~16u * |A|
    c = tensor_io.load_tensor(str(out))
    assert c.dtype == np.float32 and c.shape == (4, 4)
    assert np.all(np.abs(c.astype(np.float64) - a) <= 16 * 2.0 ** -24 * np.abs(a))


@pytest.mark.gpu
def test_cli_runs_a_tuple_entry(tmp_path):
    from paper_2503_10855_b200 import workloads as W
    args = W.bp_inputs(64, 16, 1)
    paths = []
    for i, v in enumerate(args):
        p = tmp_path / f"in{i}.json"
        tensor_io.dump_tensor(np.asarray(v), str(p))
        paths += ["--input", str(p)]
    r = subprocess.run([sys.executable, "-m", "paper_2503_10855_b200", "run", "backprop", "--dc", "64", "--dc", "16",
                        "--dc", "1", *paths, "--out-dir", str(tmp_path / "o")], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert len(json.loads(r.stdout.strip().splitlines()[-1])["outputs"]) == 6


_MATMUL_JN = """
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


def _ab_files(tmp_path, n, m, l, schedule):
    rng = np.random.default_rng(11)
    src, sch = tmp_path / "matmul.jn", tmp_path / "matmul.sch"
    src.write_text(_MATMUL_JN)
    sch.write_text(schedule)
    args = []
    for name, shape in (("a", (n, m)), ("b", (m, l))):
        p = tmp_path / f"{name}.json"
        tensor_io.dump_tensor(rng.uniform(-1, 1, shape).astype(np.float32), str(p))
        args += ["--input", str(p)]
    return ["run", "matmul", "--dc", f"n={n}", "--dc", f"m={m}", "--dc", f"l={l}", "--source", str(src),
            "--schedule", str(sch), *args]


def test_oracle_ab_runs_the_reference_interpreter(tmp_path, capsys):
    """SPEC.md:600 ``run --oracle``: the same module and inputs through the
    reference's value-semantics interpreter; the file equals what skiff's
    own oracle_execute + dump_tensor give."""
    values = _ref_values()
    from skiff.runtime.oracle import oracle_execute
    argv = _ab_files(tmp_path, 4, 6, 5, "forkify(*); forkify(*); forkify(*);")
    out = tmp_path / "o.json"
    assert cli.main(argv + ["--oracle", "-o", str(out)]) == 0
    metrics = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert metrics["kernel"] == "skiff.oracle_execute" and metrics["gpu_launches"] == 0
    mod = cli._skiff_module(str(tmp_path / "matmul.jn"), str(tmp_path / "matmul.sch"))
    a, b = tensor_io.load_tensor(str(tmp_path / "a.json")), tensor_io.load_tensor(str(tmp_path / "b.json"))
    ref = tmp_path / "ref.json"
    values.dump_tensor(oracle_execute(mod, "matmul", [4, 6, 5], [a, b]), str(ref))
    assert out.read_bytes() == ref.read_bytes()


def test_oracle_ab_constraint_error_exit_1(tmp_path, capsys):
    # SPEC.md:585 "n=6 chunk-4 -> constraint error", through the reference arm
    _ref_values()
    sch = r"forkify(*); forkify(*); forkify(*); let par = matmul@outer \ matmul@inner; fork-chunk![4](par);"
    argv = _ab_files(tmp_path, 6, 6, 6, sch)
    assert cli.main(argv + ["--oracle", "-o", str(tmp_path / "o.json")]) == 1
    assert "DynConstError" in capsys.readouterr().err


def test_oracle_needs_source(tmp_path):
    a = tmp_path / "a.json"
    tensor_io.dump_tensor(np.eye(2, dtype=np.float32), str(a))
    assert cli.main(["run", "matmul", "--dc", "2", "--dc", "2", "--dc", "2", "--input", str(a), "--input", str(a),
                     "--oracle"]) == 2


@pytest.mark.gpu
def test_oracle_ab_matches_gpu_arm(tmp_path, capsys):
    """The two arms of the A/B on a scheduled Fig. 1 matmul: the GPU kernel
    (3xTF32, re-associated k) within the fp32 bound of the interpreter."""
    _ref_values()
    argv = _ab_files(tmp_path, 64, 48, 40, r"forkify(*); forkify(*); forkify(*); fork-tile![4](matmul);")
    assert cli.main(argv + ["--oracle", "-o", str(tmp_path / "ref.json")]) == 0
    assert cli.main(argv + ["-o", str(tmp_path / "gpu.json")]) == 0
    ref = tensor_io.load_tensor(str(tmp_path / "ref.json")).astype(np.float64)
    gpu = tensor_io.load_tensor(str(tmp_path / "gpu.json")).astype(np.float64)
    a, b = (tensor_io.load_tensor(str(tmp_path / f"{x}.json")).astype(np.float64) for x in "ab")
    u, m = 2.0 ** -24, 48
    gam = m * u / (1 - m * u)
    assert np.all(np.abs(gpu - ref) <= (2 * gam + 8 * u) * (np.abs(a) @ np.abs(b)))


_ACC_JN = """
#[entry]
fn matmul<n, m, l: usize>(a: f32[n, m], b: f32[m, l]) -> f32[n, l] {
  let res : f32[n, l];
  @outer for i in 0..n {
    @middle for j in 0..l {
      let s : f32 = 0.0;
      @inner for k in 0..m {
        s += a[i, k] * b[k, j];
      }
      res[i, j] = s;
    }
  }
  return res;
}
"""


@pytest.mark.gpu
def test_cli_reduction_tree_schedule_reports_its_launch(tmp_path, capsys):
    """A reduction_tree! schedule through the CLI: the metrics line names the
    schedule-parametrised C entry and its K partials, and the result stays
    within the fp32 bound of the exact product."""
    _ref_values()
    sch = ("forkify(*); forkify(*); forkify(*); infer-attributes(*); macro reduction_tree![N](F) { "
           "fork-chunk![N](F); let (outer, inner) = fork-reshape[[0], [1]](F); monoid-reassociate(inner); "
           "let (top, bottom) = fork-fission(outer); } reduction_tree![4](matmul@inner);")
    argv = _ab_files(tmp_path, 64, 128, 96, sch)
    (tmp_path / "matmul.jn").write_text(_ACC_JN)
    assert cli.main(argv + ["-o", str(tmp_path / "gpu.json")]) == 0
    metrics = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert metrics["c_symbol"] == "jb_matmul_sched_f32" and metrics["params"]["tree"] == [4, 1]
    gpu = tensor_io.load_tensor(str(tmp_path / "gpu.json")).astype(np.float64)
    a, b = (tensor_io.load_tensor(str(tmp_path / f"{x}.json")).astype(np.float64) for x in "ab")
    u, m = 2.0 ** -24, 128
    gam = m * u / (1 - m * u)
    assert np.all(np.abs(gpu - a @ b) <= (2 * gam + 8 * u) * (np.abs(a) @ np.abs(b)))
