"""Pin the C restatement (oracle/juno_oracle.c) to the reference interpreter.

tests/golden/*.npz were produced by oracle/gen_golden.py, which runs Juno
fixture programs through skiff's ``oracle_execute``
(/root/reference/pkg/src/skiff/runtime/oracle.py:28-32).  Every comparison is
bit-exact (np.array_equal on float32 / int32 arrays).
"""
import numpy as np
import pytest

from conftest import golden


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype, (a.shape, b.shape, a.dtype, b.dtype)
    assert np.array_equal(a.view(np.uint32) if a.dtype == np.float32 else a,
                          b.view(np.uint32) if b.dtype == np.float32 else b), \
        f"max |diff| = {np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)))}"


@pytest.mark.parametrize("tag", ["8x8x8", "5x13x7", "16x16x16"])
def test_matmul_pinned(oracle, tag):
    g = golden("matmul")
    _eq(oracle.matmul(g[f"{tag}_a"], g[f"{tag}_b"]), g[f"{tag}_res"])


def test_matmul_identity_spec_example(oracle):
    # matmul(I2, A) = A
    g = golden("matmul")
    _eq(g["eye_res"], g["eye_a"])
    _eq(oracle.matmul(np.eye(2, dtype=np.float32), g["eye_a"]), g["eye_a"])


@pytest.mark.parametrize("name", ["edge_12x16_g7", "edge_9x11_g3"])
def test_edge_stages_pinned(oracle, name):
    g = golden(name)
    st = oracle.edge_frame(g["input"], g["gaussian"], g["structure"], g["sx"], g["sy"], g["theta"],
                           stages=True)
    _eq(st["smoothed"], g["smoothed"])
    _eq(st["laplacian"], g["laplacian"])
    _eq(st["zero_crossings"], g["zero_crossings"])
    _eq(st["gradient"], g["gradient"])
    assert np.float32(st["max_gradient"]).view(np.uint32) == np.float32(g["max_gradient"]).view(np.uint32)
    _eq(st["out"], g["out"])


@pytest.mark.parametrize("name", ["bfs_60", "bfs_200", "bfs_1000"])
def test_bfs_pinned(oracle, name):
    g = golden(name)
    _eq(oracle.bfs(g["starting"], g["no_of_edges"], g["edges"], int(g["source"])), g["cost"])


def test_srad_iteration_pinned(oracle):
    g = golden("srad_iter_10x13")
    _eq(oracle.srad_iter(g["J"], float(g["q0sqr"]), float(g["lam"])), g["out"])


def test_bp_stages_pinned(oracle):
    g = golden("bp_33x5")
    w, _ = oracle.bp_adjust_weights(g["delta"], g["ly"], g["w"], g["oldw"])
    # the fixture leaves column 0 (the bias unit j=0) at zero: compare j>=1
    _eq(w[:, 1:], g["adjusted"][:, 1:])
    _eq(oracle.bp_layer_sums(g["ly"], g["w"], acc64=False), g["layer_sum"])


def test_cava_stages_pinned(oracle):
    g = golden("cava_stages_6x8")
    sc = oracle.cava_stage("scale", g["raw"])
    _eq(sc, g["scaled"])
    _eq(oracle.cava_stage("transform", sc, g["tstw"]), g["transformed"])


def test_spec_known_answers(oracle):
    # SPEC.md:276 (sum of 1..8 = 36) and :326 (1..1000 = 500500) as matmul
    # reductions: ones(1,n) @ v
    for n, want in ((8, 36.0), (1000, 500500.0)):
        v = np.arange(1, n + 1, dtype=np.float32)[:, None]
        assert oracle.matmul(np.ones((1, n), np.float32), v)[0, 0] == want


def test_fixed_interpreter_accumulator_programs(oracle):
    """tests/golden/fixed_interp.npz comes from skiff's own interpreter with
    the Appendix A dependents defect fixed (oracle/gen_golden_fixed.py):
    the gaussian in its scalar-accumulator form (which the unpatched
    interpreter cannot run) must equal the restatement's smoothed stage, and
    the per-row max fold / abs-sum must equal sequential f32 folds."""
    g = golden("fixed_interp")
    e = golden("edge_12x16_g7")
    st = oracle.edge_frame(g["edge_input"], g["gaussian"], e["structure"], e["sx"], e["sy"], e["theta"],
                           stages=True)
    _eq(st["smoothed"], g["gaussian_acc"])
    x = g["x"]
    rowmax = []
    for r in x:
        mx = r[0]
        for v in r:
            if v > mx:
                mx = v
        rowmax.append(mx)
    _eq(np.asarray(g["rowmax"]), np.array(rowmax, np.float32))
    sums = []
    for r in x:
        acc = np.float32(0.0)
        for v in r:
            acc = np.float32(acc + np.float32(abs(v)))
        sums.append(acc)
    _eq(np.asarray(g["abs_sum"]), np.array(sums, np.float32))


def test_fixed_interpreter_cava_demosaic_denoise(oracle):
    """CAVA's demosaic and 3x3-median denoise as Juno programs (if/else on
    the Bayer site, insertion-sort median with a while loop), run by the
    reference interpreter with the Appendix A fix, against the restatement."""
    from paper_2503_10855_b200 import workloads as W
    g = golden("fixed_interp")
    st = oracle.cava_frame(g["cava_raw"], *W.cava_params(16), stages=True)
    _eq(st["demosaic"], g["cava_demosaic"])
    _eq(st["denoise"], g["cava_denoise"])


def test_fixed_interpreter_srad_q0sqr(oracle):
    """SRAD's q0^2 (f64 sums, one rounding to f32) as a Juno program on the
    fixed reference interpreter, against the restatement."""
    g = golden("fixed_interp")
    got = np.float32(oracle.srad_q0sqr(g["srad_J"]))
    assert got.view(np.uint32) == np.float32(g["srad_q0sqr"]).view(np.uint32), (got, g["srad_q0sqr"])


def test_fixed_interpreter_backprop_errors(oracle):
    """bpnn_output_error / bpnn_hidden_error as Juno programs on the fixed
    reference interpreter (fed the restatement's forward pass: squash needs
    exp), against the restatement's deltas and error sums."""
    g = golden("fixed_interp")
    fw = oracle.bp_train(g["bp_x"], g["bp_iw"], g["bp_hw"], g["bp_t"], g["bp_ipw"], g["bp_hpw"])
    _eq(fw["delta_o"][1:], g["bp_delta_o"][1:])
    _eq(fw["delta_h"][1:], g["bp_delta_h"][1:])
    _eq(np.float32(fw["out_err"]), np.float32(g["bp_out_err"]))
    _eq(np.float32(fw["hid_err"]), np.float32(g["bp_hid_err"]))


def test_fixed_interpreter_cava_tonemap_descale(oracle):
    """CAVA's tone map + descale as a Juno program on the fixed reference
    interpreter (fed the restatement's gamut stage: it needs sqrt)."""
    from paper_2503_10855_b200 import workloads as W
    g = golden("fixed_interp")
    st = oracle.cava_frame(g["cava_raw"], *W.cava_params(16), stages=True)
    _eq(st["gamut"], g["cava_gamut"])
    _eq(st["out"], g["cava_out"])


def test_fixed_interpreter_cava_gamut_around_sqrt(oracle):
    """CAVA's gamut map: radicands and the RBF + affine sums as Juno programs
    on the fixed reference interpreter, IEEE sqrt between them (numpy's f32
    sqrt is correctly rounded, like sqrtf): bit-identical to the
    restatement's gamut stage."""
    from paper_2503_10855_b200 import workloads as W
    g = golden("fixed_interp")
    st = oracle.cava_frame(g["cava_raw"], *W.cava_params(16), stages=True)
    _eq(st["gamut"], g["cava_gamut_juno"])


def test_fixed_interpreter_euler_around_sqrt(oracle):
    """CFD/Euler step factor and flux (walls, far field, interior faces) as
    Juno programs on the fixed reference interpreter, with IEEE sqrt between
    the radicand and sum programs: bit-identical to the restatement."""
    g = golden("fixed_interp")
    _eq(oracle.euler_step_factor(g["eu_vars"], g["eu_areas"]), g["eu_step_factor"])
    _eq(oracle.euler_flux(g["eu_nbrs"], g["eu_normals"], g["eu_ff"], g["eu_vars"]), g["eu_flux"])
    assert (g["eu_nbrs"] == -1).any() and (g["eu_nbrs"] == -2).any()  # both boundary kinds covered
