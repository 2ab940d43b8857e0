"""GPU edge cases and alternative kernel paths, against the oracle."""

import os
import subprocess
import sys

import numpy as np
import pytest

import eikfld_oracle as orc
from conftest import REPO, rng_for

pytestmark = pytest.mark.gpu


def _grid(counts, h=1.0, origin=None):
    from paper_1112_3010_b200 import GridSpec

    return GridSpec(origin or (0.0,) * len(counts), h, counts)


@pytest.mark.parametrize("counts,k,tau", [
    ((2, 2), 1, 1.0),            # smallest grid
    ((3, 17), 4, 1.3),           # odd, unequal axes
    ((17, 3), 4, 1.3),
    ((33, 64), 30, 2.0),         # non power of two c0
    ((64, 33), 30, 2.0),
    ((5, 6, 7), 9, 1.1),         # odd 3-D
    ((2, 2, 2), 2, 1.0),
    ((40,), 3, 0.7),             # 1-D
    ((2,), 1, 0.7),
])
def test_odd_and_tiny_shapes(cuda_ok, counts, k, tau):
    from paper_1112_3010_b200 import engine

    grid = _grid(counts)
    nodes = np.sort(rng_for(sum(counts)).choice(grid.num_nodes, k, replace=False))
    dt = engine.DistanceTransform(grid, tau, grad=True, hess=len(counts) == 2)
    out = dt.run_host(nodes)
    ref = orc.run_config_unchecked(nodes, counts, 1.0, tau, want_hessian=len(counts) == 2)
    keep = ref["phi"] >= 1e-5 * ref["phi"].max()
    rel = lambda a, b: (np.abs(a - b)[keep] / np.maximum(np.abs(b[keep]), 1.0)).max()  # noqa: E731
    assert rel(out["S"], ref["S"]) <= 1e-9
    for a in range(len(counts)):
        assert rel(out["grad"][a], ref["grad"][a]) <= 1e-9
    if len(counts) == 2:
        for i in range(3):
            assert rel(out["hess"][i], ref["hess"][i]) <= 1e-9


def test_every_node_a_source(cuda_ok):
    """Dense impulse field (K = N): phi >= 1 everywhere, S <= 0 (tests/test_distance.py:66-69 style)."""
    from paper_1112_3010_b200 import engine

    grid = _grid((24, 20))
    dt = engine.DistanceTransform(grid, 0.5, grad=True)
    out = dt.run_host(np.arange(grid.num_nodes))
    ref = orc.run_config_unchecked(np.arange(grid.num_nodes), grid.counts, 1.0, 0.5)
    assert np.abs(out["S"] - ref["S"]).max() <= 1e-12
    assert (out["S"] <= 1e-12).all() and out["n_underflow"] == 0


def test_sources_in_one_row_and_corner(cuda_ok):
    from paper_1112_3010_b200 import engine

    grid = _grid((48, 40))
    nodes = np.array([0, 5, 6, 39])  # row 0 only, includes both corners of the row
    dt = engine.DistanceTransform(grid, 2.0, grad=True)
    out = dt.run_host(nodes)
    ref = orc.run_config_unchecked(nodes, grid.counts, 1.0, 2.0)
    keep = ref["phi"] >= 1e-5 * ref["phi"].max()
    assert (np.abs(out["S"] - ref["S"])[keep]).max() <= 1e-9 * np.abs(ref["S"][keep]).max()


def test_invalid_inputs_rejected(cuda_ok):
    from paper_1112_3010_b200 import PointSet, PrecisionConfig, ValidationError, _native, distance

    grid = _grid((16, 16))
    plan = _native.get_plan(grid, 1.0, _native.FIELD_PHI | _native.FIELD_S)
    with pytest.raises(ValidationError):
        plan.run(np.array([3, 3], dtype=np.int64), S=np.empty(256), count=True)  # duplicate
    with pytest.raises(ValidationError):
        plan.run(np.array([256], dtype=np.int64), S=np.empty(256), count=True)   # out of grid
    with pytest.raises(ValidationError):
        plan.run(np.array([], dtype=np.int64), S=np.empty(256), count=True)      # empty
    bad = PointSet(points=np.zeros((1, 2)), snapped_indices=np.array([300]))
    with pytest.raises(ValidationError):
        distance.s_fft(bad, grid, PrecisionConfig.native64(1.0))
    # the invalid-node flag belongs to its own run: valid / invalid / valid /
    # unsorted runs back to back on one plan (the flag is never reset on the
    # device, each run compares it with its own generation)
    good = np.array([5, 77, 200], dtype=np.int64)
    ref = np.empty(256)
    plan.run(good, S=ref, count=True)
    with pytest.raises(ValidationError):
        plan.run(np.array([9, 9], dtype=np.int64), S=np.empty(256), count=True)
    again = np.empty(256)
    plan.run(good, S=again, count=True)
    assert np.array_equal(ref, again)
    with pytest.raises(ValidationError):
        plan.run(np.array([200, 5], dtype=np.int64), S=np.empty(256), count=True)  # unsorted


@pytest.mark.parametrize("env,exact", [({"EIK_ROWDFT": "0"}, False), ({"EIK_TMEM": "0"}, False),
                                       ({"EIK_ROWDFT": "0", "EIK_TMEM": "0"}, False)])
def test_alternative_kernel_paths_agree(cuda_ok, env, exact):
    """The node-list walk inside the column kernel (EIK_ROWDFT=0; exact table
    twiddles instead of the row DFT's split W^{col tl} W^{col q tpr} products)
    and the register-resident column kernel (EIK_TMEM=0, radix 8 instead of 16)
    agree with the default path to T1/T3 tolerance."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1112_3010_b200 import engine, workloads
d = workloads.c2(seed=2, n=512, k=4096, radius=150.0, tau=2.0)
dt = engine.DistanceTransform(d["grid"], 2.0, grad=True, hess=True, sign=True)
sn, sw = dt.sign_inputs(d["curve"])
o = dt.run_host(d["points"].distinct_nodes(), sign_nodes=sn, sign_weights=sw)
np.savez(sys.argv[1], S=o["S"], mu=o["mu"], h=np.stack(o["hess"]), g=np.stack(o["grad"]))
''' % REPO
    outs = []
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        for i, e in enumerate(({}, env)):
            f = os.path.join(d, f"o{i}.npz")
            subprocess.run([sys.executable, "-c", code, f], check=True, env={**os.environ, **e})
            outs.append(np.load(f))
        # T1 conditioning mask: phi/phi_max >= 1e-5  <=>  S <= S_min + tau ln(1e5)
        S0 = outs[0]["S"]
        keep = S0 <= np.nanmin(S0) + 2.0 * np.log(1e5)
        for k in ("S", "mu", "h", "g"):
            a, b = outs[0][k], outs[1][k]
            if exact:
                assert np.array_equal(a, b, equal_nan=True), k
            elif k == "mu":
                assert np.abs(a - b).max() <= 1e-12, k
            else:
                m = keep if a.ndim == 1 else np.broadcast_to(keep, a.shape)
                assert (np.abs(a - b)[m] / np.maximum(np.abs(a[m]), 1.0)).max() <= 1e-9, k


def test_tau_sweep_matches_single_tau_runs(cuda_ok):
    """One delta transform, nine tau values: each S_tau equals the single-tau
    pipeline bit for bit and the oracle to T1 tolerance."""
    from paper_1112_3010_b200 import engine

    grid = _grid((96, 80))
    nodes = np.sort(rng_for(13).choice(grid.num_nodes, 150, replace=False))
    taus = [0.5 * (i + 2) for i in range(9)]  # 1.0 .. 5.0 (> MAXC: two chunks)
    outs, n_uf = engine.TauSweep(grid, taus).run_host(nodes)
    assert len(outs) == 9
    for tau, S in zip(taus, outs):
        single = engine.DistanceTransform(grid, tau, grad=False).run_host(nodes)["S"]
        assert np.array_equal(S, single, equal_nan=True)
        ref = orc.run_config_unchecked(nodes, grid.counts, 1.0, tau)
        keep = ref["phi"] >= 1e-5 * ref["phi"].max()
        assert (np.abs(S - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1.0)).max() <= 1e-9


def test_tau_sweep_3d_matches_single_tau_runs(cuda_ok):
    """3-D sweep (shared planes pass, chunks of four tau values): every S_tau is
    bit-identical to the single-tau pipeline and within T1 of the oracle."""
    from paper_1112_3010_b200 import engine

    grid = _grid((20, 24, 18))
    nodes = np.sort(rng_for(17).choice(grid.num_nodes, 90, replace=False))
    taus = [0.75, 1.0, 1.5, 2.0, 3.0]  # two chunks
    outs, n_uf = engine.TauSweep(grid, taus).run_host(nodes)
    assert len(outs) == 5
    for tau, S in zip(taus, outs):
        single = engine.DistanceTransform(grid, tau, grad=False).run_host(nodes)["S"]
        assert np.array_equal(S, single, equal_nan=True)
        ref = orc.run_config_unchecked(nodes, grid.counts, 1.0, tau)
        keep = ref["phi"] >= 1e-5 * ref["phi"].max()
        assert (np.abs(S - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1.0)).max() <= 1e-9


@pytest.mark.parametrize("counts", [(40, 33), (17, 16, 15), (64,)])
def test_gpu_classify_matches_scipy_fill(cuda_ok, counts):
    """GPU nearest-unflagged fill + rounding == reference classify (scipy EDT), bit for bit."""
    from paper_1112_3010_b200 import ScalarField, sign

    grid = _grid(counts)
    rng = rng_for(len(counts) * 7)
    mu = rng.uniform(-0.6, 1.6, grid.num_nodes)
    mode = "winding2d" if len(counts) != 3 else "degree3d"
    for frac in (0.02, 0.3, 0.7):
        flagged = np.sort(rng.choice(grid.num_nodes, int(frac * grid.num_nodes), replace=False))
        field = ScalarField(grid, mu, flagged)
        got = sign.classify(field, mode).values
        ref = orc.classify(mu, flagged, counts, mode)
        assert np.array_equal(got, ref)
        got_t = sign.classify(field, mode, threshold=0.4).values
        assert np.array_equal(got_t, orc.classify(mu, flagged, counts, mode, threshold=0.4))
    S = rng.standard_normal(grid.num_nodes)
    sd = sign.signed_distance(ScalarField(grid, S), ScalarField(grid, got)).values
    assert np.array_equal(sd, np.where(got > 0.5, S, -S))


def test_gpu_classify_c2_full_size(cuda_ok):
    """C2: winding field + classify on the GPU vs the oracle's scipy fill on the same mu."""
    from paper_1112_3010_b200 import PrecisionConfig, sign, workloads

    d = workloads.c2()
    mu = sign.winding_field(d["curve"], d["grid"], PrecisionConfig.native64(0.5))
    got = sign.classify(mu, sign.WINDING_2D).values
    ref = orc.classify(mu.values, mu.flagged_nodes, d["grid"].counts, "winding2d")
    assert np.array_equal(got, ref)
    inside = got.mean()
    assert 0.2 < inside < 0.4  # star of radius ~600 in a 2048^2 grid


# ----------------------------------------------------------------- empty / ragged / duplicate inputs


@pytest.mark.parametrize("counts", [(48, 40), (12, 10, 9)])
def test_empty_point_set(cuda_ok, counts):
    """K = 0 is rejected with ValidationError, at the C ABI (eik_run: "empty
    point set") and at the drop-in, where the reference cannot even build the
    point set (R/grid.py:99-102).  An empty ITEM inside a batch is legal (see
    test_ragged_batch_with_empty_item)."""
    from paper_1112_3010_b200 import PointSet, ValidationError, engine

    grid = _grid(counts)
    dt = engine.DistanceTransform(grid, 1.0, grad=True)
    with pytest.raises(ValidationError):
        dt.run_host(np.zeros(0, dtype=np.int64))
    with pytest.raises(ValueError):
        PointSet(points=np.zeros((0, len(counts))), snapped_indices=np.zeros(0, dtype=np.int64))


def test_ragged_batch_with_empty_item(cuda_ok):
    """Items of different K, one of them empty, in one batched launch: each
    item equals its own single-grid run bit for bit."""
    from paper_1112_3010_b200 import engine

    grid = _grid((64, 48))
    rng = rng_for(77)
    ks = [5, 0, 300, 1, 48]
    nodes = [np.sort(rng.choice(grid.num_nodes, k, replace=False)) for k in ks]
    offs = np.cumsum([0] + ks)
    dt = engine.DistanceTransform(grid, 1.5, grad=True, hess=True)
    batch = dt.run_host(np.concatenate(nodes), item_offsets=offs)
    N = grid.num_nodes
    empty = slice(N, 2 * N)  # item 1 has no sources: phi = 0, S = NaN, every node underflows
    assert np.isnan(batch["S"][empty]).all() and batch["underflow"][empty].all()
    for i, nd in enumerate(nodes):
        if not ks[i]:
            continue
        single = dt.run_host(nd)
        sl = slice(i * N, (i + 1) * N)
        assert np.array_equal(single["S"], batch["S"][sl], equal_nan=True)
        for a in range(2):
            assert np.array_equal(single["grad"][a], batch["grad"][a][sl], equal_nan=True)
        for a in range(3):
            assert np.array_equal(single["hess"][a], batch["hess"][a][sl], equal_nan=True)
        ref = orc.run_config_unchecked(nd, grid.counts, 1.0, 1.5)
        keep = ref["phi"] >= 1e-5 * ref["phi"].max()
        assert (np.abs(single["S"] - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1)).max() <= 1e-9
    assert batch["n_underflow"] == int(batch["underflow"].sum())


@pytest.mark.parametrize("counts", [(40, 72), (12, 10, 20)])
def test_batch_row_csr_gaps(cuda_ok, counts):
    """Row CSR built by prep_nodes: empty first and last items, items whose
    only nodes sit in their first or last row (long leading / trailing gaps,
    filled warp-cooperatively), and a dense item; every item equals its own
    single run bit for bit (2-D and 3-D)."""
    from paper_1112_3010_b200 import engine

    grid = _grid(counts)
    N = grid.num_nodes
    last = counts[-1]
    rng = rng_for(91)
    items = [
        np.array([], dtype=np.int64),
        np.array([0], dtype=np.int64),                      # first row only
        np.array([N - 1], dtype=np.int64),                  # last row only
        np.array([N // 2 - 3, N // 2 + last], dtype=np.int64),
        np.sort(rng.choice(N, N // 3, replace=False)),       # dense
        np.array([], dtype=np.int64),
    ]
    offs = np.cumsum([0] + [len(x) for x in items])
    dt = engine.DistanceTransform(grid, 1.5, grad=True)
    batch = dt.run_host(np.concatenate(items), item_offsets=offs)
    for i, nd in enumerate(items):
        sl = slice(i * N, (i + 1) * N)
        if not len(nd):
            assert np.isnan(batch["S"][sl]).all()
            continue
        single = dt.run_host(nd)
        assert np.array_equal(single["S"], batch["S"][sl], equal_nan=True), i
        for a in range(len(counts)):
            assert np.array_equal(single["grad"][a], batch["grad"][a][sl], equal_nan=True), i


def test_duplicate_points_collapse(cuda_ok):
    """Duplicated (and unsnapped) points collapse to one unit impulse per
    node, as PointSet.distinct_nodes does in the reference (R/grid.py:89-121)."""
    from paper_1112_3010_b200 import GridSpec, PointSet, PrecisionConfig
    from paper_1112_3010_b200.distance import s_fft
    from paper_1112_3010_b200.grid import snap_points

    grid = GridSpec((0.0, 0.0), 0.5, (40, 36))
    pts = np.array([[3.0, 4.0], [3.1, 3.9], [3.0, 4.0], [10.2, 7.7], [10.0, 7.5]])
    ps = snap_points(pts, grid)
    assert ps.distinct_nodes().size == 2
    s_dup = s_fft(ps, grid, PrecisionConfig.native64(0.4)).values
    uniq = PointSet.from_node_indices(grid, ps.distinct_nodes())
    s_one = s_fft(uniq, grid, PrecisionConfig.native64(0.4)).values
    assert np.array_equal(s_dup, s_one)
    ref = orc.run_config_unchecked(ps.distinct_nodes(), grid.counts, 0.5, 0.4)
    keep = ref["phi"] >= 1e-5 * ref["phi"].max()  # T1 conditioning mask
    assert (np.abs(s_dup - ref["S"])[keep] / np.maximum(np.abs(ref["S"][keep]), 1.0)).max() <= 1e-9


def test_async_host_runs_match_sync(cuda_ok):
    """EIK_ASYNC: back-to-back queued host-output runs (different inputs,
    different host buffers, chunked D2H overlapping the next run's column
    passes) equal synchronous runs bit for bit once the stream is done."""
    import torch

    from paper_1112_3010_b200 import _native, engine

    grid = _grid((2048, 2048))  # >= 2^22 nodes: the chunked copy-stream path
    dt = engine.DistanceTransform(grid, 2.0, grad=True, hess=True)
    rng = rng_for(5)
    inputs = [np.sort(rng.choice(grid.num_nodes, k, replace=False)) for k in (300, 900, 50)]
    ref = [dt.run_host(nd) for nd in inputs]

    def pinned(n):
        return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()

    N = grid.num_nodes
    outs = [{"S": pinned(N), "grad": [pinned(N), pinned(N)], "hess": [pinned(N) for _ in range(3)]} for _ in inputs]
    st = torch.cuda.current_stream()
    for nd, o in zip(inputs, outs):
        dt.plan.run(nd, S=o["S"], grad=o["grad"], hess=o["hess"], host=True, stream=st.cuda_stream, wait=False)
    torch.cuda.synchronize()
    for r, o in zip(ref, outs):
        assert np.array_equal(r["S"], o["S"], equal_nan=True)
        for a in range(2):
            assert np.array_equal(r["grad"][a], o["grad"][a], equal_nan=True)
        for a in range(3):
            assert np.array_equal(r["hess"][a], o["hess"][a], equal_nan=True)
    assert _native.ASYNC == 0x40


@pytest.mark.parametrize("wave", ["1", "3"])
def test_item_waves_bit_identical(cuda_ok, wave):
    """EIK_WAVE=n (batched 2-D distance runs: column pass + row pass per wave
    of n items) is bit-identical to the whole-batch schedule, for a small
    ragged batch (one empty item) and a batch large enough for the chunked
    device-to-host path (whose item ranges the waves shift)."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1112_3010_b200 import engine
from paper_1112_3010_b200 import GridSpec
res = {}
for tag, counts, ks in (("small", (64, 48), [5, 0, 300, 1, 48, 7, 9]), ("big", (512, 512), [1000] * 20)):
    grid = GridSpec((0.0, 0.0), 1.0, counts)
    rng = np.random.default_rng(5)
    nodes = [np.sort(rng.choice(grid.num_nodes, k, replace=False)) for k in ks]
    offs = np.cumsum([0] + ks)
    dt = engine.DistanceTransform(grid, 0.5 if tag == "big" else 1.5, grad=True, hess=tag == "small")
    o = dt.run_host(np.concatenate(nodes), item_offsets=offs)
    res[tag + "_S"] = o["S"]
    res[tag + "_g"] = np.stack(o["grad"])
    if tag == "small":
        res[tag + "_h"] = np.stack(o["hess"])
    res[tag + "_uf"] = o["underflow"]
np.savez(sys.argv[1], **res)
''' % REPO
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        outs = []
        for i, e in enumerate(({"EIK_WAVE": "0"}, {"EIK_WAVE": wave})):
            f = os.path.join(d, f"o{i}.npz")
            subprocess.run([sys.executable, "-c", code, f], check=True, env={**os.environ, **e})
            outs.append(np.load(f))
        for k in outs[0].files:
            assert np.array_equal(outs[0][k], outs[1][k], equal_nan=True), k


def test_graph_replay_matches_eager(cuda_ok):
    """Repeated device-resident runs are captured once and replayed as a CUDA
    graph (eik_run): replays are bit-identical to eager host runs, read the
    current contents of the input buffers, and a changed argument (another
    output buffer) runs eagerly again."""
    import torch

    from paper_1112_3010_b200 import _native, engine

    grid = _grid((96, 80))
    N = grid.num_nodes
    rng = rng_for(123)
    na = np.sort(rng.choice(N, 60, replace=False)).astype(np.int64)
    nb = np.sort(rng.choice(N, 60, replace=False)).astype(np.int64)
    dt = engine.DistanceTransform(grid, 1.5, grad=True, hess=True)
    ref = {"a": dt.run_host(na), "b": dt.run_host(nb)}
    plan = _native.Plan(2, grid.counts, 1.0, 1.5, engine.field_bits(2, True, True, False), 0)
    dev = torch.device("cuda", 0)
    nodes = torch.from_numpy(na).to(dev)
    f = lambda: torch.empty(N, dtype=torch.float64, device=dev)  # noqa: E731
    S, S2, grad, hess = f(), f(), [f(), f()], [f(), f(), f()]
    # eager, captured, replay, replay on new buffer contents, replay, new S buffer (eager), back
    for i, (which, out) in enumerate([("a", S), ("a", S), ("a", S), ("b", S), ("a", S), ("a", S2), ("b", S)]):
        nodes.copy_(torch.from_numpy(na if which == "a" else nb))
        out.fill_(-1.0)
        plan.run(nodes, S=out, grad=grad, hess=hess, host=False)
        torch.cuda.synchronize()
        r = ref[which]
        assert np.array_equal(out.cpu().numpy(), r["S"], equal_nan=True), i
        for a in range(2):
            assert np.array_equal(grad[a].cpu().numpy(), r["grad"][a], equal_nan=True), i
        for a in range(3):
            assert np.array_equal(hess[a].cpu().numpy(), r["hess"][a], equal_nan=True), i


def test_graph_replay_with_sign_group(cuda_ok):
    """The captured graph of a 2-D run with the sign group (forked onto the
    plan's side stream and joined back) replays bit-identically."""
    import torch

    from paper_1112_3010_b200 import _native, engine, workloads

    d = workloads.c2(seed=2, n=256, k=2048, radius=80.0, tau=1.0)
    grid = d["grid"]
    N = grid.num_nodes
    dt = engine.DistanceTransform(grid, 1.0, grad=True, hess=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    nd = d["points"].distinct_nodes()
    ref = dt.run_host(nd, sign_nodes=sn, sign_weights=sw)
    plan = _native.Plan(2, grid.counts, grid.spacing, 1.0, engine.field_bits(2, True, True, True), 0)
    dev = torch.device("cuda", 0)
    nodes, snodes, sweights = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (nd, sn, sw))
    f = lambda: torch.empty(N, dtype=torch.float64, device=dev)  # noqa: E731
    S, mu, grad, hess = f(), f(), [f(), f()], [f(), f(), f()]
    mask = torch.empty(N, dtype=torch.uint8, device=dev)
    for i in range(4):
        S.fill_(-1.0)
        mu.fill_(-1.0)
        plan.run(nodes, None, 1, snodes, sweights, S=S, grad=grad, hess=hess, mu=mu, mask=mask, host=False)
        torch.cuda.synchronize()
        assert np.array_equal(S.cpu().numpy(), ref["S"], equal_nan=True), i
        assert np.array_equal(mu.cpu().numpy(), ref["mu"]), i
        assert np.array_equal(mask.cpu().numpy(), ref["mask"]), i
        for a in range(3):
            assert np.array_equal(hess[a].cpu().numpy(), ref["hess"][a], equal_nan=True), i


def test_caller_stream_capture(cuda_ok):
    """A caller capturing its own stream (torch.cuda.graph) after warm-up calls
    records eik_run's eager launches into its graph: replaying that graph
    reproduces the eager result, including the sign mask fill."""
    import torch

    from paper_1112_3010_b200 import _native, engine, workloads

    d = workloads.c2(seed=4, n=128, k=1024, radius=40.0, tau=1.0)
    grid = d["grid"]
    N = grid.num_nodes
    dt = engine.DistanceTransform(grid, 1.0, grad=True, sign=True)
    sn, sw = dt.sign_inputs(d["curve"])
    nd = d["points"].distinct_nodes()
    ref = dt.run_host(nd, sign_nodes=sn, sign_weights=sw)
    plan = _native.Plan(2, grid.counts, grid.spacing, 1.0, engine.field_bits(2, True, False, True), 0)
    dev = torch.device("cuda", 0)
    nodes, snodes, sweights = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (nd, sn, sw))
    S = torch.empty(N, dtype=torch.float64, device=dev)
    mu = torch.empty_like(S)
    grad = [torch.empty_like(S), torch.empty_like(S)]
    mask = torch.empty(N, dtype=torch.uint8, device=dev)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(3):  # warm-up: the plan's own graph is captured at the second call
            plan.run(nodes, None, 1, snodes, sweights, S=S, grad=grad, mu=mu, mask=mask, host=False,
                     stream=side.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.run(nodes, None, 1, snodes, sweights, S=S, grad=grad, mu=mu, mask=mask, host=False,
                 stream=torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        S.fill_(-1.0)
        mask.fill_(7)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(S.cpu().numpy(), ref["S"], equal_nan=True)
        assert np.array_equal(mask.cpu().numpy(), ref["mask"])
        assert np.array_equal(grad[1].cpu().numpy(), ref["grad"][1], equal_nan=True)


def test_async_host_path_validates_inputs(cuda_ok):
    """The asynchronous host path (EIK_ASYNC) rejects bad node lists and item
    offsets before queueing anything (host-side checks)."""
    import torch

    from paper_1112_3010_b200 import ValidationError, engine

    grid = _grid((64, 64))
    dt = engine.DistanceTransform(grid, 20.0, grad=False)
    S = torch.empty(grid.num_nodes, dtype=torch.float64, pin_memory=True).numpy()
    for bad in ([5, 3], [1, 1], [-1, 4], [0, grid.num_nodes]):
        with pytest.raises(ValidationError):
            dt.plan.run(np.array(bad, dtype=np.int64), S=S, host=True, wait=False)
    S2 = torch.empty(2 * grid.num_nodes, dtype=torch.float64, pin_memory=True).numpy()
    for offs in ([0, 3, 2], [1, 2, 4], [0, 2, 3]):
        with pytest.raises(ValidationError):
            dt.plan.run(np.array([1, 5, 7, 9], dtype=np.int64), np.array(offs, dtype=np.int64), 2, S=S2,
                        host=True, wait=False)
    dt.plan.run(np.array([1, 5, 7, 9], dtype=np.int64), np.array([0, 2, 4], dtype=np.int64), 2, S=S2, host=True)
    assert np.isfinite(S2).all()
    with pytest.raises(ValidationError):
        dt.plan.run(np.zeros(0, dtype=np.int64), np.zeros(65537, dtype=np.int64), 65536, S=S2, host=True)
