"""The mixed-precision time step on device against the reference.

sphx_step_mixed_device runs step_mixed (dynamics.cpp:136-203) on device-resident
state: the approach's neighbour search, EOS, Newtonian stress (three
grad_normalized), the FP64 rates, kick-drift with periodic wrap, then
update_relative + rebuild_members (approach III) or rebin (I, II). The checker is
the reference library itself (oracle/_ref, compiled from the reference's sources;
oracle.RefMixed drives its MixedState / step_mixed). Tolerance: zero -- after
every step the table, max_dx and every field (x, v, rho, p, e, RelCoords, grid
membership) must equal the reference's bit for bit.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # dim, periodic, approach, ds, n_moving_cut
    (2, (0, 0, 0), 2, 0.02, 0),
    (2, (1, 1, 0), 2, 0.025, 0),
    (2, (1, 0, 0), 2, 0.02, 37),
    (2, (0, 1, 0), 0, 0.025, 0),
    (2, (0, 0, 0), 1, 0.025, 0),
    (3, (1, 1, 1), 2, 0.0625, 0),
    (3, (0, 0, 1), 0, 0.0625, 11),
    (1, (1, 0, 0), 2, 0.004, 0),
]


@pytest.fixture(scope="module")
def ctx():
    import paper_2401_08586_b200 as P
    return P.Context(0)


def _setup(dim, periodic, approach, ds, seed=3):
    rs = O.RefSystem.lattice(dim, ds, 0.3, seed)
    ref = O.RefMixed(rs, periodic, approach)
    rng = np.random.default_rng(seed)
    h = rs.h
    for k in range(dim):
        ref.set("v", k, rng.normal(0.0, 0.2, ref.n))
    ref.set("rho", 0, 1.0 + rng.normal(0.0, 0.02, ref.n))
    ref.set("e", 0, rng.uniform(0.0, 1.0, ref.n))
    return rs, ref, h


def _device_state(ref, dim, cells, h):
    import torch
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    cell_of, start, items = ref.grid_members(cells)
    return {
        "h": h,
        "x": [t(ref.get("x", k)) for k in range(dim)],
        "v": [t(ref.get("v", k)) for k in range(dim)],
        "m": t(ref.get("m")), "rho": t(ref.get("rho")), "p": t(ref.get("p")),
        "e": t(ref.get("e")),
        "rel": [t(ref.get("rel", k)) for k in range(dim)],
        "cell": [t(ref.get("cell", k)) for k in range(dim)],
        "cell_of": t(cell_of), "cell_start": t(start), "items": t(items),
    }


def _compare(ref, st, dim, cells, approach):
    for name in ("x", "v", "rel", "cell"):
        for k in range(dim):
            got = st[name][k].cpu().numpy()
            want = ref.get(name, k)
            assert np.array_equal(got, want), f"{name}[{k}] differs"
    for name in ("rho", "p", "e"):
        assert np.array_equal(st[name].cpu().numpy(), ref.get(name)), f"{name} differs"
    cell_of, start, items = ref.grid_members(cells)
    assert np.array_equal(st["cell_start"].cpu().numpy(), start)
    assert np.array_equal(st["items"].cpu().numpy(), items)
    assert np.array_equal(st["cell_of"].cpu().numpy(), cell_of)


@pytest.mark.parametrize("dim,periodic,approach,ds,cut", CASES)
def test_step_mixed_matches_reference(ctx, dim, periodic, approach, ds, cut):
    import torch

    import paper_2401_08586_b200 as P
    rs, ref, h = _setup(dim, periodic, approach, ds)
    g = P.grid_init(dim, (0, 0, 0), (1, 1, 1), 2.0 * h, periodic)
    cells = int(np.prod([g.counts[k] for k in range(dim)]))
    st = _device_state(ref, dim, cells, h)
    n = ref.n
    cfg = dict(dt=2e-4, c_sound=10.0, rho0=1.0, mu=1e-3, body_force=(0.0, -1.0, 0.5)[:dim],
               n_moving=(n - cut) if cut else 0, evolve_density=True, compute_energy=True)
    dev = torch.device("cuda", 0)
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    items = torch.empty(200 * n, dtype=torch.int32, device=dev)
    for step in range(3):
        want_mx, want_tot = ref.step(**cfg)
        mx, tot = ctx.step_mixed_device(g, approach, st, cfg, off, items)
        torch.cuda.synchronize()
        assert tot == want_tot, f"step {step}: table size"
        woff, wit = ref.table(want_tot)
        assert np.array_equal(off.cpu().numpy(), woff), f"step {step}: offsets"
        assert np.array_equal(items[:tot].cpu().numpy(), wit), f"step {step}: items"
        assert mx == want_mx, f"step {step}: max_dx {mx!r} != {want_mx!r}"
        _compare(ref, st, dim, cells, approach)


def test_step_capacity_leaves_state_untouched(ctx):
    import torch

    import paper_2401_08586_b200 as P
    rs, ref, h = _setup(2, (0, 0, 0), 2, 0.02)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h)
    cells = int(g.counts[0] * g.counts[1])
    st = _device_state(ref, 2, cells, h)
    dev = torch.device("cuda", 0)
    off = torch.empty(ref.n + 1, dtype=torch.int64, device=dev)
    items = torch.empty(10, dtype=torch.int32, device=dev)
    x0 = st["x"][0].clone()
    with pytest.raises(RuntimeError, match="capacity"):
        ctx.step_mixed_device(g, 2, st, dict(dt=1e-4, c_sound=10.0), off, items)
    assert torch.equal(st["x"][0], x0)


def test_step_displacement_error_matches_reference(ctx):
    import torch

    import paper_2401_08586_b200 as P
    rs, ref, h = _setup(2, (1, 1, 0), 2, 0.025)
    g = P.grid_init(2, (0, 0, 0), (1, 1, 1), 2.0 * h, (1, 1, 0))
    cells = int(g.counts[0] * g.counts[1])
    st = _device_state(ref, 2, cells, h)
    dev = torch.device("cuda", 0)
    off = torch.empty(ref.n + 1, dtype=torch.int64, device=dev)
    items = torch.empty(200 * ref.n, dtype=torch.int32, device=dev)
    cfg = dict(dt=0.5, c_sound=10.0)  # displacements of several cells
    with pytest.raises(O.RefError) as want:
        ref.step(**cfg)
    with pytest.raises(RuntimeError) as got:
        ctx.step_mixed_device(g, 2, st, cfg, off, items)
    assert str(got.value) == str(want.value)
