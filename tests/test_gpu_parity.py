"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by
element, on the same seeded inputs. Run on a B200 with ``pytest -m gpu``.

Inputs come from synth (host generator for the oracle; its bit-identical device
twin for large batches). No expected value here is produced by the CUDA path.
"""
import os

import numpy as np
import pytest
import torch

import synth
from tests._parity import (boost_violations, energy_scale, find_bin_np, hist_check, hist_check_delta, mass_violations,
                           tau_of)

pytestmark = pytest.mark.gpu

LO, HI, NB = 0.25, 300.0, 1000
TDT = {np.float32: torch.float32, np.float64: torch.float64}


@pytest.fixture(scope="module")
def gvx():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2312_02756_b200 as g
    return g


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


def dev(a, dt=None):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def host(t):
    return t.detach().cpu().numpy()


def edge_events(dt):
    """Hand-built PtEtaPhiM pairs covering the degenerate cases of the method."""
    inf, nan = np.inf, np.nan
    rows = [
        # (v1, v2)
        ([30, 0.5, 1.0, 0.105], [0, 0, 0, 0]),                # single vector → m
        ([1, 0, 0, -0.5], [0, 0, 0, 0]),                      # spacelike, negative mass convention
        ([1, 0, 0, -5.0], [2, 0.3, 0.1, -3.0]),               # E² clamp on both (R2)
        ([25, 1.1, 0.3, 0], [25, -1.1, 0.3 - np.pi, 0]),      # back-to-back massless
        ([20, 2.4, -3.0, 0.105], [20, 2.39, -3.01, 0.105]),   # near-collinear
        ([40, 0.0, 0.0, 0.105], [40, 0.0, 0.0, 0.105]),       # exactly collinear
        ([50, 25.0, 0.2, 0.105], [30, -1.0, 2.0, 0.105]),     # |η| beyond the fast domain (cold path)
        ([50, -30.0, 0.2, 0.105], [30, 40.0, 2.0, 0.105]),
        ([50, 1.0, 1e5, 0.105], [30, -1.0, -2e5, 0.105]),     # |φ| ≫ π (R16)
        ([50, 1.0, 7.5, 0.105], [30, -1.0, -7.9, 0.105]),     # φ just outside (−π, π]
        ([0, 0, 0, 91.0], [0, 0, 0, 0.0]),                    # at rest
        ([0, 0, 0, 0], [0, 0, 0, 0]),                         # all zero
        ([nan, 0, 0, 0.1], [3, 0, 0, 0.1]),                   # NaN propagates
        ([3, 0, 0, 0.1], [3, inf, 0, 0.1]),                   # Inf
        ([1e3, 2.5, -3.1, 0.105], [2e3, -2.5, 3.1, 0.105]),   # high pt, edges of acceptance
        ([5, 0.3, 1.0, 10.0], [7, -0.2, -1.0, 80.0]),         # heavy
    ]
    a = np.array([r[0] for r in rows], np.float64).astype(dt)
    b = np.array([r[1] for r in rows], np.float64).astype(dt)
    return a, b


def mixed_inputs(n, dt, seed=12345, first=0):
    v1, v2 = synth.muon_pairs(np.arange(first, first + n), seed=seed, dtype=dt)
    ea, eb = edge_events(dt)
    v1 = np.concatenate([ea, v1, ea])
    v2 = np.concatenate([eb, v2, eb])
    return v1, v2


# ----------------------------------------------------------------------------
# generator twin
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("first", [0, 700_000_123])
def test_synth_device_matches_host(dt, first):
    import synth.device as sd
    n = 50_001
    v1d, v2d = sd.muon_pairs(n, first=first, dtype=TDT[dt])
    v1h, v2h = synth.muon_pairs(np.arange(first, first + n), dtype=dt)
    assert np.array_equal(host(v1d), v1h) and np.array_equal(host(v2d), v2h)
    r1d, r2d = sd.muon_pairs(n, first=first, dtype=TDT[dt], f_res=0.1)  # resonance admixture twin
    r1h, r2h = synth.muon_pairs(np.arange(first, first + n), dtype=dt, f_res=0.1)
    assert np.array_equal(host(r1d), r1h) and np.array_equal(host(r2d), r2h)
    vd, bd = sd.boost_inputs(n, first=first, dtype=TDT[dt])
    vh, bh = synth.boost_inputs(np.arange(first, first + n), dtype=dt)
    assert np.array_equal(host(vd), vh) and np.array_equal(host(bd), bh)


# ----------------------------------------------------------------------------
# K1 invariant mass
# ----------------------------------------------------------------------------

def test_cfg1_mass_65536_f64(gvx, O):
    """BASELINE configs[0]: N = 65536 PtEtaPhiM pairs, fp64, AoS, vs the oracle."""
    v1, v2 = synth.muon_pairs(np.arange(65536), dtype=np.float64)
    m = host(gvx.invariant_mass(dev(v1), dev(v2)))
    mo, e = O.invariant_mass(v1, v2)
    bad = mass_violations(m, mo, e, 1e-12)
    assert bad.size == 0, (bad[:5], m[bad[:5]], mo[bad[:5]])
    rel = np.abs(m * np.abs(m) - mo * np.abs(mo)) / e ** 2
    print(f"cfg1 max |dM2|/E2 = {rel.max():.3e}")
    # quality guard (not the parity bar): the fast f64 math is budgeted at ~1e-15 E^2
    assert rel.max() <= 1e-13


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("coords", ["ptetaphim", "pxpypze"])
def test_mass_parity_layouts(gvx, O, dt, coords):
    n = 3 * 256 * 148 + 37  # several tiles per CTA + a ragged tail
    v1, v2 = mixed_inputs(n, dt)
    if coords == "pxpypze":
        # Cartesian inputs: the boost generator's on-shell vectors, plus the edge rows as given
        a, _ = synth.boost_inputs(np.arange(v1.shape[0]), dtype=dt, seed=5)
        b, _ = synth.boost_inputs(np.arange(v1.shape[0]), dtype=dt, seed=6)
        v1, v2 = a, b
    mo, _ = O.invariant_mass(v1, v2, coords=coords)
    e = energy_scale(O, v1, v2, coords)
    tau = tau_of(dt)
    t1, t2 = dev(v1), dev(v2)
    m_aos = host(gvx.invariant_mass(t1, t2, coords=coords))
    bad = mass_violations(m_aos, mo, e, tau)
    assert bad.size == 0, (bad[:8], m_aos[bad[:8]], mo[bad[:8]])
    # SoA: 4 separate component arrays
    s1 = [t1[:, k].contiguous() for k in range(4)]
    s2 = [t2[:, k].contiguous() for k in range(4)]
    m_soa = host(gvx.invariant_mass(s1, s2, coords=coords))
    # interleaved pairs [N, 2, 4] (strided view, stride 8)
    pairs = torch.stack([t1, t2], dim=1).contiguous()
    m_pair = host(gvx.invariant_mass(pairs[:, 0, :], pairs[:, 1, :], coords=coords))
    # misaligned AoS view (offset by one vector: 16/32-byte alignment lost for f32/f64)
    big1 = torch.cat([t1[:1], t1]).contiguous()[1:]
    big2 = torch.cat([t2[:1], t2]).contiguous()[1:]
    m_mis = host(gvx.invariant_mass(big1, big2, coords=coords))
    for other in (m_soa, m_pair, m_mis):
        assert np.array_equal(other, m_aos, equal_nan=True)  # bitwise identical across layouts


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_mass_small_and_empty(gvx, O, dt):
    for n in (0, 1, 2, 3, 5, 7, 9, 255, 257):
        v1, v2 = synth.muon_pairs(np.arange(n), dtype=dt)
        mo, e = O.invariant_mass(v1, v2)
        m = host(gvx.invariant_mass(dev(v1).reshape(n, 4), dev(v2).reshape(n, 4)))
        assert m.shape == (n,)
        assert mass_violations(m, mo, e, tau_of(dt)).size == 0


def test_mass_errors(gvx):
    a = torch.zeros((4, 4), device="cuda")
    with pytest.raises(ValueError):
        gvx.invariant_mass(a, torch.zeros((5, 4), device="cuda"))
    with pytest.raises(ValueError):
        gvx.invariant_mass(a.cpu(), a.cpu())
    with pytest.raises(TypeError):
        gvx.invariant_mass(a.half(), a.half())


# ----------------------------------------------------------------------------
# K2 boost
# ----------------------------------------------------------------------------

def boost_edge_rows(dt):
    v = np.array([[0, 0, 0, 1.0], [1, 2, 3, 10], [3, 0, 4, 5], [0, 0, 0, 0], [5, -7, 9, 30]], np.float64)
    b = np.array([[0, 0, 0.6], [0, 0, 0], [0.9, 0.9, 0], [0.5, -0.5, 0.5], [np.nan, 0, 0]], np.float64)
    return v.astype(dt), b.astype(dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_boost_parity(gvx, O, dt):
    n = 2 * 256 * 148 + 11
    v, b = synth.boost_inputs(np.arange(n), dtype=dt)
    ev, eb = boost_edge_rows(dt)
    v = np.concatenate([ev, v])
    b = np.concatenate([eb, b])
    ref, s = O.boost(v, b)
    tv, tb = dev(v), dev(b)
    out = host(gvx.boost(tv, tb))
    bad = boost_violations(out, ref, s, tau_of(dt))
    assert bad.size == 0, (bad[:5], out[bad[:5]], ref[bad[:5]])
    # SoA and in-place give the same bits
    out_soa = [torch.empty(tv.shape[0], dtype=tv.dtype, device="cuda") for _ in range(4)]
    gvx.boost([tv[:, k].contiguous() for k in range(4)], [tb[:, k].contiguous() for k in range(3)], out=out_soa)
    assert np.array_equal(np.stack([host(c) for c in out_soa], 1), out, equal_nan=True)
    tv2 = tv.clone()
    gvx.boost(tv2, tb, out=tv2)
    assert np.array_equal(host(tv2), out, equal_nan=True)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_boost_uniform_parity(gvx, O, dt):
    v, _ = synth.boost_inputs(np.arange(100_003), dtype=dt)
    beta = (0.3, -0.4, 0.5)
    ref = O.boost_uniform(v, *[dt(x) for x in beta])
    out = host(gvx.boost_uniform(dev(v), beta))
    s = O.boost(v, np.tile(np.array(beta, dt), (v.shape[0], 1)))[1]
    assert boost_violations(out, ref, s, tau_of(dt)).size == 0
    with pytest.raises(gvx.DomainError):
        gvx.boost_uniform(dev(v), (0.9, 0.9, 0.0))


def test_boost_inverse_on_gpu(gvx):
    """β then −β recovers the input at 2^20 events: |Δ| ≤ τ·(S + γS'),
    bounded here by τ·4γ²E."""
    import synth.device as sd
    v, b = sd.boost_inputs(1 << 20)
    back = gvx.boost(gvx.boost(v, b), -b)
    g = 1 / torch.sqrt(1 - (b * b).sum(1))
    err = ((back - v).abs().max(1).values / (4 * g * g * v[:, 3])).max().item()
    assert err <= 1e-12


# ----------------------------------------------------------------------------
# K3 fused histogram (lab and CM)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("cm", [False, True])
def test_histogram_parity(gvx, O, dt, cm):
    n = 200_003
    v1, v2 = mixed_inputs(n, dt, seed=99)
    bins_o, mo = O.mass_histogram(v1, v2, LO, HI, NB, cm=cm)
    mlab, _ = O.invariant_mass(v1, v2)
    e = energy_scale(O, v1, v2)
    t1, t2 = dev(v1), dev(v2)
    m_out = torch.empty(v1.shape[0], dtype=TDT[dt], device="cuda")
    bo = torch.empty((2 * v1.shape[0], 4), dtype=TDT[dt], device="cuda") if cm else None
    h = host(gvx.mass_histogram(t1, t2, LO, HI, NB, cm=cm, m_out=m_out, boosted_out=bo))
    assert h.sum() == v1.shape[0]
    tau = tau_of(dt)
    mg = host(m_out)
    if cm:
        # CM NaN is possible where β_cm² rounds to 1: near-collinear pairs (reading R11/R14)
        nanp = np.isnan(mo) | (np.abs(mlab.astype(np.float64)) < (1e-2 if dt == np.float32 else 1e-6) * e)
        fails, namb = hist_check(h, mo, e, tau, LO, HI, NB, nan_possible=nanp, m_window_center=mlab)
        ok = ~nanp
        bad = mass_violations(mg[ok], mo[ok], e[ok], tau)
        assert bad.size == 0
    else:
        fails, namb = hist_check(h, mo, e, tau, LO, HI, NB)
        assert mass_violations(mg, mo, e, tau).size == 0
        # the fused kernel's mass equals the mass kernel's, bit for bit
        assert np.array_equal(mg, host(gvx.invariant_mass(t1, t2)), equal_nan=True)
    assert not fails, fails
    # the GPU's own bins agree exactly with binning its masses
    assert np.array_equal(h, np.bincount(find_bin_np(mg, LO, HI, NB), minlength=NB + 2))
    # SoA views (TMA component tiles) and a strided view give the same bins
    hs = host(gvx.mass_histogram([t1[:, k].contiguous() for k in range(4)], [t2[:, k].contiguous() for k in range(4)],
                                 LO, HI, NB, cm=cm))
    pairs = torch.stack([t1, t2], dim=1).contiguous()
    hp = host(gvx.mass_histogram(pairs[:, 0, :], pairs[:, 1, :], LO, HI, NB, cm=cm))
    assert np.array_equal(hs, h) and np.array_equal(hp, h)
    print(f"hist dt={dt.__name__} cm={cm}: ambiguous events {namb}, exact bins "
          f"{int((h == bins_o).sum())}/{NB + 2}")
    if cm and dt == np.float64:
        _, _, bref = O.cm_mass(v1, v2, want_boosted=True)
        bg = host(bo).reshape(-1, 8)
        fin = np.isfinite(bref).all(1)
        S = e[fin] ** 2 / np.maximum(np.abs(mlab[fin]), 1e-300)
        err = np.abs(bg[fin] - bref[fin]).max(1) / S
        assert err.max() <= 1e-12


def test_histogram_accumulates_and_shards(gvx):
    import synth.device as sd
    n = 1 << 21
    v1, v2 = sd.muon_pairs(n, dtype=torch.float32)
    full = gvx.mass_histogram(v1, v2)
    acc = gvx.new_bins()
    for r in range(8):
        a, b = synth.shard_range(n, r, 8)
        gvx.mass_histogram(v1[a:b], v2[a:b], bins=acc)
    assert torch.equal(full, acc)
    gvx.mass_histogram(v1, v2, bins=acc)
    assert torch.equal(acc, 2 * full)


def test_histogram_single_bin_and_specials(gvx, O):
    # every pair at rest with mass 91 → one bin (contention stress)
    v = torch.zeros((1 << 20, 4), dtype=torch.float64, device="cuda")
    v[:, 3] = 45.5
    h = host(gvx.mass_histogram(v, v, coords="pxpypze"))
    b = find_bin_np(np.array([91.0]), LO, HI, NB)[0]
    assert h[b] == 1 << 20 and h.sum() == 1 << 20
    # NaN → overflow, exact lower edge → bin 1, M = hi → overflow, negative → underflow
    rows = np.array([[np.nan, 0, 0, 1], [0, 0, 0, LO / 2], [0, 0, 0, HI / 2], [1, 0, 0, 0.0]], np.float64)
    rows2 = np.array([[0, 0, 0, 1], [0, 0, 0, LO / 2], [0, 0, 0, HI / 2], [-1, 0, 0, 0.0]], np.float64)
    hg = host(gvx.mass_histogram(dev(rows), dev(rows2), coords="pxpypze"))
    ho, _ = O.mass_histogram(rows, rows2, LO, HI, NB, coords="pxpypze")
    assert np.array_equal(hg, ho.astype(np.int64))
    assert hg[NB + 1] == 2 and hg[1] == 1


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_find_bin_bit_exact_at_edges(gvx, O, dt):
    """Reading R12: for identical mass bits the kernel's bin is the oracle's FindBin,
    also on and within a few ulp of every kind of edge (the GPU's fast binning must
    send those to the exact division). Masses are fed exactly: PxPyPzE (0,0,0,x) + 0
    has M = sqrt(x*x) = x, and (p,0,0,0) + 0 has M = -p (both sides IEEE sqrt)."""
    rng = np.random.default_rng(7)
    for lo, hi, nb in ((LO, HI, NB), (0.0, 1.0, 10), (-50.0, 50.0, 100_000), (0.1, 0.7, 3), (1e-3, 1e3, 999)):
        w = (hi - lo) / nb
        ks = np.unique(np.concatenate([[0, 1, 2, nb - 1, nb], rng.integers(0, nb + 1, 300)]))
        x = lo + ks * w
        x = np.concatenate([x, lo + (hi - lo) * ks / nb, [lo, hi, hi + w, lo - w, 2 * hi]]).astype(dt)
        xs = [x]
        for s in (1, 2, 3):
            up, dn = x.copy(), x.copy()
            for _ in range(s):
                up = np.nextafter(up, dt(np.inf))
                dn = np.nextafter(dn, dt(-np.inf))
            xs += [up, dn]
        x = np.concatenate(xs + [rng.uniform(lo - w, hi + w, 2000).astype(dt)])
        x = x[np.isfinite(x) & (np.abs(x) < (1e18 if dt == np.float32 else 1e150))]
        v1 = np.zeros((x.size + 4, 4), dt)
        pos = x >= 0
        v1[:x.size][pos, 3] = x[pos]
        v1[:x.size][~pos, 0] = -x[~pos]   # M = -|px|
        v1[x.size:] = np.array([[np.nan, 0, 0, 1], [0, 0, 0, np.inf], [np.inf, 0, 0, 0], [0, 0, 0, 0]], dt)
        v2 = np.zeros_like(v1)
        ho, mo = O.mass_histogram(v1, v2, lo, hi, nb, coords="pxpypze")
        m_out = torch.empty(v1.shape[0], dtype=TDT[dt], device="cuda")
        hg = host(gvx.mass_histogram(dev(v1), dev(v2), lo, hi, nb, coords="pxpypze", m_out=m_out))
        assert np.array_equal(host(m_out), mo, equal_nan=True), (lo, hi, nb)
        assert np.array_equal(hg, ho.astype(np.int64)), (lo, hi, nb, np.nonzero(hg != ho.astype(np.int64))[0][:10])


def test_histogram_nbins_variants(gvx, O):
    v1, v2 = synth.muon_pairs(np.arange(50_000), dtype=np.float64)
    for lo, hi, nb in ((0.0, 200.0, 1), (0.0, 200.0, 7), (-50.0, 50.0, 100_000)):
        ho, mo = O.mass_histogram(v1, v2, lo, hi, nb)
        _, e = O.invariant_mass(v1, v2)
        h = host(gvx.mass_histogram(dev(v1), dev(v2), lo, hi, nb))
        fails, _ = hist_check(h, mo, e, 1e-12, lo, hi, nb)
        assert not fails, (lo, hi, nb, fails)
    with pytest.raises(gvx.GvxError):
        gvx.mass_histogram(dev(v1), dev(v2), 1.0, 1.0, 10)


# ----------------------------------------------------------------------------
# Full-size configurations, launched as bench.py launches them: sampled outputs
# ----------------------------------------------------------------------------

def _sample_idx(n, k=4096, seed=0):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.integers(0, n, k), [0, n - 1]]))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_cfg2_mass_1e8_sampled(gvx, O, dt):
    import synth.device as sd
    n = 100_000_000
    v1, v2 = sd.muon_pairs(n, dtype=TDT[dt])
    m = gvx.invariant_mass(v1, v2)
    idx = _sample_idx(n)
    a, b = synth.muon_pairs(idx, dtype=dt)
    mo, e = O.invariant_mass(a, b)
    mg = host(m[torch.from_numpy(idx).cuda()])
    assert mass_violations(mg, mo, e, tau_of(dt)).size == 0
    # SoA at full size on the same events
    del m
    s1 = [v1[:, k].contiguous() for k in range(4)]
    del v1
    s2 = [v2[:, k].contiguous() for k in range(4)]
    del v2
    m = gvx.invariant_mass(s1, s2)
    assert mass_violations(host(m[torch.from_numpy(idx).cuda()]), mo, e, tau_of(dt)).size == 0


def test_cfg3_boost_1e8_sampled(gvx, O):
    import synth.device as sd
    n = 100_000_000
    v, b = sd.boost_inputs(n, dtype=torch.float64)
    out = gvx.boost(v, b)
    idx = _sample_idx(n, seed=1)
    vh, bh = synth.boost_inputs(idx, dtype=np.float64)
    ref, s = O.boost(vh, bh)
    assert boost_violations(host(out[torch.from_numpy(idx).cuda()]), ref, s, 1e-12).size == 0


@pytest.mark.parametrize("cm", [False, True])
def test_cfg4_cfg5_histogram_1e9_f32(gvx, O, cm):
    """configs[3]/[4] at full size on one GPU: 1e9 fp32 pairs; masses sampled vs the
    oracle, bins vs sharded (8 shards) accumulation, bitwise."""
    import synth.device as sd
    n = 1_000_000_000
    v1, v2 = sd.muon_pairs(n, dtype=torch.float32)
    m_out = torch.empty(n, dtype=torch.float32, device="cuda")
    h = gvx.mass_histogram(v1, v2, cm=cm, m_out=m_out)
    assert int(h.sum()) == n
    acc = gvx.new_bins()
    for r in range(8):
        a, b = synth.shard_range(n, r, 8)
        gvx.mass_histogram(v1[a:b], v2[a:b], cm=cm, bins=acc)
    assert torch.equal(h, acc)
    idx = _sample_idx(n, seed=2)
    a, b = synth.muon_pairs(idx, dtype=np.float32)
    mo, e = (O.cm_mass(a, b) if cm else O.invariant_mass(a, b))
    mlab, _ = O.invariant_mass(a, b)
    mg = host(m_out[torch.from_numpy(idx).cuda()])
    ok = np.isfinite(mo) & (np.abs(mlab) >= 1e-2 * e) if cm else np.ones(idx.size, bool)
    assert mass_violations(mg[ok], mo[ok], e[ok], 1e-5).size == 0
    # the bins are exactly FindBin (double, oracle order) of the kernel's own masses
    x = m_out.double()
    q = (float(NB) * (x - LO)) / (HI - LO)
    inner = 1 + torch.trunc(torch.nan_to_num(q, nan=0.0, posinf=0.0, neginf=0.0)).long()
    b = torch.where(x < LO, 0, torch.where(~(x < HI), NB + 1, inner))
    assert torch.equal(torch.bincount(b, minlength=NB + 2), h)


def test_tma_ring_kernels_all_modes():
    """The TMA bulk-copy ring kernels are routed by default only where they measured faster
    (f32 CM histogram); rerun the AoS parity tests with GVX_FORCE_TMA=1 so every mode and
    dtype of the ring kernel is checked against the oracle too."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, GVX_FORCE_TMA="1")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", os.path.join(here, "test_gpu_parity.py"),
                        "-k", "cfg1 or layouts or small_and_empty or histogram_parity or single_bin or nbins or deterministic"],
                       env=env, cwd=os.path.dirname(here), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_hostpipe_matches_device_path(gvx):
    """Transfer-inclusive mode (hostpipe) gives the same bits as the device-resident calls."""
    import synth.device as sd
    from paper_2312_02756_b200 import hostpipe
    n = (1 << 20) + 12345
    for tdt in (torch.float64, torch.float32):
        v1, v2 = sd.muon_pairs(n, dtype=tdt)
        bv, bb = sd.boost_inputs(n, dtype=tdt)
        m = gvx.invariant_mass(v1, v2)
        bo = gvx.boost(bv, bb)
        h = gvx.mass_histogram(v1, v2)
        hc = gvx.mass_histogram(v1, v2, cm=True)
        hs = [t.cpu().pin_memory() for t in (v1, v2, bv, bb)]
        pipe = hostpipe.HostPipeline(n, tdt, "cuda", chunk=1 << 18)
        hm, hbo, hbins = pipe.step(*hs)
        torch.cuda.synchronize()
        assert torch.equal(hm, m.cpu()) and torch.equal(hbo, bo.cpu())
        assert torch.equal(hbins[0], h.cpu()) and torch.equal(hbins[1], hc.cpu())


def test_sharded_histogram_single_rank(gvx):
    import synth.device as sd
    v1, v2 = sd.muon_pairs(100_000, dtype=torch.float64)
    assert torch.equal(gvx.sharded_mass_histogram(v1, v2), gvx.mass_histogram(v1, v2))


def test_boosted_output_f32(gvx, O):
    """CM boosted-pair output (diagnostic) in f32: checked at 1e-4·S for well-conditioned pairs
    (DESIGN R5/R14: fp32 CM boosts of near-collinear pairs are ill-conditioned)."""
    v1, v2 = synth.muon_pairs(np.arange(50_000), seed=3, dtype=np.float32)
    _, _, bref = O.cm_mass(v1, v2, want_boosted=True)
    mlab, e = O.invariant_mass(v1, v2)
    bo = torch.empty((2 * v1.shape[0], 4), dtype=torch.float32, device="cuda")
    gvx.mass_histogram(dev(v1), dev(v2), cm=True, boosted_out=bo)
    bg = host(bo).reshape(-1, 8).astype(np.float64)
    ok = np.isfinite(bref).all(1) & (np.abs(mlab) >= 1e-2 * e)
    S = (e[ok].astype(np.float64) ** 2) / np.abs(mlab[ok].astype(np.float64))
    assert (np.abs(bg[ok] - bref[ok]).max(1) / S).max() <= 1e-4


@pytest.mark.parametrize("dt", [torch.float64, torch.float32])
def test_repeat_runs_bitwise_deterministic(gvx, dt):
    """Same inputs, same bits, run after run — on L2-resident inputs (1M pairs), where a
    premature reuse of a TMA ring stage would show up (regression test for the missing
    generic->async proxy fence found in round 1)."""
    import synth.device as sd
    n = (1 << 20) + 12345
    v1, v2 = sd.muon_pairs(n, dtype=dt)
    m0 = gvx.invariant_mass(v1, v2)
    h0 = gvx.mass_histogram(v1, v2)
    c0 = gvx.mass_histogram(v1, v2, cm=True)
    for _ in range(12):
        assert torch.equal(gvx.invariant_mass(v1, v2), m0)
        assert torch.equal(gvx.mass_histogram(v1, v2), h0)
        assert torch.equal(gvx.mass_histogram(v1, v2, cm=True), c0)


def other_coords_inputs(n, dt, coords, seed=31):
    """Seeded pairs in PxPyPzM / PtEtaPhiE (built on the host from synth muons; both sides
    receive the same rounded values)."""
    v1, v2 = synth.muon_pairs(np.arange(n), seed=seed)
    out = []
    for v in (v1, v2):
        pt, eta, phi, m = v.T
        if coords == "pxpypzm":
            w = np.stack([pt * np.cos(phi), pt * np.sin(phi), pt * np.sinh(eta), m], 1)
        else:
            w = np.stack([pt, eta, phi, np.sqrt(m * m + (pt * np.cosh(eta)) ** 2)], 1)
        out.append(w.astype(dt))
    # degenerate rows: spacelike / clamped masses, zero vectors, out-of-fast-domain eta
    extra = np.array([[3, 4, 12, -5], [3, 4, 12, -20], [0, 0, 0, 0], [1, 25.0, 0.3, 5e10]], np.float64).astype(dt)
    return np.concatenate([extra, out[0]]), np.concatenate([extra[::-1], out[1]])


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("coords", ["pxpypzm", "ptetaphie"])
def test_other_coordinate_systems(gvx, O, dt, coords):
    v1, v2 = other_coords_inputs(150_001, dt, coords)
    mo, _ = O.invariant_mass(v1, v2, coords=coords)
    # tolerance scale: sum of max(E_i, |p_i|) from the oracle's own E and |p| (R5)
    z = np.zeros_like(v1)
    _, e1 = O.invariant_mass(v1, z, coords=coords)
    _, e2 = O.invariant_mass(v2, z, coords=coords)
    a, b = v1.astype(np.float64), v2.astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        p1 = np.sqrt((a[:, :3] ** 2).sum(1)) if coords == "pxpypzm" else np.abs(a[:, 0]) * np.cosh(a[:, 1])
        p2 = np.sqrt((b[:, :3] ** 2).sum(1)) if coords == "pxpypzm" else np.abs(b[:, 0]) * np.cosh(b[:, 1])
    e = np.fmax(e1.astype(np.float64), p1) + np.fmax(e2.astype(np.float64), p2)
    tau = tau_of(dt)
    t1, t2 = dev(v1), dev(v2)
    m = host(gvx.invariant_mass(t1, t2, coords=coords))
    bad = mass_violations(m, mo, e, tau)
    assert bad.size == 0, (bad[:5], m[bad[:5]], mo[bad[:5]])
    m_soa = host(gvx.invariant_mass([t1[:, k].contiguous() for k in range(4)],
                                    [t2[:, k].contiguous() for k in range(4)], coords=coords))
    assert np.array_equal(m_soa, m, equal_nan=True)
    for cm in (False, True):
        h = host(gvx.mass_histogram(t1, t2, coords=coords, cm=cm))
        ho, mho = O.mass_histogram(v1, v2, LO, HI, NB, cm=cm, coords=coords)
        mlab = mo
        nanp = (np.isnan(mho) | (np.abs(mlab.astype(np.float64)) < (1e-2 if dt == np.float32 else 1e-6) * e)) if cm else None
        fails, _ = hist_check(h, mho, e, tau, LO, HI, NB, nan_possible=nanp, m_window_center=mlab if cm else None)
        assert not fails, (cm, fails)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_dimuon_histogram_parity(gvx, O, dt):
    mu, q, off = synth.jagged_events(0, 400_003, seed=8, dtype=dt)
    bins_o, mo, sel = O.dimuon_histogram(mu, q, off, LO, HI, NB)
    tm, tq, to = dev(mu), dev(q), dev(off)
    m_out = torch.empty(off.size - 1, dtype=TDT[dt], device="cuda")
    h = host(gvx.dimuon_histogram(tm, tq, to, m_out=m_out))
    mg = host(m_out)
    assert int(h.sum()) == sel
    assert np.array_equal(np.isnan(mg), np.isnan(mo))
    ok = ~np.isnan(mo)
    # tolerance scale: the selected pair's E_lab from the oracle
    first = off[:-1][ok]
    _, e = O.invariant_mass(mu[first], mu[first + 1])
    assert mass_violations(mg[ok], mo[ok], e, tau_of(dt)).size == 0
    fails, _ = hist_check(h, mo[ok], e, tau_of(dt), LO, HI, NB)
    assert not fails, fails
    # SoA view of the muons gives the same bits; the device generator twin gives the same events
    hs = host(gvx.dimuon_histogram([tm[:, k].contiguous() for k in range(4)], tq, to))
    assert np.array_equal(hs, h)
    import synth.device as sd
    dmu, dq, doff = sd.jagged_events(0, off.size - 1, seed=8, dtype=TDT[dt])
    assert torch.equal(dmu, tm) and torch.equal(dq, tq) and torch.equal(doff, to)
    # repeat runs are bitwise stable (TMA column ring), and the plain-load kernel (TMA off) agrees
    for _ in range(5):
        assert np.array_equal(host(gvx.dimuon_histogram(tm, tq, to)), h)
    # a tile whose muon range overflows the stage buffer: one event with many muons in the middle
    big = np.concatenate([mu[: off[5000]], np.tile(mu[:1], (3000, 1)), mu[off[5000]:]])
    bq = np.concatenate([q[: off[5000]], np.ones(3000, np.int32), q[off[5000]:]])
    boff = np.concatenate([off[:5001], off[5000:] + 3000])
    boff[5000] = off[5000]  # event 5000 gets 3000 extra muons (never selected); later offsets shift
    hb_o, mb_o, sel_b = O.dimuon_histogram(big, bq, boff, LO, HI, NB)
    mb = torch.empty(boff.size - 1, dtype=TDT[dt], device="cuda")
    hb = host(gvx.dimuon_histogram(dev(big), dev(bq), dev(boff), m_out=mb))
    assert int(hb.sum()) == sel_b and np.array_equal(np.isnan(host(mb)), np.isnan(mb_o))
    # charges beyond +-1 (R21 selects on the sign of the 64-bit product q0 q1): zero, large
    # magnitudes and the int32 extremes, whose 32-bit product would overflow
    rng = np.random.default_rng(5)
    qx = rng.choice(np.array([0, 1, -1, 7, -7, 1 << 30, -(1 << 30), 2**31 - 1, -2**31], np.int64),
                    size=q.size).astype(np.int32)
    hx_o, mx_o, sel_x = O.dimuon_histogram(mu, qx, off, LO, HI, NB)
    mx = torch.empty(off.size - 1, dtype=TDT[dt], device="cuda")
    hx = host(gvx.dimuon_histogram(tm, dev(qx), to, m_out=mx))
    assert int(hx.sum()) == sel_x and np.array_equal(np.isnan(host(mx)), np.isnan(mx_o))
    assert sel_x > 1000 and sel_x != sel


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_dimuon_carried_list_edges(gvx, O, dt):
    """The default dimuon kernel (k_dimuon_carry: consecutive-event selection, a circular
    list carried across tiles, L2 prefetch) against the oracle on the shapes that stress
    its bookkeeping: batches below / at / just above one tile (512 f64, 1024 f32 events)
    and with a ragged last tile, every event selected (the list at its 2 ET + NT bound),
    none selected, offsets that are 8- but not 32-byte aligned (the scalar offset loads),
    with and without m_out (the same bins)."""
    mu, q, off = synth.jagged_events(0, 70_001, seed=31, dtype=dt)
    for n in (1, 3, 511, 512, 513, 1023, 1024, 1025, 2049, 9_999, 70_001):
        o = off[: n + 1]
        h_o, m_o, sel = O.dimuon_histogram(mu, q, o, LO, HI, NB)
        m_out = torch.empty(n, dtype=TDT[dt], device="cuda")
        h = host(gvx.dimuon_histogram(dev(mu), dev(q), dev(o), m_out=m_out))
        mg = host(m_out)
        assert int(h.sum()) == sel and np.array_equal(np.isnan(mg), np.isnan(m_o)), n
        ok = ~np.isnan(m_o)
        if ok.any():
            first = o[:-1][ok]
            _, e = O.invariant_mass(mu[first], mu[first + 1])
            assert mass_violations(mg[ok], m_o[ok], e, tau_of(dt)).size == 0, n
            fails, _ = hist_check(h, m_o[ok], e, tau_of(dt), LO, HI, NB)
            assert not fails, (n, fails)
        assert np.array_equal(host(gvx.dimuon_histogram(dev(mu), dev(q), dev(o))), h), n
    # offsets starting at event 1 (8-byte aligned, not 32): the same events, shifted
    to = dev(off)
    for s0 in (1, 2, 3):
        sub = to[s0:]
        h_o, _, sel = O.dimuon_histogram(mu, q, off[s0:], LO, HI, NB)
        h = host(gvx.dimuon_histogram(dev(mu), dev(q), sub))
        assert int(h.sum()) == sel
        assert np.array_equal(h, host(gvx.dimuon_histogram(dev(mu), dev(q), dev(off[s0:].copy()))))
    # every event a selected pair (list at capacity), then no event selected
    n = 20_000
    pm = mu[:2 * n].copy()  # event i owns rows 2i, 2i + 1
    qa = np.tile(np.array([1, -1], np.int32), n)
    oa = np.arange(0, 2 * n + 1, 2, dtype=np.int64)
    h_o, m_o, sel = O.dimuon_histogram(pm, qa, oa, LO, HI, NB)
    assert sel == n
    m_out = torch.empty(n, dtype=TDT[dt], device="cuda")
    h = host(gvx.dimuon_histogram(dev(pm), dev(qa), dev(oa), m_out=m_out))
    _, e = O.invariant_mass(pm[0::2], pm[1::2])
    assert int(h.sum()) == n and mass_violations(host(m_out), m_o, e, tau_of(dt)).size == 0
    fails, _ = hist_check(h, m_o, e, tau_of(dt), LO, HI, NB)
    assert not fails, fails
    h = host(gvx.dimuon_histogram(dev(pm), dev(np.ones(2 * n, np.int32)), dev(oa), m_out=m_out))
    assert int(h.sum()) == 0 and bool(torch.isnan(m_out).all())


def test_dimuon_muon_span_beyond_32_bits(gvx):
    """k_dimuon_carry keeps 32-bit list entries (muon offset - offsets[0]) while a launch's
    muons span < 2^32 and switches to 64-bit entries on half-size tiles otherwise. A first
    event owning 2^32 + 7 muons (never selected: not two muons) pushes the span past 2^32;
    the events after it must give the same bins and masses as the same events on their own
    (which take the 32-bit path). f32, ~86 GB of muon columns (only the tail is written)."""
    mu, q, off = synth.jagged_events(0, 100_003, seed=41, dtype=np.float32)
    m = off[-1]
    big = (1 << 32) + 7
    free, _ = torch.cuda.mem_get_info()
    need = (big + m) * (16 + 4) + (1 << 30)
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB of free device memory")
    ref_m = torch.empty(off.size - 1, dtype=torch.float32, device="cuda")
    ref = host(gvx.dimuon_histogram(dev(mu), dev(q), dev(off), m_out=ref_m))
    bm = torch.empty((big + m, 4), dtype=torch.float32, device="cuda")
    bq = torch.empty(big + m, dtype=torch.int32, device="cuda")
    bm[big:] = dev(mu)
    bq[big:] = dev(q)
    boff = torch.cat([torch.zeros(1, dtype=torch.int64, device="cuda"), dev(off) + big])
    got_m = torch.empty(off.size, dtype=torch.float32, device="cuda")
    got = host(gvx.dimuon_histogram(bm, bq, boff, m_out=got_m))
    assert np.array_equal(got, ref)
    assert bool(torch.isnan(got_m[0])) and torch.equal(torch.isnan(got_m[1:]), torch.isnan(ref_m))
    ok = ~torch.isnan(ref_m)
    assert torch.equal(got_m[1:][ok], ref_m[ok])
    del bm, bq
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_lorentz_transform_parity(gvx, O, dt):
    v, beta = synth.boost_inputs(np.arange(200_003), dtype=dt, seed=23)
    b = (0.3, -0.4, 0.5)
    c, s_ = np.cos(0.7), np.sin(0.7)
    R = np.array([[c, -s_, 0, 0], [s_, c, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]])
    Lb = O.boost(np.eye(4), np.array([b] * 4))[0].T
    L = Lb @ R
    ref = O.lorentz_transform(v, L)
    out = host(gvx.lorentz_transform(dev(v), L))
    S = (np.abs(L) @ np.abs(v.astype(np.float64)).T).T.max(1)  # bound on |L||v| per vector
    assert boost_violations(out, ref, S, tau_of(dt)).size == 0
    # in place and SoA give the same bits; a non-Lorentz matrix is a domain error
    tv = dev(v)
    gvx.lorentz_transform(tv, L, out=tv)
    assert np.array_equal(host(tv), out)
    with pytest.raises(gvx.DomainError):
        gvx.lorentz_transform(dev(v), 2 * np.eye(4))


def test_cuda_graph_capture(gvx):
    """The ABI only enqueues on the caller's stream (no allocation, no sync), so a whole step
    can be captured into a CUDA graph and replayed — the launch-bound small-N regime's answer."""
    import synth.device as sd
    n = 50_000
    v1, v2 = sd.muon_pairs(n, dtype=torch.float64)
    bv, bb = sd.boost_inputs(n, dtype=torch.float64)
    m = torch.empty(n, dtype=torch.float64, device="cuda")
    bo = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    bins = gvx.new_bins()
    binc = gvx.new_bins()

    def step():
        bins.zero_()
        binc.zero_()
        gvx.invariant_mass(v1, v2, out=m)
        gvx.boost(bv, bb, out=bo)
        gvx.mass_histogram(v1, v2, bins=bins)
        gvx.mass_histogram(v1, v2, bins=binc, cm=True)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()  # warm-up outside capture (occupancy queries, smem opt-in)
    torch.cuda.current_stream().wait_stream(s)
    ref = [t.clone() for t in (m, bo, bins, binc)]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    m.zero_()
    bo.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip((m, bo, bins, binc), ref):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dt", [torch.float64, torch.float32])
def test_physics_invariants_full_size(gvx, dt):
    """Properties that hold at any size, checked on all 1e8 pairs of the bench batch:
    pair symmetry (bitwise: every step of the formula is symmetric), and invariance of M
    under a common rotation about z (φ → φ + δ) and under the reflection η → −η of both
    vectors (within the north-star tolerance, scale E_lab² ≤ (2 Σ pt cosh η)²)."""
    import synth.device as sd
    n = 100_000_000
    v1, v2 = sd.muon_pairs(n, dtype=dt)
    m = gvx.invariant_mass(v1, v2)
    assert torch.equal(gvx.invariant_mass(v2, v1), m)
    tau = 1e-12 if dt == torch.float64 else 1e-5
    e = (v1[:, 0] * torch.cosh(v1[:, 1]) + v2[:, 0] * torch.cosh(v2[:, 1])).double() + 1.0
    for k, delta in ((2, 0.37), (1, None)):
        w1, w2 = v1.clone(), v2.clone()
        if delta is None:
            w1[:, 1].neg_()
            w2[:, 1].neg_()
        else:
            w1[:, 2] += delta
            w2[:, 2] += delta
        mr = gvx.invariant_mass(w1, w2)
        md, mrd = m.double(), mr.double()
        err = (md * md.abs() - mrd * mrd.abs()).abs() / (e * e)
        assert err.max().item() <= tau, (k, err.max().item())
        del w1, w2, mr


def _layout_views(t, kind, rng):
    """Return a view of the [n, 4] CUDA tensor t with the requested memory layout (same values)."""
    n = t.shape[0]
    if kind == "aos":
        return t
    if kind == "aos_offset":  # misaligned base (one scalar offset)
        buf = torch.empty(n * 4 + 1, dtype=t.dtype, device=t.device)
        v = buf[1:].view(n, 4)
        v.copy_(t)
        return v
    if kind == "soa":
        return [t[:, k].contiguous() for k in range(4)]
    if kind == "soa_offset":
        out = []
        for k in range(4):
            buf = torch.empty(n + 3, dtype=t.dtype, device=t.device)
            buf[3:].copy_(t[:, k])
            out.append(buf[3:])
        return out
    if kind.startswith("strided"):
        s = int(kind[len("strided"):])
        buf = torch.zeros((n, s), dtype=t.dtype, device=t.device)
        buf[:, :4].copy_(t)
        return buf[:, :4]
    raise ValueError(kind)


def test_dispatch_fuzz(gvx, O):
    """Random sizes x layouts x coordinate systems x dtypes x operations against the oracle —
    exercises every dispatch branch (TMA ring AoS/SoA, LDG AoS/SoA/strided, tails, misaligned
    views) with the same parity predicates as the targeted tests."""
    rng = np.random.default_rng(2024)
    kinds = ["aos", "aos_offset", "soa", "soa_offset", "strided5", "strided8"]
    for trial in range(36):
        dt = [np.float32, np.float64][trial % 2]
        coords = ["ptetaphim", "pxpypze", "pxpypzm", "ptetaphie"][rng.integers(4)]
        n = int(rng.choice([0, 1, 3, 31, 257, 4097, int(rng.integers(1, 300_000))]))
        kind1, kind2 = rng.choice(kinds, 2)
        op = ["mass", "hist", "cm"][trial % 3]
        v1, v2 = synth.muon_pairs(np.arange(n), seed=100 + trial, dtype=dt)
        if coords == "pxpypze":
            v1, _ = synth.boost_inputs(np.arange(n), seed=200 + trial, dtype=dt)
            v2, _ = synth.boost_inputs(np.arange(n), seed=300 + trial, dtype=dt)
        elif coords == "pxpypzm":
            a, _ = synth.boost_inputs(np.arange(n), seed=200 + trial, dtype=dt)
            b, _ = synth.boost_inputs(np.arange(n), seed=300 + trial, dtype=dt)
            v1 = np.concatenate([a[:, :3], np.full((n, 1), synth.MUON_MASS, dt)], 1).astype(dt)
            v2 = np.concatenate([b[:, :3], np.full((n, 1), synth.MUON_MASS, dt)], 1).astype(dt)
        elif coords == "ptetaphie":
            v1 = v1.copy()
            v2 = v2.copy()
            v1[:, 3] = (v1[:, 0] * np.cosh(v1[:, 1].astype(np.float64)) * 1.01).astype(dt)
            v2[:, 3] = (v2[:, 0] * np.cosh(v2[:, 1].astype(np.float64)) * 1.01).astype(dt)
        t1 = _layout_views(torch.from_numpy(v1).cuda().reshape(n, 4), kind1, rng)
        t2 = _layout_views(torch.from_numpy(v2).cuda().reshape(n, 4), kind2, rng)
        tag = (trial, dt.__name__, coords, n, kind1, kind2, op)
        z = np.zeros_like(v1)
        _, e1 = O.invariant_mass(v1, z, coords=coords)
        _, e2 = O.invariant_mass(v2, z, coords=coords)
        e = np.abs(e1.astype(np.float64)) + np.abs(e2.astype(np.float64)) + 1e-30
        if coords in ("pxpypze", "pxpypzm"):
            e = e + np.sqrt((v1[:, :3].astype(np.float64) ** 2).sum(1)) + np.sqrt((v2[:, :3].astype(np.float64) ** 2).sum(1))
        if op == "mass":
            mo, _ = O.invariant_mass(v1, v2, coords=coords)
            m = host(gvx.invariant_mass(t1, t2, coords=coords))
            assert mass_violations(m, mo, e, tau_of(dt)).size == 0, tag
        else:
            cm = op == "cm"
            h = host(gvx.mass_histogram(t1, t2, coords=coords, cm=cm))
            ho, mo = O.mass_histogram(v1, v2, LO, HI, NB, cm=cm, coords=coords)
            assert int(h.sum()) == n, tag
            if cm:
                mlab, _ = O.invariant_mass(v1, v2, coords=coords)
                nanp = np.isnan(mo) | (np.abs(mlab.astype(np.float64)) < (1e-2 if dt == np.float32 else 1e-6) * e)
                fails, _ = hist_check(h, mo, e, tau_of(dt), LO, HI, NB, nan_possible=nanp, m_window_center=mlab)
            else:
                fails, _ = hist_check(h, mo, e, tau_of(dt), LO, HI, NB)
            assert not fails, (tag, fails)


# ----------------------------------------------------------------------------
# CM decay angle cos θ* (reading R22)
# ----------------------------------------------------------------------------

def _costheta_reference(O, v1, v2, dt, coords="ptetaphim"):
    """Oracle cos θ*, its tolerance window δ = 2 τ_b S/|p'1| (S = E_lab²/|M_lab|, the CM
    boost's γE scale; τ_b = 1e-12 f64, 1e-4 f32 as for the boosted vectors), and the
    events whose CM boost is ill-conditioned (f32: M_lab/E_lab < 1e-2; any: oracle NaN)."""
    mb, cb, mo, co = O.cm_costheta(v1, v2, c_axis=(-1.0, 1.0, 100), coords=coords)
    _, _, bo = O.cm_mass(v1, v2, coords=coords, want_boosted=True)
    mlab, _ = O.invariant_mass(v1, v2, coords=coords)
    e = energy_scale(O, v1, v2, coords)
    tau_b = 1e-12 if dt == np.float64 else 1e-4
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        pstar = np.sqrt((bo[:, :3].astype(np.float64) ** 2).sum(1))
        S = e * e / np.maximum(np.abs(mlab.astype(np.float64)), 1e-300)
        delta = 2 * tau_b * S / pstar
    small = np.abs(mlab.astype(np.float64)) < (1e-2 if dt == np.float32 else 1e-6) * e
    nanp = np.isnan(co) | np.isnan(mo) | small
    return mb, cb, mo, co, delta, nanp, mlab, e


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("layout", ["aos", "soa", "pairs"])
def test_cm_costheta_parity(gvx, O, dt, layout):
    n = 200_003 if layout == "aos" else 3 * 256 * 148 + 37
    v1, v2 = mixed_inputs(n, dt, seed=17)
    mb_o, cb_o, mo, co, delta, nanp, mlab, e = _costheta_reference(O, v1, v2, dt)
    t1, t2 = dev(v1), dev(v2)
    if layout == "soa":
        a = [t1[:, k].contiguous() for k in range(4)]
        b = [t2[:, k].contiguous() for k in range(4)]
    elif layout == "pairs":  # interleaved [N][2][4]: the generic strided kernel
        pr = torch.stack([t1, t2], 1).contiguous()
        a, b = pr[:, 0], pr[:, 1]
    else:
        a, b = t1, t2
    N = v1.shape[0]
    m_out = torch.empty(N, dtype=TDT[dt], device="cuda")
    c_out = torch.empty(N, dtype=TDT[dt], device="cuda")
    mb, cb = gvx.cm_costheta_histogram(a, b, c_axis=(-1.0, 1.0, 100), m_out=m_out, cos_out=c_out)
    mb, cb, mg, cg = host(mb), host(cb), host(m_out), host(c_out)
    assert mb.sum() == N and cb.sum() == N
    # the mass axis is the CM mass histogram, bit for bit (same arithmetic, same binning)
    m_ref = torch.empty(N, dtype=TDT[dt], device="cuda")
    h_cm = host(gvx.mass_histogram(t1, t2, cm=True, m_out=m_ref))
    assert np.array_equal(mb, h_cm) and np.array_equal(mg, host(m_ref), equal_nan=True)
    # cos θ* element-wise within the window, class-equal (finite <=> finite) where well conditioned
    ok = ~nanp
    c64, g64 = co.astype(np.float64), cg.astype(np.float64)
    fin = np.isfinite(c64[ok])
    assert np.array_equal(fin, np.isfinite(g64[ok]))
    err = np.abs(g64[ok][fin] - c64[ok][fin])
    assert np.all(err <= delta[ok][fin]), (err / delta[ok][fin]).max()
    fails, namb = hist_check_delta(cb, co, delta, -1.0, 1.0, 100, nan_possible=nanp)
    assert not fails, (fails, namb)
    assert np.abs(g64[np.isfinite(g64)]).max() <= 1 + 1e-6


def test_cm_costheta_cartesian_and_closed_form(gvx, O):
    """PxPyPzE input: rest-frame decays boosted into the lab recover their angle on the GPU too."""
    rng = np.random.default_rng(11)
    n = 50_000
    th = np.arccos(rng.uniform(-1, 1, n))
    ph = rng.uniform(-np.pi, np.pi, n)
    ps = rng.uniform(5, 50, n)
    E = np.sqrt(ps ** 2 + synth.MUON_MASS ** 2)
    p1 = np.stack([ps * np.sin(th) * np.cos(ph), ps * np.sin(th) * np.sin(ph), ps * np.cos(th), E], 1)
    p2 = p1 * np.array([-1, -1, -1, 1])
    d = rng.normal(size=(n, 3))
    beta = 0.9 * rng.uniform(size=(n, 1)) ** (1 / 3) * d / np.linalg.norm(d, axis=1, keepdims=True)
    l1, _ = O.boost(p1, beta)
    l2, _ = O.boost(p2, beta)
    c_out = torch.empty(n, dtype=torch.float64, device="cuda")
    _, cb = gvx.cm_costheta_histogram(dev(l1), dev(l2), c_axis=(-1.0, 1.0, 20), cos_out=c_out, coords="pxpypze")
    assert np.abs(host(c_out) - np.cos(th)).max() <= 1e-11
    _, cbo, _, co = O.cm_costheta(l1, l2, c_axis=(-1.0, 1.0, 20), coords="pxpypze")
    assert np.abs(host(c_out) - co).max() <= 1e-12
    # uniform in cos θ: every one of the 20 bins holds 5 % ± 5σ
    h = host(cb)[1:21]
    assert np.all(np.abs(h - n / 20) <= 5 * np.sqrt(n / 20))


def test_cm_costheta_errors(gvx):
    v = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(gvx.GvxError):
        gvx.cm_costheta_histogram(v, v, c_axis=(1.0, -1.0, 10))
    with pytest.raises(gvx.GvxError):
        gvx.cm_costheta_histogram(v, v, m_axis=(0.0, 1.0, 0))
    with pytest.raises(ValueError):
        gvx.cm_costheta_histogram(v, v[:3])
    mb, cb = gvx.cm_costheta_histogram(v[:0], v[:0])
    assert int(mb.sum()) == 0 and int(cb.sum()) == 0
    # zero vectors: invalid CM boost -> both overflow bins
    mb, cb = gvx.cm_costheta_histogram(v, v, coords="pxpypze", c_axis=(-1.0, 1.0, 10))
    assert int(mb[-1]) == 4 and int(cb[-1]) == 4


def test_cfg5_costheta_1e9_f32(gvx, O):
    """cos θ* (R22) at CFG5's per-GPU size, launched as bench.py launches it: 1e9 fp32 pairs.
    Sampled values vs the oracle; the mass axis equals the CM histogram bit for bit; the
    angle axis is exactly FindBin of the kernel's own cos θ*; 8-shard accumulation equal."""
    import synth.device as sd
    n = 1_000_000_000
    v1, v2 = sd.muon_pairs(n, dtype=torch.float32)
    m_out = torch.empty(n, dtype=torch.float32, device="cuda")
    c_out = torch.empty(n, dtype=torch.float32, device="cuda")
    mb, cb = gvx.cm_costheta_histogram(v1, v2, m_out=m_out, cos_out=c_out)
    assert int(mb.sum()) == n and int(cb.sum()) == n
    assert torch.equal(mb, gvx.mass_histogram(v1, v2, cm=True))
    x = c_out.double()
    q = (100.0 * (x + 1.0)) / 2.0
    inner = 1 + torch.trunc(torch.nan_to_num(q, nan=0.0, posinf=0.0, neginf=0.0)).long()
    b = torch.where(x < -1.0, 0, torch.where(~(x < 1.0), 101, inner))
    assert torch.equal(torch.bincount(b, minlength=102), cb)
    del x, q, inner, b
    am, ac = gvx.new_bins(), gvx.new_bins(100)
    for r in range(8):
        lo, hi = synth.shard_range(n, r, 8)
        gvx.cm_costheta_histogram(v1[lo:hi], v2[lo:hi], m_bins=am, c_bins=ac)
    assert torch.equal(am, mb) and torch.equal(ac, cb)
    idx = _sample_idx(n, seed=5)
    a, bb = synth.muon_pairs(idx, dtype=np.float32)
    _, _, mo, co, delta, nanp, _, _ = _costheta_reference(O, a, bb, np.float32)
    sel = torch.from_numpy(idx).cuda()
    cg = host(c_out[sel]).astype(np.float64)
    ok = ~nanp & np.isfinite(co)
    assert np.all(np.abs(cg[ok] - co[ok]) <= delta[ok])


def test_dimuon_1e8_full_size(gvx, O):
    """Jagged dimuon (f4) at the bench size (1e8 events, f64), launched as bench.py does:
    the selected count equals the selection rule evaluated by torch on the device columns,
    the bins are FindBin of the kernel's own masses, sampled events match the oracle."""
    import synth.device as sd
    n = 100_000_000
    mu, q, off = sd.jagged_events(0, n, dtype=torch.float64)
    m_out = torch.empty(n, dtype=torch.float64, device="cuda")
    h = gvx.dimuon_histogram(mu, q, off, m_out=m_out)
    k = off[1:] - off[:-1]
    first = off[:-1].clamp(max=q.numel() - 2)
    sel = (k == 2) & (q[first].long() * q[first + 1].long() < 0)
    assert int(h.sum()) == int(sel.sum())
    assert torch.equal(torch.isnan(m_out), ~sel)
    x = m_out.double()
    qq = (float(NB) * (x - LO)) / (HI - LO)
    inner = 1 + torch.trunc(torch.nan_to_num(qq, nan=0.0, posinf=0.0, neginf=0.0)).long()
    b = torch.where(x < LO, 0, torch.where(~(x < HI), NB + 1, inner))[sel]
    assert torch.equal(torch.bincount(b, minlength=NB + 2), h)
    del x, qq, inner, b
    ev = _sample_idx(n, seed=9)
    ev = ev[host(sel[torch.from_numpy(ev).cuda()])]
    assert ev.size > 300
    for e0 in ev[:400]:
        hm, hq, ho = synth.jagged_events(int(e0), 1, dtype=np.float64)
        _, mo, s = O.dimuon_histogram(hm, hq, ho, LO, HI, NB)
        assert s == 1
        _, e = O.invariant_mass(hm[:1], hm[1:2])
        assert mass_violations(host(m_out[int(e0):int(e0) + 1]), mo, e, 1e-12).size == 0


# ----------------------------------------------------------------------------
# Cross-GPU bin reduction fused into the kernel tail
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("cm", [False, True])
def test_mass_histogram_peers_simulated(gvx, dt, cm):
    """gvx_mass_histogram_peers adds every CTA's counts to each array of the peer list: with
    three 'peers' that are local buffers, each receives the whole histogram (what every rank of
    an all-reduce receives), bit-equal to the plain fused histogram, for the TMA ring (AoS),
    the register kernel (strided pairs) and several launches' worth of accumulation."""
    import synth.device as sd
    n = 3 * 1024 * 148 + 77
    v1, v2 = sd.muon_pairs(n, dtype=TDT[dt])
    ref = gvx.mass_histogram(v1, v2, cm=cm)
    pr = torch.stack([v1, v2], 1).contiguous()
    for a, b in ((v1, v2), (pr[:, 0], pr[:, 1])):
        peers = [gvx.new_bins() for _ in range(3)]
        ptrs = torch.tensor([t.data_ptr() for t in peers], dtype=torch.int64, device="cuda")
        gvx.mass_histogram_peers(a, b, ptrs.data_ptr(), 3, cm=cm)
        torch.cuda.synchronize()
        for t in peers:
            assert torch.equal(t, ref)
        gvx.mass_histogram_peers(a, b, ptrs.data_ptr(), 3, cm=cm)  # accumulates like the plain call
        torch.cuda.synchronize()
        assert torch.equal(peers[1], 2 * ref)
    with pytest.raises(gvx.GvxError):
        gvx.mass_histogram_peers(v1, v2, 0, 3)
    with pytest.raises(gvx.GvxError):
        gvx.mass_histogram_peers(v1, v2, ptrs.data_ptr(), 0)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_mass_histogram_peers_prereduce_workspace(gvx, dt):
    """The pre-reduced sink: CTAs add into the caller's workspace and the last CTA of each launch
    pushes the totals to the peers and clears it — so the workspace is all zero after every call
    (and its ticket re-armed), and back-to-back calls of different sizes and paths (TMA ring,
    register kernel, lab and CM) sharing one workspace each deliver exactly the plain histogram."""
    import synth.device as sd
    work = torch.zeros(gvx.DEFAULT_NBINS + 3, dtype=torch.int64, device="cuda")
    peers = [gvx.new_bins() for _ in range(2)]
    ptrs = torch.tensor([t.data_ptr() for t in peers], dtype=torch.int64, device="cuda")
    for n in (1, 4097, 300_000, 3 * 1536 * 148 + 5):
        v1, v2 = sd.muon_pairs(n, first=n, dtype=TDT[dt])
        pr = torch.stack([v1, v2], 1).contiguous()
        for a, b in ((v1, v2), (pr[:, 0], pr[:, 1])):
            for cm in (False, True):
                ref = gvx.mass_histogram(a, b, cm=cm)
                for t in peers:
                    t.zero_()
                gvx.mass_histogram_peers(a, b, ptrs.data_ptr(), 2, cm=cm, work=work)
                torch.cuda.synchronize()
                assert int(work.abs().sum()) == 0, (n, cm)
                for t in peers:
                    assert torch.equal(t, ref), (n, cm)
    with pytest.raises(ValueError):
        gvx.mass_histogram_peers(v1, v2, ptrs.data_ptr(), 2, work=work[:10])


def test_allreduce_mass_histogram_symmetric_memory_world1():
    """The symmetric-memory plumbing (rendezvous, peer pointer array, device barriers) on a
    one-rank NCCL group: the fused all-reduce equals the plain histogram."""
    import subprocess
    import sys
    code = r'''
import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29731")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
import paper_2312_02756_b200 as gvx, synth.device as sd
v1, v2 = sd.muon_pairs(1_000_003, dtype=torch.float64)
for cm in (False, True):
    ref = gvx.mass_histogram(v1, v2, cm=cm)
    got = gvx.allreduce_mass_histogram(v1, v2, cm=cm).clone()
    torch.cuda.synchronize()
    assert torch.equal(got, ref), (cm, (got - ref).abs().sum().item())
dist.destroy_process_group()
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, PYTHONPATH=root))
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_bench_step_histograms_full_size(gvx, O, dt):
    """The bench step's two histogram kernels at its size (1e8 pairs, default launch: the
    two-event TMA rings): sampled masses vs the oracle (lab and CM), bins == FindBin of the
    kernel's own masses over all 1e8 events, and 4-shard accumulation bit-equal."""
    import synth.device as sd
    n = 100_000_000
    v1, v2 = sd.muon_pairs(n, dtype=TDT[dt])
    idx = _sample_idx(n, seed=13)
    a, b = synth.muon_pairs(idx, dtype=dt)
    sel = torch.from_numpy(idx).cuda()
    tau = tau_of(dt)
    for cm in (False, True):
        m_out = torch.empty(n, dtype=TDT[dt], device="cuda")
        h = gvx.mass_histogram(v1, v2, cm=cm, m_out=m_out)
        assert int(h.sum()) == n
        x = m_out.double()
        q = (float(NB) * (x - LO)) / (HI - LO)
        inner = 1 + torch.trunc(torch.nan_to_num(q, nan=0.0, posinf=0.0, neginf=0.0)).long()
        bb = torch.where(x < LO, 0, torch.where(~(x < HI), NB + 1, inner))
        assert torch.equal(torch.bincount(bb, minlength=NB + 2), h), cm
        del x, q, inner, bb
        acc = gvx.new_bins()
        for r in range(4):
            lo_, hi_ = synth.shard_range(n, r, 4)
            gvx.mass_histogram(v1[lo_:hi_], v2[lo_:hi_], cm=cm, bins=acc)
        assert torch.equal(acc, h), cm
        mo, e = (O.cm_mass(a, b) if cm else O.invariant_mass(a, b))
        mlab, _ = O.invariant_mass(a, b)
        mg = host(m_out[sel])
        if cm:
            ok = np.isfinite(mo) & (np.abs(mlab.astype(np.float64)) >= (1e-2 if dt == np.float32 else 1e-6) * e)
        else:
            ok = np.ones(idx.size, bool)
        assert mass_violations(mg[ok], mo[ok], e[ok], tau).size == 0, cm
        del m_out


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_bench_step_fused_pass_full_size(gvx, O, dt):
    """The bench step's fused pair pass (gvx_pair_histograms) at its size and launch
    configuration (1e8 pairs, two-event TMA ring): both histograms == FindBin of the kernel's own
    lab / CM masses over all 1e8 events, sampled lab and CM masses vs the oracle, and the
    histograms and masses equal to the separate kernels' bit for bit."""
    import synth.device as sd
    n = 100_000_000
    v1, v2 = sd.muon_pairs(n, dtype=TDT[dt])
    m, mc = (torch.empty(n, dtype=TDT[dt], device="cuda") for _ in range(2))
    lab, cmb = gvx.pair_histograms(v1, v2, m_out=m, cm_m_out=mc)
    for h, mm in ((lab, m), (cmb, mc)):
        assert int(h.sum()) == n
        x = mm.double()
        q = (float(NB) * (x - LO)) / (HI - LO)
        inner = 1 + torch.trunc(torch.nan_to_num(q, nan=0.0, posinf=0.0, neginf=0.0)).long()
        bb = torch.where(x < LO, 0, torch.where(~(x < HI), NB + 1, inner))
        assert torch.equal(torch.bincount(bb, minlength=NB + 2), h)
        del x, q, inner, bb
    idx = _sample_idx(n, seed=17)
    a, b = synth.muon_pairs(idx, dtype=dt)
    sel = torch.from_numpy(idx).cuda()
    tau = tau_of(dt)
    mlab, e = O.invariant_mass(a, b)
    mo, ec = O.cm_mass(a, b)
    assert mass_violations(host(m[sel]), mlab, e, tau).size == 0
    ok = np.isfinite(mo) & (np.abs(mlab.astype(np.float64)) >= (1e-2 if dt == np.float32 else 1e-6) * e)
    assert mass_violations(host(mc[sel])[ok], mo[ok], ec[ok], tau).size == 0
    ref = torch.empty_like(m)
    bits = (lambda t: t.view(torch.int64)) if dt == np.float64 else (lambda t: t.view(torch.int32))
    assert torch.equal(gvx.mass_histogram(v1, v2, m_out=ref), lab) and torch.equal(bits(ref), bits(m))
    assert torch.equal(gvx.mass_histogram(v1, v2, cm=True, m_out=ref), cmb) and torch.equal(bits(ref), bits(mc))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_fast_domain_edges(gvx, O, dt):
    """Inputs just inside (and just outside) the fast-path domain of the GPU arithmetic
    (|eta| < 20, |phi| < 1024 f64 / 8 f32, 2^-200 (f64) / 2^-40 (f32) <= pt, pt and |m| large):
    lab mass, CM mass and cos theta* within the north-star tolerance of the oracle."""
    rng = np.random.default_rng(23)
    n = 20_000
    phimax = 1023.9 if dt == np.float64 else 7.99
    ptmin = 2.0 ** -199 if dt == np.float64 else 2.0 ** -39

    def vecs():
        v = np.empty((n, 4))
        v[:, 0] = np.exp(rng.uniform(np.log(1e-3), np.log(1e4), n))
        v[:, 1] = rng.choice([-1, 1], n) * rng.uniform(15.0, 20.5, n)       # some beyond 20: cold path
        v[:, 2] = rng.choice([-1, 1], n) * rng.uniform(0.9, 1.02, n) * phimax
        v[:, 3] = rng.uniform(-5.0, 100.0, n)
        v[: n // 20, 0] = ptmin * rng.uniform(0.5, 4.0, n // 20)          # around the pt lower bound
        return v.astype(dt)

    v1, v2 = vecs(), vecs()
    tau = tau_of(dt)
    e = energy_scale(O, v1, v2)
    mo, _ = O.invariant_mass(v1, v2)
    m = host(gvx.invariant_mass(dev(v1), dev(v2)))
    assert mass_violations(m, mo, e, tau).size == 0
    mcm, _ = O.cm_mass(v1, v2)
    m_out = torch.empty(n, dtype=TDT[dt], device="cuda")
    gvx.mass_histogram(dev(v1), dev(v2), cm=True, m_out=m_out)
    mlab = mo.astype(np.float64)
    ok = np.isfinite(mcm) & (np.abs(mlab) >= (1e-2 if dt == np.float32 else 1e-6) * e)
    assert mass_violations(host(m_out)[ok], mcm[ok], e[ok], tau).size == 0


def test_cm_costheta_large_axes(gvx, O):
    """Axes too large for shared-memory privatisation take the global-atomics kernel; counts
    still match the oracle's histograms (well-separated bins: no edge ambiguity at 1e-3 width)."""
    v1, v2 = synth.muon_pairs(np.arange(30_000), seed=41, dtype=np.float64)
    mb, cb = gvx.cm_costheta_histogram(dev(v1), dev(v2), m_axis=(0.0, 300.0, 60_000), c_axis=(-1.0, 1.0, 2_000))
    mbo, cbo, mo, co = O.cm_costheta(v1, v2, m_axis=(0.0, 300.0, 60_000), c_axis=(-1.0, 1.0, 2_000))
    _, _, _, _, delta, nanp, mlab, e = _costheta_reference(O, v1, v2, np.float64)
    fails, _ = hist_check_delta(host(cb), co, delta, -1.0, 1.0, 2_000, nan_possible=nanp)
    assert not fails, fails
    fails, _ = hist_check(host(mb), mo, e, 1e-12, 0.0, 300.0, 60_000, nan_possible=nanp, m_window_center=mlab)
    assert not fails, fails


def test_boost_high_beta_f64(gvx, O):
    """fp64 boosts at |β| = 0.999 … 0.9999 (reading R10's stress set) within τ·S of the oracle."""
    rng = np.random.default_rng(78)
    n = 100_000
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    beta = d * rng.uniform(0.999, 0.9999, size=(n, 1))
    v, _ = synth.boost_inputs(np.arange(n), seed=4)
    ref, S = O.boost(v, beta)
    out = host(gvx.boost(dev(v), dev(beta)))
    assert boost_violations(out, ref, S, 1e-12).size == 0


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("layout", ["aos", "soa", "pairs"])
def test_pair_histograms_fused_equals_separate(gvx, dt, layout):
    """gvx_pair_histograms (one pass) == invariant_mass + mass_histogram + mass_histogram(cm),
    bit for bit: masses, lab bins, CM masses, CM bins — TMA two-event ring (AoS/SoA, n above the
    small-batch threshold) and the two-pass fallback (strided pairs); edge rows included."""
    n = 300_000 + 7
    v1, v2 = mixed_inputs(n, dt, seed=5)
    t1, t2 = dev(v1), dev(v2)
    if layout == "soa":
        a = [t1[:, k].contiguous() for k in range(4)]
        b = [t2[:, k].contiguous() for k in range(4)]
    elif layout == "pairs":
        pr = torch.stack([t1, t2], 1).contiguous()
        a, b = pr[:, 0], pr[:, 1]
    else:
        a, b = t1, t2
    N = v1.shape[0]
    m, mc = (torch.empty(N, dtype=TDT[dt], device="cuda") for _ in range(2))
    lab, cmb = gvx.pair_histograms(a, b, m_out=m, cm_m_out=mc)
    m_ref = gvx.invariant_mass(t1, t2)
    mc_ref = torch.empty_like(m_ref)
    h_ref = gvx.mass_histogram(t1, t2)
    hc_ref = gvx.mass_histogram(t1, t2, cm=True, m_out=mc_ref)
    assert torch.equal(lab, h_ref) and torch.equal(cmb, hc_ref)
    assert np.array_equal(host(m), host(m_ref), equal_nan=True)
    assert np.array_equal(host(mc), host(mc_ref), equal_nan=True)
    lab2, cmb2 = gvx.pair_histograms(a, b, lab_bins=lab.clone(), cm_bins=cmb.clone())  # accumulates
    assert torch.equal(lab2, 2 * h_ref) and torch.equal(cmb2, 2 * hc_ref)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["pxpypze", "pxpypzm", "wide_axis", "small_n", "empty", "ragged_ring"])
def test_pair_histograms_other_branches(gvx, dt, case):
    """The fused pass's other dispatch branches equal the separate kernels bit for bit:
    Cartesian input through the TMA ring (PxPyPzE) and the two-pass fallback (PxPyPzM), an axis
    too wide for two shared-memory histograms (nbins = 40000: fallback), a batch below the
    small-batch threshold, n = 0 (nothing launched, bins untouched) and a ring whose last stage
    is ragged (n = one stage x 148 CTAs + 1)."""
    coords, nb, n = "ptetaphim", NB, 300_007
    if case in ("pxpypze", "pxpypzm"):
        coords = case
    elif case == "wide_axis":
        nb = 40_000
    elif case == "small_n":
        n = 1_001
    elif case == "empty":
        n = 0
    elif case == "ragged_ring":
        n = (1536 if dt == np.float64 else 1792) * 148 + 1
    if coords == "ptetaphim":
        v1, v2 = mixed_inputs(max(n, 1), dt, seed=9)
        v1, v2 = v1[:n], v2[:n]
    else:
        v1, _ = synth.boost_inputs(np.arange(n), dtype=dt, seed=5)
        v2, _ = synth.boost_inputs(np.arange(n), dtype=dt, seed=6)
        if coords == "pxpypzm":  # same momenta, the 4th component the (signed) mass
            for v in (v1, v2):
                v[:, 3] = np.sqrt(np.maximum(v[:, 3] ** 2 - (v[:, :3] ** 2).sum(1), 0.0))
    t1, t2 = dev(v1), dev(v2)
    N = t1.shape[0]
    m, mc = (torch.empty(N, dtype=TDT[dt], device="cuda") for _ in range(2))
    lab0 = torch.arange(nb + 2, dtype=torch.int64, device="cuda")
    lab, cmb = gvx.pair_histograms(t1, t2, LO, HI, nb, lab_bins=lab0.clone(), cm_bins=lab0.clone(), m_out=m,
                                   cm_m_out=mc, coords=coords)
    m_ref, mc_ref = torch.empty_like(m), torch.empty_like(mc)
    h_ref = gvx.mass_histogram(t1, t2, LO, HI, nb, bins=lab0.clone(), m_out=m_ref, coords=coords)
    hc_ref = gvx.mass_histogram(t1, t2, LO, HI, nb, cm=True, bins=lab0.clone(), m_out=mc_ref, coords=coords)
    assert torch.equal(lab, h_ref) and torch.equal(cmb, hc_ref)
    assert np.array_equal(host(m), host(m_ref), equal_nan=True)
    assert np.array_equal(host(mc), host(mc_ref), equal_nan=True)
    if n == 0:
        assert torch.equal(lab, lab0) and torch.equal(cmb, lab0)
    else:
        assert int((lab - lab0).sum()) == n and int((cmb - lab0).sum()) == n


@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("sizes", [((1 << 20) + 37, (1 << 20) + 11), ((1 << 21) + 5, (1 << 20) + 3),
                                   ((1 << 20) + 1, (1 << 22) + 7), (1000, 5000)])
def test_pair_histograms_boost_one_launch(gvx, dt, sizes):
    """gvx_pair_histograms_boost (the step in one launch: pair ring + boost ring on every SM) ==
    gvx_pair_histograms + gvx_boost bit for bit — bins, lab and CM masses, boosted vectors —
    with ragged pair and boost tails, unequal batch sizes (either one finishing first) and a
    small batch (the two-call fallback)."""
    n, nb = sizes
    v1, v2 = mixed_inputs(n, dt, seed=21)
    n = v1.shape[0]
    t1, t2 = dev(v1), dev(v2)
    x, beta = synth.boost_inputs(np.arange(nb), dtype=dt, seed=8)
    tx, tb = dev(x), dev(beta)
    m, mc, m_ref, mc_ref = (torch.empty(n, dtype=TDT[dt], device="cuda") for _ in range(4))
    lab, cmb, out = gvx.pair_histograms_boost(t1, t2, tx, tb, m_out=m, cm_m_out=mc)
    lab_ref, cmb_ref = gvx.pair_histograms(t1, t2, m_out=m_ref, cm_m_out=mc_ref)
    out_ref = gvx.boost(tx, tb)
    assert torch.equal(lab, lab_ref) and torch.equal(cmb, cmb_ref)
    assert int(lab.sum()) == n and int(cmb.sum()) == n
    assert np.array_equal(host(m), host(m_ref), equal_nan=True)
    assert np.array_equal(host(mc), host(mc_ref), equal_nan=True)
    assert np.array_equal(host(out), host(out_ref), equal_nan=True)


def test_one_launch_step_repeat_bitwise(gvx):
    """Ring-reuse stress for k_step (the check that caught the missing proxy fence in the pair
    ring): L2-sized batches (2^20 pairs, 2^20 boosts: each CTA cycles both rings many times with
    L2-resident refills) run 40 times; every run equals the two-call result bit for bit."""
    import synth.device as sd
    n = nb = 1 << 20
    v1, v2 = sd.muon_pairs(n, dtype=torch.float64)
    bv, bb = sd.boost_inputs(nb, dtype=torch.float64)
    m_ref = torch.empty(n, dtype=torch.float64, device="cuda")
    lab_ref, cm_ref = gvx.pair_histograms(v1, v2, m_out=m_ref)
    out_ref = gvx.boost(bv, bb)
    m = torch.empty_like(m_ref)
    out = torch.empty_like(out_ref)
    for _ in range(40):
        lab, cmb, _o = gvx.pair_histograms_boost(v1, v2, bv, bb, m_out=m, out=out)
        assert torch.equal(lab, lab_ref) and torch.equal(cmb, cm_ref)
        assert torch.equal(m.view(torch.int64), m_ref.view(torch.int64))
        assert torch.equal(out.view(torch.int64), out_ref.view(torch.int64))


# ----------------------------------------------------------------------------
# Mixed-coordinate pairs (ABI v7; "any 4-dimensional coordinate system")
# ----------------------------------------------------------------------------
SYSTEMS = ("ptetaphim", "pxpypze", "pxpypzm", "ptetaphie")


def as_system(v, system):
    """Rewrite PtEtaPhiM vectors (f64) in `system` (numpy f64; input preparation, not the method)."""
    pt, eta, phi, m = v[:, 0], v[:, 1], v[:, 2], v[:, 3]
    px, py, pz = pt * np.cos(phi), pt * np.sin(phi), pt * np.sinh(eta)
    E = np.sqrt(m * m + (pt * np.cosh(eta)) ** 2)
    return {"ptetaphim": v, "pxpypze": np.stack([px, py, pz, E], 1), "pxpypzm": np.stack([px, py, pz, m], 1),
            "ptetaphie": np.stack([pt, eta, phi, E], 1)}[system]


def scale_of(O, v, system):
    """max(E, |p|) of each vector in its own system (reading R5)."""
    _, e = O.invariant_mass(v, np.zeros_like(v), coords=system)
    a = v.astype(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        p = np.abs(a[:, 0]) * np.cosh(a[:, 1]) if system.startswith("pt") else np.sqrt((a[:, :3] ** 2).sum(1))
    return np.fmax(e.astype(np.float64), p)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_mixed_coordinate_pairs(gvx, O, dt):
    """All 16 (system of v1, system of v2) combinations against the oracle: lab masses (AoS, SoA,
    strided views), lab and CM histograms (R14), the fused pair pass and the one-call step; equal
    systems through the mixed entry points are bit-identical to the single-system calls."""
    n = 40_003
    base1, base2 = synth.muon_pairs(np.arange(n), seed=404)
    ea, eb = edge_events(np.float64)
    tau = tau_of(dt)
    for s1 in SYSTEMS:
        for s2 in SYSTEMS:
            with np.errstate(invalid="ignore", over="ignore"):
                v1 = np.concatenate([as_system(ea, s1), as_system(base1, s1)]).astype(dt)
                v2 = np.concatenate([as_system(eb, s2), as_system(base2, s2)]).astype(dt)
            mo, _ = O.invariant_mass(v1, v2, coords=s1, coords2=s2)
            e = scale_of(O, v1, s1) + scale_of(O, v2, s2)
            t1, t2 = dev(v1), dev(v2)
            m = host(gvx.invariant_mass(t1, t2, coords=s1, coords2=s2))
            bad = mass_violations(m, mo, e, tau)
            assert bad.size == 0, (s1, s2, bad[:5], m[bad[:5]], mo[bad[:5]])
            soa = lambda t: [t[:, k].contiguous() for k in range(4)]  # noqa: E731
            assert np.array_equal(host(gvx.invariant_mass(soa(t1), soa(t2), coords=s1, coords2=s2)), m, equal_nan=True)
            pairs = torch.stack([t1, t2], dim=1).contiguous()
            assert np.array_equal(host(gvx.invariant_mass(pairs[:, 0, :], pairs[:, 1, :], coords=s1, coords2=s2)), m,
                                  equal_nan=True)
            if s1 == s2:
                assert np.array_equal(m, host(gvx.invariant_mass(t1, t2, coords=s1)), equal_nan=True)
            for cm in (False, True):
                mg = torch.empty(v1.shape[0], dtype=TDT[dt], device="cuda")
                h = host(gvx.mass_histogram(t1, t2, cm=cm, coords=s1, coords2=s2, m_out=mg))
                ho, mho = O.mass_histogram(v1, v2, LO, HI, NB, cm=cm, coords=s1, coords2=s2)
                nanp = (np.isnan(mho) | (np.abs(mo.astype(np.float64)) < (1e-2 if dt == np.float32 else 1e-6) * e)) \
                    if cm else None
                fails, _ = hist_check(h, mho, e, tau, LO, HI, NB, nan_possible=nanp, m_window_center=mo if cm else None)
                assert not fails, (s1, s2, cm, fails)
                ok = ~nanp if cm else np.ones(v1.shape[0], bool)
                assert mass_violations(host(mg)[ok], mho[ok], e[ok], tau).size == 0, (s1, s2, cm)
                assert np.array_equal(h, np.bincount(find_bin_np(host(mg), LO, HI, NB), minlength=NB + 2))
            # the fused pair pass and the one-call step: the same bins and masses as the calls above
            ml, mc = (torch.empty(v1.shape[0], dtype=TDT[dt], device="cuda") for _ in range(2))
            lab, cmb = gvx.pair_histograms(t1, t2, coords=s1, coords2=s2, m_out=ml, cm_m_out=mc)
            assert np.array_equal(host(ml), m, equal_nan=True)
            mcs = torch.empty_like(mc)
            assert torch.equal(gvx.mass_histogram(t1, t2, coords=s1, coords2=s2), lab)
            assert torch.equal(gvx.mass_histogram(t1, t2, cm=True, coords=s1, coords2=s2, m_out=mcs), cmb)
            assert np.array_equal(host(mc), host(mcs), equal_nan=True), (s1, s2)
            bv, bb = synth.boost_inputs(np.arange(1000), dtype=dt)
            lab2, cmb2, out = gvx.pair_histograms_boost(t1, t2, dev(bv), dev(bb), coords=s1, coords2=s2)
            assert torch.equal(lab2, lab) and torch.equal(cmb2, cmb), (s1, s2)
            assert np.array_equal(host(out), host(gvx.boost(dev(bv), dev(bb))), equal_nan=True), (s1, s2)


def test_mixed_coordinate_pair_closed_form(gvx):
    """SPEC.md:88's vector (PtEtaPhiM) against its mirror image in PxPyPzE as S:88 prints it:
    back to back with equal energies, M = 2E (f64 to τ·E²)."""
    a = torch.tensor([[10.0, 1.2, 0.5, 0.105]] * 5, dtype=torch.float64, device="cuda")
    b = torch.tensor([[-8.7758256189037271612, -4.7942553860420300027, -15.09461355412172616,
                       18.106860118426809386]] * 5, dtype=torch.float64, device="cuda")
    m = host(gvx.invariant_mass(a, b, coords="ptetaphim", coords2="pxpypze"))
    E = 2 * 18.106860118426809386
    assert np.all(np.abs(m * m - E * E) <= 1e-12 * E * E), m
    mc = torch.empty(5, dtype=torch.float64, device="cuda")
    gvx.mass_histogram(a, b, cm=True, coords="ptetaphim", coords2="pxpypze", m_out=mc)
    assert np.all(np.abs(host(mc) ** 2 - E * E) <= 1e-12 * E * E)


def test_bench_two_ranks_self_check():
    """bench.py's N > 1 path end to end on one GPU: two torchrun ranks (gloo, both mapped to
    cuda:0 by GVX_BENCH_SAME_DEVICE — plumbing only, never numbers) shard the index space,
    all-reduce the bins, and rank 0's self-check recomputes the one-GPU histogram of all global
    indices: the line must report bins_equal and n_gpus 2."""
    import json
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--events", "1000003", "--dist-backend", "gloo", "--no-e2e", "--no-per-op"]
    for extra in ([], ["--two-launch"]):
        r = subprocess.run(cmd + extra, cwd=root, capture_output=True, text=True, timeout=900,
                           env=dict(os.environ, GVX_BENCH_SAME_DEVICE="1", PYTHONPATH=root))
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
        line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
        assert line["n_gpus"] == 2 and line["self_check"]["bins_equal"], line.get("self_check")
        assert line["self_check"]["events"] == 2 * 1000003
