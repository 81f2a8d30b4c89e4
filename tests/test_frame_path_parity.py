"""Bit-exact order and binning of the BENCHMARKED frame path (sc_render_composed /
sc_render_survivors), not only of the stage-level sc_bin_sort.

The frame path quantises depth keys over the instance spheres' depth range,
re-orders equal keys by (f64 depth, survivor index) and bins (splat, 8x4
pixel block) entries instead of (splat, 16x16 tile) entries.  Given the
oracle's survivor set (injected with sc_render_survivors), these tests assert
against the oracle (reference-pinned, tests/test_oracle_golden.py):

  (i)   the (depth, index) order of the passed survivors equals the oracle's
        argsort(depth, kind="stable") (sc/raster.py:319) exactly;
  (ii)  with exact projection, every (tile, block) list equals the oracle's
        bin_tiles segment of that tile (sc/_kernels.py:137-165) filtered to the
        entries whose product pixel window touches the block, with the same
        clipped window code, entry for entry;
  (iii) the product window never drops a pixel the reference composites: an
        entry of the tile segment whose reference window (sc/_kernels.py:224-227)
        touches the block but that is missing from the block list composites at
        none of the block's pixels under the oracle's f64 power / opacity tests
        (sc/_kernels.py:215-247);
  (iv)  with the default f32-covariance projection, every list is an in-order
        subsequence of the reference-window-filtered segment that contains the
        exact-projection list.
"""

import math

import numpy as np
import pytest

from oracle import raster_ref as rr
from oracle import scene_ref as sr

pytestmark = pytest.mark.gpu

LN_MIN_ALPHA = math.log(1.0 / 255.0)


def _blocks(counts, entry_idx, x0, x1, y0, y1, width, height):
    """(block id, entry, code) triples of the tile segments, block-major, entry order
    inside a block.  x0..y1 are per-entry pixel windows (before the tile clip)."""
    n_tx = (width + 15) // 16
    tile = np.repeat(np.arange(counts.size - 1, dtype=np.int64), np.diff(counts))
    ty, tx = tile // n_tx, tile % n_tx
    cx0 = np.maximum(np.maximum(x0, 16 * tx), 0)
    cx1 = np.minimum(np.minimum(x1, 16 * tx + 15), width - 1)
    cy0 = np.maximum(np.maximum(y0, 16 * ty), 0)
    cy1 = np.minimum(np.minimum(y1, 16 * ty + 15), height - 1)
    ids, codes, touch = [], [], []
    for b in range(8):
        bx0 = 16 * tx + 8 * (b & 1)
        by0 = 16 * ty + 4 * (b >> 1)
        a0, a1 = np.maximum(cx0, bx0), np.minimum(cx1, bx0 + 7)
        b0, b1 = np.maximum(cy0, by0), np.minimum(cy1, by0 + 3)
        touch.append((a0 <= a1) & (b0 <= b1))
        ids.append(8 * tile + b)
        codes.append((a0 - bx0) | ((a1 - bx0) << 3) | ((b0 - by0) << 6) | ((b1 - by0) << 8))
    touch = np.stack(touch, 1).reshape(-1)
    ids = np.stack(ids, 1).reshape(-1)[touch]
    codes = np.stack(codes, 1).reshape(-1)[touch]
    ent = np.repeat(entry_idx, 8)[touch]
    pos = np.repeat(np.arange(entry_idx.size), 8)[touch]   # position in the tile-binned list
    o = np.argsort(ids, kind="stable")
    return ids[o], ent[o], codes[o], pos[o]


def _offsets(ids, n_blocks):
    return np.searchsorted(ids, np.arange(n_blocks + 1), side="left")


def _product_windows(dscene, surv_inst, surv_gid, cam, opts):
    from paper_2511_19202_b200 import stages

    p = stages.project(dscene, surv_inst, surv_gid, cam, opts)
    w = p["windows"].cpu().numpy().view(np.int16).reshape(-1, 4).astype(np.int64)
    return w[:, 0], w[:, 1], w[:, 2], w[:, 3]


def _reference_windows(st):
    m, r = st.proj.mean2d, st.proj.radius
    return (np.floor(m[:, 0] - r).astype(np.int64), np.floor(m[:, 0] + r).astype(np.int64) + 1,
            np.floor(m[:, 1] - r).astype(np.int64), np.floor(m[:, 1] + r).astype(np.int64) + 1)


def _composites_somewhere(st, ent, bid, width, height):
    """Per (entry, block): does the oracle composite the entry at any pixel of the
    block inside its reference window (the power / opacity tests of
    sc/_kernels.py:215-247; T-independent)?"""
    n_tx = (width + 15) // 16
    tile, b = bid // 8, bid % 8
    bx0 = 16 * (tile % n_tx) + 8 * (b & 1)
    by0 = 16 * (tile // n_tx) + 4 * (b >> 1)
    rx0, rx1, ry0, ry1 = (w[ent] for w in _reference_windows(st))
    op = st.opacity[ent]
    p_min = LN_MIN_ALPHA - np.log(np.maximum(op, 1e-300))
    ha, bb, hc = 0.5 * st.proj.conic[ent, 0], st.proj.conic[ent, 1], 0.5 * st.proj.conic[ent, 2]
    mx, my = st.proj.mean2d[ent, 0], st.proj.mean2d[ent, 1]
    hit = np.zeros(ent.size, bool)
    for lane in range(32):
        px, py = bx0 + (lane & 7), by0 + (lane >> 3)
        inside = (px >= rx0) & (px <= rx1) & (py >= ry0) & (py <= ry1) & (px < width) & (py < height)
        dx, dy = px - mx, py - my
        power = -(ha * dx * dx + hc * dy * dy) - bb * dx * dy
        hit |= inside & (op >= 1.0 / 255.0) & ~(power > 0.0) & ~(power < p_min)
    return hit


def _pair_keys(ids, ent):
    return ids.astype(np.int64) * (1 << 32) + ent.astype(np.int64)


def _subsequence_check(got_ids, got_ent, ids, ent, pos):
    """got (block id, entry) pairs are a subset of (ids, ent) with entries in list order per block."""
    k_all = _pair_keys(ids, ent)
    o = np.argsort(k_all, kind="stable")
    ks, ps = k_all[o], pos[o]
    k_got = _pair_keys(got_ids, got_ent)
    j = np.minimum(np.searchsorted(ks, k_got), ks.size - 1)
    assert np.all(ks[j] == k_got), "block list holds an entry that is not in the tile's bin_tiles segment"
    gp = ps[j]
    same = got_ids[1:] == got_ids[:-1]
    assert np.all(gp[1:][same] > gp[:-1][same]), "block list out of (depth, index) order"


def _contains(big_ids, big_ent, small_ids, small_ent):
    kb = np.sort(_pair_keys(big_ids, big_ent))
    ksm = _pair_keys(small_ids, small_ent)
    j = np.minimum(np.searchsorted(kb, ksm), max(kb.size - 1, 0))
    return ksm.size == 0 or (kb.size > 0 and bool(np.all(kb[j] == ksm)))


def check_frame_path(scene, cam, surv_inst, surv_gid, **render_kw):
    """Inject the oracle's survivors into the frame path and check (i)-(iv) against the
    oracle rendering the same survivors."""
    import torch

    from paper_2511_19202_b200.scene import RenderOptions, Renderer

    tabs = sr.SceneTables(scene)
    m, ls, q, op, sh, deg = sr.instantiate(tabs, cam, surv_inst, surv_gid)
    st = rr.Stages()
    oracle_kw = {k: v for k, v in render_kw.items() if k not in ("use_mlp", "frustum")}
    ref = rr.render_arrays(m, ls, q, op, sh, deg, cam, stages=st, **oracle_kw)
    r = Renderer(scene)
    dev = r.dscene.device
    surv = torch.from_numpy(np.stack([surv_inst, surv_gid], 1).astype(np.uint32).view(np.int32)).to(dev)
    W, H = int(cam.width), int(cam.height)
    n_blocks = 8 * ((W + 15) // 16) * ((H + 15) // 16)
    res = {}
    for exact in (True, False):
        opts = RenderOptions(exact_projection=exact, **render_kw)
        _frame, fst, dbg = r.render(cam, opts, to_host=False, survivors=surv, debug=True)
        assert fst.passed == ref.passed_count
        # (i) order
        np.testing.assert_array_equal(dbg["order"], st.order_idx)
        np.testing.assert_array_equal(dbg["block_offsets"][-1], fst.block_entries)
        got_ids = dbg["block_codes"] >> 10
        got_codes = dbg["block_codes"] & 0x3FF
        np.testing.assert_array_equal(_offsets(got_ids, n_blocks), dbg["block_offsets"])
        res[exact] = (got_ids, dbg["block_entries"], got_codes)
        if exact:
            # (ii) exact lists: the oracle's segments filtered by the product window
            x0, x1, y0, y1 = _product_windows(r.dscene, surv_inst, surv_gid, cam, opts)
            e = st.entry_idx
            ids, ent, codes, _pos = _blocks(st.counts, e, x0[e], x1[e], y0[e], y1[e], W, H)
            np.testing.assert_array_equal(got_ids, ids)
            np.testing.assert_array_equal(dbg["block_entries"], ent)
            np.testing.assert_array_equal(got_codes, codes)
            # (iii) entries the window clipped away composite nowhere in the block
            rx0, rx1, ry0, ry1 = _reference_windows(st)
            rids, rent, _rc, rpos = _blocks(st.counts, e, rx0[e], rx1[e], ry0[e], ry1[e], W, H)
            kk = np.sort(_pair_keys(ids, ent))
            kr = _pair_keys(rids, rent)
            j = np.minimum(np.searchsorted(kk, kr), max(kk.size - 1, 0))
            miss = ~(kk[j] == kr) if kk.size else np.ones(kr.size, bool)
            if miss.any():
                hit = _composites_somewhere(st, rent[miss], rids[miss], W, H)
                assert not hit.any(), f"{int(hit.sum())} dropped (entry, block) pairs composite a pixel"
            ref_lists = (rids, rent, rpos)
    # (iv) fast projection: exact lists <= fast lists <= reference-window lists, in order
    fi, fe, _fc = res[False]
    ei, ee, _ec = res[True]
    rids, rent, rpos = ref_lists
    _subsequence_check(fi, fe, rids, rent, rpos)
    assert _contains(fi, fe, ei, ee), "fast projection dropped an exact-path entry"
    return ref, st


def pkg_render(sc, cam):
    import paper_2511_19202_b200 as pkg

    return pkg.render_composed(sc, cam, use_mlp=False)


def _single(asset):
    from paper_2511_19202_b200.scene import ComposedScene, InstanceTransform

    sc = ComposedScene()
    sc.add_asset(asset)
    sc.add_instance(0, InstanceTransform())
    return sc


def test_frame_path_goldens(golden):
    name, asset, cam, opts, z = golden
    if opts.get("tile_size", 16) != 16:
        pytest.skip("block lists are compared with 16x16 reference tiles")
    kw = {k: v for k, v in opts.items() if k != "record_contributions"}
    n = len(asset)
    ref, st = check_frame_path(_single(asset), cam, np.zeros(n, np.int64), np.arange(n), use_mlp=False,
                               frustum="off", **kw)
    np.testing.assert_array_equal(st.order_idx, z["order_idx"])   # the oracle is the reference here
    np.testing.assert_array_equal(st.entry_idx, z["entry_idx"])


@pytest.mark.parametrize("cam_i", [0, 1, 2])
def test_frame_path_composed_scenes(cam_i):
    from conftest import look_at
    from test_gpu_parity import CAMS, _multi_scene

    sc = _multi_scene(with_model=True)
    cam = look_at(*CAMS[cam_i])
    c = sr.cull(sr.SceneTables(sc), cam)
    check_frame_path(sc, cam, c.surv_inst, c.surv_gid, use_mlp=True)


@pytest.mark.parametrize("view", [0, 1, 2], ids=["near", "mid", "far"])
def test_frame_path_config3_views(view):
    from paper_2511_19202_b200.workloads import config3

    wl = config3(n_per=6_000, n_instances=150, width=480, height=270)
    cam = wl.cameras[view]
    c = sr.cull(sr.SceneTables(wl.scene), cam)
    check_frame_path(wl.scene, cam, c.surv_inst, c.surv_gid)


@pytest.mark.parametrize("tilt, n", [(2e-12, 1_500), (0.0, 20_000), (2e-12, 60_000)],
                         ids=["tilted-unsorted-run", "head-on-equal-run", "tilted-unsorted-60k-run"])
def test_frame_path_tie_runs(tilt, n):
    from paper_2511_19202_b200.camera import Camera
    from test_gpu_parity import _plane_asset

    asset = _plane_asset(n, seed=5)
    cam = Camera.look_at((0.0, 0.0, 3.0), (tilt, 0.0, 0.0), math.radians(50.0), 96, 96, up=(0.0, 1.0, 0.0))
    check_frame_path(_single(asset), cam, np.zeros(n, np.int64), np.arange(n), use_mlp=False, frustum="off")


def test_frame_path_deep_scene():
    """Depth range >= 1e4 x the splat spacing: one instance at depth ~2, one ~4e6
    away, so the 32-bit keys over the whole range resolve ~1e-3 while the near
    asset's splats lie ~1e-4 apart in depth: they collide into tie runs that
    the (f64 depth, index) tie-fix must order exactly."""
    from paper_2511_19202_b200 import synth
    from paper_2511_19202_b200.asset import prepare
    from paper_2511_19202_b200.camera import Camera
    from paper_2511_19202_b200.scene import ComposedScene, InstanceTransform

    sc = ComposedScene()
    a = prepare(synth.make_random_cloud(30_000, seed=21))
    sc.add_asset(a)
    sc.add_instance(0, InstanceTransform([0.0, 0.0, 0.0], [1, 0, 0, 0], 1.0))
    sc.add_instance(0, InstanceTransform([0.0, 4.0e6, 0.0], [1, 0, 0, 0], 1.5e5))
    cam = Camera.look_at((0.0, -2.0, 0.0), (0.0, 0.0, 0.0), math.radians(60.0), 160, 120)
    c = sr.cull(sr.SceneTables(sc), cam)
    assert np.unique(c.surv_inst).size == 2
    ref, _st = check_frame_path(sc, cam, c.surv_inst, c.surv_gid)
    assert ref.passed_count > 10_000
    _out, st = pkg_render(sc, cam)
    assert st.max_tie_run >= 8, st   # the near asset's keys really collide


def test_frame_path_record_and_image_match_oracle():
    """The injected-survivor frame equals the oracle's image within the blend tolerance."""
    from conftest import look_at
    from test_gpu_parity import CAMS, _image_close, _multi_scene

    from paper_2511_19202_b200.scene import RenderOptions, Renderer

    import torch

    sc = _multi_scene(with_model=True)
    cam = look_at(*CAMS[0])
    c = sr.cull(sr.SceneTables(sc), cam)
    m, ls, q, op, sh, deg = sr.instantiate(sr.SceneTables(sc), cam, c.surv_inst, c.surv_gid)
    ref = rr.render_arrays(m, ls, q, op, sh, deg, cam, record_contributions=True)
    r = Renderer(sc)
    surv = torch.from_numpy(np.stack([c.surv_inst, c.surv_gid], 1).astype(np.int32)).to(r.dscene.device)
    out, st = r.render(cam, RenderOptions(record_contributions=True), survivors=surv)
    _image_close(out.image, ref.image)
    np.testing.assert_allclose(out.contribution_max, ref.contribution_max, atol=5e-3)
    assert st.passed == ref.passed_count


_CFG2 = {}


def _cfg2():
    if "wl" not in _CFG2:
        from paper_2511_19202_b200.workloads import config2

        _CFG2["wl"] = config2()
    return _CFG2["wl"]


@pytest.mark.parametrize("frame", [0, 24, 48, 72, 96])
def test_config2_full_size(frame):
    """BASELINE config 2 at full size (100K shell x 16 instances, 1080p, orbit frames;
    SURVEY §4 / §8d): with the oracle's survivors injected, order and (tile, block)
    lists are bit-exact (i)-(iv) and the image is within the blend tolerance of the
    oracle rendering the same survivors; the whole pipeline (GPU cull + MLP) is
    >= 45 dB against the oracle's whole pipeline."""
    import torch

    import paper_2511_19202_b200 as pkg
    from paper_2511_19202_b200.scene import RenderOptions, Renderer
    from test_gpu_parity import _image_close

    wl = _cfg2()
    cam = wl.cameras[frame]
    tabs = sr.SceneTables(wl.scene)
    c = sr.cull(tabs, cam)
    assert c.surv_inst.size > 100_000
    ref, _st = check_frame_path(wl.scene, cam, c.surv_inst, c.surv_gid)
    r = Renderer(wl.scene)
    surv = torch.from_numpy(np.stack([c.surv_inst, c.surv_gid], 1).astype(np.int32)).to(r.dscene.device)
    out, _fst = r.render(cam, RenderOptions(), survivors=surv)
    _image_close(out.image, ref.image)
    whole, st = pkg.render_composed(wl.scene, cam)
    assert st.frustum_passed == int(np.count_nonzero(c.flags & 1))
    # MLP decisions may differ only within the fp16 logit margin of the threshold
    assert abs(st.instantiated - c.surv_inst.size) <= max(3, int(1e-4 * c.surv_inst.size))
    assert rr.psnr(whole.image, ref.image, cap=None) >= 45.0
    assert rr.ssim(whole.image, ref.image) >= 0.995


@pytest.mark.parametrize("log2", [0, 5, 9])
@pytest.mark.parametrize("view", [0, 2], ids=["near", "far"])
def test_long_lists_cta_walk(monkeypatch, log2, view):
    """Lists of >= 2^log2 entries are walked by a whole CTA (segments composited
    from T = 1, combined in order, the retiring segment re-composited exactly;
    blend.cu coop_list).  Forced onto every list of a small config-3 view with
    SPLATCULL_B200_LONG_LIST_LOG2: the image equals the per-warp serial walk within
    fp32 reassociation, and the oracle (sc/_kernels.py:190-275 on the same
    survivors) within the blend tolerance; bands stay bit-identical to the whole
    frame; record mode keeps the serial walk (its contributions need the true T)."""
    import torch

    from test_gpu_parity import _image_close

    from paper_2511_19202_b200 import sharding
    from paper_2511_19202_b200.scene import RenderOptions, Renderer
    from paper_2511_19202_b200.workloads import config3

    wl = config3(n_per=6_000, n_instances=150, width=480, height=270)
    cam = wl.cameras[view]
    r = Renderer(wl.scene)
    monkeypatch.setenv("SPLATCULL_B200_LONG_LIST_LOG2", "40")
    serial, sst = r.render(cam, return_survivors=True)
    monkeypatch.setenv("SPLATCULL_B200_LONG_LIST_LOG2", str(log2))
    coop, cst = r.render(cam, return_survivors=True)
    assert cst.block_entries == sst.block_entries and cst.passed == sst.passed
    d = np.abs(coop.image.astype(np.float64) - serial.image)
    assert d.max() <= 2e-4, d.max()
    assert np.abs(coop.final_transmittance.astype(np.float64) - serial.final_transmittance).max() <= 2e-4
    s = coop.survivors
    m, ls, q, op, sh, deg = sr.instantiate(sr.SceneTables(wl.scene), cam, s[:, 0], s[:, 1])
    ref = rr.render_arrays(m, ls, q, op, sh, deg, cam)
    _image_close(coop.image, ref.image)
    # bands: the same lists, so the same walk decisions
    full, _ = r.render(cam, RenderOptions(), to_host=False)
    img = full.image.clone()
    bounds = sharding.split_rows(sharding.tile_rows(cam.height), 3)
    for b in range(len(bounds) - 1):
        y0, y1 = sharding.band_pixels(bounds, b, cam.height)
        band, _ = r.render(cam, RenderOptions(band=(y0, y1)), to_host=False)
        assert torch.equal(band.image[y0:y1], img[y0:y1]), b
    # record mode: serial walk whatever the threshold
    rec, _ = r.render(cam, RenderOptions(record_contributions=True))
    monkeypatch.setenv("SPLATCULL_B200_LONG_LIST_LOG2", "40")
    rec40, _ = r.render(cam, RenderOptions(record_contributions=True))
    np.testing.assert_array_equal(rec.image, rec40.image)
    np.testing.assert_array_equal(rec.contribution_max, rec40.contribution_max)
