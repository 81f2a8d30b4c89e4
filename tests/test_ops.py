"""torch.library boundary (BASELINE north_star: "PyTorch custom ops over a thin C-ABI").

CPU: every op is registered under torch.ops.splatcull with a fake kernel, so
the path traces under FakeTensorMode without a GPU.  GPU: the frame op runs
inside a captured CUDA graph and under torch.compile(fullgraph=True) with
results identical to eager, and torch.library.opcheck validates the schemas.
"""

import numpy as np
import pytest
import torch

OPS = ["render_frame_", "render_frame", "cull_mlp", "project", "bin_sort", "blend", "vis_mlp_forward",
       "encode_features", "visibility_labels_or_"]


def test_ops_registered():
    import paper_2511_19202_b200.ops  # noqa: F401

    for name in OPS:
        assert hasattr(torch.ops.splatcull, name), name


def test_fake_kernels_shapes():
    """Shapes and dtypes from the fake (meta) kernels, no device code runs."""
    from torch._subclasses.fake_tensor import FakeTensorMode

    from paper_2511_19202_b200 import _native as nat
    from paper_2511_19202_b200 import ops

    with FakeTensorMode():
        dev = torch.device("cuda", 0)
        scene = [torch.empty(4, device=dev) for _ in range(9)]
        ws = torch.empty(1024, dtype=torch.uint8, device=dev)
        cam_f, cam_i = [0.0] * 16, [320, 180]
        opt_f, opt_i = [0.0, 1 / 255, 1.0, 1.0, 1.0, 0.3, 1.0], [16, -1, 0, 1, 0, 0, 0, 0]
        img, tr, st = torch.ops.splatcull.render_frame(scene, [1, 3, 1, 1, 0, 1], cam_f, cam_i, opt_f, opt_i, ws,
                                                       [1, 1, 1, 1])
        assert img.shape == (180, 320, 3) and tr.shape == (180, 320) and st.shape == (nat.STATS_BYTES,)
        assert img.dtype == torch.float32 and st.dtype == torch.uint8
        surv = torch.empty((10, 2), dtype=torch.int32, device=dev)
        sp, win, dbg, rect, flags, pst = ops.project(scene, [1, 3, 1, 1, 0, 1], surv, cam_f, cam_i, opt_f, opt_i)
        assert sp.shape == (10, nat.SPLAT_BYTES) and dbg.shape == (10, 8) and dbg.dtype == torch.float64
        opt_i8 = [8] + opt_i[1:]
        out = ops.bin_sort(scene, [1, 3, 1, 1, 0, 1], surv, cam_f, cam_i, opt_f, opt_i8, ws, [1, 1, 10, 64])
        assert out[2].shape == (64,) and out[3].shape == (40 * 23 + 1,)
        x = torch.empty((7, 16), device=dev)
        assert ops.vis_mlp_forward(torch.empty(8, dtype=torch.uint8, device=dev), x).shape == (7,)
        f = ops.encode_features(torch.empty(8, device=dev), torch.empty((5, 14), device=dev))
        assert f.shape == (5, 8) and f.dtype == torch.float16


def _small_scene():
    from paper_2511_19202_b200.workloads import config3

    return config3(n_per=5_000, n_instances=80, width=320, height=180)


@pytest.mark.gpu
def test_cuda_graph_replays_frame():
    """A whole frame (cull, MLP, projection, sort, blend) captured once in a CUDA graph and
    replayed: no host synchronisation inside the path, results equal to eager."""
    from paper_2511_19202_b200.scene import RenderOptions, Renderer

    wl = _small_scene()
    r = Renderer(wl.scene)
    for cam in wl.cameras:
        ref, st = r.render(cam, RenderOptions(), to_host=False)   # sizes the workspace
        want = ref.image.clone()
        out = r.render_device(cam, RenderOptions())
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            r.render_device(cam, RenderOptions(), out=out)
        for _ in range(2):
            out.image.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(out.image, want)


@pytest.mark.gpu
def test_torch_compile_fullgraph():
    from paper_2511_19202_b200 import ops
    from paper_2511_19202_b200.scene import RenderOptions, Renderer

    wl = _small_scene()
    r = Renderer(wl.scene)
    cam = wl.cameras[2]
    ref, _st = r.render(cam, RenderOptions(), to_host=False)
    ws = r.workspace(cam)
    cam_f, cam_i = ops.pack_camera(cam)
    opt_f, opt_i = ops.pack_opts(RenderOptions().struct(cam))
    scene, meta, ws_meta = r.dscene.op_scene, r.dscene.op_meta, ws.op_meta

    def frame(buf):
        img, tr, st = torch.ops.splatcull.render_frame(scene, meta, cam_f, cam_i, opt_f, opt_i, buf, ws_meta)
        return img * tr[..., None]

    eager = frame(ws.buf)
    compiled = torch.compile(frame, fullgraph=True)(ws.buf)
    torch.cuda.synchronize()
    assert torch.equal(eager, compiled)
    assert torch.equal(eager, ref.image * ref.trans[..., None])


@pytest.mark.gpu
def test_opcheck_mlp_ops():
    from paper_2511_19202_b200 import nn, ops, synth
    from paper_2511_19202_b200.asset import prepare
    from paper_2511_19202_b200 import _native as nat
    from paper_2511_19202_b200.scene import feature_params, vis_weights_struct
    from paper_2511_19202_b200.workloads import calibrated_model

    a = prepare(synth.make_shell(1000, seed=1))
    m = calibrated_model(a, seed=1)
    w = nat.struct_tensor(vis_weights_struct(m), "cuda")
    x = torch.rand((1000, 16), device="cuda") * 2 - 1
    torch.library.opcheck(torch.ops.splatcull.vis_mlp_forward.default, (w, x))
    p = torch.from_numpy(feature_params(m)).cuda()
    xf = torch.from_numpy(nn.feature_inputs(a, m.mean_scale)).cuda()
    torch.library.opcheck(torch.ops.splatcull.encode_features.default, (p, xf))
    np.testing.assert_array_equal(ops.vis_mlp_forward(w, x).cpu().numpy(), nn.forward(m, x)[:, 0].cpu().numpy())
