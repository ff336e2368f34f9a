"""tcgen05 GEMM (Darknet layer core) vs a plain PyTorch fp32 reference.

The operands are bf16; the reference upcasts the SAME bf16 values to fp32
and multiplies in fp32, so the only difference is accumulation order inside
the tensor core: fp32 outputs must agree to 1e-5 relative (plus an absolute
floor scaled by sqrt(K) for cancellation near zero).
"""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
W = pytest.importorskip("paper_2107_08538_b200.workloads")


def ref(a, b, bias, act):
    y = a.float() @ b.float().T
    if bias is not None:
        y = y + bias
    if act:
        y = torch.where(y > 0, y, 0.1 * y)
    return y


SHAPES = [(128, 128, 64), (256, 64, 128), (128, 32, 64), (384, 256, 256), (1000, 255, 1152),
          (173, 100, 72), (4096, 512, 2304), (13 * 13 * 8, 1024, 4608)]


@pytest.mark.parametrize("m,n,k", SHAPES, ids=[f"{m}x{n}x{k}" for m, n, k in SHAPES])
@pytest.mark.parametrize("act", [0, 1])
def test_gemm_fp32_out_matches_torch(m, n, k, act):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    a = torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    bias = torch.randn(n, device="cuda", generator=g)
    got = W.gemm_bf16(a, b, bias, act=act)
    torch.cuda.synchronize()
    want = ref(a, b, bias, act)
    atol = 1e-5 * (k ** 0.5)
    torch.testing.assert_close(got, want, rtol=1e-5, atol=atol)


def test_gemm_bf16_out_rounds_like_torch():
    m, n, k = 512, 192, 320
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.05).to(torch.bfloat16)
    got = W.gemm_bf16(a, b, None, act=1, out_f32=False)
    torch.cuda.synchronize()
    want = ref(a, b, None, 1).to(torch.bfloat16)
    # one bf16 ulp where fp32 accumulation order flips the rounding
    torch.testing.assert_close(got.float(), want.float(), rtol=2 ** -7, atol=1e-3)


def test_gemm_strided_output_writes_a_channel_slice():
    """Route/concat layers write a GEMM into a column slice of a wider NHWC tensor."""
    m, n, k = 256, 64, 128
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.05).to(torch.bfloat16)
    wide = torch.full((m, 3 * n), 7.0, device="cuda")
    W.gemm_bf16(a, b, None, out=wide[:, n:2 * n])
    torch.cuda.synchronize()
    torch.testing.assert_close(wide[:, n:2 * n], ref(a, b, None, 0), rtol=1e-5, atol=1e-4)
    assert torch.all(wide[:, :n] == 7.0) and torch.all(wide[:, 2 * n:] == 7.0)


@pytest.mark.parametrize("S,N", [(64, 2), (96, 1)])
def test_yolov3_tiny_job_matches_torch_reference(S, N):
    """The whole Darknet YOLOv3-tiny job (im2row + tcgen05 GEMM + pools +
    route/upsample + YOLO heads) against torch fp32 with bf16 rounding at
    the same points.  Tolerance: a bf16 rounding flip (2^-8 relative) of an
    intermediate activation may propagate; outputs are logistic / linear
    O(1) values, so demand max |err| < 5e-2 and mean |err| < 2e-3."""
    import yolo_ref

    job = W.Job("yolo", n=S, m=N, iters=1, seed=11)
    got, rec = W.run_solo(job)
    assert rec.state == 0 and rec.n_kernels > 13
    want = yolo_ref.forward(S, N, 11).cpu().numpy()
    err = abs(got.astype("float64") - want.astype("float64"))
    assert got.shape == want.shape
    assert err.max() < 5e-2 and err.mean() < 2e-3, (err.max(), err.mean())


def test_yolo_probe_matches_host_footprint_and_reports_gemm_smem():
    from paper_2107_08538_b200 import catalog as C

    job = W.Job("yolo", n=416, m=4, iters=1, seed=1)
    p = W.probe(job)
    assert p.mem_bytes == C.host_footprint(job)
    assert p.smem_per_block > 64 * 1024  # the tcgen05 GEMM's dynamic shared-memory ring is counted


@pytest.mark.parametrize("S,N", [(64, 2), (96, 1)])
def test_resnet50_job_matches_torch_reference(S, N):
    """ResNet-50 job (im2row with strides + tcgen05 GEMM with the fused
    shortcut + ReLU epilogue, max / average pools, FC) against torch fp32
    with bf16 rounding at the same points.  Random He-init residual stacks
    grow the activations, so the bar is relative to the largest logit:
    max error < 5e-2, mean < 5e-3 of max |logit|."""
    import yolo_ref

    job = W.Job("resnet", n=S, m=N, iters=1, seed=13)
    got, rec = W.run_solo(job)
    assert rec.state == 0 and rec.n_kernels > 53
    want = yolo_ref.resnet50_forward(S, N, 13).cpu().numpy()
    scale = float(abs(want).max())
    err = abs(got.reshape(-1).astype("float64") - want.astype("float64")) / scale
    assert err.max() < 5e-2 and err.mean() < 5e-3, (err.max(), err.mean(), scale)


def test_resnet_probe_matches_host_footprint():
    from paper_2107_08538_b200 import catalog as C

    job = W.Job("resnet", n=224, m=4, iters=1, seed=1)
    assert W.probe(job).mem_bytes == C.host_footprint(job)
