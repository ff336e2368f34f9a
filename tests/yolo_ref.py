"""PyTorch fp32 reference of the YOLOv3-tiny job (csrc/gs_darknet.cu).

Regenerates the job's synthetic image, filters and biases on the host with
the shared counter hash (include/gs_work.h, restated in kernels_ref.py),
then runs Darknet's yolov3-tiny.cfg forward in fp32 NCHW with torch,
rounding every activation to bf16 exactly where the GPU job stores bf16.
"""

from __future__ import annotations

import numpy as np

import kernels_ref as R

# (kind, cin, cout, k) in the job's plan order; "pool2" / "pool1" are
# maxpool size 2 stride 2 / stride 1
CONVS = [(3, 16, 3), (16, 32, 3), (32, 64, 3), (64, 128, 3), (128, 256, 3), (256, 512, 3), (512, 1024, 3),
         (1024, 256, 1), (256, 512, 3), (512, 255, 1), (256, 128, 1), (384, 256, 3), (256, 255, 1)]


def filters(seed: int, li: int, cin: int, cout: int, k: int):
    kdim = k * k * cin
    kpad = (kdim + 7) // 8 * 8
    u = R.unit(seed + 100 + li, np.arange(cout * kpad, dtype=np.uint64)).reshape(cout, kpad)
    s = np.sqrt(np.float32(6.0) / np.float32(kdim)).astype(np.float32)
    w = ((np.float32(2.0) * u - np.float32(1.0)) * s).astype(np.float32)[:, :kdim]
    b = (np.float32(0.1) * (np.float32(2.0) * R.unit(seed + 200 + li, np.arange(cout, dtype=np.uint64))
                            - np.float32(1.0))).astype(np.float32)
    return w.reshape(cout, k, k, cin), b  # [cout][kh][kw][cin]


def forward(S: int, N: int, seed: int, device="cuda"):
    import torch
    import torch.nn.functional as F

    def bf(t):
        return t.to(torch.bfloat16).float()

    img = R.unit(seed, np.arange(N * S * S * 3, dtype=np.uint64)).reshape(N, S, S, 3)
    x = bf(torch.from_numpy(img).to(device).permute(0, 3, 1, 2).contiguous())
    params = []
    for li, (cin, cout, k) in enumerate(CONVS):
        w, b = filters(seed, li, cin, cout, k)
        params.append((bf(torch.from_numpy(w).to(device).permute(0, 3, 1, 2).contiguous()),
                       torch.from_numpy(b).to(device), k))

    def conv(x, li, act):
        w, b, k = params[li]
        y = F.conv2d(x, w, b, padding=k // 2)
        if act == "leaky":
            return bf(torch.where(y > 0, y, 0.1 * y))
        # YOLO head: logistic on everything but w, h of each 85-channel anchor group
        e = torch.arange(y.shape[1], device=y.device) % 85
        keep = ((e == 2) | (e == 3)).view(1, -1, 1, 1)
        return torch.where(keep, y, torch.sigmoid(y))

    def pool2(x):
        return F.max_pool2d(x, 2, 2)

    def pool1(x):
        return F.max_pool2d(F.pad(x, (0, 1, 0, 1), value=float("-inf")), 2, 1)

    x = pool2(conv(x, 0, "leaky"))
    x = pool2(conv(x, 1, "leaky"))
    x = pool2(conv(x, 2, "leaky"))
    x = pool2(conv(x, 3, "leaky"))
    l8 = conv(x, 4, "leaky")
    x = pool2(l8)
    x = pool1(conv(x, 5, "leaky"))
    x = conv(x, 6, "leaky")
    l13 = conv(x, 7, "leaky")
    x = conv(l13, 8, "leaky")
    det1 = conv(x, 9, "yolo")
    l18 = conv(l13, 10, "leaky")
    cat = torch.cat([F.interpolate(l18, scale_factor=2, mode="nearest"), l8], dim=1)
    x = conv(cat, 11, "leaky")
    det2 = conv(x, 12, "yolo")
    return torch.cat([det1.permute(0, 2, 3, 1).reshape(-1), det2.permute(0, 2, 3, 1).reshape(-1)])


def resnet50_forward(S: int, N: int, seed: int, device="cuda"):
    """ResNet-50 (v1.5, folded batch-norm) job reference: same filters /
    biases as csrc/gs_darknet.cu resnet50_plan (conv li from seed+100+li /
    seed+200+li, plan order), bf16 rounding wherever the job stores bf16
    (every activation, the pooled features); logits in fp32."""
    import torch
    import torch.nn.functional as F

    from paper_2107_08538_b200.catalog import resnet50_convs

    def bf(t):
        return t.to(torch.bfloat16).float()

    img = R.unit(seed, np.arange(N * S * S * 3, dtype=np.uint64)).reshape(N, S, S, 3)
    x = bf(torch.from_numpy(img).to(device).permute(0, 3, 1, 2).contiguous())
    convs = resnet50_convs(S)
    params = []
    for li, (_, cin, cout, k, stride, _) in enumerate(convs):
        w, b = filters(seed, li, cin, cout, k)
        params.append((bf(torch.from_numpy(w).to(device).permute(0, 3, 1, 2).contiguous()),
                       torch.from_numpy(b).to(device), k, stride))
    it = iter(range(len(convs)))

    def conv(x, act="relu", res=None):
        w, b, k, stride = params[next(it)]
        y = F.conv2d(x, w, b, stride=stride, padding=k // 2)
        if res is not None:
            y = y + res
        if act == "relu":
            y = torch.relu(y)
        return bf(y)

    x = conv(x)                                      # stem 7x7/2
    x = F.max_pool2d(x, 3, 2, 1)
    for mid, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for bi in range(blocks):
            a = conv(x)
            b = conv(a)
            sc = conv(x, act=None) if bi == 0 else x
            x = conv(b, res=sc)
    pooled = bf(x.mean(dim=(2, 3)))
    w, b, _, _ = params[next(it)]
    return (pooled @ w.view(w.shape[0], -1).T + b).reshape(-1)
