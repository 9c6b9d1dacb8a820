"""Independent cross-check of the FP32 C oracle (the reference has no forward
pass to pin it against): the oracle's exported layer list and weights are
executed by torch.nn.functional (different conv/pool implementations,
NCHW, different summation order), and the resulting logits are committed as
fixtures tests/golden/xcheck_<model>.npz. test_oracle.py then requires the
C oracle to reproduce them. Run from make_golden.py --xcheck (needs torch).
"""
import ctypes
import os
import sys

import numpy as np
import torch
import torch.nn.functional as F

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle  # noqa: E402

K_CONV, K_DW, K_MAXPOOL, K_AVGPOOL, K_GAP, K_FC = range(6)
IMAGES = {"synthetic_cnn": 8, "mobilenet_v1": 4, "resnet50_v1": 2, "inception_v3": 2}


def lib():
    L = oracle.fwd()
    L.oracle_num_ops.argtypes = [ctypes.c_char_p]
    L.oracle_num_buffers.argtypes = [ctypes.c_char_p]
    L.oracle_buffer_shape.argtypes = [ctypes.c_char_p, ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 3
    L.oracle_op.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p]
    L.oracle_op_params.restype = ctypes.c_long
    L.oracle_op_params.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return L


def bf16(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def torch_forward(model: str, images: np.ndarray) -> np.ndarray:
    L = lib()
    mid = model.encode()
    nb = L.oracle_num_buffers(mid)
    shapes = []
    for b in range(nb):
        h, w, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        L.oracle_buffer_shape(mid, b, ctypes.byref(h), ctypes.byref(w), ctypes.byref(c))
        shapes.append((h.value, w.value, c.value))
    n = images.shape[0]
    x = torch.from_numpy(images.astype(np.float32)).permute(0, 3, 1, 2)  # NCHW
    bufs = {0: bf16((x - 127.5) / 63.75)}
    logits = None
    for i in range(L.oracle_num_ops(mid)):
        f = np.zeros(14, np.int32)
        L.oracle_op(mid, i, f.ctypes.data)
        kind, bi, bo, coff, res, kh, kw, sh, sw, ph, pw, relu, cin, cout = f.tolist()
        x = bufs[bi]
        if bo not in bufs:
            h, w, c = shapes[bo]
            bufs[bo] = torch.zeros(n, c, h, w)
        if kind in (K_CONV, K_DW, K_FC):
            cnt = L.oracle_op_params(mid, i, None, None)
            wt = np.empty(cnt, np.float32)
            bias = np.empty(cout, np.float32)
            L.oracle_op_params(mid, i, wt.ctypes.data, bias.ctypes.data)
            bias_t = torch.from_numpy(bias)
        if kind == K_CONV:
            wt_t = torch.from_numpy(wt.reshape(cout, kh, kw, cin)).permute(0, 3, 1, 2)
            y = F.conv2d(x, wt_t, bias_t, stride=(sh, sw), padding=(ph, pw))
            if res >= 0:
                y = y + bufs[res]
            if relu:
                y = F.relu(y)
            bufs[bo][:, coff:coff + cout] = y
        elif kind == K_DW:
            c = cout
            wt_t = torch.from_numpy(wt.reshape(3, 3, c)).permute(2, 0, 1).unsqueeze(1)
            y = F.relu(F.conv2d(x, wt_t, bias_t, stride=sh, padding=1, groups=c))
            bufs[bo][:] = y
        elif kind == K_MAXPOOL:
            y = F.max_pool2d(x, 3, stride=sh, padding=ph)
            bufs[bo][:, coff:coff + x.shape[1]] = y
        elif kind == K_AVGPOOL:
            y = F.avg_pool2d(x, 3, stride=sh, padding=ph, count_include_pad=True)
            bufs[bo][:, coff:coff + x.shape[1]] = y
        elif kind == K_GAP:
            bufs[bo] = x.mean(dim=(2, 3), keepdim=True)
        elif kind == K_FC:
            logits = F.linear(x.flatten(1), torch.from_numpy(wt.reshape(cout, cin)), bias_t)
    return logits.numpy()


def main():
    torch.set_num_threads(8)
    for model, count in IMAGES.items():
        imgs = oracle.images(model, 0, count)
        with torch.no_grad():
            ref = torch_forward(model, imgs)
        ours = oracle.forward(model, imgs, bf16_storage=False)
        rel = np.abs(ours - ref).max(1) / np.abs(ref).max(1)
        print(f"{model}: oracle vs torch max rel {rel.max():.2e}")
        np.savez_compressed(os.path.join(HERE, f"xcheck_{model}.npz"), image_first=0,
                            logits=ref.astype(np.float32))


if __name__ == "__main__":
    main()
