"""Run tools/tc_probe.cu on the GPU and compare with numpy (bring-up of tcgen05 kind::i8)."""
import ctypes
import os
import subprocess
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libtcprobe.so")
if not os.path.exists(SO):
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                    "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "tc_probe.cu")], check=True)
lib = ctypes.CDLL(SO)
ok = True
for N, K in [(256, 128), (128, 128), (256, 256), (64, 128)]:
    rng = np.random.default_rng(N + K)
    A = rng.integers(-128, 128, size=(128, K)).astype(np.int8)
    B = rng.integers(-128, 128, size=(N, K)).astype(np.int8)
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c = torch.zeros((128, N), dtype=torch.int32, device="cuda")
    rc = lib.tc_probe(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(c.data_ptr()), N, K)
    got = c.cpu().numpy()
    good = rc == 0 and np.array_equal(got, ref)
    ok &= good
    nbad = int((got != ref).sum())
    print(f"N={N} K={K} rc={rc} exact={good} mismatches={nbad}")
    if not good and rc == 0:
        bad = np.argwhere(got != ref)[:5]
        for r, cidx in bad:
            print("  ", r, cidx, got[r, cidx], ref[r, cidx])
sys.exit(0 if ok else 1)
