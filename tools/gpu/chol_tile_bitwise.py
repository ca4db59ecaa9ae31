# the split-tile (64x64 / 64x128) factor must equal the 128x128 one bitwise
# (same K order per element; C - acc either way), run after run
import os, sys, subprocess
import numpy as np
code = r'''
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_13209_b200 as hs
from paper_2605_13209_b200 import hsolve as H
rt = hs.Runtime(stream=torch.cuda.current_stream().cuda_stream)
n, b = int(sys.argv[2]), int(sys.argv[3])
m = hs.generate_spd_device(rt, n, b, seed=7)
w = hs.DeviceMatrix(rt, n, b); w.copy_from(m)
H.potrf_device(rt, w)
L = w.download()
N = n // b
parts = []
for i in range(N):
    for j in range(i + 1):
        t = i * (i + 1) // 2 + j
        T = L[t * b * b:(t + 1) * b * b].reshape(b, b)
        parts.append((np.tril(T) if i == j else T).ravel())
np.save(sys.argv[1], np.concatenate(parts))
'''
def run(env, out, n, b):
    subprocess.run([sys.executable, "-c", code, out, str(n), str(b)],
                   env=dict(os.environ, **env), check=True)
for n, b in [(8192, 512), (16384, 512), (32768, 512), (16384, 256)]:
    run({"HS_GEMM64": "0"}, "/tmp/L0.npy", n, b)
    L0 = np.load("/tmp/L0.npy")
    d = []
    for rep in range(3):
        run({"HS_GEMM64": "1"}, "/tmp/L1.npy", n, b)
        d.append(float(np.max(np.abs(np.load("/tmp/L1.npy") - L0))))
    print(n, b, "max |L(split tiles) - L(128x128)| per run:", d, flush=True)
