"""The single-GPU bf16 layer reads fc1's and the fc1 weight gradient's input
rows straight from x with TMA tile::gather4 (local_scatter
folded into the GEMM A-load; tc_gemm.cuh Params::gather_rows) instead of
scattering them into xs first.  The gathered rows are the scattered rows, so
every result must equal the scatter path's byte for byte.  (The gathered
loads are off by default -- ~3x slower on these tensor-bound GEMMs,
profiles/r02q_gather_ab.log -- and enabled here with FMOE_TC_GATHER=1):
y, d_x, all gradients, for single-CTA (128-row) and CTA-pair (256-row) expert
blocks, gated and injected (routed) forwards, and the xs the operator-level
cache view materialises on request (fmoe_layer_activations)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import ctypes as C, hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2103_13262_b200 as fm
from paper_2103_13262_b200 import _lib
from paper_2103_13262_b200.workloads import zipf_routing
n, d, h, e, k, routed = (int(a) for a in sys.argv[2:8])
layer = fm.MoELayer(fm.MoEConfig(n, d, h, k, e, 1, 9), dtype=torch.bfloat16)
g = torch.Generator(device="cuda").manual_seed(4)
x = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
dy = (torch.rand(n, d, device="cuda", generator=g) * 2 - 1).bfloat16()
y = torch.empty_like(x); dx = torch.empty_like(x)
if routed:
    idx, sc = zipf_routing(n, e, k, 1.1, seed=3)
    idx = torch.as_tensor(idx, device="cuda"); sc = torch.as_tensor(sc, device="cuda")
for _ in range(2):
    if routed:
        layer.forward_routed(x, idx, sc, y)
    else:
        layer.forward(x, y)
    xs_p = C.c_void_p()
    _lib.check(_lib.lib.fmoe_layer_activations(layer.h, C.byref(xs_p), None, None, None))
    layer.backward(dy, dx)
torch.cuda.synchronize()
# the xs the cache view materialises (last forward), copied out through cudaMemcpy
align = 256 if n * k >= 1024 * e else 128
cap, scr = C.c_int64(), C.c_int64()
_lib.check(_lib.lib.fmoe_plan_sizes(n, k, e, align, C.byref(cap), C.byref(scr)))
xs = torch.empty(cap.value * d, dtype=torch.bfloat16, device="cuda")
cudart = C.CDLL("libcudart.so.12")  # already loaded by torch
assert cudart.cudaMemcpy(C.c_void_p(xs.data_ptr()), xs_p, C.c_size_t(cap.value * d * 2), 3) == 0
gr = layer.grads
parts = [y, dx, gr.d_w1, gr.d_w2, gr.d_b1, gr.d_b2, layer.d_wg, xs]
print(hashlib.sha256(b"".join(t.detach().cpu().contiguous().view(torch.uint8).numpy().tobytes()
      for t in parts)).hexdigest())
"""


def _run(args, env):
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, *map(str, args)], capture_output=True, text=True,
                       timeout=600, env={**os.environ, **env})
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("n,d,h,e,k,routed", [
    (4096, 128, 256, 64, 2, 0),    # ~128 rows per expert: 128-row blocks, single-CTA tiles
    (16384, 256, 512, 8, 2, 0),    # 4096 rows per expert: 256-row blocks, CTA pairs
    (20000, 128, 256, 16, 1, 1),   # injected Zipf routing (cfg5 path), ragged experts
    (777, 64, 128, 8, 2, 0),       # ragged n, padding rows in every block
])
def test_gathered_a_loads_equal_the_scatter_path(n, d, h, e, k, routed):
    assert _run((n, d, h, e, k, routed), {"FMOE_TC_GATHER": "1"}) == _run((n, d, h, e, k, routed), {})
