"""The cross-process EP data planes on the one GPU this run has: 2 and 4 rank
PROCESSES (tests/mp_ep_worker.py), each with its own CUDA context, created with
moe_layer_create_hostcoll (counts + the one-time cudaIpc mapping over a gloo
group).  Rows move on the layer's own planes (put kernels, a2a_p2p = 1;
copy engines, a2a_p2p = 2) into the peers' REAL cudaIpc mappings, and only
the st.release.sys / ld.acquire.sys epoch flags order a rank's puts before its
peers' reads (no host barrier, no CUDA event across ranks).  The contexts
time-slice the GPU, so a spinning flag wait yields to the peer's put.

y must equal the EP = 1 layer's bit for bit (R6), over several forwards on the
same layers (epochs advance, buffers are reused without resets)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from gen import Inputs
from paper_2410_12247_b200 import MOE_GEMM_GROUPED, make_plan

from .gpu_util import dev_bf16, layer_from_inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "mp_ep_worker.py")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_ranks(D, plane, N, forwards, tmp_path, extra=()):
    port = _free_port()
    procs, outs = [], []
    for r in range(D):
        out = str(tmp_path / f"rank{r}.npz")
        outs.append(out)
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(D), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   LOCAL_RANK="0")
        procs.append(subprocess.Popen([sys.executable, WORKER, out, str(plane), str(N), str(forwards), *extra],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:  # pragma: no cover
            for q in procs:
                q.kill()
            raise AssertionError("multi-process EP forward hung")
        logs.append(o)
    for p, o in zip(procs, logs):
        assert p.returncode == 0, o[-3000:]
    return [np.load(o) for o in outs]


def _ep1(forwards, fp8=False):
    from tests.mp_ep_worker import CASE, inputs
    base = inputs(1)
    L = layer_from_inputs(base, CASE["k"], 0, dispatch_fp8=fp8)
    ys = []
    for f in range(forwards):
        y = L.forward(dev_bf16(inputs(1 + f).x), plan=make_plan(1, MOE_GEMM_GROUPED))
        torch.cuda.synchronize()
        ys.append(y.view(torch.int16).cpu().numpy())
    L.close()
    return ys


@pytest.mark.parametrize("plane", [1, 2])
@pytest.mark.parametrize("D,N", [(2, 3), (4, 2)])
def test_multiprocess_ep_equals_ep1(D, N, plane, tmp_path):
    forwards = 3
    res = _run_ranks(D, plane, N, forwards, tmp_path)
    ref = _ep1(forwards)
    for f in range(forwards):
        y = np.concatenate([r[f"arr_{f}"] for r in res])
        assert np.array_equal(y, ref[f]), (D, N, plane, f)
    # every rank saw the same global histogram, and rows sent == rows received by the peer
    gh = res[0]["global_hist"]
    for r in range(D):
        assert np.array_equal(res[r]["global_hist"], gh)
        for p in range(D):
            assert np.array_equal(res[r]["chunk_rows"][0, :N, p], res[p]["chunk_rows"][1, :N, r])


def test_multiprocess_ep_fp8_dispatch(tmp_path):
    """NEXT-2 across processes: packed FP8 rows through the peer mappings,
    dequantised on arrival == the EP = 1 FP8 round trip, bit for bit."""
    res = _run_ranks(2, 1, 2, 2, tmp_path, extra=("fp8",))
    ref = _ep1(2, fp8=True)
    for f in range(2):
        assert np.array_equal(np.concatenate([r[f"arr_{f}"] for r in res]), ref[f])


def test_multiprocess_ep_local_reduce(tmp_path):
    """NEXT-3 across processes: dedup rows + meta out, LocalReduce partials
    back through the peer mappings; y within the oracle's R16 tolerance."""
    import oracle
    from tests.mp_ep_worker import CASE, inputs

    from .gpu_util import assert_close
    res = _run_ranks(4, 1, 2, 1, tmp_path, extra=("lr",))
    inp = inputs(1)
    ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=CASE["k"], norm_topk=0,
                           ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down, D=4, N=2,
                           local_reduce=True)
    y = np.concatenate([r["arr_0"] for r in res]).view(np.uint16)
    assert_close(oracle.bf16_bits_to_f64(y), ref["y"], "multiprocess LR EP4")


def test_in_process_flags_only_ep2(tmp_path):
    """The in-process test group with the event ordering off
    (EPSMOE_LOCAL_P2P_EVENTS=0): with CUDA_DEVICE_MAX_CONNECTIONS=32 the ranks'
    streams do not share hardware queues, so the device flags alone order the
    puts; y == EP = 1.  (Run in a subprocess: a hang would trap the context.)"""
    code = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch
from gen import Inputs
from paper_2410_12247_b200 import MOE_GEMM_GROUPED, make_plan
from tests.test_gpu_ep import _ep_forward, _ep1_forward
for plane in (1, 2):
    inp = Inputs(E=16, k=4, H=256, F=256, S=1, Fs=128, T=919, seed=5, grid=True)
    y, _ = _ep_forward(inp, 4, 1, 2, make_plan(2, MOE_GEMM_GROUPED), p2p=plane)
    y1 = _ep1_forward(inp, 4, 1, make_plan(1, MOE_GEMM_GROUPED))
    assert np.array_equal(y, y1), plane
print("ok")
'''
    env = dict(os.environ, EPSMOE_LOCAL_P2P_EVENTS="0", CUDA_DEVICE_MAX_CONNECTIONS="32", ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
