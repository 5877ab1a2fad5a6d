"""One EP rank in its own process (tests/test_gpu_multiproc.py): the layer is
created with moe_layer_create_hostcoll (counts and the one-time cudaIpc
mapping over a torch.distributed gloo group), rows move on the layer's own
peer-memory plane, and NOTHING orders one rank's puts before another rank's
waits except the device flags (separate processes, separate CUDA contexts).

  python tests/mp_ep_worker.py <out.npz> <plane> <N> <forwards> [fp8] [lr]
  (env: RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402  (token shards only: the input recipe)
from gen import Inputs  # noqa: E402
from paper_2410_12247_b200 import MOE_GEMM_GROUPED, HostAllgather, MoELayer, make_plan  # noqa: E402

CASE = dict(E=16, k=4, H=256, F=256, S=1, Fs=128, T=997)


def inputs(seed):
    return Inputs(E=CASE["E"], k=CASE["k"], H=CASE["H"], F=CASE["F"], S=CASE["S"], Fs=CASE["Fs"], T=CASE["T"],
                  seed=seed, grid=True)


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


def main():
    out, plane, N, forwards = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    fp8 = "fp8" in sys.argv[5:]
    lr = "lr" in sys.argv[5:]
    rank, D = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    E, k, H, F, T = CASE["E"], CASE["k"], CASE["H"], CASE["F"], CASE["T"]
    E_loc = E // D
    start = oracle.token_shards(T, D)
    inp = inputs(1)
    w = dict(w_router=dev(inp.w_router), w_gate=dev(inp.w_gate[rank * E_loc:(rank + 1) * E_loc]),
             w_up=dev(inp.w_up[rank * E_loc:(rank + 1) * E_loc]), w_down=dev(inp.w_down[rank * E_loc:(rank + 1) * E_loc]),
             ws_gate=dev(inp.ws_gate), ws_up=dev(inp.ws_up), ws_down=dev(inp.ws_down))
    layer = MoELayer(E, k, H, F, w, S=1, Fs=128, ep=D, rank=rank, max_tokens=int(np.diff(start).max()), norm_topk=0,
                     a2a_p2p=plane, dispatch_fp8=fp8, local_reduce=lr, host_allgather=HostAllgather())
    ys = []
    for f in range(forwards):                   # new x every forward: epochs advance, buffers are reused
        x = dev(inputs(1 + f).x[start[rank]:start[rank + 1]])
        d, b = layer.debug_buffers(x.shape[0])
        y = layer.forward(x, plan=make_plan(N, MOE_GEMM_GROUPED), debug=d)
        torch.cuda.synchronize()
        ys.append(y.view(torch.int16).cpu().numpy())
    np.savez(out, *ys, chunk_rows=b["chunk_rows"], global_hist=b["global_hist"])
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
