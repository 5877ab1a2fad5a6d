"""Multi-process (gloo, CPU) coverage of the EP host logic: two ranks agree on
the plan from the allgathered histogram, their moe_exchange_layout tables are
mirror images, and a real all2all driven by those tables (per (peer, expert)
p2p messages, in Algorithm 1's chunk order) reproduces the oracle's layer
output bit-exactly.  The expert math here is the oracle's (CPU); the GPU path
uses the same tables with NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from gen import Inputs
from paper_2410_12247_b200 import abi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, E, k, H, F, T, N, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        inp = Inputs(E=E, k=k, H=H, F=F, S=1, Fs=128, T=T, seed=99)
        start = oracle.token_shards(T, world)
        t0, t1 = int(start[rank]), int(start[rank + 1])
        E_loc = E // world
        # local routing (each rank routes only its own tokens)
        logits = oracle.router_logits(inp.x[t0:t1], inp.w_router)
        idx, w = oracle.topk_gating(logits, k, 0)
        hist = np.array([np.count_nonzero(idx == e) for e in range(E)], np.int32)
        allh = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allh, torch.from_numpy(hist))
        gh = torch.stack(allh).numpy()
        cfg = abi.make_config(E, k, H, F, 1, 128, ep=world, rank=rank, max_tokens=T)
        cost = abi.moe_cost_model_t()
        cost.n_points = 2
        cost.m_points[0], cost.m_points[1] = 64.0, 4096.0
        for kind in (0, 1):
            cost.gemm_ms[kind][0], cost.gemm_ms[kind][1] = 0.01, 0.64
        cost.a2a_fixed_ms, cost.a2a_gbps, cost.k_ms, cost.b_ms = 0.0, 0.5, 0.001, 0.0
        plan = abi.plan_compute(cfg, T, gh, cost)
        pb = torch.frombuffer(bytearray(bytes(plan)), dtype=torch.uint8)
        allp = [torch.zeros_like(pb) for _ in range(world)]
        dist.all_gather(allp, pb)
        same_plan = all(torch.equal(p, allp[0]) for p in allp)
        if N:
            plan = abi.make_plan(N)
        send_off, recv_off, cs, cr = abi.exchange_layout(cfg, plan, gh)
        allcs = [torch.zeros(cs.shape, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allcs, torch.from_numpy(cs))
        mirror = all(allcs[d][c, rank].item() == cr[c, d] for c in range(cs.shape[0]) for d in range(world))
        # split: send rows expert-major in token order (R6)
        pos = np.zeros_like(idx)
        nxt = send_off[:-1].copy()
        for t in range(idx.shape[0]):
            for j in range(k):
                pos[t, j] = nxt[idx[t, j]]
                nxt[idx[t, j]] += 1
        send = np.zeros((int(send_off[-1]), H), np.uint16)
        for t in range(idx.shape[0]):
            for j in range(k):
                send[pos[t, j]] = inp.x[t0 + t]
        recv = np.zeros((int(recv_off[-1]), H), np.uint16)
        o_recv = np.zeros((int(recv_off[-1]), H), np.float32)
        comb = np.zeros((int(send_off[-1]), H), np.float32)
        gb = list(plan.group_begin[:plan.num_chunks + 1])
        if gb[-1] == 0:   # caller-built plan: the library fills balanced groups (R8)
            gb = oracle.chunk_groups(E_loc, plan.num_chunks).tolist()
        for c in range(plan.num_chunks):
            # dispatch chunk c: per (peer, expert) messages
            ops = []
            for peer in range(world):
                for el in range(gb[c], gb[c + 1]):
                    ex = peer * E_loc + el
                    ns = int(gh[rank, ex])
                    if ns:
                        buf = torch.from_numpy(send[send_off[ex]:send_off[ex] + ns].view(np.int16).copy())
                        ops.append(dist.isend(buf, peer) if peer != rank else None)
                        if peer == rank:
                            s = recv_off[el * world + rank]
                            recv[s:s + ns] = send[send_off[ex]:send_off[ex] + ns]
                    nr = int(gh[peer, rank * E_loc + el])
                    if nr and peer != rank:
                        rb = torch.zeros((nr, H), dtype=torch.int16)
                        ops.append((dist.irecv(rb, peer), rb, int(recv_off[el * world + peer]), nr))
            for op in ops:
                if isinstance(op, tuple):
                    op[0].wait()
                    recv[op[2]:op[2] + op[3]] = op[1].numpy().view(np.uint16)
                elif op is not None:
                    op.wait()
            # ComputeMoE(c) on the received rows of chunk c's experts
            for el in range(gb[c], gb[c + 1]):
                a, b = int(recv_off[el * world]), int(recv_off[(el + 1) * world])
                if b > a:
                    e = rank * E_loc + el
                    o_recv[a:b] = oracle.expert_ffn(recv[a:b], inp.w_gate[e], inp.w_up[e], inp.w_down[e])
            # combine chunk c: mirror messages back to the home ranks
            ops = []
            for peer in range(world):
                for el in range(gb[c], gb[c + 1]):
                    nb = int(gh[peer, rank * E_loc + el])
                    s = int(recv_off[el * world + peer])
                    if nb:
                        if peer == rank:
                            ex = rank * E_loc + el
                            comb[send_off[ex]:send_off[ex] + nb] = o_recv[s:s + nb]
                        else:
                            ops.append(dist.isend(torch.from_numpy(o_recv[s:s + nb].copy()), peer))
                    ex = peer * E_loc + el
                    nh = int(gh[rank, ex])
                    if nh and peer != rank:
                        rb = torch.zeros((nh, H), dtype=torch.float32)
                        ops.append((dist.irecv(rb, peer), rb, int(send_off[ex]), nh))
            for op in ops:
                if isinstance(op, tuple):
                    op[0].wait()
                    comb[op[2]:op[2] + op[3]] = op[1].numpy()
                else:
                    op.wait()
        s_sh = oracle.expert_ffn(inp.x[t0:t1], inp.ws_gate, inp.ws_up, inp.ws_down)
        y = oracle.combine(s_sh, comb[pos], w)
        ref = oracle.moe_layer(inp.x, inp.w_router, inp.w_gate, inp.w_up, inp.w_down, k=k, norm_topk=0,
                               ws_gate_bits=inp.ws_gate, ws_up_bits=inp.ws_up, ws_down_bits=inp.ws_down)["y"]
        q.put((rank, same_plan, mirror, bool(np.array_equal(y, ref[t0:t1])), plan.num_chunks))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e), False, 0))


@pytest.mark.parametrize("N", [0, 1, 3])
def test_two_rank_exchange_matches_oracle(N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    E, k, H, F, T = 8, 2, 64, 128, 37
    procs = [ctx.Process(target=_worker, args=(r, 2, port, E, k, H, F, T, N, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, same_plan, mirror, ok, n in res:
        assert same_plan is True, res
        assert mirror is True, res
        assert ok, res
