"""Multi-process communicator on real hardware: two processes (torchrun
style, gloo for the rendezvous-id broadcast) share ONE B200 -- the only
multi-process topology a 1-GPU box offers.  NVLS cannot bind two ranks to one
device, so AUTO must fall back (collectively) to the PEER transport over
cudaIpc-mapped buffers; K1 then runs as two per-rank launches from two
processes whose in-kernel barrier meets across process boundaries."""
import json
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from tests.conftest import ROOT
from tests.helpers import assert_bf16_close, bf16_round, group_inputs

pytestmark = pytest.mark.gpu

WORKER = textwrap.dedent("""
    import ctypes, json, os, sys
    sys.path.insert(0, {root!r})
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2505_11329_b200 as tw
    from paper_2505_11329_b200 import _lib
    from tools.bench_tp import rendezvous_id
    from tests.helpers import group_inputs, bf16_round
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    T, H = {T}, {H}
    torch.cuda.set_device(0)
    rid = rendezvous_id(dist)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_create_mp(world, rank, 0, T * H * 2, rid.encode(), _lib.TW_TRANSPORT_AUTO,
                                          ctypes.byref(h)))
    w_, tr, nb = ctypes.c_int(), ctypes.c_int(), ctypes.c_size_t()
    _lib.check(_lib.lib.tw_comm_info(h, ctypes.byref(w_), ctypes.byref(tr), ctypes.byref(nb)))
    inputs, residual, weight = group_inputs(5, world, T, H)
    inputs, residual = bf16_round(inputs), bf16_round(residual)
    p = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_INPUT, ctypes.byref(p)))
    buf = torch.as_tensor(tw._DevBuf(p.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    buf.copy_(torch.from_numpy(inputs[rank]).bfloat16())
    ranges = tw.token_shard_map(T, world)
    b, e = ranges[rank]
    shard = torch.from_numpy(np.ascontiguousarray(residual[b:e])).cuda().bfloat16()
    wt = torch.from_numpy(weight).cuda()
    torch.cuda.synchronize()
    dist.barrier()
    flat = (ctypes.c_int64 * (2 * world))(*[v for rg in ranges for v in rg])
    for _ in range({reps}):
        shard.copy_(torch.from_numpy(np.ascontiguousarray(residual[b:e])).bfloat16())
        torch.cuda.synchronize()
        dist.barrier()
        _lib.check(_lib.lib.tw_fused_allreduce_rmsnorm(h, T, H, 0, flat, shard.data_ptr(), wt.data_ptr(), 1e-5,
                                                       _lib.TW_BF16, 2, 0, None))
        torch.cuda.synchronize()
    _lib.check(_lib.lib.tw_comm_check(h))
    _lib.check(_lib.lib.tw_comm_buffer(h, rank, _lib.TW_BUF_OUTPUT, ctypes.byref(p)))
    out = torch.as_tensor(tw._DevBuf(p.value, (T * H,), "<i2"), device="cuda").view(torch.bfloat16).view(T, H)
    np.save({outdir!r} + f"/out{{rank}}.npy", out.float().cpu().numpy())
    np.save({outdir!r} + f"/res{{rank}}.npy", shard.float().cpu().numpy())
    print(json.dumps({{"rank": rank, "transport": _lib.TRANSPORT_NAMES[tr.value]}}), flush=True)
    dist.barrier()
    _lib.lib.tw_comm_destroy(h)
    dist.destroy_process_group()
""")


WEAVE_WORKER = textwrap.dedent("""
    import ctypes, json, os, sys
    sys.path.insert(0, {root!r})
    import torch
    import torch.distributed as dist
    from paper_2505_11329_b200 import _lib, weave
    from tools.bench_tp import rendezvous_id
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    T, H = 512, 1024
    rid = rendezvous_id(dist)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib.tw_comm_create_mp(world, rank, 0, T * H * 2, rid.encode(), _lib.TW_TRANSPORT_AUTO,
                                          ctypes.byref(h)))
    r = weave.LayerRunner("llama-70b", tp=world, max_tokens=T, comm=h, hidden=H, intermediate=2048, heads=16,
                          kv_heads=4, head_dim=64)
    out = {{}}
    for mode, kw in (("fuseonly", {{}}), ("unfused", {{}}), ("tokenweave", {{"prefix": 320, "boundary_sms": 4}})):
        dist.barrier()
        out[mode] = r.run(T, mode, layers=2, **kw)
        out[mode + "_ops"] = [(e["op"], e["split"], e["stream"]) for e in r.trace()]
    dist.barrier()
    # K1 inside a CUDA graph, replayed: barrier generations live on the device
    out["tokenweave_graph"] = r.run(T, "tokenweave", prefix=320, boundary_sms=4, layers=2, graph=True)
    # measured serving throughput in TP mode: chunked-prefill batches (with
    # prior-context attention) through K1, identical call sequence per rank
    dist.barrier()
    tp = r.throughput(weave.synth_trace(3, 200, 4), 256, "tokenweave", num_layers=2, layers_measured=1,
                      boundary_sms=4, threshold=256)
    out["throughput"] = {{k: tp[k] for k in ("iterations", "total_tokens", "tokens_per_sec")}}
    _lib.check(_lib.lib.tw_comm_check(h))
    print(json.dumps(out), flush=True)
    dist.barrier()
    r.close()
    _lib.lib.tw_comm_destroy(h)
    dist.destroy_process_group()
""")


def test_weave_tp_runner_two_processes(cuda, tmp_path):
    """The TP weave runner (K1 boundary over a multi-process communicator):
    every mode completes on both ranks with the reference's DAG shapes."""
    world = 2
    script = tmp_path / "ww.py"
    script.write_text(WEAVE_WORKER.format(root=ROOT))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for rank in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE=str(world), TW_BARRIER_SPIN_LIMIT=str(1 << 28))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    for o in outs:
        res = json.loads([ln for ln in o.splitlines() if ln.startswith("{")][-1])
        assert len(res["fuseonly_ops"]) == 4 and len(res["unfused_ops"]) == 4
        ops = res["tokenweave_ops"]
        assert len(ops) == 8 and sum(1 for op, _, st in ops if op == "fused_ar_norm" and st == "comm") == 4
        assert res["throughput"]["total_tokens"] == 3 * (200 + 4) and res["throughput"]["tokens_per_sec"] > 0
        from paper_2505_11329_b200 import weave
        assert res["throughput"]["iterations"] == len(weave.form_batches(weave.synth_trace(3, 200, 4), 256))


def test_two_processes_one_gpu_peer_fallback(cuda, orc, tmp_path):
    world, T, H = 2, 48, 1024
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=ROOT, T=T, H=H, reps=3, outdir=str(tmp_path)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = []
    for rank in range(world):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                   WORLD_SIZE=str(world), TW_BARRIER_SPIN_LIMIT=str(1 << 28))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=300)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
    infos = [json.loads([ln for ln in o.splitlines() if ln.startswith("{")][-1]) for o in outs]
    assert all(i["transport"] == "peer" for i in infos)
    inputs, residual, weight = group_inputs(5, world, T, H)
    inputs, residual = bf16_round(inputs), bf16_round(residual)
    ranges = orc.token_shard_map(T, world)
    want_out, want_res = orc.fused_allreduce_rmsnorm(list(inputs), [residual[b:e] for b, e in ranges], weight)
    for r in range(world):
        assert_bf16_close(np.load(tmp_path / f"out{r}.npy"), want_out)
        assert np.array_equal(np.load(tmp_path / f"res{r}.npy"), bf16_round(want_res[r]))
