"""Small launches of the kernels added in r01f for compute-sanitizer: a5 with
the P~ stores + a7 from P~ (ragged V and N), the fused-Adam epilogues, the
fused VP path at world 1 (peer stores, scatter epilogue, slot sum, barrier),
the fused DP path at world 1 (arena scatter, sharded Adam), a Layer step (RoPE
table in the q/k epilogues and the attention-backward stores), 16-byte
transposes with a ragged tail."""
import sys
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import eesynth as S
import paper_2402_00518_b200 as ee
from harness import gpu_step
from paper_2402_00518_b200.parallel import (GpuPhases, LocalComm, PeerBuffers, ShardedDPHeads,
                                            vocab_parallel_step_fused)

ee.load()
# ragged tune step (a5 P~ stores / a7 from P~ / transposes with n = 77)
cfg = S.Cfg(name="small", hidden=192, vocab=2056, ffn=384, arch="mlp", tokens=77, layers=2,
            after=[1, 2], init="random", seed=11)
hid, tg, prm = S.hidden_states(cfg, 77), S.targets(cfg, 77), S.head_params(cfg)
_, _, _, st = gpu_step(ee, cfg, hid, tg, prm, [1.0, 0.5])
assert st == (0, -1), st
# fused Adam (both epilogue instantiations)
hd = ee.ExitHeads(ee.HeadSpec(192, 2056, 384, 2, "mlp"), 77)
hd.init("copy", copy_src=[{k: v.cuda().float().contiguous() for k, v in p.items()} for p in prm],
        src_dtype=torch.float32)
hd.step_adam([x.cuda() for x in hid], tg.cuda(), 1e-3)
# fused VP at world 1
c1 = ee.make_config(192, 2056, 384, 1, "mlp", 1e-5, 0, 2056)
ws = torch.zeros(ee.ee_workspace_size(c1, 77), dtype=torch.uint8, device="cuda")
pb = PeerBuffers(0, 1, 77, 192)
pb.connect_local([pb])
W = torch.tensor([int((tg != -1).sum())], dtype=torch.int64, device="cuda")
loss = torch.zeros(1, device="cuda")
bufs = {"key": torch.zeros(77, dtype=torch.int64, device="cuda"),
        "sums": torch.zeros(77, 2, device="cuda")}
ops = [{k: (v.cuda().float() if k.startswith("g_") else v.cuda().bfloat16()).contiguous()
        for k, v in prm[0].items()}]
grd = [{k: torch.zeros(v.shape, device="cuda") for k, v in prm[0].items()}]
vocab_parallel_step_fused(GpuPhases(ee, c1, ws), LocalComm(), pb, "mlp", [hid[0].cuda()],
                          tg.cuda(), ops, grd, loss, [1.0], W, bufs)
# fused DP at world 1
dp = ShardedDPHeads(ee.HeadSpec(192, 2056, 384, 2, "mlp"), 77, 0, 1)
dp.connect_local([dp])
dp.init("copy", copy_src=[{k: v.cuda().float().contiguous() for k, v in p.items()} for p in prm],
        src_dtype=torch.float32)
dp.step([x.cuda() for x in hid], tg.cuda(), 1e-3)
# Layer exit step (RoPE table)
cl = S.get_cfg("tiny_layer")
_, _, _, st = gpu_step(ee, cl, S.hidden_states(cl), S.targets(cl), S.head_params(cl), [1.0, 0.5])
assert st == (0, -1), st
torch.cuda.synchronize()
print("sanitize run ok")
# VP with the sharded exit body at world 1 (tensor mask, arenas without W_out)
from paper_2402_00518_b200.parallel import ShardedVPHeads
zs = ShardedVPHeads(ee.HeadSpec(192, 2056, 384, 2, "mlp"), 77, 0, 1)
zs.connect_local([zs])
zs.init("copy", copy_src=[{k: v.cuda().float().contiguous() for k, v in p.items()} for p in prm],
        src_dtype=torch.float32)
pb2 = PeerBuffers(0, 1, 77, 192)
pb2.connect_local([pb2])
zs.set_lr(1e-3)
vocab_parallel_step_fused(GpuPhases(ee, zs.exit_cfg, zs.workspace), LocalComm(), pb2, "mlp",
                          [x.cuda() for x in hid], tg.cuda(), zs.operand, zs.grads, zs.loss,
                          [1.0, 0.5], W, {"key": torch.zeros(77, dtype=torch.int64, device="cuda"),
                                          "sums": torch.zeros(77, 2, device="cuda")}, body=zs)
torch.cuda.synchronize()
print("sanitize run 2 ok")
