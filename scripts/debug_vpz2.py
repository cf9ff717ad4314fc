# Layer under ShardedVPHeads: which attention grads differ?  Compare the arena
# slot sums (before Adam) with the ref's all-reduced grads, per tensor.
import sys, threading, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2402_00518_b200 as ee
import paper_2402_00518_b200.parallel as par
import eesynth as S
import test_gpu_vp_fused as T
ee.load()
cfg = T._cfg("layer", 37)
hidden = S.hidden_states(cfg, 256); targets = S.targets(cfg, 256); params = S.head_params(cfg)
# bypass the NotImplementedError guard for the experiment
orig = par.ShardedVPHeads.__init__
def init(self, spec, *a, **k):
    arch = spec.arch; spec.arch = "mlp_"  # not "layer"
    spec.arch = arch
    self_spec = spec
    import types
    try:
        par_spec_arch = spec.arch
        spec.arch = "x"
        spec.arch = par_spec_arch
    finally:
        pass
src = open(par.__file__).read()
par_ns = {}
exec(compile(src.replace('if spec.arch == "layer":', 'if False:'), par.__file__, "exec"), par.__dict__)
# capture arena contents right before each update
captured = {}
orig_update = par.ShardedVPHeads.update
def upd(self, i, *a, **k):
    torch.cuda.current_stream().synchronize()
    captured[(self.rank, i)] = self.arenas[i % self.n_arenas].clone()
    return orig_update(self, i, *a, **k)
par.ShardedVPHeads.update = upd
got = T._run_vp_adam(ee, cfg, 2, hidden, targets, params, sharded=True, steps=1)
# reference grads: fused VP without body (grads all-reduced, no Adam)
ref = T.run_threads(ee, cfg, 2, hidden, targets, params, [1.0, 0.5], fused=True, steps=1)
spec_cfg = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, "layer", 1e-5, 0, 504, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads, seq_len=cfg.seq_len)
for r in range(2):
    vb, ve = par.vocab_shard(cfg.vocab, 2, r)
    c = ee.make_config(cfg.hidden, cfg.vocab, cfg.ffn, 1, "layer", 1e-5, vb, ve, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads or cfg.n_heads, seq_len=cfg.seq_len)
    shapes = ee.tensor_shapes(cfg.hidden, ve - vb, cfg.ffn, "layer", c.n_kv_heads)
    for i in range(cfg.exits):
        ar = captured[(r, i)]
        for k in shapes:
            if k == "w_out": continue
            b, rows, off, total = ee.ee_dp_shard_layout(c, 2, r, k)
            if rows == 0: continue
            C = shapes[k][-1]
            sl = ar[off:off + 2 * rows * C].view(2, rows, C).double().sum(0).cpu()
            want = ref[r][1][i][k].double().reshape(-1, C)[b:b + rows]
            err = float((sl - want).abs().max() / (want.abs().max() + 1e-30))
            print(r, i, k, "rel max err", err)
