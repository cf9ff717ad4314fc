"""Multi-GPU host orchestration of the exit-head step: data
parallelism over tokens (`data_parallel_step` over NCCL; `ShardedDPHeads`, the
fused ZeRO-1 path over peer memory), vocab-parallel W_out
(`vocab_parallel_step`; `vocab_parallel_step_fused` with `PeerBuffers` and
`ShardedVPHeads`) and the forward-communication-only pipeline
(`pipeline_forward_only_step`).  All compute runs in the CUDA library; these
functions only order its calls and the collectives between them.

Data parallelism: EE-Tuning's exits are independent and every token
contributes independently to an exit's loss, so the step shards
along the flat token axis: rank r owns tokens [r*N/P, (r+1)*N/P).  The only
exchanges of the NCCL path are

  1. the global number of valid tokens W (one int64 all-reduce), so every
     rank normalises its loss and gradients by the *global* W (A16);
  2. each exit's fp32 parameter gradients (sum all-reduce), issued
     asynchronously right after that exit's backward so it overlaps the next
     exit's compute on the GPU (NCCL runs on its own stream);
  3. the per-exit partial losses (sum all-reduce) for reporting.

The compute is injected (`run_exit`), so the same orchestration drives the CUDA
library on GPUs (NCCL) and is tested on CPUs with the oracle (gloo,
tests/test_dp_gloo.py).
"""

from __future__ import annotations

from typing import Callable, Iterable

import torch
import torch.distributed as dist


def shard_range(n_global: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """Contiguous token shard of `rank`, in units of `align` tokens (sizes differ
    by at most one unit).  Layer exits couple the tokens of a sequence, so their
    shards are whole sequences: align = seq_len (n_global a multiple of it)."""
    if n_global % align:
        raise ValueError("n_global must be a multiple of align")
    base, rem = divmod(n_global // align, world)
    start = rank * base + min(rank, rem)
    return start * align, (start + base + (1 if rank < rem else 0)) * align


def data_parallel_step(n_exits: int, count_local: Callable[[], torch.Tensor] | None,
                       run_exit: Callable[[int, torch.Tensor | None], None],
                       grads_of: Callable[[int], Iterable[torch.Tensor]],
                       loss: torch.Tensor, optimizer_step: Callable[[], None] | None = None,
                       group=None, weight_sums: torch.Tensor | None = None,
                       normalize: Callable[[int], None] | None = None) -> torch.Tensor:
    """One data-parallel EE-Tuning step.

    Uniform token weights: count_local() -> int64 tensor [1] with the local
    valid-token count; run_exit(i, W) computes exit i's loss (into loss[i]) and
    gradients on the local tokens, normalised by the global count W (A16).
    Confidence weights (weight_sums = float tensor [E]): run_exit(i,
    None) computes the UNNORMALISED sum_t c_t loss_t, its gradient and
    weight_sums[i] = sum_t c_t on the local tokens (EE_WEIGHT_CONFIDENCE_SUM);
    after the SUM all-reduces, normalize(i) divides exit i by the global
    sum_t c_t (ee_normalize_exit).  grads_of(i) yields exit i's gradient
    tensors; optimizer_step() applies the update after all reductions.
    Returns W (uniform) or the global weight sums (confidence).
    """
    conf = weight_sums is not None
    W = None
    if not conf:
        W = count_local()
        dist.all_reduce(W, group=group)
    handles = []
    for i in range(n_exits):
        run_exit(i, W)
        for t in grads_of(i):
            handles.append(dist.all_reduce(t, group=group, async_op=True))
    handles.append(dist.all_reduce(loss, group=group, async_op=True))
    if conf:
        handles.append(dist.all_reduce(weight_sums, group=group, async_op=True))
    for h in handles:
        h.wait()
    if conf:
        for i in range(n_exits):
            normalize(i)
    if optimizer_step is not None:
        optimizer_step()
    return weight_sums if conf else W


# ---------------------------------------------------------------------------
# Data parallel with the gradient reduce-scatter fused into the weight-gradient
# GEMMs and a sharded Adam whose operand stores are the all-gather (ZeRO-1)
# ---------------------------------------------------------------------------

def _peer_tables(rank, local_tensors, group=None, ranks=None):
    """Per-tensor peer pointer lists: from the other ranks' objects (ranks, one
    process) or by exchanging CUDA IPC handles over the process group.
    Returns (tables, opened) with tables[j] = [ptr of rank q's tensor j]."""
    import paper_2402_00518_b200 as ee
    if ranks is not None:
        return [[r_tensors[j].data_ptr() for r_tensors in ranks]
                for j in range(len(local_tensors))], []
    world = dist.get_world_size(group)
    mine = [ee.ee_ipc_get_handle(t) for t in local_tensors]
    allh = [None] * world
    dist.all_gather_object(allh, mine, group=group)
    tabs, opened = [], []
    for j, t in enumerate(local_tensors):
        row = []
        for q in range(world):
            if q == rank:
                row.append(t.data_ptr())
            else:
                p = ee.ee_ipc_open(*allh[q][j])
                opened.append((p, allh[q][j][1]))
                row.append(p)
        tabs.append(row)
    return tabs, opened


class ShardedDPHeads:
    """Exit heads of one rank under the fused data-parallel path
    (include/ee.h ee_tune_step_rs / ee_adam_update_sharded).

    Every rank holds the full bf16 operands (fp32 gains) of every exit, but
    only its row shard of the fp32 masters and Adam moments (1/P of the
    optimizer state), and `n_arenas` gradient arenas in which the other ranks'
    weight-gradient GEMMs deposit their partials of this rank's rows.  step():
    exit by exit, tune with the gradient rows routed to their owners,
    peer barrier, sharded Adam that stores the new operand rows into every
    rank -- no NCCL on the bulk path; only the valid-token count and the
    per-exit losses (8 B each) use `comm_all_reduce`."""

    def __init__(self, spec, max_tokens: int, rank: int, world: int, device="cuda",
                 n_arenas: int = 2):
        import paper_2402_00518_b200 as ee
        self.ee, self.spec, self.rank, self.world = ee, spec, rank, world
        self.conf = spec.token_weighting == "confidence"   # dynamic weights
        wt = "confidence_sum" if self.conf else "uniform"
        self.cfg = ee.make_config(spec.hidden, spec.vocab, spec.ffn, spec.num_exits, spec.arch,
                                  spec.norm_eps, token_weighting=wt, **spec.attn_kwargs())
        self.exit_cfg = ee.make_config(spec.hidden, spec.vocab, spec.ffn, 1, spec.arch,
                                       spec.norm_eps, token_weighting=wt, **spec.attn_kwargs())
        shapes = ee.tensor_shapes(spec.hidden, spec.vocab, spec.ffn, spec.arch,
                                  self.cfg.n_kv_heads)
        self.names = [k for k in ee.TENSOR_NAMES if k in shapes]
        self.shapes = shapes
        dev = torch.device(device)
        E = spec.num_exits
        self.layout = {k: ee.ee_dp_shard_layout(self.exit_cfg, world, rank, k)
                       for k in self.names}
        total = self.layout[self.names[0]][3]

        def shard(k):
            rows = self.layout[k][1]
            C = shapes[k][-1]
            return torch.zeros(rows, C, dtype=torch.float32, device=dev)

        self.operand = [{k: torch.zeros(shapes[k], device=dev,
                                        dtype=torch.float32 if k.startswith("g_")
                                        else torch.bfloat16) for k in self.names}
                        for _ in range(E)]
        self.master = [{k: shard(k) for k in self.names} for _ in range(E)]
        self.m = [{k: shard(k) for k in self.names} for _ in range(E)]
        self.v = [{k: shard(k) for k in self.names} for _ in range(E)]
        self.n_arenas = max(1, min(int(n_arenas), E))
        self.arenas = [torch.zeros(max(total, 4), dtype=torch.float32, device=dev)
                       for _ in range(self.n_arenas)]
        self.sig = torch.zeros(8, dtype=torch.int32, device=dev)
        self.epoch = 0
        self.workspace = torch.zeros(ee.ee_workspace_size(self.cfg, max_tokens),
                                     dtype=torch.uint8, device=dev)
        self.workspace_tokens = int(max_tokens)
        self.loss = torch.zeros(E, dtype=torch.float32, device=dev)
        self.wsum = torch.zeros(E, dtype=torch.float32, device=dev)   # sum_t c_t per exit
        self.step_count = 0
        self._opened = []

    def _locals(self):
        ts = list(self.arenas) + [self.sig]
        for d in self.operand:
            ts += [d[k] for k in self.names]
        return ts

    def _set_tables(self, tabs):
        ee = self.ee
        na = self.n_arenas
        self.arena_sets = [ee.peer_set(self.rank, tabs[j]) for j in range(na)]
        self.sig_set = ee.peer_set(self.rank, tabs[na])
        nt = len(self.names)
        self.operand_sets = [{k: ee.peer_set(self.rank, tabs[na + 1 + i * nt + j])
                              for j, k in enumerate(self.names)}
                             for i in range(self.spec.num_exits)]

    def connect_local(self, ranks: list["ShardedDPHeads"]):
        tabs, _ = _peer_tables(self.rank, self._locals(), ranks=[r._locals() for r in ranks])
        self._set_tables(tabs)

    def connect_ipc(self, group=None):
        tabs, self._opened = _peer_tables(self.rank, self._locals(), group=group)
        self._set_tables(tabs)

    def close(self):
        for p, off in self._opened:
            self.ee.ee_ipc_close(p, off)
        self._opened = []

    def init(self, mode="copy", copy_src=None, seed=0, std=0.02, src_dtype=torch.bfloat16):
        """Initialise through full-size fp32 staging masters (Copy and Random
        are deterministic, so every rank builds the same operands) and keep
        this rank's rows.  Copy stages one exit at a time; Random stages all
        exits at once (its streams are keyed by exit index)."""
        ee = self.ee
        dev = self.loss.device
        E = self.spec.num_exits

        def staging():
            return {k: torch.zeros(self.shapes[k], dtype=torch.float32, device=dev)
                    for k in self.names}

        def keep(i, full):
            for k in self.names:
                b, rows = self.layout[k][0], self.layout[k][1]
                if rows:
                    self.master[i][k].copy_(full[k].reshape(-1, self.shapes[k][-1])[b:b + rows])
                if k.startswith("g_"):
                    self.operand[i][k].copy_(full[k])

        if mode == "random":
            full = [staging() for _ in range(E)]
            ee.ee_init_heads(self.cfg, "random", None, full, self.operand, seed=seed, std=std)
            for i in range(E):
                keep(i, full[i])
            return
        for i in range(E):
            full = staging()
            ee.ee_init_heads(self.exit_cfg, mode, copy_src[i:i + 1], [full],
                             self.operand[i:i + 1], src_dtype=src_dtype)
            keep(i, full)
            del full

    def barrier(self, stream=None):
        self.epoch += 1
        self.ee.ee_peer_barrier(self.sig_set, self.epoch, self.workspace, stream)

    def status(self):
        return self.ee.ee_get_status(self.workspace)

    def step(self, hidden, targets, lr, all_reduce=None, exit_weights=None, beta1=0.9,
             beta2=0.95, eps=1e-5, weight_decay=0.0):
        """One tuning step + Adam on this rank's tokens.  all_reduce(t) sums a
        small tensor over the ranks in place (the valid-token count before the
        step, the per-exit losses after); None = one rank."""
        return self._step(lambda i: hidden[i], None, targets, lr, all_reduce, exit_weights,
                          beta1, beta2, eps, weight_decay)

    def step_host(self, hidden_host, targets_host, lr, all_reduce=None, exit_weights=None,
                  beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0):
        """step() with this rank's hidden states and targets in pinned host
        memory: exit i + 1's H2D copy overlaps exit i's compute (HostStager)."""
        ee = self.ee
        dev = self.loss.device
        st = torch.cuda.current_stream(dev)
        if getattr(self, "_stager", None) is None:
            self._stager = ee.HostStager(self.workspace_tokens, self.spec.hidden, dev)
        stg = self._stager
        tg = stg.begin(hidden_host, targets_host, st)
        return self._step(lambda i: stg.get(i, st), lambda i: stg.release(i, st), tg, lr,
                          all_reduce, exit_weights, beta1, beta2, eps, weight_decay)

    def _step(self, hidden_of, release, targets, lr, all_reduce, exit_weights, beta1, beta2,
              eps, weight_decay):
        ee = self.ee
        E = self.spec.num_exits
        w = exit_weights if exit_weights is not None else [1.0] * E
        W = None
        if not self.conf:
            W = torch.zeros(1, dtype=torch.int64, device=self.loss.device)
            ee.ee_count_valid(targets, self.spec.vocab, W, self.workspace)
            if all_reduce is not None:
                all_reduce(W)
        self.step_count += 1
        self.barrier()                       # previous update's operand stores are complete
        for i in range(E):
            j = i % self.n_arenas
            aux = [{"weight_sum": self.wsum[i:i + 1]}] if self.conf else None
            ee.ee_tune_step_rs(self.exit_cfg, [hidden_of(i)], targets, w[i:i + 1],
                               self.operand[i:i + 1], [self.arena_sets[j]],
                               self.loss[i:i + 1], self.workspace, aux=aux, valid_count=W)
            if release is not None:
                release(i)
            if self.conf and all_reduce is not None:
                all_reduce(self.wsum[i:i + 1])   # global sum_t c_t: the gradient divisor
            self.barrier()                   # every rank's partials of exit i have landed
            ee.ee_adam_update_sharded(self.exit_cfg, self.world, self.rank, [self.arenas[j]],
                                      self.master[i:i + 1], self.m[i:i + 1], self.v[i:i + 1],
                                      self.operand_sets[i:i + 1], lr, self.step_count, beta1,
                                      beta2, eps, weight_decay,
                                      grad_divisor=self.wsum[i:i + 1] if self.conf else None)
            if self.n_arenas == 1 and i + 1 < E:
                self.barrier()               # arena read by every owner before it is rewritten
        if all_reduce is not None:
            all_reduce(self.loss)
        if self.conf:                        # L_i = sum c_t loss_t / sum c_t over all ranks
            for i in range(E):
                ee.ee_normalize_exit(self.exit_cfg, None, self.loss[i:i + 1],
                                     self.wsum[i:i + 1])
        return self.loss


# ---------------------------------------------------------------------------
# Vocab-parallel W_out (BASELINE configs[3]: "vocab-parallel W_out over 8 GPUs")
# ---------------------------------------------------------------------------

EXIT_BODY = ("g_a", "w_gate", "w_up", "w_down", "g_f",    # replicated; W_out is sharded
             "g_att", "w_q", "w_k", "w_v", "w_o")


class TorchComm:
    """Collectives of the vocab-parallel step over a torch.distributed group
    (NCCL on GPUs, gloo on CPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather_into(self, out, inp):
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def all_reduce(self, t, op="sum", async_op=False):
        o = dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM
        return dist.all_reduce(t, op=o, group=self.group, async_op=async_op)

    def reduce_scatter(self, out, inp):
        dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM, group=self.group)


class LocalComm:
    """World of one: every collective is the identity (P = 1)."""
    rank, world = 0, 1

    def all_gather_into(self, out, inp):
        if inp.data_ptr() != out.data_ptr():
            out[:inp.shape[0]].copy_(inp)

    def all_reduce(self, t, op="sum", async_op=False):
        return None

    def reduce_scatter(self, out, inp):
        out.copy_(inp[:out.shape[0]])


def vocab_shard(V: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous W_out row shard of `rank`; widths are multiples of 8 (TMA row
    stride rule), the last shard takes the remainder."""
    w = ((V // world + 7) // 8) * 8
    b = min(V, rank * w)
    e = V if rank == world - 1 else min(V, (rank + 1) * w)
    return b, e


class GpuPhases:
    """The five ee_vp_* phases of the CUDA library for one rank."""

    def __init__(self, ee, cfg, workspace, stream=None):
        self.ee, self.cfg, self.ws, self.stream = ee, cfg, workspace, stream

    def exit_forward(self, hidden, params, z_out, n_all):
        self.ee.ee_vp_exit_forward(self.cfg, hidden, n_all, params, z_out, self.ws, self.stream)

    def vocab_stats(self, z_all, targets_all, params, key, sums):
        self.ee.ee_vp_vocab_stats(self.cfg, z_all, targets_all, params, key, sums, self.ws,
                                  self.stream)

    def rescale(self, key, sums):
        self.ee.ee_vp_rescale(self.cfg, key.numel(), key, sums, self.ws, self.stream)

    def vocab_backward(self, i, z_all, targets_all, key, sums, alpha, W, params, grads,
                       dz_partial, loss_slot, accumulate, aux=None):
        self.ee.ee_vp_vocab_backward(self.cfg, z_all, targets_all, key, sums, alpha, params, grads,
                                     dz_partial, loss_slot, self.ws, valid_count=W,
                                     accumulate=accumulate, aux=aux, exit_index=i,
                                     stream=self.stream)

    def exit_backward(self, hidden, params, dz_local, grads, accumulate, n_all):
        self.ee.ee_vp_exit_backward(self.cfg, hidden, n_all, params, dz_local, grads, self.ws,
                                    accumulate=accumulate, stream=self.stream)

    # fused peer-memory variants (vocab_parallel_step_fused)
    def exit_forward_ag(self, hidden, params, peer, n_all):
        self.ee.ee_vp_exit_forward_ag(self.cfg, hidden, n_all, params, peer.z_set, self.ws,
                                      self.stream)

    def vocab_backward_rs(self, i, z_all, targets_all, key, sums, alpha, W, params, grads, peer,
                          loss_slot, accumulate, aux=None):
        self.ee.ee_vp_vocab_backward_rs(self.cfg, z_all, targets_all, key, sums, alpha, params,
                                        grads, peer.slot_set, loss_slot, self.ws, valid_count=W,
                                        accumulate=accumulate, aux=aux, exit_index=i,
                                        stream=self.stream)

    def exit_backward_slots(self, hidden, params, peer, grads, accumulate, n_all,
                            grad_arenas=None):
        self.ee.ee_vp_exit_backward_slots(self.cfg, hidden, n_all, params, peer.slots,
                                          peer.world, grads, self.ws, accumulate=accumulate,
                                          grad_arenas=grad_arenas, stream=self.stream)

    def barrier(self, peer):
        peer.epoch += 1
        self.ee.ee_peer_barrier(peer.sig_set, peer.epoch, self.ws, self.stream)


def vocab_parallel_step(phases, comm, arch: str, hidden_local, targets_all, params, grads,
                        loss: torch.Tensor, exit_weights, W: torch.Tensor, bufs: dict,
                        accumulate: bool = False, aux=None):
    """One EE-Tuning step with W_out sharded by vocabulary rows over the ranks
    of `comm` and tokens sharded for the exit bodies (equal shards, n_all =
    world * n_local).  Per exit: all-gather z, the distributed softmax-CE
    (MAX all-reduce of the (max, argmax) key, SUM all-reduce of the rescaled
    sum-exp and target logit), local dW_out shard, reduce-scatter of dz back
    to the token owners, and an async SUM all-reduce of the exit-body grads.

    bufs: z_all [n_all x h] (exit-head input dtype), key [n_all] int64,
    sums [n_all x 2] fp32, dz_partial [n_all x h] fp32, dz_local [n_local x h].
    W: global valid-token count (int64 [1]).  loss[i] = global mean loss.
    """
    r = comm.rank
    z_all, key, sums = bufs["z_all"], bufs["key"], bufs["sums"]
    n_all = z_all.shape[0]
    n_local = n_all // comm.world
    if n_local * comm.world != n_all:
        raise ValueError("vocab-parallel step needs equal token shards")
    dz_partial = bufs.get("dz_partial") if arch != "embedding" else None
    dz_local = bufs.get("dz_local") if arch != "embedding" else None
    handles = []
    for i in range(len(hidden_local)):
        mine = z_all[r * n_local:(r + 1) * n_local]
        phases.exit_forward(hidden_local[i], params[i], mine, n_all)            # a1-a4
        comm.all_gather_into(z_all, mine)
        phases.vocab_stats(z_all, targets_all, params[i], key, sums)            # a5
        comm.all_reduce(key, "max")
        phases.rescale(key, sums)
        comm.all_reduce(sums, "sum")
        phases.vocab_backward(i, z_all, targets_all, key, sums, exit_weights[i], W, params[i],
                              grads[i], dz_partial, loss[i:i + 1], accumulate,
                              None if aux is None else aux[i])                  # a6-a9
        if dz_partial is not None:
            comm.reduce_scatter(dz_local, dz_partial)
        phases.exit_backward(hidden_local[i], params[i], dz_local, grads[i], accumulate,
                             n_all)                                             # a10-a13
        for k in EXIT_BODY:
            if grads[i].get(k) is not None:
                handles.append(comm.all_reduce(grads[i][k], "sum", async_op=True))
    for h in handles:
        if h is not None:
            h.wait()


# ---------------------------------------------------------------------------
# Vocab-parallel step with the z all-gather and the dz reduce-scatter fused
# into the producing kernels over peer memory (SURVEY §8(e) "fused variants")
# ---------------------------------------------------------------------------

class PeerBuffers:
    """The symmetric buffers of the fused vocab-parallel collectives on one
    rank: z_all [n_all x h] bf16 (every rank's a4 kernel stores its z rows
    here), dz slots [world x n_local x h] fp32 (every rank's a8 epilogue stores
    its dz partial rows for this rank's tokens into slot [its rank]) and the
    int32 signal array of ee_peer_barrier.  ptr tables: connect_ipc (one
    process per GPU, CUDA IPC handles exchanged over the process group) or
    connect_local (ranks emulated inside one process)."""

    def __init__(self, rank: int, world: int, n_all: int, h: int, device="cuda",
                 z_dtype=torch.bfloat16):
        if n_all % world:
            raise ValueError("fused vocab-parallel step needs equal token shards")
        self.rank, self.world, self.n_all, self.n_local = rank, world, n_all, n_all // world
        self.z_all = torch.zeros(n_all, h, dtype=z_dtype, device=device)
        self.slots = torch.zeros(world, self.n_local, h, dtype=torch.float32, device=device)
        self.sig = torch.zeros(8, dtype=torch.int32, device=device)
        self.epoch = 0
        self._opened = []
        self.z_set = self.slot_set = self.sig_set = None

    def _tables(self, z, sl, sg):
        from paper_2402_00518_b200 import peer_set
        self.z_set, self.slot_set, self.sig_set = (peer_set(self.rank, z), peer_set(self.rank, sl),
                                                   peer_set(self.rank, sg))

    def connect_local(self, ranks: list["PeerBuffers"]):
        self._tables([b.z_all for b in ranks], [b.slots for b in ranks], [b.sig for b in ranks])

    def connect_ipc(self, group=None):
        tabs, self._opened = _peer_tables(self.rank, [self.z_all, self.slots, self.sig],
                                          group=group)
        self._tables(*tabs)

    def close(self):
        import paper_2402_00518_b200 as ee
        for p, off in self._opened:
            ee.ee_ipc_close(p, off)
        self._opened = []


class ShardedVPHeads:
    """Exit heads of one rank under the fused vocab-parallel path with the
    replicated exit body updated ZeRO-1 style (vocab_parallel_step_fused(...,
    body=self)): W_out is this rank's [V/P x h] shard (full master, moments,
    gradient); the body (norm gains, MLP, attention) is held in full as bf16
    operands (fp32 gains) on every rank but only this rank's row blocks of its
    fp32 masters and moments, and `n_arenas` arenas collect the other ranks'
    body-gradient rows (include/ee.h ee_vp_exit_backward_slots grad_arenas,
    ee_adam_update_sharded tensor_mask).  Call set_lr() before each step."""

    def __init__(self, spec, n_all: int, rank: int, world: int, device="cuda", n_arenas: int = 2):
        import paper_2402_00518_b200 as ee
        self.ee, self.spec, self.rank, self.world = ee, spec, rank, world
        vb, ve = vocab_shard(spec.vocab, world, rank)
        kw = spec.attn_kwargs()
        self.cfg = ee.make_config(spec.hidden, spec.vocab, spec.ffn, spec.num_exits, spec.arch,
                                  spec.norm_eps, vb, ve, **kw)
        self.exit_cfg = ee.make_config(spec.hidden, spec.vocab, spec.ffn, 1, spec.arch,
                                       spec.norm_eps, vb, ve, **kw)
        self.wcfg = ee.make_config(spec.hidden, spec.vocab, 0, 1, "embedding", spec.norm_eps,
                                   vb, ve, ds_mode=spec.ds_mode)                     # the W_out shard alone
        shapes = ee.tensor_shapes(spec.hidden, ve - vb, spec.ffn, spec.arch,
                                  self.cfg.n_kv_heads)
        self.shapes = shapes
        self.names = [k for k in ee.TENSOR_NAMES if k in shapes]
        self.body = [k for k in self.names if k != "w_out"]
        dev = torch.device(device)
        E = spec.num_exits
        self.layout = {k: ee.ee_dp_shard_layout(self.exit_cfg, world, rank, k) for k in self.names}
        total = self.layout[self.names[0]][3]    # (no W_out block under a vocab shard)

        def master_like(k):
            if k == "w_out":
                return torch.zeros(shapes[k], dtype=torch.float32, device=dev)
            return torch.zeros(self.layout[k][1], shapes[k][-1], dtype=torch.float32, device=dev)

        self.operand = [{k: torch.zeros(shapes[k], device=dev,
                                        dtype=torch.float32 if k.startswith("g_")
                                        else torch.bfloat16) for k in self.names}
                        for _ in range(E)]
        self.master = [{k: master_like(k) for k in self.names} for _ in range(E)]
        self.m = [{k: master_like(k) for k in self.names} for _ in range(E)]
        self.v = [{k: master_like(k) for k in self.names} for _ in range(E)]
        self.grads = [{"w_out": torch.zeros(shapes["w_out"], device=dev)} for _ in range(E)]
        self.n_arenas = max(1, min(int(n_arenas), E))
        self.arenas = [torch.zeros(max(total, 4), dtype=torch.float32, device=dev)
                       for _ in range(self.n_arenas)]
        self.workspace = torch.zeros(ee.ee_workspace_size(self.cfg, n_all), dtype=torch.uint8,
                                     device=dev)
        self.loss = torch.zeros(E, dtype=torch.float32, device=dev)
        self.step_count = 0
        self.lr = 0.0
        self._opened = []

    def _locals(self):
        ts = list(self.arenas)
        for d in self.operand:
            ts += [d[k] for k in self.body]
        return ts

    def _set_tables(self, tabs):
        ee = self.ee
        na, nb = self.n_arenas, len(self.body)
        self.arena_sets = [ee.peer_set(self.rank, tabs[j]) for j in range(na)]
        self.operand_sets = [{k: ee.peer_set(self.rank, tabs[na + i * nb + j])
                              for j, k in enumerate(self.body)}
                             for i in range(self.spec.num_exits)]

    def connect_local(self, ranks):
        tabs, _ = _peer_tables(self.rank, self._locals(), ranks=[r._locals() for r in ranks])
        self._set_tables(tabs)

    def connect_ipc(self, group=None):
        tabs, self._opened = _peer_tables(self.rank, self._locals(), group=group)
        self._set_tables(tabs)

    def close(self):
        for p, off in self._opened:
            self.ee.ee_ipc_close(p, off)
        self._opened = []

    def init(self, mode="copy", copy_src=None, seed=0, std=0.02, src_dtype=torch.bfloat16):
        """Copy / Random through full-size staging masters (deterministic, so
        every rank builds the same body operands); keeps this rank's rows."""
        ee = self.ee
        dev = self.loss.device
        E = self.spec.num_exits
        staging = lambda: {k: torch.zeros(self.shapes[k], dtype=torch.float32, device=dev)
                           for k in self.names}
        if mode == "random":
            full = [staging() for _ in range(E)]
            ee.ee_init_heads(self.cfg, "random", None, full, self.operand, seed=seed, std=std)
        else:
            full = []
            for i in range(E):
                f = staging()
                ee.ee_init_heads(self.exit_cfg, mode, copy_src[i:i + 1], [f],
                                 self.operand[i:i + 1], src_dtype=src_dtype)
                full.append(f)
        for i in range(E):
            for k in self.names:
                if k == "w_out":
                    self.master[i][k].copy_(full[i][k])
                    continue
                b, rows = self.layout[k][0], self.layout[k][1]
                if rows:
                    self.master[i][k].copy_(full[i][k].reshape(-1, self.shapes[k][-1])[b:b + rows])
                if k.startswith("g_"):
                    self.operand[i][k].copy_(full[i][k])

    def set_lr(self, lr):
        self.lr = lr
        self.step_count += 1

    def arena_set(self, i):
        return self.arena_sets[i % self.n_arenas]

    def update(self, i, beta1=0.9, beta2=0.95, eps=1e-5, weight_decay=0.0):
        """Exit i: sharded Adam of the body rows this rank owns (+ their stores
        into every rank's operands) and Adam of the local W_out shard."""
        ee = self.ee
        if self.body:                                  # (Embedding exits have no body)
            ee.ee_adam_update_sharded(self.exit_cfg, self.world, self.rank,
                                      [self.arenas[i % self.n_arenas]], self.master[i:i + 1],
                                      self.m[i:i + 1], self.v[i:i + 1],
                                      self.operand_sets[i:i + 1], self.lr, self.step_count,
                                      beta1, beta2, eps, weight_decay, tensors=self.body)
        w = lambda d: [{"w_out": d[i]["w_out"]}]
        ee.ee_adam_update(self.wcfg, w(self.master), w(self.operand), w(self.grads), w(self.m),
                          w(self.v), self.lr, self.step_count, beta1, beta2, eps, weight_decay)

    def status(self):
        return self.ee.ee_get_status(self.workspace)


def vocab_parallel_step_fused(phases, comm, peer: PeerBuffers, arch: str, hidden_local,
                              targets_all, params, grads, loss: torch.Tensor, exit_weights,
                              W: torch.Tensor, bufs: dict, accumulate: bool = False, aux=None,
                              body=None):
    """vocab_parallel_step with the two bulk exchanges inside the kernels:
    a4 stores z into every rank's z_all (all-gather), the a8 epilogue stores
    dz rows into their owners' slots (reduce-scatter; the owner's a10 kernel
    sums the slots in rank order).  Peer barriers (ee_peer_barrier) order the
    stores against the readers: once before the first exit (the previous
    step's readers), after each all-gather and after each reduce-scatter.  The
    CE statistics (8 B + 8 B per token) stay on `comm`, as do the exit-body
    gradient all-reduces (async).  bufs: key [n_all] int64, sums [n_all x 2].

    body (ShardedVPHeads): the replicated exit body is updated ZeRO-1 style
    instead -- its gradient rows go to their owners' arenas in the a11/a12
    epilogues, and after one more barrier body.update(i) runs the sharded
    Adam (whose stores are the body operands' all-gather) and the local Adam
    of the W_out shard; no body all-reduce."""
    key, sums = bufs["key"], bufs["sums"]
    n_all = peer.n_all
    handles = []
    phases.barrier(peer)
    for i in range(len(hidden_local)):
        phases.exit_forward_ag(hidden_local[i], params[i], peer, n_all)         # a1-a4 + AG
        phases.barrier(peer)
        phases.vocab_stats(peer.z_all, targets_all, params[i], key, sums)       # a5
        comm.all_reduce(key, "max")
        phases.rescale(key, sums)
        comm.all_reduce(sums, "sum")
        phases.vocab_backward_rs(i, peer.z_all, targets_all, key, sums, exit_weights[i], W,
                                 params[i], grads[i], peer, loss[i:i + 1], accumulate,
                                 None if aux is None else aux[i])               # a6-a9 + RS
        phases.barrier(peer)
        if body is not None:                                  # sharded body update
            if arch != "embedding":
                phases.exit_backward_slots(hidden_local[i], params[i], peer, None, False,
                                           n_all, grad_arenas=body.arena_set(i))  # a10-a13
            phases.barrier(peer)                              # every partial has landed
            body.update(i)
            continue
        if arch != "embedding":
            phases.exit_backward_slots(hidden_local[i], params[i], peer, grads[i], accumulate,
                                       n_all)                                   # a10-a13
        for k in EXIT_BODY:
            if grads[i].get(k) is not None:
                handles.append(comm.all_reduce(grads[i][k], "sum", async_op=True))
    for h in handles:
        if h is not None:
            h.wait()


# ---------------------------------------------------------------------------
# Forward-communication-only pipeline schedule (Fig. 3; NEXT #3)
# ---------------------------------------------------------------------------

def pipeline_forward_only_step(stage: int, n_stages: int, n_micro: int,
                               run_stage_forward: Callable[[int, torch.Tensor | None], torch.Tensor],
                               run_stage_exits: Callable[[int], None],
                               send: Callable[[int, torch.Tensor], object] | None,
                               recv: Callable[[int], torch.Tensor] | None,
                               optimizer_step: Callable[[], None] | None = None) -> None:
    """One EE-Tuning iteration of the paper's customised pipeline schedule
    "with forward communication only": the backbone is split into
    n_stages consecutive layer ranges; for each microbatch m, stage s receives
    the activation from stage s-1 (stage 0 reads its input), runs its backbone
    layers forward (run_stage_forward -> the activation for stage s+1; it also
    keeps the hidden states at this stage's exits), sends it on, and then --
    "as soon as the forward pass of the Transformer backbone within that stage
    is completed" -- runs forward, loss and backward of its own exits
    (run_stage_exits, gradients accumulated over microbatches).  No backbone
    activations are kept and nothing is sent backward.  optimizer_step()
    updates this stage's exits after the last microbatch.

    send(m, t) may return a handle with .wait() (isend); recv(m) returns the
    received activation.  Sends are waited for at the end of the iteration so
    stage s's exit work overlaps the transfer to stage s+1."""
    pending = []
    for m in range(n_micro):
        x_in = recv(m) if stage > 0 else None
        x_out = run_stage_forward(m, x_in)
        if stage + 1 < n_stages:
            pending.append(send(m, x_out))
        run_stage_exits(m)
    for h in pending:
        if h is not None and hasattr(h, "wait"):
            h.wait()
    if optimizer_step is not None:
        optimizer_step()


class TorchP2P:
    """Point-to-point transport of the forward-only pipeline over a
    torch.distributed group (NCCL on GPUs, gloo in the CPU tests)."""

    def __init__(self, stage: int, shape, dtype, device, group=None):
        self.stage, self.shape, self.dtype, self.device, self.group = stage, shape, dtype, device, group

    def send(self, m: int, t: torch.Tensor):
        return dist.isend(t.contiguous(), dst=self.stage + 1, group=self.group)

    def recv(self, m: int) -> torch.Tensor:
        buf = torch.empty(self.shape, dtype=self.dtype, device=self.device)
        dist.recv(buf, src=self.stage - 1, group=self.group)
        return buf
