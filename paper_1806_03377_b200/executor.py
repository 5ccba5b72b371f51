"""``run(cfg, ctx, schedule=None, *, model=...) -> SimResult`` on B200s.

This is the drop-in for ``pipesim.run`` (simulator.py:401-411).  Same inputs
(``SimConfig`` with a plan and a mode, a ``CostContext``, an optional explicit
``Schedule``), same output types; the difference is that the schedule is
*executed*: every stage of the plan trains a real MLP slice on a B200 with the
tcgen05 GEMM kernels of libpd_b200.so, and the trace holds measured device
times.  ``model=`` (an ``MLPSpec``) is the one required addition: the reference
has no tensors to run.

Layout in HBM (per hosted stage):
  w_master[l]  fp32 [out,in]            latest weights (SGD target)
  w_ring[l]    dtype [depth,out,in]     weight versions; slot from program.py
  b_master/b_ring                       same for biases (fp32)
  act[l]       dtype [act_depth,B,d]    stashed layer inputs of in-flight minibatches
  act_in       dtype [in_depth,B,d_0]   activation inbox (stage 0: resident data blocks)
  grad_in      dtype [grad_depth,B,d_L] gradient inbox
  dz_last      dtype [act_depth,B,d_L]  loss gradient (last stage)
PyTorch only allocates these; all math runs in the library.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import SimulationError, ValidationError
from .ledger import Mode, SimConfig, SimResult, TraceEvent, VersionLedger, build_report
from .models import ConvNetSpec, GPTSpec, MLPSpec, init_params_any, make_data_any
from .orders import Direction, Schedule, build_schedule, stage_inflight_caps
from .program import Program, compile_program

HOST_INIT_LIMIT = 64 * 1024 * 1024  # parameters; above this, weights/data are drawn on the device


def _torch():
    import torch

    return torch


@dataclass
class _StageBuf:
    wid: int
    stage: int
    dims: list[int]
    ring_depth: int
    init_slot: int
    act_depth: int
    in_depth: int
    grad_depth: int
    tensors: dict = field(default_factory=dict)
    desc: object = None
    keep: list = field(default_factory=list)  # ctypes arrays referenced by desc
    geoms: list | None = None  # layered stages: LayerGeom per layer


def _validate(cfg: SimConfig, ctx, model: MLPSpec) -> None:
    plan = cfg.plan
    if ctx is not None and plan.num_layers != ctx.num_layers:
        raise ValidationError(f"plan covers {plan.num_layers} layers, profile has {ctx.num_layers}")
    if plan.num_layers != model.num_layers:
        raise ValidationError(f"plan covers {plan.num_layers} layers, model has {model.num_layers}")
    if cfg.num_minibatches >= 65536:
        raise ValidationError("num_minibatches must be below 65536 (device flag values are epoch * 65536 + mb)")
    if any(st.replication > 16 for st in plan.stages):
        raise ValidationError("at most 16 replicas per stage")
    for s, st in enumerate(plan.stages):
        if st.replication > 1 and cfg.num_minibatches % st.replication:
            raise ValidationError(
                f"stage {s} is replicated {st.replication}x: num_minibatches ({cfg.num_minibatches}) must be a "
                "multiple of the replication so every allreduce round is complete (DESIGN.md §5)"
            )


class Executor:
    """Allocates one pipeline's device state and runs its compiled program repeatedly."""

    def __init__(self, cfg: SimConfig, ctx=None, schedule: Schedule | None = None, *, model: MLPSpec,
                 device: int | None = None, init: str | None = None, group=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise nat.NativeError("no CUDA device: the B200 executor has no CPU fallback")
        _validate(cfg, ctx, model)
        self.cfg, self.ctx, self.model = cfg, ctx, model
        self.schedule = schedule or build_schedule(cfg.plan, cfg.num_minibatches, cfg.max_inflight)
        dist = torch.distributed
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if device is None:
            device = (int(os.environ.get("LOCAL_RANK", self.rank)) % torch.cuda.device_count()
                      if self.world > 1 else torch.cuda.current_device())
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        self.program: Program = compile_program(self.schedule, cfg.mode, n_blocks=model.n_blocks,
                                                world_size=self.world)
        self.hosted = [wp for wp in self.program.workers if self.program.device_of[wp.wid] == self.rank]
        self.dtype = torch.float32 if model.dtype == "fp32" else torch.bfloat16
        self.pd_dtype = nat.PD_F32 if model.dtype == "fp32" else nat.PD_BF16
        self.layered = isinstance(model, (ConvNetSpec, GPTSpec))
        self.is_gpt = isinstance(model, GPTSpec)
        self.geoms = model.geoms() if self.layered else None
        n_params = (model.n_params() if self.layered
                    else sum(a * b for a, b in zip(model.widths[:-1], model.widths[1:])))
        self.init = init or ("host" if n_params <= HOST_INIT_LIMIT else "device")
        self._alloc()
        self._exchange()
        self._build_runtime()
        self.runs = 0
        if self.world == 1 and os.environ.get("PD_GRAPHS", "1") != "0":
            self.set_graph(True)

    # ------------------------------------------------------------------ setup
    KINDS = {"linear": nat.PD_LAYER_LINEAR, "conv": nat.PD_LAYER_CONV3, "embed": nat.PD_LAYER_EMBED,
             "block": nat.PD_LAYER_BLOCK, "head": nat.PD_LAYER_HEAD}

    def _layer_desc(self, x, argmax=None, cols=None, save=None, work=None):
        d = nat.LayerDesc()
        d.kind = self.KINDS[x.kind]
        d.relu, d.pool, d.im2col = int(x.relu), int(x.pool), int(x.im2col)
        d.h, d.w, d.c_in, d.c_out = x.h, x.w, x.c_in, x.c_out
        d.ffn, d.vocab = x.ffn, x.vocab
        if save is not None:
            a = self._parr([p.data_ptr() for p in save])
            self._keep.append(a)
            d.save = ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))
        if work is not None:
            d.work = work.data_ptr()
        if argmax is not None:
            a = self._parr([p.data_ptr() for p in argmax])
            self._keep.append(a)
            d.argmax = ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))
        if cols is not None:
            a = self._parr([p.data_ptr() for p in cols])
            self._keep.append(a)
            d.cols = ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))
        return d

    def _scratch_floats(self, x) -> int:
        self._keep = getattr(self, "_keep", [])
        d = self._layer_desc(x)
        return int(nat.lib().pd_layer_scratch_floats(ctypes.byref(d), self.model.batch))

    def _layer_bytes(self, x, which: str) -> int:
        d = self._layer_desc(x)
        fn = nat.lib().pd_layer_save_bytes if which == "save" else nat.lib().pd_layer_work_bytes
        return int(fn(ctypes.byref(d), self.model.batch))

    @staticmethod
    def _device_init(x, g, dev, torch, layers: int):
        """Seeded on-device initialisation of one layer's (W, b) for models too large for the host."""
        if x.kind in ("conv", "linear"):
            fan = 9 * x.c_in if x.kind == "conv" else x.c_in
            W = torch.randn(*x.w_shape, device=dev, generator=g) * math.sqrt(2.0 / fan)
            if x.im2col:
                W[9 * x.c_in:] = 0.0
            return W, torch.randn(x.c_out, device=dev, generator=g) * 0.01
        W = torch.randn(*x.w_shape, device=dev, generator=g) * 0.02
        d = x.c_in if x.kind != "embed" else x.c_out
        if x.kind == "block":
            f = x.ffn
            flat = W.view(-1)
            scale = 1.0 / math.sqrt(2.0 * layers)
            flat[3 * d * d: 4 * d * d] *= scale
            flat[4 * d * d + f * d:] *= scale
            b = torch.zeros(x.b_numel, device=dev)
            b[5 * d + f: 6 * d + f] = 1.0
            b[7 * d + f: 8 * d + f] = 1.0
            return W, b
        if x.kind == "head":
            return W, torch.cat([torch.ones(d, device=dev), torch.zeros(d, device=dev)])
        return W, torch.zeros(0, device=dev)

    def _alloc(self) -> None:
        torch = _torch()
        dev, dt, m = self.device, self.dtype, self.model
        plan = self.cfg.plan
        if self.init == "host":
            params = init_params_any(m)
            X, T = make_data_any(m)
        else:
            params = None

            def gen(key: int):
                # one stream per global layer (key = layer id) or data tensor (key < 0): every
                # replica of a stage draws identical weights, and the model does not depend on
                # which rank hosts which stage
                return torch.Generator(device=dev).manual_seed(m.seed * 1_000_003 + 1000 + key)
        self.bufs: dict[int, _StageBuf] = {}
        workers = self.program.workers
        for wp in self.hosted:
            st = plan.stages[wp.stage]
            dims = list(m.widths[st.first_layer - 1: st.last_layer + 1])
            b = _StageBuf(wid=wp.wid, stage=wp.stage, dims=dims, ring_depth=wp.ring_depth,
                          init_slot=wp.ring_slot[0], act_depth=wp.act_depth, in_depth=wp.in_depth,
                          grad_depth=wp.grad_depth)
            L = len(dims) - 1
            t = b.tensors
            geo = self.geoms[st.first_layer - 1: st.last_layer] if self.layered else None
            b.geoms = geo
            t["w_master"], t["b_master"], t["w_ring"], t["b_ring"] = [], [], [], []
            for l in range(L):
                din, dout = dims[l], dims[l + 1]
                wshape = geo[l].w_shape if geo else (dout, din)
                nb = geo[l].b_numel if geo else dout
                gl = st.first_layer - 1 + l
                if params is not None:
                    W = torch.from_numpy(params[gl][0]).float().to(dev)
                    bias = torch.from_numpy(params[gl][1]).float().to(dev)
                elif geo:
                    W, bias = self._device_init(geo[l], gen(gl), dev, torch, getattr(m, "layers", 0))
                else:
                    g = gen(gl)
                    W = torch.randn(*wshape, device=dev, generator=g) * math.sqrt(2.0 / din)
                    bias = torch.randn(nb, device=dev, generator=g) * 0.01
                t["w_master"].append(W.contiguous())
                t["b_master"].append(bias.contiguous())
                t["w_ring"].append(torch.empty(b.ring_depth, *wshape, device=dev, dtype=dt))
                t["b_ring"].append(torch.empty(b.ring_depth, nb, device=dev, dtype=torch.float32))
            t["act"] = [torch.empty(b.act_depth, m.batch, dims[l + 1], device=dev, dtype=dt) for l in range(L - 1)]
            if wp.stage == 0 and self.is_gpt:  # int32 token ids
                if params is not None:
                    t["act_in"] = torch.from_numpy(X).to(dev).to(torch.int32).contiguous()
                else:
                    t["act_in"] = torch.randint(0, m.vocab, (m.n_blocks, m.batch, m.seq), device=dev, generator=gen(-1),
                                                dtype=torch.int32)
            elif wp.stage == 0:
                if params is not None:
                    t["act_in"] = torch.from_numpy(X.reshape(m.n_blocks, m.batch, -1)).to(dev).to(dt).contiguous()
                else:
                    t["act_in"] = torch.randn(m.n_blocks, m.batch, dims[0], device=dev, generator=gen(-1)).to(dt)
            else:
                t["act_in"] = torch.zeros(b.in_depth, m.batch, dims[0], device=dev, dtype=dt)
            if wp.stage < plan.num_stages - 1:
                t["grad_in"] = torch.zeros(b.grad_depth, m.batch, dims[-1], device=dev, dtype=dt)
            else:
                t["dz_last"] = torch.empty(b.act_depth, m.batch, dims[-1], device=dev, dtype=dt)
                if self.is_gpt:  # next-token labels and fp32 logits [tokens, padded vocab]
                    if params is not None:
                        t["target"] = torch.from_numpy(T).to(dev).to(torch.int32).contiguous()
                    else:
                        t["target"] = torch.randint(0, m.vocab, (m.n_blocks, m.batch, m.seq), device=dev,
                                                    generator=gen(-2), dtype=torch.int32)
                    t["logits"] = torch.empty(m.tokens, m.vocab_pad, device=dev, dtype=torch.float32)
                elif self.layered:  # cross-entropy: int32 labels and fp32 logits
                    if params is not None:
                        t["target"] = torch.from_numpy(T).to(dev).to(torch.int32).contiguous()
                    else:
                        t["target"] = torch.randint(0, m.classes, (m.n_blocks, m.batch), device=dev, generator=gen(-2),
                                                    dtype=torch.int32)
                    t["logits"] = torch.empty(m.batch, m.classes, device=dev, dtype=torch.float32)
                elif params is not None:
                    t["target"] = torch.from_numpy(T).float().to(dev).contiguous()
                else:
                    t["target"] = torch.randn(m.n_blocks, m.batch, dims[-1], device=dev, generator=gen(-2))
                t["loss"] = torch.zeros(self.cfg.num_minibatches + 1, device=dev, dtype=torch.float32)
            if self.fused_bias(wp.stage):  # fp32 column-sum partials [ceil(B/32), width] per consumed dZ
                nrb = -(-m.batch // 32)
                f32 = dict(device=dev, dtype=torch.float32)
                t["bpart"] = [torch.zeros(nrb, dims[l + 1], **f32) for l in range(L - 1)]
                if wp.stage < plan.num_stages - 1:
                    t["grad_bpart"] = torch.zeros(b.grad_depth, nrb, dims[-1], **f32)
                else:
                    t["dz_bpart"] = torch.zeros(b.act_depth, nrb, dims[-1], **f32)
            tmp_feat = (max(max(x.pre_features for x in geo), max(x.in_features for x in geo)) if geo
                        else max(dims))
            t["tmp"] = [torch.empty(m.batch, tmp_feat, device=dev, dtype=dt) for _ in range(2)]
            if geo:
                t["argmax"] = [torch.empty(b.act_depth, m.batch, x.out_features, device=dev, dtype=torch.uint8)
                               if x.pool else None for x in geo]
                t["cols"] = [torch.empty(b.act_depth, m.batch * x.h * x.w, 64, device=dev, dtype=dt)
                             if x.im2col else None for x in geo]
                scratch = max([self._scratch_floats(x) for x in geo] + [1])
                t["part"] = torch.empty(scratch, device=dev, dtype=torch.float32)
                t["save"] = [[torch.empty(self._layer_bytes(x, "save"), device=dev, dtype=torch.uint8)
                              for _ in range(b.act_depth)] if self._layer_bytes(x, "save") else None for x in geo]
                work = max([self._layer_bytes(x, "work") for x in geo] + [0])
                t["work"] = torch.empty(max(work, 256), device=dev, dtype=torch.uint8)
            t["err"] = torch.zeros(1, device=dev, dtype=torch.int32)
            t["sync"] = torch.zeros(16, device=dev, dtype=torch.int32)
            # receiver-owned inbox flags (zero = nothing delivered yet); used when a producer is remote
            i32 = dict(device=dev, dtype=torch.int32)
            if wp.stage > 0:
                t["act_ready"] = torch.zeros(b.in_depth, **i32)
                t["act_ack"] = torch.zeros(b.in_depth, **i32)
            if wp.stage < plan.num_stages - 1:
                t["grad_ready"] = torch.zeros(b.grad_depth, **i32)
                t["grad_ack"] = torch.zeros(b.grad_depth, **i32)
            if st.replication > 1:  # round-parity gradient buffers + reduction flags
                t["red_grad"] = [[torch.zeros(*t["w_master"][l].shape, device=dev) for _ in range(2)] for l in range(L)]
                t["red_bgrad"] = [[torch.zeros(t["b_master"][l].numel(), device=dev) for _ in range(2)]
                                  for l in range(L)]
                t["red_flags"] = torch.zeros(2, **i32)
                t["red_lflags"] = torch.zeros(2, L, **i32)  # per-layer ready / updated rounds
            self.bufs[wp.wid] = b

    EXPORTS = ("act_in", "grad_in", "act_ready", "act_ack", "grad_ready", "grad_ack", "red_flags", "grad_bpart")

    def fused_bias(self, stage: int) -> bool:
        """Bias gradients fused into the GEMM epilogues (include/pd_b200.h pd_stage_desc.fused_bias):
        bf16 MLP stages with replication 1 and every width a multiple of 32 (PD_FUSED_BIAS=0: off)."""
        if self.layered or self.model.dtype != "bf16" or os.environ.get("PD_FUSED_BIAS", "1") == "0":
            return False
        st = self.cfg.plan.stages[stage]
        widths = self.model.widths[st.first_layer - 1: st.last_layer + 1]
        return st.replication == 1 and all(w % 32 == 0 for w in widths)

    def _exchange(self) -> None:
        """Publish CUDA IPC handles of this rank's inboxes, flags and reduction buffers."""
        self._remote: dict[int, dict] = {}
        if self.world == 1:
            return
        torch = _torch()

        def export(t):
            h, off = nat.ipc_export(t)
            slot = t[0].numel() * t.element_size() if t.dim() > 1 else t.element_size()
            return (h, off, slot, t.shape[0])

        mine = {}
        for b in self.bufs.values():
            ent = {}
            for name in self.EXPORTS:
                if name == "act_in" and b.stage == 0:
                    continue
                if name in b.tensors:
                    ent[name] = export(b.tensors[name])
            if "red_grad" in b.tensors:
                ent["red_grad"] = [[export(g) for g in pair] for pair in b.tensors["red_grad"]]
                ent["red_bgrad"] = [[export(g) for g in pair] for pair in b.tensors["red_bgrad"]]
                ent["w_master"] = [export(w) for w in b.tensors["w_master"]]
                ent["b_master"] = [export(x) for x in b.tensors["b_master"]]
                ent["red_lflags"] = export(b.tensors["red_lflags"])
            mine[b.wid] = ent
        gathered = [None] * self.world
        torch.distributed.all_gather_object(gathered, mine, group=self.group)
        for part in gathered:
            for wid, ent in part.items():
                if self.program.device_of[wid] != self.rank:
                    self._remote[wid] = ent

    def _addr(self, wid: int, name: str) -> list[int]:
        """Per-slot device addresses of worker wid's buffer `name` (local or peer-mapped)."""
        if self.program.device_of[wid] == self.rank:
            t = self.bufs[wid].tensors.get(name)
            if t is None:
                return []
            return [x.data_ptr() for x in t] if t.dim() > 1 else [t.data_ptr() + 4 * k for k in range(t.shape[0])]
        ent = self._remote[wid].get(name)
        if ent is None:
            return []
        h, off, slot, count = ent
        base = nat.ipc_import(h, off)
        return [base + k * slot for k in range(count)]

    def _list_addrs(self, wid: int, name: str) -> list[int]:
        """Addresses of worker wid's per-layer tensor list `name` (local or peer-mapped)."""
        if self.program.device_of[wid] == self.rank:
            return [x.data_ptr() for x in self.bufs[wid].tensors[name]]
        return [nat.ipc_import(h, off) for (h, off, _s, _c) in self._remote[wid][name]]

    def _red_addrs(self, wid: int, name: str) -> list[int]:
        if self.program.device_of[wid] == self.rank:
            return [g.data_ptr() for pair in self.bufs[wid].tensors[name] for g in pair]
        return [nat.ipc_import(h, off) for pair in self._remote[wid][name] for (h, off, _s, _c) in pair]

    @staticmethod
    def _parr(ptrs) -> ctypes.Array:
        return (ctypes.c_void_p * max(1, len(ptrs)))(*[int(p) for p in ptrs])

    def _build_runtime(self) -> None:
        L = nat.lib()
        plan = self.cfg.plan
        n = plan.num_stages
        rt = ctypes.c_void_p()
        nat.check(L.pd_rt_create(self.device.index, ctypes.byref(rt)), "pd_rt_create")
        self._rt = rt
        self._keep = getattr(self, "_keep", [])

        def arr(ptrs):
            a = self._parr(ptrs)
            self._keep.append(a)
            return ctypes.cast(a, ctypes.POINTER(ctypes.c_void_p))

        def iptr(addrs):
            return addrs[0] if addrs else None

        # views of every worker the hosted ones talk to (all workers: cheap, and replicas need them)
        for wp in self.program.workers:
            wid = wp.wid
            v = nat.WorkerView()
            v.worker = wid
            v.remote = int(self.program.device_of[wid] != self.rank)
            v.in_depth, v.grad_depth = wp.in_depth, wp.grad_depth
            st = plan.stages[wp.stage]
            v.n_layers = st.last_layer - st.first_layer + 1
            if wp.stage > 0:
                v.act_in = arr(self._addr(wid, "act_in"))
                v.act_ready, v.act_ack = iptr(self._addr(wid, "act_ready")), iptr(self._addr(wid, "act_ack"))
            if wp.stage < n - 1:
                v.grad_in = arr(self._addr(wid, "grad_in"))
                v.grad_ready, v.grad_ack = iptr(self._addr(wid, "grad_ready")), iptr(self._addr(wid, "grad_ack"))
            if wp.stage < n - 1 and self.fused_bias(wp.stage):
                v.fused_bias = 1
                v.grad_bpart = arr(self._addr(wid, "grad_bpart"))
            if st.replication > 1:
                v.red_grad = arr(self._red_addrs(wid, "red_grad"))
                v.red_bgrad = arr(self._red_addrs(wid, "red_bgrad"))
                fl = self._addr(wid, "red_flags")
                v.red_ready, v.red_done = fl[0], fl[1]
                v.w_master = arr(self._list_addrs(wid, "w_master"))
                v.b_master = arr(self._list_addrs(wid, "b_master"))
                lf = self._addr(wid, "red_lflags")  # rows: ready, updated
                v.red_lready, v.red_lupd = lf[0], lf[1]
            self._keep.append(v)
            nat.check(L.pd_rt_add_view(rt, ctypes.byref(v)), "pd_rt_add_view")

        reps = [st.replication for st in plan.stages]
        for b in self.bufs.values():
            t = b.tensors
            wp = self.program.workers[b.wid]
            nl = len(b.dims) - 1
            dims = (ctypes.c_int64 * len(b.dims))(*b.dims)
            self._keep.append(dims)
            is_first, is_last = b.stage == 0, b.stage == n - 1
            d = nat.StageDesc()
            d.worker, d.stage, d.replica, d.rep = b.wid, b.stage, wp.replica, reps[b.stage]
            d.first_worker = self.schedule.worker_id(b.stage, 0)
            d.n_layers, d.dims, d.batch, d.dtype = nl, dims, self.model.batch, self.pd_dtype
            d.is_first, d.is_last, d.relu_last = int(is_first), int(is_last), int(not is_last)
            d.ring_depth, d.init_slot, d.act_depth = b.ring_depth, b.init_slot, b.act_depth
            d.in_depth, d.grad_depth, d.lr = b.in_depth, b.grad_depth, self.model.lr
            d.n_data_blocks = self.model.n_blocks
            # does any producer of my inboxes live in another process?
            if not is_first:
                prev = [self.schedule.worker_id(b.stage - 1, r) for r in range(reps[b.stage - 1])]
                d.remote_prev = int(any(self.program.device_of[w] != self.rank for w in prev))
            if not is_last:
                nxt = [self.schedule.worker_id(b.stage + 1, r) for r in range(reps[b.stage + 1])]
                d.remote_next = int(any(self.program.device_of[w] != self.rank for w in nxt))
            d.w_master = arr([w.data_ptr() for w in t["w_master"]])
            d.b_master = arr([x.data_ptr() for x in t["b_master"]])
            d.w_ring = arr([t["w_ring"][l][k].data_ptr() for l in range(nl) for k in range(b.ring_depth)])
            d.b_ring = arr([t["b_ring"][l][k].data_ptr() for l in range(nl) for k in range(b.ring_depth)])
            d.act = arr([t["act"][l][k].data_ptr() for l in range(nl - 1) for k in range(b.act_depth)])
            d.act_in = arr([x.data_ptr() for x in t["act_in"]])
            if not is_last:
                d.grad_in = arr([x.data_ptr() for x in t["grad_in"]])
                d.grad_ready, d.grad_ack = t["grad_ready"].data_ptr(), t["grad_ack"].data_ptr()
            else:
                d.dz_last = arr([x.data_ptr() for x in t["dz_last"]])
                d.target = arr([x.data_ptr() for x in t["target"]])
                d.loss = t["loss"].data_ptr()
            if not is_first:
                d.act_ready, d.act_ack = t["act_ready"].data_ptr(), t["act_ack"].data_ptr()
            if d.rep > 1:
                d.red_grad = arr([g.data_ptr() for pair in t["red_grad"] for g in pair])
                d.red_bgrad = arr([g.data_ptr() for pair in t["red_bgrad"] for g in pair])
                d.red_ready, d.red_done = t["red_flags"].data_ptr(), t["red_flags"].data_ptr() + 4
                d.red_lready, d.red_lupd = t["red_lflags"][0].data_ptr(), t["red_lflags"][1].data_ptr()
            d.tmp[0], d.tmp[1] = t["tmp"][0].data_ptr(), t["tmp"][1].data_ptr()
            d.err_word = t["err"].data_ptr()
            d.sync = t["sync"].data_ptr()
            if self.fused_bias(b.stage):
                d.fused_bias = 1
                d.bpart = arr([x.data_ptr() for x in t["bpart"]])
                if is_last:
                    d.dz_bpart = arr([x.data_ptr() for x in t["dz_bpart"]])
                else:
                    d.grad_bpart = arr([x.data_ptr() for x in t["grad_bpart"]])
            if self.layered:
                descs = (nat.LayerDesc * nl)(*[self._layer_desc(x, t["argmax"][l], t["cols"][l], t["save"][l],
                                                                t["work"]) for l, x in enumerate(b.geoms)])
                self._keep.append(descs)
                d.layers = ctypes.cast(descs, ctypes.POINTER(nat.LayerDesc))
                d.part = t["part"].data_ptr()
                if is_last:
                    d.loss_kind = nat.PD_LOSS_CE
                    d.logits = t["logits"].data_ptr()
            b.desc = d
            nat.check(L.pd_rt_add_stage(rt, ctypes.byref(d)), "pd_rt_add_stage")
        prog = np.ascontiguousarray(self.program.items_for_rank(self.rank))
        self._prog = prog
        nat.check(L.pd_rt_load_program(rt, prog.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), prog.shape[0]),
                  "pd_rt_load_program")
        # device pass records of traced runs: timestamps, the version tag each pass read, bytes
        # stored into peer inboxes, commits (include/pd_b200.h pd_rt_set_records)
        torch = _torch()
        self._rec = torch.zeros((1 + prog.shape[0]) * nat.REC_WIDTH, device=self.device, dtype=torch.int64)
        self._tags = torch.full((64 * max(1, len(self.bufs)),), -1, device=self.device, dtype=torch.int32)
        nat.check(L.pd_rt_set_records(rt, self._rec.data_ptr(), prog.shape[0], self._tags.data_ptr()),
                  "pd_rt_set_records")

    # ------------------------------------------------------------------ execution
    def step(self, stream=None, trace: bool = False) -> None:
        """Enqueue one execution of the whole schedule behind ``stream`` (async)."""
        torch = _torch()
        s = stream or torch.cuda.current_stream(self.device)
        nat.check(nat.lib().pd_rt_run(self._rt, int(s.cuda_stream), int(trace)), "pd_rt_run")
        self.runs += 1
        self._traced = trace

    def load_inputs(self, X_host, T_host, stream=None) -> None:
        """Copy host (pinned) input / target blocks into the resident data buffers (e2e path)."""
        torch = _torch()
        s = stream or torch.cuda.current_stream(self.device)
        # Replicas of a stage hosted here hold the same resident blocks: one host->device copy,
        # then device-to-device copies to the other replicas' buffers.
        with torch.cuda.stream(s):
            first = {}
            for b in self.bufs.values():
                for want, src, key in ((0, X_host, "act_in"), (self.cfg.plan.num_stages - 1, T_host, "target")):
                    if b.stage != want or src is None:
                        continue
                    dst = b.tensors[key]
                    if key in first and first[key].device == dst.device:
                        dst.copy_(first[key], non_blocking=True)
                    else:
                        dst.copy_(src, non_blocking=True)
                        first.setdefault(key, dst)

    def hosts_stage(self, s: int) -> bool:
        return any(b.stage == s for b in self.bufs.values())

    def losses(self) -> list[float] | None:
        last = [b for b in self.bufs.values() if b.stage == self.cfg.plan.num_stages - 1]
        return last[0].tensors["loss"][1:].float().cpu().tolist() if last else None

    def loss_tensor(self):
        last = [b for b in self.bufs.values() if b.stage == self.cfg.plan.num_stages - 1]
        return last[0].tensors["loss"] if last else None

    def weights(self) -> dict[int, tuple[np.ndarray, np.ndarray]]:
        """Final fp32 (W, b) per global 1-based layer id."""
        out = {}
        plan = self.cfg.plan
        for b in self.bufs.values():
            st = plan.stages[b.stage]
            for l, (W, bias) in enumerate(zip(b.tensors["w_master"], b.tensors["b_master"])):
                out[st.first_layer + l] = (W.cpu().numpy().astype(np.float64), bias.cpu().numpy().astype(np.float64))
        return out

    # ------------------------------------------------------------------ checkpoints
    def save_checkpoint(self, directory) -> list[str]:
        """Per-stage weight checkpoint, written by each process for the workers it hosts without
        any global coordination: one .npz per worker with the fp32 master
        weights and biases of its layers and the number of completed runs."""
        import pathlib

        torch = _torch()
        torch.cuda.synchronize(self.device)
        out = pathlib.Path(directory)
        out.mkdir(parents=True, exist_ok=True)
        paths = []
        for b in self.bufs.values():
            arrays = {}
            for l, (W, bias) in enumerate(zip(b.tensors["w_master"], b.tensors["b_master"])):
                arrays[f"W{l}"] = W.cpu().numpy()
                arrays[f"b{l}"] = bias.cpu().numpy()
            path = out / f"stage{b.stage:02d}_worker{b.wid:02d}.npz"
            np.savez(path, runs=np.int64(self.runs), **arrays)
            paths.append(str(path))
        return paths

    def load_checkpoint(self, directory) -> None:
        """Restore the hosted workers' master weights from ``save_checkpoint`` files (the next run
        refreshes version 0 of every ring from them)."""
        import pathlib

        torch = _torch()
        src = pathlib.Path(directory)
        for b in self.bufs.values():
            path = src / f"stage{b.stage:02d}_worker{b.wid:02d}.npz"
            if not path.exists():
                raise ValidationError(f"no checkpoint for worker {b.wid} (stage {b.stage}) in {src}")
            data = np.load(path)
            for l, (W, bias) in enumerate(zip(b.tensors["w_master"], b.tensors["b_master"])):
                w, bb = data[f"W{l}"], data[f"b{l}"]
                if w.shape != tuple(W.shape) or bb.shape != tuple(bias.shape):
                    raise ValidationError(f"checkpoint {path.name}: layer {l} shape mismatch")
                W.copy_(torch.from_numpy(w).to(W.device))
                bias.copy_(torch.from_numpy(bb).to(bias.device))
        torch.cuda.synchronize(self.device)

    def set_graph(self, on: bool) -> None:
        """Replay single-process runs from a captured CUDA graph (the first eligible run captures)."""
        nat.check(nat.lib().pd_rt_set_graph(self._rt, int(on)), "pd_rt_set_graph")

    def set_serial(self, on: bool) -> None:
        """Issue every hosted stage on one stream in program order (single-GPU timing mode)."""
        nat.check(nat.lib().pd_rt_set_serial(self._rt, int(on)), "pd_rt_set_serial")

    def kernel_timing(self, on: bool) -> None:
        """Per-GEMM CUDA events on the launching stage streams (resets the counters)."""
        nat.check(nat.lib().pd_rt_kernel_timing(self._rt, int(on)), "pd_rt_kernel_timing")

    KERNEL_CLASSES = ("fwd", "dgrad", "wgrad_sgd", "attention", "layernorm", "loss", "update", "other")

    def kernel_stats(self, worker: int = -1) -> dict:
        """{class: launches, avg ms, algorithmic flops per launch, total ms} per kernel class
        (GEMM passes fwd / dgrad / wgrad_sgd, then attention, layernorm, loss, update, other),
        over all hosted workers or one (``worker``)."""
        n = len(self.KERNEL_CLASSES)
        buf = (ctypes.c_double * (3 * n))()
        nat.check(nat.lib().pd_rt_kernel_stats(self._rt, worker, buf, n), "pd_rt_kernel_stats")
        out = {}
        for i, name in enumerate(self.KERNEL_CLASSES):
            n, ms, fl = buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]
            if n:
                out[name] = {"launches": int(n), "avg_ms": ms / n, "flops_per_launch": fl / n, "total_ms": ms,
                             "total_flops": fl}
        return out

    def launch_count(self) -> int:
        v = ctypes.c_int64(0)
        nat.check(nat.lib().pd_rt_launch_count(self._rt, ctypes.byref(v)), "pd_rt_launch_count")
        return int(v.value)

    def records(self) -> list[tuple[int, float, float]]:
        L = nat.lib()
        n = self._prog.shape[0]
        recs = (nat.Record * n)()
        got = ctypes.c_int(0)
        nat.check(L.pd_rt_records(self._rt, recs, n, ctypes.byref(got)), "pd_rt_records")
        err = [int(b.tensors["err"].item()) for b in self.bufs.values()]
        if any(err):
            raise SimulationError(f"flag wait timed out (values {err}): a neighbour never delivered")
        return [(r.item, r.t_start_ms, r.t_end_ms) for r in recs[: got.value]]

    def device_records(self) -> tuple[int, list[tuple]]:
        """(run-start %globaltimer ns, [(program row, t_start ns, t_end ns, version at start, version at
        end, peer bytes stored, committed version)]) of the last traced run, as the device wrote them."""
        self.records()  # raises SimulationError if a flag wait timed out
        rec = self._rec.cpu().numpy().reshape(-1, nat.REC_WIDTH)
        rows = [(self._prog[i], *[int(x) for x in rec[1 + i, :6]]) for i in range(self._prog.shape[0])]
        return int(rec[0, 0]), rows

    def trace(self, t0_ns: int | None = None) -> list[TraceEvent]:
        """Passes of the last traced run in seconds since ``t0_ns`` (default: this rank's run start),
        with the weight version each pass observed on the device."""
        start, rows = self.device_records()
        base = start if t0_ns is None else t0_ns
        evs = []
        for row, t0, t1, v0, _v1, _b, _c in rows:
            if row[nat.IT_OP] == 2:  # replica reduction: part of the backward round, not a pass
                continue
            evs.append(TraceEvent(
                time_start=(t0 - base) * 1e-9, time_end=(t1 - base) * 1e-9, worker=int(row[nat.IT_WORKER]),
                minibatch=int(row[nat.IT_MB]), stage=int(row[nat.IT_STAGE]),
                direction=Direction.FORWARD if row[nat.IT_OP] == 0 else Direction.BACKWARD,
                version_used=v0,
            ))
        return evs

    def device_ledger(self, rows) -> VersionLedger:
        """The reference's VersionLedger (simulator.py:69-99, recorded at pass start :256-264) rebuilt
        from the version tags the device passes read; a slot overwritten under a pass (tag at the end
        differs from the start) is a protocol failure and raises SimulationError."""
        plan = self.cfg.plan
        led = VersionLedger(n_stages=plan.num_stages, stage_replications=tuple(st.replication for st in plan.stages))
        for s in range(plan.num_stages):
            led.latest[s] = 0
        for row, _t0, _t1, v0, v1, _b, commit in sorted(rows, key=lambda r: r[1]):
            op, s, mb = int(row[nat.IT_OP]), int(row[nat.IT_STAGE]), int(row[nat.IT_MB])
            if commit >= 0:
                led.latest[s] = max(led.latest[s], commit)
            if op == 2:
                continue
            d = Direction.FORWARD if op == 0 else Direction.BACKWARD
            if v0 < 0 or v0 != v1:
                raise SimulationError(f"worker {int(row[nat.IT_WORKER])} (stage {s}): ring slot {int(row[nat.IT_WSLOT])} "
                                      f"held version {v0} at the start of {d.value} of minibatch {mb} and {v1} at its end")
            led.record(s, mb, d, v0)
        return led

    def comm_bytes(self) -> float:
        """The reference's communication count (simulator.py:288 and :320-321) over the executed program:
        each forward crossing adds the boundary activation bytes, each backward crossing the same bytes,
        and each backward of a replicated stage (rep - 1) x the stage's weight bytes.  With a
        CostContext the sizes are the profile's (activation_elems, prefix_W_bytes, hw.bytes_per_elem)
        exactly as the reference computes them; without one they are the model's own."""
        m, plan, ctx = self.model, self.cfg.plan, self.ctx
        n = plan.num_stages
        if ctx is not None:
            bpe = ctx.hw.bytes_per_elem
            act = [ctx.profile.layers[st.last_layer - 1].activation_elems * bpe for st in plan.stages[:-1]]
            wb = [ctx.prefix_W_bytes[st.last_layer] - ctx.prefix_W_bytes[st.first_layer - 1] for st in plan.stages]
        else:
            bpe = m.bytes_per_elem
            if self.layered:
                act = [m.batch * self.geoms[st.last_layer - 1].out_features * bpe for st in plan.stages[:-1]]
                wb = [sum(x.w_numel + x.b_numel for x in self.geoms[st.first_layer - 1: st.last_layer]) * bpe
                      for st in plan.stages]
            else:
                act = [m.batch * m.widths[st.last_layer] * bpe for st in plan.stages[:-1]]
                wb = [sum(a * b + b for a, b in zip(m.widths[st.first_layer - 1: st.last_layer],
                                                    m.widths[st.first_layer: st.last_layer + 1])) * bpe
                      for st in plan.stages]
        total = 0.0
        for row in self._prog:
            op, s = int(row[nat.IT_OP]), int(row[nat.IT_STAGE])
            if op == 0 and s < n - 1:
                total += act[s]
            if op == 1:
                if plan.stages[s].replication > 1:
                    total += (plan.stages[s].replication - 1) * wb[s]
                if s > 0:
                    total += act[s - 1]
        return float(total)

    def gpu_utilization(self, trace, rank: int | None = None, whole_run: bool = False) -> float:
        """Fraction of the steady window during which GPU `rank` runs at least one pass.

        The reference's per-worker utilisation (simulator.py:379-385) is kept in the report;
        with several stages per GPU the device-level bubble is 1 - (union of their busy time).
        whole_run: over the GPU's own first pass start .. last pass end (fill and drain included).
        """
        from .ledger import steady_window

        rank = self.rank if rank is None else rank
        if whole_run:
            mine = [ev for ev in trace if self.program.device_of[ev.worker] == rank]
            if not mine:
                return 0.0
            t1, t2 = min(ev.time_start for ev in mine), max(ev.time_end for ev in mine)
        else:
            k1, k2 = steady_window(self.cfg, self.cfg.plan.num_stages, self.cfg.plan.stages[0].replication)
            done = {ev.minibatch: ev.time_end for ev in trace if ev.stage == 0 and ev.direction is Direction.BACKWARD}
            t1, t2 = done[k1], done[k2]
        iv = sorted((max(ev.time_start, t1), min(ev.time_end, t2)) for ev in trace
                    if self.program.device_of[ev.worker] == rank and ev.time_end > t1 and ev.time_start < t2)
        busy, cur_lo, cur_hi = 0.0, None, None
        for lo, hi in iv:
            if cur_hi is None or lo > cur_hi:
                if cur_hi is not None:
                    busy += cur_hi - cur_lo
                cur_lo, cur_hi = lo, hi
            else:
                cur_hi = max(cur_hi, hi)
        if cur_hi is not None:
            busy += cur_hi - cur_lo
        return busy / (t2 - t1)

    def result(self) -> SimResult:
        """SimResult of the last run; with several ranks every rank returns the merged result."""
        torch = _torch()
        torch.cuda.synchronize(self.device)
        traced = getattr(self, "_traced", False)
        start, rows = self.device_records() if traced else (0, [])
        # bytes the replicas' sharded reductions read from each other (counted by the kernels)
        red = int(self._rec[1].item()) if traced else 0  # row 0, field 1 (include/pd_b200.h)
        losses, weights, comm = self.losses(), self.weights(), self.comm_bytes()
        if self.world > 1:
            parts = [None] * self.world
            torch.distributed.all_gather_object(parts, (start, rows, losses, weights, comm, red), group=self.group)
            red = sum(p[5] for p in parts)
            # one time base for the merged trace: the earliest run start over the ranks (every rank
            # stamps %globaltimer, a node-wide clock, so the ranks' events line up)
            start = min(p[0] for p in parts) if traced else 0
            rows = [r for p in parts for r in p[1]]
            losses = next((p[2] for p in parts if p[2] is not None), None)
            weights = {k: v for p in parts for k, v in p[3].items()}
            comm = parts[0][4]  # the program-wide count is the same on every rank
        trace, ledger, p2p, p2p_by = [], self.program.ledger, 0, {}
        if traced:
            trace = sorted((TraceEvent(time_start=(t0 - start) * 1e-9, time_end=(t1 - start) * 1e-9,
                                       worker=int(row[nat.IT_WORKER]), minibatch=int(row[nat.IT_MB]),
                                       stage=int(row[nat.IT_STAGE]),
                                       direction=Direction.FORWARD if row[nat.IT_OP] == 0 else Direction.BACKWARD,
                                       version_used=v0)
                            for row, t0, t1, v0, _v1, _b, _c in rows if row[nat.IT_OP] != 2),
                           key=lambda e: (e.time_start, e.worker))
            ledger = self.device_ledger(rows)
            p2p = sum(b for *_r, b, _c in rows)
            for row, *_x, b, _c in rows:
                if b:
                    k = int(row[nat.IT_STAGE]) - (0 if row[nat.IT_OP] == 0 else 1)
                    p2p_by[k] = p2p_by.get(k, 0) + int(b)
        report = build_report(self.cfg, trace, len(self.schedule.workers), comm) if trace else None
        bubble, gpu_util, bubble_run = None, None, None
        if report is not None:
            gpu_util = sum(self.gpu_utilization(trace, r) for r in range(self.world)) / self.world
            bubble = 1.0 - gpu_util
        if trace:
            bubble_run = 1.0 - sum(self.gpu_utilization(trace, r, whole_run=True) for r in range(self.world)) / self.world
        return SimResult(report=report, ledger=ledger, trace=trace, losses=losses, weights=weights,
                         extras={"bubble_fraction": bubble, "gpu_utilization": gpu_util,
                                 "bubble_fraction_whole_run": bubble_run,
                                 "ledger_source": "device" if traced else "program",
                                 "p2p_bytes_measured": p2p if traced else None,
                                 "p2p_bytes_by_boundary": p2p_by if traced else None,
                                 "replica_reduce_bytes_measured": red if traced else None,
                                 "ring_depths": {b.stage: b.ring_depth for b in self.bufs.values()},
                                 "device_of_worker": list(self.program.device_of),
                                 "device": str(self.device), "runs": self.runs})

    def close(self) -> None:
        if getattr(self, "_rt", None) is not None:
            nat.lib().pd_rt_destroy(self._rt)
            self._rt = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def run(cfg: SimConfig, ctx=None, schedule: Schedule | None = None, *, model: MLPSpec, trace: bool = True,
        device: int | None = None, init: str | None = None) -> SimResult:
    """Execute ``cfg`` on the GPU and return the reference's ``SimResult`` shape (simulator.py:401-411)."""
    ex = Executor(cfg, ctx, schedule, model=model, device=device, init=init)
    try:
        ex.step(trace=trace)
        return ex.result()
    finally:
        ex.close()
