"""Python front end (glue only) over the native Reducer.

Mirrors the paper's Python layer (§4.1: constructor
knobs ``process_group`` / ``bucket_cap_mb``, the ``no_sync`` context manager)
for the gradient path only.  PyTorch is used for device memory (symmetric
memory for the peer-mapped bucket storage), streams, the process group that
carries the NCCL unique id, and the autograd hook mechanism
(``register_post_accumulate_grad_hook``, the AccumulateGrad post-hook of
P:L186 / L306).  Every step of the synchronization runs in
``libb200ddp.so``: this module only marshals arguments.
"""

from __future__ import annotations

import contextlib
import dataclasses
from typing import Dict, Iterable, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _lib as L

MIB = 1 << 20
_DTYPES = {torch.float32: L.FP32, torch.bfloat16: L.BF16, "fp32": L.FP32, "bf16": L.BF16}


def _group_info(group) -> tuple:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _broadcast_id(nccl_id: Optional[bytes], rank: int, group, device) -> bytes:
    """Rank 0's NCCL unique id to every rank through the torch process group
    (PAPER.md L278 rendezvous).  Works with gloo (CPU) and nccl (CUDA)."""
    backend = dist.get_backend(group)
    dev = torch.device("cpu") if backend == "gloo" else device
    t = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_id), dtype=torch.uint8))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().tolist())


class GradReducer:
    """One native Reducer context bound to the current CUDA device.

    ``numels``: per-parameter element counts in registration order.
    ``options``: {key: value} of ``_lib.OPT_*`` applied before binding (must
    be identical on every rank).
    """

    def __init__(self, numels: Sequence[int], dtype="fp32", bucket_cap_bytes: int = 25 * MIB,
                 group=None, device: Optional[torch.device] = None,
                 options: Optional[Dict[int, int]] = None, comm_stream: Optional[torch.cuda.Stream] = None,
                 scan_order: Optional[Sequence[int]] = None):
        self.rank, self.world = _group_info(group)
        self.group = group
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.numels = [int(n) for n in numels]
        self.dtype = _DTYPES[dtype]
        self.ctx = L.ddp_create_ordered(self.numels, scan_order, self.dtype, bucket_cap_bytes, self.world, self.rank)
        try:
            for k, v in (options or {}).items():
                L.ddp_set_option(self.ctx, k, v)
            self.storage_bytes = L.ddp_storage_bytes(self.ctx)
            low = bool((options or {}).get(L.OPT_LOW_PRIORITY, 1))   # the library's default
            self.comm_stream = comm_stream or torch.cuda.Stream(device=self.device, priority=0 if low else -1)
            nccl_id = L.ddp_get_nccl_id() if self.rank == 0 else None
            mc = 0
            if self.world > 1:
                nccl_id = _broadcast_id(nccl_id, self.rank, group, self.device)
                self._storage, peers, mc = self._symmetric_storage()
                want = (options or {}).get(L.OPT_MULTICAST)
                ok = self._all_agree(mc != 0)          # NVLS only if every rank has multicast
                if want and not ok:
                    raise RuntimeError("OPT_MULTICAST requested but NVSwitch multicast is unavailable")
                if want is None and ok:
                    L.ddp_set_option(self.ctx, L.OPT_MULTICAST, 1)
                    assert L.ddp_storage_bytes(self.ctx) <= self.storage_bytes
                if not L.ddp_get_option(self.ctx, L.OPT_MULTICAST):
                    mc = 0
            else:
                self._storage = torch.empty(self.storage_bytes, dtype=torch.uint8, device=self.device)
                peers = [self._storage.data_ptr()]
            self.multicast = bool(mc)
            L.ddp_bind_device(self.ctx, self.device.index, nccl_id, self.comm_stream.cuda_stream, peers, mc)
        except Exception:
            L.ddp_destroy(self.ctx)
            self.ctx = None
            raise

    def _symmetric_storage(self):
        import torch.distributed._symmetric_memory as symm_mem
        t = symm_mem.empty(self.storage_bytes, dtype=torch.uint8, device=self.device)
        h = symm_mem.rendezvous(t, self.group if self.group is not None else dist.group.WORLD)
        base = h.buffer_ptrs[self.rank]
        delta = t.data_ptr() - base
        self._symm_handle = h
        mc = 0
        if getattr(h, "has_multicast_support", False) and h.multicast_ptr:
            mc = int(h.multicast_ptr) + delta
        return t, [int(p) + delta for p in h.buffer_ptrs], mc

    def _all_agree(self, flag: bool) -> bool:
        t = torch.tensor([1 if flag else 0], dtype=torch.int32, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return bool(t.item())

    # ---- introspection -------------------------------------------------------
    @property
    def num_buckets(self) -> int:
        return L.ddp_num_buckets(self.ctx)

    def bucket_algos(self) -> List[str]:
        return [L.ALGO_NAMES[L.ddp_bucket_algo(self.ctx, b)] for b in range(self.num_buckets)]

    def bucket_numels(self) -> List[int]:
        return [L.ddp_bucket_info(self.ctx, b)[0] for b in range(self.num_buckets)]

    # ---- hot path --------------------------------------------------------------
    def grad_ready(self, param_idx: int, grad: torch.Tensor, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.ddp_grad_ready(self.ctx, param_idx, grad.data_ptr(), s.cuda_stream)

    def grads_ready(self, batch: "L.ReadyBatch", stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.ddp_grads_ready(self.ctx, batch, s.cuda_stream)

    def mark_unused(self, param_idx: int, grad: Optional[torch.Tensor],
                    stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.ddp_mark_unused(self.ctx, param_idx, 0 if grad is None else grad.data_ptr(), s.cuda_stream)

    def ready_order(self) -> List[int]:
        return L.ddp_ready_order(self.ctx)

    def broadcast(self, tensors: Sequence[torch.Tensor], root: int = 0,
                  stream: Optional[torch.cuda.Stream] = None):
        """In-place broadcast of contiguous device tensors from `root` (one NCCL group)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.ddp_broadcast(self.ctx, [t.data_ptr() for t in tensors],
                        [t.numel() * t.element_size() for t in tensors], root, s.cuda_stream)

    def global_unused(self) -> List[bool]:
        return L.ddp_global_unused(self.ctx, len(self.numels))

    def finalize(self, stream: Optional[torch.cuda.Stream] = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        L.ddp_finalize_backward(self.ctx, s.cuda_stream)

    @contextlib.contextmanager
    def no_sync(self):
        L.ddp_no_sync_begin(self.ctx)
        try:
            yield
        finally:
            L.ddp_no_sync_end(self.ctx)

    def set_option(self, key: int, value: int):
        L.ddp_set_option(self.ctx, key, value)

    def profile_read(self):
        return L.ddp_profile_read(self.ctx)

    def check_errors(self):
        L.ddp_check_device_errors(self.ctx)

    def close(self):
        if self.ctx:
            L.ddp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dense(t: torch.Tensor) -> bool:
    """t covers exactly numel consecutive elements from its data pointer (any
    dimension order: contiguous, channels_last, ...).  The average is elementwise,
    so such a gradient is synchronized as a flat array; every rank's replica has
    the same layout (same model, same memory format), hence the same element order."""
    if t.is_contiguous():
        return True
    dims = sorted((st, sz) for st, sz in zip(t.stride(), t.size()) if sz != 1)
    expect = 1
    for st, sz in dims:
        if st != expect:
            return False
        expect *= sz
    return True


def _tensors(x):
    """Every tensor inside a (nested) forward output: tensors, sequences,
    mappings and dataclass-like objects (e.g. HF ModelOutput)."""
    if isinstance(x, torch.Tensor):
        yield x
    elif isinstance(x, dict):
        for v in x.values():
            yield from _tensors(v)
    elif isinstance(x, (list, tuple)):
        for v in x:
            yield from _tensors(v)
    elif dataclasses.is_dataclass(x) and not isinstance(x, type):
        for f in dataclasses.fields(x):
            yield from _tensors(getattr(x, f.name))


class DistributedDataParallel(torch.nn.Module):
    """Wraps a module; gradients of its parameters are bucketed, averaged across
    the process group and written back into ``.grad`` during backward.

    Constructor: ``process_group``, ``bucket_cap_mb``
    (default 25, read as MiB, C-5).  ``broadcast_parameters``: rank 0's
    parameters (and buffers) are copied to every rank at construction (Alg. 1
    L214-L215) through the library's communicator (``ddp_broadcast``).
    ``find_unused_parameters``: Alg. 1 forward L224-L225.
    ``rebuild_buckets``: gradient order prediction — after the
    first synced backward, rank 0's traced ready order is broadcast and the
    parameter-to-bucket map is rebuilt from it once, at the next forward.
    ``gradient_as_bucket_view`` (§8(f) N-3, zero-copy): after the first synced
    backward every ``.grad`` is a view of its bucket slot in the library's
    storage, so the buckets are averaged in place (``DDP_OPT_GRAD_VIEW``: no
    pack / unpack).  Clear gradients with ``zero_grad(set_to_none=False)`` to
    keep the views; a re-created ``.grad`` is copied into its slot and the view
    re-attached at the end of the pass.  The buckets synced beside backward then
    use the copy engines in place (CE at world 2, CE2 wider) under the fp32 overlap
    policy, the last bucket (and every bucket under the bf16 policy) the fused
    two-shot in place (include/b200ddp.h, DDP_OPT_GRAD_VIEW).
    The exchange policy for hook-driven passes is ``DDP_OPT_PREFER_OVERLAP``:
    1 (copy engines) for fp32 models, 2 (SM kernels) otherwise, unless
    ``options`` sets it.
    """

    def __init__(self, module: torch.nn.Module, process_group=None, bucket_cap_mb: float = 25,
                 broadcast_parameters: bool = True, options: Optional[Dict[int, int]] = None,
                 find_unused_parameters: bool = False, rebuild_buckets: bool = False,
                 gradient_as_bucket_view: bool = False):
        super().__init__()
        if gradient_as_bucket_view and find_unused_parameters:
            raise ValueError("gradient_as_bucket_view with find_unused_parameters is not supported")
        gradient_as_bucket_view = gradient_as_bucket_view or bool((options or {}).get(L.OPT_GRAD_VIEW))
        self.gradient_as_bucket_view = gradient_as_bucket_view
        self.find_unused_parameters = find_unused_parameters
        self.process_group = process_group
        self.bucket_cap_mb = bucket_cap_mb
        self._rebuild = rebuild_buckets
        self._new_order: Optional[List[int]] = None
        options = dict(options or {})
        if find_unused_parameters:
            options[L.OPT_FIND_UNUSED] = 1
        if gradient_as_bucket_view:
            options[L.OPT_GRAD_VIEW] = 1
        # DDP's buckets are synced while backward still runs, so an overlap policy
        # applies unless the caller chose.  Measured (profiles/r01_n2.md, r01_n4.md):
        # fp32 models hide the exchange best with the copy engines (BERT-large W=4
        # 8.7% -> 4.3% exposed), bf16 models — a backward half as long — with the SM
        # kernels (W=2: CE 10.6-11.6% vs one-shot 6.7%; W=4: CE2 15-31% vs two-shot 8.8%)
        dtypes_ = {p.dtype for p in module.parameters() if p.requires_grad}
        options.setdefault(L.OPT_PREFER_OVERLAP, 1 if dtypes_ == {torch.float32} else 2)
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        dtypes = {p.dtype for p in self.params}
        if len(dtypes) != 1:
            raise ValueError("one gradient dtype per reducer (reading C-11)")
        self._dtype = dtypes.pop()
        self._options = options
        self.reducer = GradReducer([p.numel() for p in self.params], self._dtype,
                                   int(bucket_cap_mb * MIB), group=process_group,
                                   device=self.params[0].device, options=options)
        self._views = self._make_views()
        if broadcast_parameters and self.reducer.world > 1:
            # every parameter and buffer; a non-dense one travels as a contiguous copy
            # that is copied back (no state may start out different on some rank)
            states = list(module.parameters()) + list(module.buffers())
            with torch.no_grad():
                bufs = [t.data if _dense(t) else t.data.contiguous() for t in states]
                self.reducer.broadcast(bufs, root=0)
                for t, b in zip(states, bufs):
                    if b.data_ptr() != t.data_ptr():
                        t.data.copy_(b)
        self._pass_open = False
        self._in_no_sync = False
        self._unused_bufs: Dict[int, torch.Tensor] = {}
        self._param_index = {id(p): i for i, p in enumerate(self.params)}
        self._hooks = [p.register_post_accumulate_grad_hook(self._make_hook(i))
                       for i, p in enumerate(self.params)]

    def _make_views(self) -> Optional[List[torch.Tensor]]:
        """Each parameter's bucket slot in this rank's storage, shaped like the
        parameter (DDP_OPT_GRAD_VIEW; ddp_param_storage_offset)."""
        if not self.gradient_as_bucket_view:
            return None
        st, views = self.reducer._storage, []
        for i, p in enumerate(self.params):
            o = L.ddp_param_storage_offset(self.reducer.ctx, i)
            views.append(st[o:o + p.numel() * p.element_size()].view(p.dtype).view(p.shape))
        return views

    def _make_hook(self, idx: int):
        def hook(p: torch.Tensor):
            if not self._pass_open:
                self._pass_open = True
                # finalize when the autograd engine finishes this backward
                torch.autograd.Variable._execution_engine.queue_callback(self._finalize)
            g = p.grad
            if not _dense(g):
                raise ValueError("gradients must be dense (contiguous, channels_last, ... : no gaps or overlaps)")
            self.reducer.grad_ready(idx, g)
        return hook

    def _finalize(self):
        self._pass_open = False
        self.reducer.finalize()
        if self._views is not None and not self._in_no_sync:
            # the slots hold the averages of every gradient (in place): attach them
            for p, v in zip(self.params, self._views):
                if p.grad is not None and p.grad.data_ptr() != v.data_ptr():
                    p.grad = v
        if self._rebuild and not self._in_no_sync:
            self._rebuild = False
            order = torch.tensor(self.reducer.ready_order(), dtype=torch.int32, device=self.params[0].device)
            if self.reducer.world > 1:
                dist.broadcast(order, src=dist.get_global_rank(self.process_group, 0)
                               if self.process_group is not None else 0, group=self.process_group)
            self._new_order = order.tolist()
        if self._unused_bufs:
            # locally-unused params without a .grad got a zero buffer as their
            # destination; attach it only where some rank used the param (the
            # bitmap read blocks on the extra allreduce, as P:L310 implies)
            gu = self.reducer.global_unused()
            for i, buf in self._unused_bufs.items():
                if not gu[i]:
                    self.params[i].grad = buf
            self._unused_bufs = {}

    def _rebuild_reducer(self):
        """Rebuild the parameter-to-bucket map from the agreed traced order (rare;
        re-allocates the symmetric storage, a collective)."""
        order, self._new_order = self._new_order, None
        self.reducer.close()
        self.reducer = GradReducer([p.numel() for p in self.params], self._dtype,
                                   int(self.bucket_cap_mb * MIB), group=self.process_group,
                                   device=self.params[0].device, options=self._options, scan_order=order)
        self._views = self._make_views()

    def forward(self, *args, **kwargs):
        if self._new_order is not None:
            self._rebuild_reducer()
        out = self.module(*args, **kwargs)
        if self.find_unused_parameters and torch.is_grad_enabled():
            self._mark_unused(out)
        return out

    def _mark_unused(self, out):
        """Alg. 1 forward (L224-L225): traverse the autograd graph from the
        outputs; parameters not reached get no gradient this pass and are
        marked ready now."""
        used = set()
        stack, seen = [], set()
        for t in _tensors(out):
            if t.requires_grad:
                if t.grad_fn is not None:
                    stack.append(t.grad_fn)
                elif id(t) in self._param_index:
                    used.add(id(t))
        while stack:
            fn = stack.pop()
            if fn in seen:
                continue
            seen.add(fn)
            var = getattr(fn, "variable", None)
            if var is not None:
                used.add(id(var))
            for nxt, _ in fn.next_functions:
                if nxt is not None:
                    stack.append(nxt)
        for i, p in enumerate(self.params):
            if id(p) in used:
                continue
            g = p.grad
            if g is None and not self._in_no_sync:
                g = self._unused_bufs[i] = torch.zeros_like(p)
            self.reducer.mark_unused(i, g)

    @contextlib.contextmanager
    def no_sync(self):
        with self.reducer.no_sync():
            self._in_no_sync = True
            try:
                yield
            finally:
                self._in_no_sync = False

    def close(self):
        """Removes the hooks and releases the native context (the module can be
        wrapped again, e.g. with another bucket cap)."""
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.reducer.close()
