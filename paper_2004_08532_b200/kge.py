"""Thin ctypes binding of libkge.so (include/kge.h): argument marshalling only.

Every step of the training path runs in the library's CUDA kernels; this module converts numpy arrays to host
pointers, hands PyTorch's caching allocator and current stream to the library, and raises KgeError on a non-OK status.
There is no CPU fallback: if libkge.so is missing or no sm_100 device is present, calls raise.
Names mirror the C entry points: init (kge_init), Handle.sample (kge_sample), Handle.train_step (kge_train_step),
Handle.train_batch (kge_train_batch), Handle.score (kge_score), get_rows / set_rows, step, sync, destroy.
"""
from __future__ import annotations

import atexit
import ctypes
import os
import weakref
from dataclasses import dataclass

import numpy as np

from .build import LIB

# Kernels are force-loaded at kge_init; eager loading (when set before CUDA initialises) is belt and braces for the
# multi-rank device barriers (a lazily loaded kernel may wait for a spinning barrier kernel).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

MODELS = {"transe_l1": 0, "transe_l2": 1, "distmult": 2, "complex": 3, "rotate": 4, "transr": 5, "rescal": 6}
CORRUPT = {"tail": 0, "head": 1, "alternate": 2}
PRECISION = {"fp32": 0, "tf32": 1, "bf16": 2, "3xtf32": 3}
LOSS = {"logistic": 0, "pairwise": 1}
STATUS = {0: "KGE_OK", -1: "KGE_EINVAL", -2: "KGE_ERANGE", -3: "KGE_ENOMEM", -4: "KGE_ECUDA", -5: "KGE_ENCCL",
          -6: "KGE_ENONFINITE", -7: "KGE_ESTATE", -8: "KGE_EUNSUPPORTED"}
KERNELS = ["k_sample", "k_gather", "k_neg_fwd", "k_neg_bwd", "k_chain", "k_update"]
OPTIONS = {"ffma_splitk": 0, "capture_neg": 1, "barrier_ms": 2}  # kge_set_option (include/kge.h)

ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)


class KgeError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_int32), ("model", ctypes.c_int32),
                ("n_entities", ctypes.c_int64), ("n_relations", ctypes.c_int64),
                ("dim", ctypes.c_int32), ("batch_size", ctypes.c_int32), ("chunk_size", ctypes.c_int32),
                ("neg_k", ctypes.c_int32), ("gamma", ctypes.c_float), ("lr", ctypes.c_float),
                ("adagrad_eps", ctypes.c_float), ("init_bound", ctypes.c_float), ("seed", ctypes.c_uint64),
                ("corrupt", ctypes.c_int32), ("neg_precision", ctypes.c_int32), ("rotate_variant", ctypes.c_int32),
                ("lag", ctypes.c_int32), ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("nccl_comm", ctypes.c_void_p), ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p),
                ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("neg_deg_k", ctypes.c_int32), ("neg_local", ctypes.c_int32), ("loss", ctypes.c_int32),
                ("repartition", ctypes.c_int32), ("placement", ctypes.c_int32)]


_lib = None
P = ctypes.POINTER
_i64p = P(ctypes.c_int64)
_i32p = P(ctypes.c_int32)
_fp = P(ctypes.c_float)


def lib():
    """Load libkge.so. Raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"libkge.so not built at {LIB}; run __graft_entry__.build() (there is no CPU fallback)")
        L = ctypes.CDLL(LIB)
        L.kge_config_default.argtypes = [P(_Config)]
        L.kge_init.argtypes = [P(ctypes.c_void_p), P(_Config), _i64p, _i64p, _i64p, ctypes.c_int64]
        L.kge_sample.argtypes = [ctypes.c_void_p, ctypes.c_int64, _i64p, _i64p, P(ctypes.c_int8), _i64p, _i64p, _i32p,
                                 _i64p, _i64p, _i32p]
        L.kge_train_step.argtypes = [ctypes.c_void_p, ctypes.c_int64, _fp]
        L.kge_train_batch.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, _fp]
        # raw addresses (ints): the pipelined path is called once per step, ctypes.cast per argument costs more than
        # the C call
        L.kge_train_batch_async.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p]
        L.kge_score.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, _fp]
        L.kge_rank.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int32, _i64p, _i64p,
                               _i64p, _i64p, _i64p]
        L.kge_rank_sampled.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, _i64p]
        L.kge_link_metrics.argtypes = [_i64p, ctypes.c_int64, P(ctypes.c_double)]
        L.kge_locality_order.argtypes = [_i64p, _i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _i64p, _i64p]
        L.kge_get_rows.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i64p, ctypes.c_int64, _fp]
        L.kge_set_rows.argtypes = [ctypes.c_void_p, ctypes.c_int32, _i64p, ctypes.c_int64, _fp]
        L.kge_table_width.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.kge_table_width.restype = ctypes.c_int32
        L.kge_step.argtypes = [ctypes.c_void_p]
        L.kge_step.restype = ctypes.c_int64
        L.kge_set_step.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.kge_flush.argtypes = [ctypes.c_void_p]
        L.kge_sync.argtypes = [ctypes.c_void_p]
        L.kge_profile_begin.argtypes = [ctypes.c_void_p]
        L.kge_profile_end.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_double), _i64p]
        L.kge_neg_path.argtypes = [ctypes.c_void_p]
        L.kge_neg_path.restype = ctypes.c_int32
        L.kge_launch_count.argtypes = [ctypes.c_void_p]
        L.kge_launch_count.restype = ctypes.c_int64
        L.kge_destroy.argtypes = [ctypes.c_void_p]
        L.kge_read_losses.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, _fp]
        L.kge_partition.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _i32p, _i64p,
                                    _i64p]
        L.kge_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(ctypes.c_size_t)]
        L.kge_connect.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        L.kge_connect_local.argtypes = [P(ctypes.c_void_p), ctypes.c_int32]
        L.kge_relation_owner.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        L.kge_relation_owner.restype = ctypes.c_int
        L.kge_last_error.restype = ctypes.c_char_p
        L.kge_set_option.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64]
        L.kge_debug_neg_scores.argtypes = [ctypes.c_void_p, _fp]
        L.kge_kernel_name.argtypes = [ctypes.c_int32]
        L.kge_kernel_name.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise KgeError(rc, lib().kge_last_error().decode())
    return rc


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _ptr(a, ct):
    return a.ctypes.data_as(P(ct)) if a is not None else None


@dataclass
class Config:
    """Mirror of kge_config (include/kge.h); defaults = kge_config_default."""
    model: str = "transe_l2"
    n_entities: int = 0
    n_relations: int = 0
    dim: int = 400
    batch_size: int = 1024
    chunk_size: int = 256
    neg_k: int = 256
    gamma: float = 12.0
    lr: float = 0.1
    adagrad_eps: float = 1e-10
    init_bound: float = 0.0
    seed: int = 1
    corrupt: str = "alternate"
    neg_precision: str = "tf32"
    rotate_variant: int = 0
    lag: int = 0
    world_size: int = 1
    neg_deg_k: int = 0  # degree-based in-batch negatives per chunk
    neg_local: int = 0  # 1: local-shard negatives when world_size > 1
    loss: str = "logistic"  # or "pairwise"
    repartition: int = 0  # 1: a randomised relation partition every epoch when world_size > 1
    placement: int = 0  # 1: head-owner triple placement when world_size > 1
    rank: int = 0

    @property
    def C(self):
        return self.batch_size // self.chunk_size

    @property
    def n_occ(self):
        return 2 * self.batch_size + self.C * self.neg_k


class _TorchAllocator:
    """Hands PyTorch's caching allocator to the library (kge_config.dev_alloc / dev_free)."""

    def __init__(self, device, stream):
        import torch
        _alloc = torch.cuda.caching_allocator_alloc
        _delete = torch.cuda.caching_allocator_delete
        self.device = device
        self.stream = stream

        def alloc(nbytes, ctx):
            try:
                return _alloc(int(nbytes), device, stream)
            except Exception:
                return None

        def free(ptr, ctx):
            try:
                _delete(ptr)
            except Exception:
                pass

        self.alloc_fn = ALLOC_FN(alloc)
        self.free_fn = FREE_FN(free)


_live = weakref.WeakSet()


@atexit.register
def _destroy_live_handles():
    # free device memory through torch's allocator before the interpreter tears torch down
    for h in list(_live):
        h.destroy()


class Handle:
    def __init__(self, ptr, cfg: Config, keep):
        self._h = ptr
        self._tba = lib().kge_train_batch_async  # bound once (per-step pipelined entry point)
        self.cfg = cfg
        self._keep = keep
        _live.add(self)

    def __del__(self):
        self.destroy()

    def destroy(self):
        if getattr(self, "_h", None):
            lib().kge_destroy(self._h)
            self._h = None

    # kge_sample
    def sample(self, step):
        c = self.cfg
        pos = np.zeros(c.batch_size, np.int64)
        neg = np.zeros(c.C * c.neg_k, np.int64)
        mode = np.zeros(c.C, np.int8)
        ue = np.zeros(c.n_occ, np.int64)
        ie = np.zeros(c.n_occ, np.int32)
        ur = np.zeros(c.batch_size, np.int64)
        ir = np.zeros(c.batch_size, np.int32)
        ne, nr = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().kge_sample(self._h, step, _ptr(pos, ctypes.c_int64), _ptr(neg, ctypes.c_int64),
                                _ptr(mode, ctypes.c_int8), _ptr(ue, ctypes.c_int64), ctypes.byref(ne),
                                _ptr(ie, ctypes.c_int32), _ptr(ur, ctypes.c_int64), ctypes.byref(nr),
                                _ptr(ir, ctypes.c_int32)))
        return dict(pos=pos, neg=neg, mode=mode, uniq_ent=ue[:ne.value], inv_ent=ie, uniq_rel=ur[:nr.value],
                    inv_rel=ir)

    # kge_train_step
    def train_step(self, n_steps=1, return_loss=True):
        if return_loss:
            out = np.zeros(n_steps, np.float32)
            _check(lib().kge_train_step(self._h, n_steps, _ptr(out, ctypes.c_float)))
            return out
        _check(lib().kge_train_step(self._h, n_steps, None))
        return None

    # kge_train_batch
    def train_batch(self, heads, rels, tails, return_loss=True):
        h, r, t = _i64(heads), _i64(rels), _i64(tails)
        assert len(h) == self.cfg.batch_size
        if return_loss:
            out = np.zeros(1, np.float32)
            _check(lib().kge_train_batch(self._h, _ptr(h, ctypes.c_int64), _ptr(r, ctypes.c_int64),
                                         _ptr(t, ctypes.c_int64), _ptr(out, ctypes.c_float)))
            return float(out[0])
        _check(lib().kge_train_batch(self._h, _ptr(h, ctypes.c_int64), _ptr(r, ctypes.c_int64),
                                     _ptr(t, ctypes.c_int64), None))
        return None

    def train_batch_ptr(self, hp, rp, tp, loss_ptr):
        """Raw-pointer variant (host int64 buffers, e.g. pinned torch tensors)."""
        _check(lib().kge_train_batch(self._h, ctypes.cast(hp, _i64p), ctypes.cast(rp, _i64p), ctypes.cast(tp, _i64p),
                                     ctypes.cast(loss_ptr, _fp) if loss_ptr else None))

    # kge_train_batch_async
    def train_batch_async_ptr(self, hp, rp, tp, loss_ptr):
        """Pipelined variant: enqueue the step (H2D batch, step, D2H loss into the pinned float at loss_ptr) and
        return; the loss is valid after sync()."""
        rc = self._tba(self._h, hp, rp, tp, loss_ptr or None)
        if rc:
            _check(rc)

    # kge_rank
    def rank(self, hs, rs, ts, head=False, candidates=None, filters=None):
        """Link-prediction ranks (PAPER.md:652-665 [5.3]) of the true tail (head=True: head; head="both": one list with
        both corruption sides). candidates / filters: None or a CSR pair (offsets, ids) -- see kge_rank in
        include/kge.h (head="both": 2n filter lists, the tail side's first)."""
        hs, rs, ts = _i64(hs), _i64(rs), _i64(ts)
        if not (len(hs) == len(rs) == len(ts)):
            raise ValueError("hs, rs, ts must have the same length")
        side = 2 if isinstance(head, str) and head == "both" else (1 if head else 0)
        out = np.zeros(len(hs), np.int64)
        co, ci = (None, None) if candidates is None else (_i64(candidates[0]), _i64(candidates[1]))
        fo, fi = (None, None) if filters is None else (_i64(filters[0]), _i64(filters[1]))
        for name, off, ids, nl in (("candidates", co, ci, len(hs)), ("filters", fo, fi, len(hs) * (2 if side == 2 else 1))):
            # CSR size contract of kge_rank: offsets[n_lists + 1], ids[max offset] (value errors: the library)
            if off is None:
                continue
            if off.ndim != 1 or len(off) != nl + 1:
                raise ValueError(f"{name}: offsets must have {nl + 1} entries, got {off.shape}")
            if len(ids) < max(int(off.max()), 0):
                raise ValueError(f"{name}: {len(ids)} ids but offsets reach {off.max()}")
        p = lambda a: None if a is None else _ptr(a, ctypes.c_int64)
        _check(lib().kge_rank(self._h, p(hs), p(rs), p(ts), len(hs), side, p(co), p(ci), p(fo), p(fi), p(out)))
        return out

    # kge_rank_sampled
    def rank_sampled(self, hs, rs, ts, head=False, n_uniform=1000, n_degree=1000, seed=0):
        """Second protocol: candidates drawn on the device (reading c.15')."""
        hs, rs, ts = _i64(hs), _i64(rs), _i64(ts)
        side = 2 if isinstance(head, str) and head == "both" else (1 if head else 0)
        out = np.zeros(len(hs), np.int64)
        p = lambda a: _ptr(a, ctypes.c_int64)
        _check(lib().kge_rank_sampled(self._h, p(hs), p(rs), p(ts), len(hs), side, n_uniform, n_degree, seed, p(out)))
        return out

    # kge_score
    def score(self, hs, rs, ts):
        hs, rs, ts = _i64(hs), _i64(rs), _i64(ts)
        out = np.zeros(len(hs), np.float32)
        _check(lib().kge_score(self._h, _ptr(hs, ctypes.c_int64), _ptr(rs, ctypes.c_int64), _ptr(ts, ctypes.c_int64),
                               len(hs), _ptr(out, ctypes.c_float)))
        return out

    # kge_set_option
    def set_option(self, name, value):
        _check(lib().kge_set_option(self._h, OPTIONS[name] if isinstance(name, str) else name, int(value)))

    # kge_debug_neg_scores: [B, k] negative pair scores of the last captured step
    def neg_scores(self):
        c = self.cfg
        out = np.zeros((c.batch_size, c.neg_k), np.float32)
        _check(lib().kge_debug_neg_scores(self._h, _ptr(out, ctypes.c_float)))
        return out

    def width(self, table):
        return lib().kge_table_width(self._h, table)

    def get_rows(self, table, ids):
        ids = _i64(ids)
        out = np.zeros((len(ids), self.width(table)), np.float32)
        _check(lib().kge_get_rows(self._h, table, _ptr(ids, ctypes.c_int64), len(ids), _ptr(out, ctypes.c_float)))
        return out

    def set_rows(self, table, ids, rows):
        ids = _i64(ids)
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        _check(lib().kge_set_rows(self._h, table, _ptr(ids, ctypes.c_int64), len(ids), _ptr(rows, ctypes.c_float)))

    @property
    def step(self):
        return lib().kge_step(self._h)

    @property
    def neg_path(self):
        """Arithmetic of the negative contraction: "ffma", "tf32" or "bf16" (tcgen05), see kge_neg_path."""
        return {0: "ffma", 1: "tf32", 2: "bf16", 3: "3xtf32"}[lib().kge_neg_path(self._h)]

    def read_losses(self, first_step, n):
        out = np.zeros(n, np.float32)
        _check(lib().kge_read_losses(self._h, first_step, n, _ptr(out, ctypes.c_float)))
        return out

    def relation_owner(self, r):
        return lib().kge_relation_owner(self._h, int(r))

    def export(self) -> bytes:
        n = ctypes.c_size_t(0)
        _check(lib().kge_export(self._h, None, ctypes.byref(n)))
        buf = (ctypes.c_char * n.value)()
        _check(lib().kge_export(self._h, buf, ctypes.byref(n)))
        return bytes(buf)

    def connect(self, blobs):
        joined = b"".join(blobs)
        buf = ctypes.create_string_buffer(joined, len(joined))
        _check(lib().kge_connect(self._h, buf, len(blobs)))

    def flush(self):
        """kge_flush: lag = 1, apply the held-back entity update of the last step."""
        _check(lib().kge_flush(self._h))

    def set_step(self, s):
        _check(lib().kge_set_step(self._h, s))

    def sync(self):
        _check(lib().kge_sync(self._h))

    def profile_begin(self):
        _check(lib().kge_profile_begin(self._h))

    def profile_end(self):
        avg = (ctypes.c_double * len(KERNELS))()
        cnt = (ctypes.c_int64 * len(KERNELS))()
        _check(lib().kge_profile_end(self._h, len(KERNELS), avg, cnt))
        return {KERNELS[i]: (avg[i], cnt[i]) for i in range(len(KERNELS))}

    @property
    def launch_count(self):
        return lib().kge_launch_count(self._h)


def init(cfg: Config, heads, rels, tails, use_torch_allocator=True, stream=None) -> Handle:
    """kge_init. heads/rels/tails: host int64 arrays of the whole graph (copied to the device)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("kge.init needs a CUDA (sm_100a) device; there is no CPU fallback")
    c = _Config()
    lib().kge_config_default(ctypes.byref(c))
    c.model = MODELS[cfg.model] if isinstance(cfg.model, str) else cfg.model
    c.n_entities, c.n_relations, c.dim = cfg.n_entities, cfg.n_relations, cfg.dim
    c.batch_size, c.chunk_size, c.neg_k = cfg.batch_size, cfg.chunk_size, cfg.neg_k
    c.gamma, c.lr, c.adagrad_eps, c.init_bound = cfg.gamma, cfg.lr, cfg.adagrad_eps, cfg.init_bound
    c.seed = cfg.seed
    c.corrupt = CORRUPT[cfg.corrupt] if isinstance(cfg.corrupt, str) else cfg.corrupt
    c.neg_precision = PRECISION[cfg.neg_precision] if isinstance(cfg.neg_precision, str) else cfg.neg_precision
    c.rotate_variant, c.lag, c.world_size, c.rank = cfg.rotate_variant, cfg.lag, cfg.world_size, cfg.rank
    c.neg_deg_k = cfg.neg_deg_k
    c.neg_local = cfg.neg_local
    c.loss = LOSS[cfg.loss] if isinstance(cfg.loss, str) else cfg.loss
    c.repartition = cfg.repartition
    c.placement = cfg.placement
    dev = torch.cuda.current_device()
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    c.cuda_stream = s.cuda_stream
    keep = [c]
    if use_torch_allocator:
        al = _TorchAllocator(dev, s)
        c.dev_alloc, c.dev_free = al.alloc_fn, al.free_fn
        keep.append(al)
    h, r, t = _i64(heads), _i64(rels), _i64(tails)
    out = ctypes.c_void_p()
    _check(lib().kge_init(ctypes.byref(out), ctypes.byref(c), _ptr(h, ctypes.c_int64), _ptr(r, ctypes.c_int64),
                          _ptr(t, ctypes.c_int64), len(h)))
    return Handle(out.value, cfg, keep)


def locality_order(heads, tails, n_entities, world_size):
    """kge_locality_order: the entity renumbering (new_id[e]) of the BFS-grown balanced parts and the edge cut."""
    h, t = _i64(heads), _i64(tails)
    nid = np.zeros(n_entities, np.int64)
    cut = np.zeros(1, np.int64)
    _check(lib().kge_locality_order(_ptr(h, ctypes.c_int64), _ptr(t, ctypes.c_int64), len(h), n_entities, world_size,
                                    _ptr(nid, ctypes.c_int64), _ptr(cut, ctypes.c_int64)))
    return nid, int(cut[0])


def partition(rels, n_relations, world_size, rank):
    """kge_partition (host-only, no GPU needed): relation owner per relation (-1 = split) and this rank's triples."""
    rels = _i64(rels)
    owner = np.zeros(n_relations, np.int32)
    n = ctypes.c_int64()
    _check(lib().kge_partition(_ptr(rels, ctypes.c_int64), len(rels), n_relations, world_size, rank,
                               _ptr(owner, ctypes.c_int32), None, ctypes.byref(n)))
    lst = np.zeros(n.value, np.int64)
    _check(lib().kge_partition(_ptr(rels, ctypes.c_int64), len(rels), n_relations, world_size, rank, None,
                               _ptr(lst, ctypes.c_int64), ctypes.byref(n)))
    return owner, lst


def exchange_and_connect(handle: Handle, all_gather_object):
    """World-size > 1: gather every rank's IPC blob with the caller's collective (torch.distributed.all_gather_object)
    and connect. Host-side plumbing only; the exchange itself runs in the library's kernels over NVLink."""
    mine = handle.export()
    world = handle.cfg.world_size
    blobs = [None] * world
    all_gather_object(blobs, mine)
    handle.connect(blobs)
    return blobs


def init_distributed(cfg: Config, heads, rels, tails, stream=None) -> Handle:
    """One process per GPU (torchrun): kge_init on this rank, then IPC exchange through torch.distributed."""
    import torch.distributed as dist
    h = init(cfg, heads, rels, tails, use_torch_allocator=True, stream=stream)
    exchange_and_connect(h, dist.all_gather_object)
    return h


def init_local_group(cfg: Config, world_size: int, heads, rels, tails):
    """Single-process emulation of world_size ranks on the current device (one handle and stream per rank), connected
    directly (kge_connect_local). Used by the one-GPU parity tests of the multi-rank path."""
    import dataclasses

    import torch
    hs = []
    for w in range(world_size):
        c = dataclasses.replace(cfg, world_size=world_size, rank=w)
        hs.append(init(c, heads, rels, tails, stream=torch.cuda.Stream()))
    arr = (ctypes.c_void_p * world_size)(*[h._h for h in hs])
    _check(lib().kge_connect_local(arr, world_size))
    return hs


def link_metrics(ranks):
    """Hit@1/3/10, MR, MRR (PAPER.md:660-664 [5.3]), computed by the library (kge_link_metrics)."""
    r = _i64(ranks)
    out = np.zeros(5, np.float64)
    _check(lib().kge_link_metrics(_ptr(r, ctypes.c_int64), len(r), out.ctypes.data_as(P(ctypes.c_double))))
    return dict(zip(["Hit@1", "Hit@3", "Hit@10", "MR", "MRR"], out.tolist()))


def filter_lists(known, hs, rs, ts, head=False):
    """CSR filter lists of the first protocol (PAPER.md:654-655 [5.3]): for query i, the entities e such that the
    corrupted triple (h_i, r_i, e) -- head=True: (e, r_i, t_i) -- is a known triple. known: (heads, rels, tails).
    head="both": the 2n lists of kge_rank's pooled protocol (the tail side's n lists, then the head side's)."""
    if isinstance(head, str) and head == "both":
        ot, it = filter_lists(known, hs, rs, ts, head=False)
        oh, ih = filter_lists(known, hs, rs, ts, head=True)
        return np.concatenate([ot, oh[1:] + ot[-1]]), np.concatenate([it, ih])
    kh, kr, kt = (np.asarray(a, np.int64) for a in known)
    fixed_a, fixed_b, free = (kr, kt, kh) if head else (kh, kr, kt)
    qa, qb = (np.asarray(rs, np.int64), np.asarray(ts, np.int64)) if head else (np.asarray(hs, np.int64),
                                                                                 np.asarray(rs, np.int64))
    order = np.lexsort((free, fixed_b, fixed_a))
    ka, kb, kf = fixed_a[order], fixed_b[order], free[order]
    key = lambda a, b: a * (int(max(kb.max(initial=0), qb.max(initial=0))) + 1) + b
    kk, qk = key(ka, kb), key(qa, qb)
    lo, hi = np.searchsorted(kk, qk, "left"), np.searchsorted(kk, qk, "right")
    off = np.zeros(len(qk) + 1, np.int64)
    off[1:] = np.cumsum(hi - lo)
    ids = np.concatenate([kf[a:b] for a, b in zip(lo, hi)]) if len(qk) else np.zeros(0, np.int64)
    return off, ids
