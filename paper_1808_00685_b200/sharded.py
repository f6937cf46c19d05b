"""Multi-GPU correlation: one process per GPU (torchrun), each rank owning a
band of output rows.

The reference's only parallelism is output row-block ownership
(engine_core.py:106-127: ``row_blocks`` linspace bounds, one block per
worker, concatenated at the end).  Here the workers are GPUs:

* ownership -- rank r owns the rows [r0, r1) of ``engine_core.band_partition``.
  A homo map is symmetric, so the rank owns only the UPPER-triangle part of its
  rows (columns >= r0) and the bands are balanced by that area; the lower
  triangle is the mirror and is implied (materialised on the host by
  ``gather``).  Each rank allocates only its band: (r1 - r0) x (n - r0)
  elements, ~1/P of the map.  A hetero map is split into equal row bands.
* spectra -- K1 runs on the rank's own channel chunk (its band rows; for a
  hetero map also a chunk of the second dataset), then every chunk is
  NCCL-broadcast by its owner (``spectra="broadcast"``, the north-star scheme)
  -- or every rank runs K1 over all channels and nothing crosses GPUs
  (``spectra="recompute"``).
* contraction -- the band's diagonal square first (a homo contraction on local
  spectra, mirrored inside the band), overlapping the broadcasts; then one
  rectangle piece per later owner, each launched as soon as that owner's
  spectra landed.  Every piece is an ordinary whole-map call of the same C ABI
  on pointer-offset operands, so every element has the bits of the one-GPU map.
* nothing else crosses GPUs: the outputs stay in the owning rank's HBM; the
  per-rank max|.| / finite / status words are all-reduced (a few bytes).
"""

from __future__ import annotations

import numpy as np

from . import _abi, engine
from .dataset import CorrelationSpectra
from .engine_core import assemble_bands, band_partition, band_pieces
from .errors import DataError, NumericError


def _dist():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise DataError("distributed=True needs an initialised torch.distributed process group "
                        "(one process per GPU, e.g. under torchrun)")
    return dist


def _is_nccl(group):
    return _dist().get_backend(group) == "nccl"


def _broadcast(t, src, group):
    """In-place broadcast of a device tensor from global rank `src`: one NCCL
    broadcast over NVLink (async; returns the work handle), or, for the gloo
    backend (CPU tests, several ranks sharing one GPU), a synchronous staged
    copy through the host (returns None)."""
    dist = _dist()
    if t.numel() == 0:
        return None
    if _is_nccl(group):
        return dist.broadcast(t, src=src, group=group, async_op=True)
    if t.is_cuda:
        engine.torch().cuda.current_stream().synchronize()
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)
    return None


def _allreduce(t, op, group):
    dist = _dist()
    if _is_nccl(group) or not t.is_cuda:
        dist.all_reduce(t, op=op, group=group)
        return
    h = t.cpu()
    dist.all_reduce(h, op=op, group=group)
    t.copy_(h)


class ShardedCorrelationPlan:
    """Device pipeline of one rank: K1 on its chunk, spectra exchange, band
    contraction.  ``launch()`` enqueues everything on the current stream (NCCL
    broadcasts on NCCL's stream, ordered by events); ``finish()`` synchronises
    and raises the reference's errors."""

    def __init__(self, *, n1, n2, m, recipe1, recipe2, norm, dtype="float64", group=None,
                 spectra="broadcast", device=None):
        dist = _dist()
        self.lib, self.dev = engine.require_device(device)
        t = engine.torch()
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.global_ranks = [dist.get_global_rank(group, q) if group is not None else q for q in range(self.world)]
        if spectra not in ("broadcast", "recompute"):
            raise DataError(f"spectra must be 'broadcast' or 'recompute', got {spectra!r}")
        self.spectra = spectra
        self.homo = recipe2 is None
        if self.homo and n1 != n2:
            raise DataError("homo correlation needs n1 == n2")
        self.n1, self.n2, self.m = int(n1), int(n2), int(m)
        self.recipe1, self.recipe2 = recipe1, recipe2
        self.norm = float(norm)
        self.dtype = np.dtype(dtype)
        if self.dtype == np.float64:
            self.pack_kind, odt, pdt = engine.f64_pack_kind(), t.float64, t.float64
        elif self.dtype == np.float32:
            self.pack_kind, odt, pdt = engine.fp32_pack_kind(), t.float32, t.bfloat16
        else:
            raise DataError(f"unsupported compute dtype {dtype}")
        self.tc = self.pack_kind in (_abi.PACK_BF16X2, _abi.PACK_F16F8)
        self.mp = self.lib.corr2d_packed_depth(self.m, self.pack_kind)
        if self.mp <= 0:
            _abi.check(_abi.ERR_DATA, self.lib)
        self.ld_pack = 2 * self.mp + 64 if self.tc else self.mp
        self.bands = band_partition(self.n1, self.world, self.homo)
        self.col_bands = None if self.homo else band_partition(self.n2, self.world, False)
        self.r0, self.r1 = self.bands[self.rank]
        self.c0 = self.r0 if self.homo else 0
        self.pieces = band_pieces(self.bands, self.rank, self.homo, self.col_bands)
        dev = self.dev
        # packed operands for every channel (the exchange fills the other ranks' chunks)
        z = t.zeros
        self.a_phi = z((self.n1, self.ld_pack), dtype=pdt, device=dev)
        gauss = self.pack_kind == _abi.PACK_F64_GAUSS
        self.a_psi = None if (self.tc or gauss) else z((self.n1, self.ld_pack), dtype=pdt, device=dev)
        if self.homo:
            self.b = self.a_phi if self.tc else z((self.n1, self.ld_pack), dtype=pdt, device=dev)
        else:
            self.b = z((self.n2, self.ld_pack), dtype=pdt, device=dev)
        self.ref1 = z(self.n1, dtype=t.float64, device=dev)
        self.ref2 = None if self.homo else z(self.n2, dtype=t.float64, device=dev)
        want_sigma = recipe1.alpha > 0.0
        self.sigma1 = z(self.n1, dtype=t.float64, device=dev) if want_sigma else None
        self.sigma2 = z(self.n2, dtype=t.float64, device=dev) if (want_sigma and not self.homo) else None
        rows, cols = self.r1 - self.r0, self.n2 - self.c0
        try:
            self.phi = t.empty((rows, cols), dtype=odt, device=dev)
            self.psi = t.empty((rows, cols), dtype=odt, device=dev)
        except t.cuda.OutOfMemoryError:
            raise NumericError(
                f"out of memory assembling this rank's band of the correlation matrix; it needs "
                f"{2 * rows * cols * self.dtype.itemsize / 1e9:.2f} GB") from None
        self.stats = t.zeros((max(1, len(self.pieces)), 4), dtype=t.int64, device=dev)
        self.status = t.zeros((2, 4), dtype=t.int32, device=dev)
        self.raw1 = self.raw2 = None
        self._works = {}

    # ---------------------------------------------------------------- inputs
    def bind(self, raw1, raw2=None):
        if raw1.shape[1] != self.n1 or (raw2 is not None and raw2.shape[1] != self.n2):
            raise DataError("bound inputs do not match the plan's shape")
        self.raw1, self.raw2 = raw1, raw2
        return self

    # ------------------------------------------------------------------- K1
    def _k1(self, raw, recipe, c0, c1, roles, a_phi, a_psi, b, ref, sigma, status):
        import dataclasses
        if c1 <= c0:
            return
        sl = dataclasses.replace(
            recipe, ref_in=None if recipe.ref_in is None else recipe.ref_in[c0:c1],
            sigma_in=None if recipe.sigma_in is None else recipe.sigma_in[c0:c1])
        rows = (lambda x: None if x is None else x[c0:c1])
        engine.launch_prep(self.lib, raw[:, c0:c1], sl, norm=self.norm, pack_kind=self.pack_kind, roles=roles,
                           a_phi=rows(a_phi), a_psi=rows(a_psi), b=rows(b), ld_pack=self.ld_pack,
                           ref_out=rows(ref), sigma_out=rows(sigma), status=status)

    def _roles1(self):
        if self.homo:
            return _abi.ROLE_A if self.tc else (_abi.ROLE_A | _abi.ROLE_B)
        return _abi.ROLE_A

    def launch_prep(self):
        """K1 of this rank's chunk(s) (recompute: of every channel), then the
        owners' broadcasts of their chunks (async on NCCL's stream)."""
        self.status.zero_()
        b1 = self.b if (self.homo and not self.tc) else None
        if self.spectra == "recompute":
            self._k1(self.raw1, self.recipe1, 0, self.n1, self._roles1(), self.a_phi, self.a_psi, b1,
                     self.ref1, self.sigma1, self.status[0])
            if not self.homo:
                self._k1(self.raw2, self.recipe2, 0, self.n2, _abi.ROLE_B, None, None, self.b,
                         self.ref2, self.sigma2, self.status[1])
            return
        self._k1(self.raw1, self.recipe1, self.r0, self.r1, self._roles1(), self.a_phi, self.a_psi, b1,
                 self.ref1, self.sigma1, self.status[0])
        if not self.homo:
            c0, c1 = self.col_bands[self.rank]
            self._k1(self.raw2, self.recipe2, c0, c1, _abi.ROLE_B, None, None, self.b,
                     self.ref2, self.sigma2, self.status[1])
        # owners broadcast their chunks: the buffers the contraction reads first
        # (later owners' column operands, in launch order), then the vectors
        self._works = {}
        if self.homo:
            order = [q for q in range(1, self.world)] + [0]
            for q in order:
                q0, q1 = self.bands[q]
                ws = [_broadcast(buf[q0:q1], self.global_ranks[q], self.group)
                      for buf in self._unique(self.a_phi, self.a_psi, self.b)]
                self._works[q] = ws
        else:
            for q in range(self.world):
                q0, q1 = self.col_bands[q]
                self._works[q] = [_broadcast(self.b[q0:q1], self.global_ranks[q], self.group)]
        vecs = []
        for q in range(self.world):
            q0, q1 = self.bands[q]
            vecs += [_broadcast(v[q0:q1], self.global_ranks[q], self.group) for v in (self.ref1, self.sigma1)
                     if v is not None]
            if not self.homo:
                c0, c1 = self.col_bands[q]
                vecs += [_broadcast(v[c0:c1], self.global_ranks[q], self.group) for v in (self.ref2, self.sigma2)
                         if v is not None]
        self._vec_works = vecs

    @staticmethod
    def _unique(*bufs):
        seen, out = set(), []
        for b in bufs:
            if b is not None and b.data_ptr() not in seen:
                seen.add(b.data_ptr())
                out.append(b)
        return out

    # ---------------------------------------------------------- contraction
    def _contract(self, k, a_rows, b_rows, homo, out_col):
        """One piece: operand rows a_rows = (a0, a1) of A, b_rows = (b0, b1) of B,
        written to the band's columns [out_col, out_col + b1 - b0)."""
        a0, a1 = a_rows
        b0, b1 = b_rows
        n1p, n2p = a1 - a0, b1 - b0
        ld_out = self.phi.shape[1]
        phi = self.phi[:, out_col:]
        psi = self.psi[:, out_col:]
        st = self.stats[k]
        if self.tc:
            code = self.lib.corr2d_contract_tc(
                self.pack_kind, engine.ptr(self.a_phi[a0:]), engine.ptr(self.b[b0:]), self.ld_pack,
                n1p, n2p, self.mp, self.m, 1 if homo else 0, 0, n1p, 0, -1,
                engine.ptr(phi), engine.ptr(psi), ld_out, engine.ptr(st), engine.stream_handle())
            _abi.check(code, self.lib)
        else:
            engine.launch_contract_f64(
                self.lib, self.pack_kind, self.a_phi[a0:], None if self.a_psi is None else self.a_psi[a0:],
                self.b[b0:], self.ld_pack, n1p, n2p, self.mp, 1 if homo else 0, 0, n1p, 0, -1,
                phi, psi, ld_out, st)

    def launch_contract(self):
        for k, (kind, owner, c0, c1) in enumerate(self.pieces):
            for w in self._works.get(owner, []) if owner != self.rank else []:
                if w is not None:
                    w.wait()          # this stream waits for the owner's spectra (no host sync)
            if kind == "diag":
                self._contract(k, (self.r0, self.r1), (self.r0, self.r1), True, 0)
            else:
                self._contract(k, (self.r0, self.r1), (c0, c1), False, c0 - self.c0)

    def launch(self):
        self.launch_prep()
        self.launch_contract()

    launch_prep_only = launch_prep          # the CorrelationPlan name bench.py drives

    @property
    def gauss(self) -> bool:
        return self.pack_kind == _abi.PACK_F64_GAUSS

    def tile_count(self) -> int:
        """Contraction-kernel tiles this rank launches (all pieces)."""
        total = 0
        for kind, _, c0, c1 in self.pieces:
            n1p, n2p = self.r1 - self.r0, c1 - c0
            homo = 1 if kind == "diag" else 0
            n = self.lib.corr2d_contract_tile_count(self.pack_kind, n1p, n2p, homo, 0, n1p, self.phi.shape[1])
            if n < 0:
                raise DataError("bad contraction shape")
            total += int(n)
        return total

    @property
    def launches_per_step(self) -> int:
        """Kernels of ours one launch() enqueues: K1 per dataset + one
        contraction per band piece."""
        return (1 if self.homo else 2) + len(self.pieces)

    # ------------------------------------------------------------- checks
    def finish(self, axes=(None, None), labels=("first", "second")):
        """Synchronise; all-reduce status / stats; raise the reference's errors.
        Returns (ref1, ref2, sigma1, sigma2, info) with the GLOBAL max|.|."""
        dist = _dist()
        t = engine.torch()
        for w in getattr(self, "_vec_works", []):
            if w is not None:
                w.wait()
        for ws in self._works.values():
            for w in ws:
                if w is not None:
                    w.wait()
        engine.sync()
        status = self.status.clone()
        if self.spectra == "broadcast":
            _allreduce(status[:, :2], dist.ReduceOp.SUM, self.group)
            _allreduce(status[:, 2:3], dist.ReduceOp.MAX, self.group)
        local = self.stats[:len(self.pieces)] if self.pieces else self.stats[:0]
        red = t.zeros(3, dtype=t.int64, device=self.dev)
        if local.numel():
            red[0] = local[:, 0].max()
            red[1] = local[:, 1].max()
            red[2] = local[:, 2].sum()
        # non-negative doubles order like their bit patterns: a MAX over int64 is the max|.|
        _allreduce(red, dist.ReduceOp.MAX, self.group)
        st = status.cpu().numpy()
        for k, lab in ((0, labels[0]), (1, labels[1])):
            if k == 1 and self.homo:
                break
            if int(st[k, _abi.ST_NONFINITE]):
                raise NumericError(f"{lab} dynamic-spectra matrix contains non-finite values")
        sig = []
        for recipe, sdev, axis in ((self.recipe1, self.sigma1, axes[0]), (self.recipe2, self.sigma2, axes[1])):
            if recipe is None or sdev is None:
                sig.append(None)
                continue
            sig.append(engine.handle_zero_variance(axis, sdev.cpu().numpy(), recipe.alpha, recipe.substitute))
        r = red.cpu().numpy()
        if int(r[2]):
            raise NumericError("correlation produced non-finite values")
        info = {"max_abs_sync": float(r[0:1].view(np.float64)[0]),
                "max_abs_async": float(r[1:2].view(np.float64)[0])}
        ref1 = self.ref1.cpu().numpy()
        ref2 = ref1 if self.homo else self.ref2.cpu().numpy()
        if self.homo:
            sig[1] = sig[0]
        return ref1, ref2, sig[0], sig[1], info


class ShardedCorrelationSpectra:
    """This rank's band of a multi-GPU correlation (``distributed=True``).

    ``sync`` / ``asyn``: CUDA tensors of the band, rows ``rows = (r0, r1)`` x
    columns ``cols = (c0, n2)`` of the map (homo: c0 = r0, the upper part; the
    lower triangle is the mirror).  ``gather(root)`` -- a collective -- returns
    the whole map as a ``CorrelationSpectra`` on `root` (None elsewhere)."""

    def __init__(self, plan: ShardedCorrelationPlan, meta):
        self._plan = plan
        self.sync, self.asyn = plan.phi, plan.psi
        self.rows = (plan.r0, plan.r1)
        self.cols = (plan.c0, plan.n2)
        self.rank, self.world = plan.rank, plan.world
        self.bands = plan.bands
        self.meta = meta
        self.stats = meta.get("stats")

    @property
    def band_bytes(self) -> int:
        return 2 * self.sync.numel() * self.sync.element_size()

    def band_to_host(self):
        """This rank's band planes as numpy arrays (pinned D2H)."""
        t = engine.torch()
        if not self.sync.is_cuda:
            return self.sync.numpy(), self.asyn.numpy()
        hs = t.empty(self.sync.shape, dtype=self.sync.dtype, pin_memory=True)
        ha = t.empty(self.asyn.shape, dtype=self.asyn.dtype, pin_memory=True)
        engine.copy_d2h([(hs, self.sync), (ha, self.asyn)])
        return hs.numpy(), ha.numpy()

    def gather(self, root: int = 0, out=None):
        """Collective: every rank sends its band to `root` (NCCL point-to-point,
        or gloo through the host), which assembles the whole map -- mirror
        included -- on the host.  Returns the CorrelationSpectra on `root`,
        None on the other ranks."""
        dist = _dist()
        t = engine.torch()
        plan = self._plan
        group = plan.group
        nccl = _is_nccl(group)
        groot = plan.global_ranks[root]
        n1, n2 = plan.n1, plan.n2
        if self.rank != root:
            for pl in (self.sync, self.asyn):
                if pl.numel():
                    dist.send(pl.contiguous() if nccl else pl.cpu(), dst=groot, group=group)
            return None
        odt = np.float32 if plan.dtype == np.float32 else np.float64
        if out is None:
            hs, ha = np.empty((n1, n2), dtype=odt), np.empty((n1, n2), dtype=odt)
        else:
            hs, ha = out
        for q, (r0, r1) in enumerate(self.bands):
            if r1 <= r0:
                continue
            c0 = r0 if plan.homo else 0
            if q == root:
                bs, ba = self.band_to_host()
            else:
                shape = (r1 - r0, n2 - c0)
                planes = []
                for _ in range(2):
                    if nccl:
                        buf = t.empty(shape, dtype=self.sync.dtype, device=plan.dev)
                        dist.recv(buf, src=plan.global_ranks[q], group=group)
                        planes.append(buf.cpu().numpy())
                    else:
                        buf = t.empty(shape, dtype=self.sync.dtype)
                        dist.recv(buf, src=plan.global_ranks[q], group=group)
                        planes.append(buf.numpy())
                bs, ba = planes
            assemble_bands(n1, n2, plan.homo, [(r0, r1, c0, bs, ba)], out=(hs, ha))
        return CorrelationSpectra._trusted(sync=hs, asyn=ha, **self.meta)


def run(plan: ShardedCorrelationPlan, meta, axes, labels=("first", "second")):
    """Launch, check and wrap one sharded correlation."""
    plan.launch()
    ref1, ref2, _, _, info = plan.finish(axes=axes, labels=labels)
    meta = dict(meta)
    meta.setdefault("ref1", ref1)
    meta.setdefault("ref2", ref2)
    meta["stats"] = info
    return ShardedCorrelationSpectra(plan, meta)
