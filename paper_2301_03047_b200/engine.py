"""Device-resident GLR iteration engine behind gap_solve / regularize_dispatch.

Everything the reference's hot loop touches (glr/solvers.py:170-308) stays
on the GPU between iterations: the iterate x (fp64, (H, W, C)), the
measurement, the masks, the edge stack, the heat map, the match positions,
the int64 fixed-point aggregation numerator and the int32 counter. One
iteration is a fixed sequence of libglr_b200 launches on one stream:

  refresh (every match_refresh_interval iterations, solvers.py:185-203)
      Sobel -> corner response -> NMS corners -> anchors (+ uniform grid)
      sign-split edge stack
      heat map (tcgen05) -> exact top-K positions       [per exemplar shard]
      counter of covered pixels                         [+ all-reduce]
  every iteration (solvers.py:204-210, 298-301)
      fused gather + WNNM + fixed-point scatter          [per exemplar shard]
      all-reduce of the numerator (multi-GPU only)
      fused normalise + GAP projection + clip + residual

Exemplars shard across ranks as contiguous anchor blocks; the
integer all-reduce makes every rank count bitwise identical.
"""

from __future__ import annotations

import numpy as np

from . import _device as D
from . import _native as N
from .lowrank import KMAX, frac_bits_for


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous anchor block [lo, hi) of ``rank`` out of ``world``."""
    return (n * rank) // world, (n * (rank + 1)) // world


def sticky_owners(prev_owner: np.ndarray, world: int) -> np.ndarray:
    """Owner rank of each anchor of a refresh (reference anchor order).
    ``prev_owner[i]`` is the rank that held anchor i at the previous refresh,
    or -1 for a new anchor. Persisting anchors keep their rank; new anchors
    go, in anchor order, to the ranks below their share of the contiguous
    split (n*r//world .. n*(r+1)//world). Deterministic in its inputs, so
    every rank computes the same assignment."""
    owner = np.asarray(prev_owner, dtype=np.int64).copy()
    owner[owner >= world] = -1
    n = owner.size
    target = np.diff([(n * r) // world for r in range(world + 1)])
    have = np.bincount(owner[owner >= 0], minlength=world)
    need = np.maximum(target - have, 0)
    pending = np.nonzero(owner < 0)[0]
    owner[pending] = np.repeat(np.arange(world), need)[:pending.size]
    return owner


class DeviceOperator:
    """Device copy of a SensingOperator, rebuilt from kind + meta
    (operators.py plug point; the Python lambdas are never called)."""

    def __init__(self, op, clip_policy: bool | None = None):
        t = D.torch()
        self.kind = op.kind
        h, w, c = op.x_shape
        self.shape = (h, w, c)
        if op.kind in ("cacti", "msfa"):
            u8 = op.meta.get("masks_u8")
            if u8 is not None and (op.meta.get("masks_u8_of") != id(op.meta["masks"])
                                   or u8.shape != (h, w, c)):
                u8 = None  # meta["masks"] replaced since the operator was built
            if u8 is not None and op.kind == "cacti":
                # binary masks: 1-byte upload, widened on device; gram = sum_t M_t^2
                # = the count of ones (exact), formed on device as well
                m8 = D.to_dev(np.ascontiguousarray(u8))
                self.masks = m8.to(t.float64)
                self.gram = m8.sum(dim=2, dtype=t.int32).to(t.float64).contiguous()
            elif u8 is not None:
                self.masks = D.to_dev(np.ascontiguousarray(u8)).to(t.float64)
                self.gram = D.f64(np.asarray(op.gram_diag, dtype=np.float64).reshape(h, w))
            else:
                self.masks = D.f64(np.asarray(op.meta["masks"], dtype=np.float64))
                self.gram = D.f64(np.asarray(op.gram_diag, dtype=np.float64).reshape(h, w))
            self.y_shape = (h, w, 1)
        elif op.kind == "fourier":
            self.mask = D.f64(np.asarray(op.meta["mask"], dtype=np.float64))
            self.y_shape = (h, w)
            self.fft_ws = D.empty((N.query("glr_fft_workspace", h, w),), t.uint8)
        else:
            raise ValueError(f"unsupported operator kind {op.kind!r}")
        # complex (re, im) images are not clipped
        self.clip = (c != 2) if clip_policy is None else bool(clip_policy)

    def upload_y(self, y: np.ndarray):
        y = np.asarray(y)
        if self.kind == "fourier":
            yc = np.stack([y.real, y.imag], axis=2) if np.iscomplexobj(y) else \
                np.stack([y, np.zeros_like(y)], axis=2)
            return D.f64(yc)
        return D.f64(np.asarray(y, dtype=np.float64).reshape(self.shape[0], self.shape[1]))

    def adjoint(self, y_d, x_d):
        h, w, c = self.shape
        if self.kind == "fourier":
            N.call("glr_fourier_adjoint", y_d.data_ptr(), self.mask.data_ptr(), h, w, c,
                   x_d.data_ptr(), self.fft_ws.data_ptr(), D.stream())
        else:
            N.call("glr_masksum_adjoint", y_d.data_ptr(), self.masks.data_ptr(), h, w, c,
                   x_d.data_ptr(), D.stream())

    def init_x(self, y_d, x_d, init: str = "adjoint"):
        """solvers.py:229-254 (_init_x / _interp_init) into x_d. "interp":
        MSFA normalised Gaussian inpainting (bit-identical to scipy's
        gaussian_filter(sigma=1.5)), CACTI adjoint / max(gram, 1e-12),
        plain adjoint otherwise."""
        if init == "zero":
            x_d.zero_()
            return
        if init == "interp" and self.kind == "msfa":
            t = D.torch()
            h, w, c = self.shape
            if getattr(self, "_xt", None) is None:
                self._xt = D.empty((h, w, c), t.float64)
                self._interp_ws = D.empty((4 * h * w * c,), t.float64)
                # scipy.ndimage _gaussian_kernel1d(sigma=1.5, radius=int(4*1.5+0.5))
                radius = int(4.0 * 1.5 + 0.5)
                xs = np.arange(-radius, radius + 1)
                phi = np.exp(-0.5 / (1.5 * 1.5) * xs ** 2)
                self._gauss = np.ascontiguousarray(phi / phi.sum(), dtype=np.float64)
                self._gauss_r = radius
            self.adjoint(y_d, self._xt)
            wts = self._gauss.ctypes.data_as(N.C.POINTER(N.C.c_double))
            N.call("glr_interp_msfa", self._xt.data_ptr(), self.masks.data_ptr(), h, w, c, wts,
                   self._gauss_r, x_d.data_ptr(), self._interp_ws.data_ptr(), D.stream())
            return
        if init == "interp" and self.kind == "cacti":
            t = D.torch()
            h, w, c = self.shape
            if getattr(self, "_xt", None) is None:
                self._xt = D.empty((h, w, c), t.float64)
            self.adjoint(y_d, self._xt)
            N.call("glr_interp_cacti", self._xt.data_ptr(), self.gram.data_ptr(), h, w, c,
                   x_d.data_ptr(), D.stream())
            return
        self.adjoint(y_d, x_d)

    def gap_update(self, acc, cnt, frac, x_in, y_d, lo, hi, x_out, resid_out, ws, rho=0.0):
        """x_out = clip(z + A^T safe_div(y - A z, gram)); resid_out = ||y - A x_out||^2,
        z = acc/cnt where covered else x_in (acc None: z = x_in)."""
        h, w, c = self.shape
        ap = acc.data_ptr() if acc is not None else None
        cp = cnt.data_ptr() if cnt is not None else None
        if self.kind == "fourier":
            N.call("glr_gap_fourier", ap, cp, frac, x_in.data_ptr(), self.mask.data_ptr(),
                   y_d.data_ptr(), h, w, c, 1 if self.clip else 0, lo, hi, float(rho),
                   x_out.data_ptr(), resid_out.data_ptr(), self.fft_ws.data_ptr(), D.stream())
        else:
            N.call("glr_gap_masksum", ap, cp, frac, x_in.data_ptr(), self.masks.data_ptr(),
                   y_d.data_ptr(), self.gram.data_ptr(), h, w, c, lo, hi, float(rho),
                   x_out.data_ptr(), resid_out.data_ptr(), ws.data_ptr(), D.stream())


class GlrEngine:
    """Device state of one GLR reconstruction (one rank of a sharded run)."""

    def __init__(self, shape, match, peak: float = 1.0, c_weight: float = 2.0 * np.sqrt(2.0),
                 eps: float = 1e-16, process_group=None, heat_budget_bytes: int = 24 << 30,
                 low_memory_match: bool | None = None, regularizer: str = "glr"):
        t = D.torch()
        h, w, c = shape
        self.shape = (h, w, c)
        self.mc = match
        if regularizer not in ("glr", "nlr-bm", "nlr-corner-bm", "nlr-corner-uniform-bm"):
            raise ValueError(f"regularizer {regularizer!r} has no nonlocal match stage")
        # solvers.py:154-167: exemplar sources per regularizer; "nlr-*" match
        # by local block matching (matching.py:256-283) instead of the heat map
        self.regularizer = regularizer
        self.global_match = regularizer == "glr"
        self.use_corners = regularizer != "nlr-bm"
        self.p = match.patch_size
        self.k = match.group_size
        # K <= 64: the fast WNNM kernels with per-group eigenvector warm
        # starts; wider groups take the generic path (cold, no cache)
        self.use_vcache = self.k <= KMAX
        if self.p > min(h, w):
            raise ValueError(f"patch size {self.p} exceeds image {h}x{w}")
        self.c_weight = c_weight
        self.eps = eps
        self.frac = frac_bits_for(peak)
        self.pg = process_group
        self.rank, self.world = 0, 1
        if process_group is not None:
            import torch.distributed as dist
            self.rank = dist.get_rank(process_group)
            self.world = dist.get_world_size(process_group)
        p = self.p
        self.oh, self.ow = h - p + 1, w - p + 1
        self.grid_interval = {"nlr-bm": match.exemplar_stride, "nlr-corner-bm": 0}.get(
            regularizer, 3 * match.exemplar_stride)
        g = self.grid_interval
        n_grid = ((h - p) // g + 1) * ((w - p) // g + 1) if g > 0 else 0
        self.max_anchors = (match.max_corners if self.use_corners else 0) + n_grid
        self.expand = N.query("glr_heat_expand_factor", c, p)
        self.max_score = 4 * c * p * p
        self.stride = N.query("glr_heat_stride", h, w, p)
        # buffers
        self.resp = D.empty((h, w), t.float64)
        if self.global_match or self.use_corners:  # Sobel gradients: corners + edge stack
            self.gh = D.empty((h, w, c), t.float64)
            self.gv = D.empty((h, w, c), t.float64)
        if self.global_match:
            self.stack = D.empty((h * w * 2 * c * self.expand,), t.uint8)  # packed fp4
        self.corners = D.empty((max(match.max_corners, 1), 2), t.int32)
        self.n_corners = D.zeros((1,), t.int32)
        self.anchors = D.empty((self.max_anchors, 2), t.int32)
        self.tags = D.empty((self.max_anchors,), t.uint8)
        self.n_anchors = D.zeros((1,), t.int32)
        # match positions, double-buffered so a refresh can re-index the cached
        # eigenvectors of groups that keep their anchor (glr_vcache_remap)
        self._pos = [D.empty((self.max_anchors, self.k, 2), t.int32) for _ in range(2)]
        self._pcur = 0
        self.positions = self._pos[0]
        self.padded = D.empty((self.max_anchors,), t.int32)
        self.acc = D.zeros((h, w, c), t.int64)
        # the numerator's consumers (glr_gap_masksum / glr_gap_fourier /
        # glr_normalize) read AND clear it, so no per-iteration memset is
        # needed; acc_dirty marks a numerator that was produced but not consumed
        self.acc_dirty = False
        self.cnt = D.zeros((h, w), t.int32)
        self.gap_ws = D.empty((N.query("glr_gap_workspace", h, w),), t.uint8)
        self.ws_corner = D.empty((N.query("glr_corner_workspace", h, w, c),), t.uint8)
        self.ws_nms = D.empty((N.query("glr_nms_workspace", h, w),), t.uint8)
        self.ws_anchor = D.empty((N.query("glr_anchor_workspace", h, w),), t.uint8)
        self.ws_edge = D.empty((64,), t.uint8)
        # heat map chunking over exemplars (the heat map is never communicated)
        # heat map + top-K, chunked over exemplars beyond the memory budget.
        # Default: the dense u16 map (glr_heat_map + glr_topk, faster on B200).
        # low_memory_match: the fused glr_heat_topk -- per-exemplar candidate
        # lists of `cand_cap` entries instead of the map (8x less memory); the
        # dense path runs only for the exemplars it hands back.
        self.heat_budget = heat_budget_bytes
        import os
        mode = os.environ.get("GLR_MATCH_MODE", "")  # dev A/B switch: dense | fused
        if mode in ("dense", "fused"):
            low_memory_match = mode == "fused"
        if low_memory_match is None:
            # auto: the fused path (candidate lists, no dense map) wherever the
            # dense map would be large -- measured per refresh: C5 P = 8, 16k
            # exemplars 43 vs 127 ms, C2 11.1 vs 11.7 ms; for maps of ~1 GB and
            # below the dense map + single-pass top-K is as fast or faster
            # (C4 105.7 vs 105.0 ms per solve, C1 26.8 vs 24.7) and C3's sparse
            # phantom maps (the pool reaches score 0) fall back anyway
            p_ = match.patch_size
            g_ = 3 * match.exemplar_stride
            n_est = match.max_corners + ((h - p_) // g_ + 1) * ((w - p_) // g_ + 1)
            low_memory_match = n_est * (h - p_ + 1) * (w - p_ + 1) * 2 > (4 << 30)
        self.low_memory_match = bool(low_memory_match)
        self.heat = None
        self.ws_dense = None
        self.n_fallback = 0     # exemplars that took the dense path (last refresh)
        if not self.global_match:
            pass
        elif self.low_memory_match:
            # list capacity: 32 pool-sizes (the sampled floor aims at ~8), and
            # room for the 32-row sampled pre-pass it aliases
            pool = self.k * (2 * match.sep + 1) ** 2 + 1
            self.cand_cap = int(min(max(32 * pool, 8192, -(-32 * self.ow // 4)),
                                    self.oh * self.ow, 1 << 17))
            per = 8 * self.cand_cap + N.query("glr_heat_topk_workspace", c, p, 1, 0)
            self.heat_chunk = max(1, min(self.max_anchors, heat_budget_bytes // per))
            self.ws_heat = D.empty((N.query("glr_heat_topk_workspace", c, p, self.heat_chunk,
                                            self.cand_cap),), t.uint8)
            self.fallback = D.zeros((self.heat_chunk,), t.uint8)
        else:
            self.heat_chunk = max(1, min(self.max_anchors, heat_budget_bytes // (2 * self.stride)))
            self.heat = D.empty((self.heat_chunk, self.stride), t.int16)
            self.ws_dense = D.empty((N.query("glr_heat_workspace", c, p, self.heat_chunk),),
                                    t.uint8)
            self.ws_topk = D.empty((N.query("glr_topk_workspace", self.heat_chunk, self.k,
                                            match.sep),), t.uint8)
        self.ws_wnnm = D.empty((N.query("glr_wnnm_workspace", self.max_anchors, self.k),),
                               t.uint8)
        # per-group Jacobi eigenvectors, warm start between refreshes
        # (double-buffered so a refresh can carry them over by anchor, see
        # glr_vcache_remap); warm: 0 cold, 1 all groups, 2 per-group flags
        vrows = self.max_anchors if self.use_vcache else 1
        self._vc = [D.empty((vrows, KMAX, KMAX), t.float64) for _ in range(2)]
        self._vcur = 0
        self.vcache_valid = False
        self.warm_flags = D.zeros((self.max_anchors,), t.uint8)
        self.anchor_map = D.empty((h * w,), t.int32).fill_(-1)
        self._anc = [self.anchors, D.empty((self.max_anchors, 2), t.int32)]
        self._acur = 0
        self.warm = 0
        self.timing = None  # list of (name, start, end) CUDA events when profiling
        self._side = None  # side stream for the edge stack (refresh)
        self.n = 0          # anchors in the current match state (all ranks)
        self.lo = self.hi = 0
        self.has_positions = False
        # sticky sharding state (world > 1): the anchors' owner ranks of the
        # last refresh, and the permutation from reference to shard order
        self._owner_map = None
        self._owner_flat = None
        self.perm = None

    @property
    def vcache(self):
        return self._vc[self._vcur]

    def _ev(self):
        if self.timing is None:
            return None
        e = D.torch().cuda.Event(enable_timing=True)
        e.record()
        return e

    def _log(self, name, start):
        if start is not None:
            self.timing.append((name, start, self._ev()))

    def _edge_stack_side(self):
        """glr_edge_stack on the side stream after the Sobel pass; returns the
        event the main stream waits on before matching."""
        torch = D.torch()
        h, w, c = self.shape
        main = torch.cuda.current_stream()
        if self._side is None:
            self._side = torch.cuda.Stream()
        side = self._side
        grads = torch.cuda.Event()
        grads.record(main)
        side.wait_event(grads)
        e0 = e1 = None
        if self.timing is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(side)
        N.call("glr_edge_stack", self.gh.data_ptr(), self.gv.data_ptr(), h, w, c,
               float(self.mc.edge_threshold), 1, self.expand, None, self.stack.data_ptr(),
               self.ws_edge.data_ptr(), side.cuda_stream)
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(side)
            self.timing.append((("edge_stack", 1), e0, e1))
        done = torch.cuda.Event()
        done.record(side)
        return done

    # -- refresh: solvers.py:154-167 + 187-203 ---------------------------------
    def refresh(self, x_d) -> int:
        """Exemplars, edge stack, heat map and top-K for this rank's shard.
        Returns the total anchor count."""
        h, w, c = self.shape
        mc = self.mc
        s = D.stream()
        stack_ready = None
        if self.use_corners or self.global_match:
            # one Sobel pass feeds both the corner response and the edge stack
            e = self._ev()
            N.call("glr_sobel", x_d.data_ptr(), h, w, c, self.gh.data_ptr(), self.gv.data_ptr(),
                   s)
            self._log(("sobel", 1), e)
        if self.global_match:
            # the edge stack needs only the gradients: it runs on a side stream
            # beside the corner response and the (single-CTA) greedy NMS
            stack_ready = self._edge_stack_side()
        if self.use_corners:
            e = self._ev()
            N.call("glr_corner_response_grad", self.gh.data_ptr(), self.gv.data_ptr(), h, w, c,
                   self.resp.data_ptr(), self.ws_corner.data_ptr(), s)
            self._log(("corner_response", 1), e)
            e = self._ev()
            N.call("glr_corners", self.resp.data_ptr(), h, w, mc.max_corners, mc.nms,
                   float(mc.corner_quality), self.corners.data_ptr(), self.n_corners.data_ptr(),
                   self.ws_nms.data_ptr(), self.ws_nms.numel(), s)
            self._log(("corners_nms", 1), e)
        else:
            self.n_corners.zero_()
        old_anchors, old_n, old_lo, old_hi = self.anchors, self.n, self.lo, self.hi
        self._acur ^= 1
        self.anchors = self._anc[self._acur]
        N.call("glr_select_anchors", self.corners.data_ptr(), self.n_corners.data_ptr(),
               mc.max_corners, h, w, self.p, self.grid_interval, self.max_anchors,
               self.anchors.data_ptr(), self.tags.data_ptr(), self.n_anchors.data_ptr(),
               self.ws_anchor.data_ptr(), s)
        n = int(self.n_anchors.item())  # one host sync per refresh
        self.n = n
        if self.world > 1:
            self._assign_shards(n)
        else:
            self.lo, self.hi = 0, n
        self.has_positions = True
        self.warm = 0
        carry = bool(n and old_n and self.vcache_valid and self.use_vcache)
        self.vcache_valid = False
        old_positions = self.positions
        self._pcur ^= 1
        self.positions = self._pos[self._pcur]
        if n == 0:
            return 0
        if self.global_match:
            D.torch().cuda.current_stream().wait_event(stack_ready)
            self.match_shard()
            if mc.rerank_pixel and self.hi > self.lo:
                e = self._ev()
                N.call("glr_rerank_pixel", x_d.data_ptr(), h, w, c, self.p,
                       self.positions[self.lo:self.hi].data_ptr(), self.hi - self.lo, self.k, s)
                self._log(("rerank", self.hi - self.lo), e)
        elif self.hi > self.lo:
            e = self._ev()
            N.call("glr_block_match", x_d.data_ptr(), h, w, c, self.p,
                   self.anchors[self.lo:self.hi].data_ptr(), self.hi - self.lo,
                   int(mc.bm_window), int(mc.bm_stride), self.k,
                   self.positions[self.lo:self.hi].data_ptr(),
                   self.padded[self.lo:self.hi].data_ptr(), s)
            self._log(("block_match", self.hi - self.lo), e)
        if carry:
            # groups keeping their anchor start from their old eigenvectors,
            # coordinates re-indexed to the refreshed positions
            vc_old = self._vc[self._vcur]
            self._vcur ^= 1
            N.call("glr_vcache_remap", old_anchors.data_ptr(), old_lo, old_hi,
                   self.anchors.data_ptr(), self.lo, self.hi, h, w, vc_old.data_ptr(),
                   self.vcache.data_ptr(), self.warm_flags.data_ptr(),
                   self.anchor_map.data_ptr(), old_positions.data_ptr(),
                   self.positions.data_ptr(), self.k, s)
            self.warm = 2
        self.count()
        return n

    def _assign_shards(self, n: int) -> None:
        """Sticky exemplar sharding (world > 1). An anchor that persists across
        a refresh stays on the rank that held it, so the rank finds the
        group's cached eigenvectors locally (glr_vcache_remap) and every group
        starts its Jacobi sweeps from exactly the state it has at world 1:
        the sharded solve is then bitwise identical to the single-rank one.
        New anchors fill the ranks below their n/world share in anchor order.
        Every rank computes the same assignment (identical anchors and
        history); the anchors are permuted so each rank's block is contiguous
        ([lo, hi)), and positions_host() restores the reference order."""
        h, w, _ = self.shape
        world = self.world
        anc = D.host(self.anchors[:n]).astype(np.int64)
        flat = anc[:, 0] * w + anc[:, 1]
        if self._owner_map is None:
            self._owner_map = np.full(h * w, -1, dtype=np.int32)
        owner = sticky_owners(self._owner_map[flat], world)
        perm = np.argsort(owner, kind="stable")
        bounds = np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=world))])
        self.lo, self.hi = int(bounds[self.rank]), int(bounds[self.rank + 1])
        if self._owner_flat is not None:
            self._owner_map[self._owner_flat] = -1
        self._owner_map[flat] = owner
        self._owner_flat = flat
        if np.array_equal(perm, np.arange(n)):
            self.perm = None
            return
        self.perm = perm
        perm_d = D.to_dev(perm)
        self.anchors[:n].copy_(self.anchors[:n].index_select(0, perm_d))
        self.tags[:n].copy_(self.tags[:n].index_select(0, perm_d))

    def match_shard(self):
        h, w, c = self.shape
        s = D.stream()
        t = D.torch()
        self.n_fallback = 0
        for a in range(self.lo, self.hi, self.heat_chunk):
            b = min(self.hi, a + self.heat_chunk)
            nb = b - a
            anc = self.anchors[a:b]
            if not self.low_memory_match:
                e = self._ev()
                N.call("glr_heat_map", self.stack.data_ptr(), h, w, c, self.p, self.expand,
                       anc.data_ptr(), nb, None, self.heat.data_ptr(), self.ws_dense.data_ptr(),
                       self.ws_dense.numel(), s)
                self._log(("heat_map", nb), e)
                e = self._ev()
                N.call("glr_topk", self.heat.data_ptr(), nb, None, self.oh, self.ow,
                       self.max_score, anc.data_ptr(), self.k, self.mc.sep,
                       self.positions[a:b].data_ptr(), self.padded[a:b].data_ptr(),
                       self.ws_topk.data_ptr(), self.ws_topk.numel(), s)
                self._log(("topk", nb), e)
                continue
            e = self._ev()
            N.call("glr_heat_topk", self.stack.data_ptr(), h, w, c, self.p, self.expand,
                   anc.data_ptr(), nb, self.k, self.mc.sep, self.cand_cap,
                   self.positions[a:b].data_ptr(), self.padded[a:b].data_ptr(),
                   self.fallback.data_ptr(), self.ws_heat.data_ptr(), self.ws_heat.numel(), s)
            self._log(("heat_topk", nb), e)
            fb = t.nonzero(self.fallback[:nb]).flatten()  # one host sync per chunk
            if fb.numel():
                self._dense_match(a, fb)

    def _dense_match(self, a, fb):
        """Full heat rows + glr_topk for the exemplars the fused path handed back."""
        h, w, c = self.shape
        s = D.stream()
        t = D.torch()
        self.n_fallback += int(fb.numel())
        rows = max(1, min(int(fb.numel()), self.heat_budget // (2 * self.stride)))
        if self.heat is None or self.heat.shape[0] < rows:
            self.heat = D.empty((rows, self.stride), t.int16)
            self.ws_dense = D.empty((N.query("glr_heat_workspace", c, self.p, rows),), t.uint8)
        for i in range(0, int(fb.numel()), rows):
            idx = fb[i:i + rows] + a
            nb = int(idx.numel())
            anc = self.anchors.index_select(0, idx).contiguous()
            pos = D.empty((nb, self.k, 2), t.int32)
            pad = D.empty((nb,), t.int32)
            e = self._ev()
            N.call("glr_heat_map", self.stack.data_ptr(), h, w, c, self.p, self.expand,
                   anc.data_ptr(), nb, None, self.heat.data_ptr(), self.ws_dense.data_ptr(),
                   self.ws_dense.numel(), s)
            self._log(("heat_map", nb), e)
            e = self._ev()
            N.call("glr_topk", self.heat.data_ptr(), nb, None, self.oh, self.ow, self.max_score,
                   anc.data_ptr(), self.k, self.mc.sep, pos.data_ptr(), pad.data_ptr(), None, 0,
                   s)
            self._log(("topk", nb), e)
            self.positions.index_copy_(0, idx, pos)
            self.padded.index_copy_(0, idx, pad)

    def count(self):
        h, w, c = self.shape
        self.cnt.zero_()
        nloc = self.hi - self.lo
        if nloc > 0:
            N.call("glr_scatter_count", self.positions[self.lo:self.hi].data_ptr(), nloc, None,
                   self.k, self.p, h, w, self.cnt.data_ptr(), D.stream())
        self._all_reduce(self.cnt)

    def set_positions(self, anchors: np.ndarray, positions: np.ndarray):
        """Inject a match state (positions-locked parity)."""
        n = len(anchors)
        self.n = n
        self.lo, self.hi = shard_bounds(n, self.rank, self.world)
        self.perm = None
        self.has_positions = True
        self.warm = 0
        self.vcache_valid = False
        if n:
            self.anchors[:n].copy_(D.i32(np.asarray(anchors).reshape(n, 2)))
            self.positions[:n].copy_(D.i32(np.asarray(positions).reshape(n, self.k, 2)))
        self.count()

    # -- every iteration: lowrank.py:68-87 --------------------------------------
    def regularize(self, x_d, sigma: float) -> bool:
        """acc <- fixed-point sum of WNNM-denoised patches of this shard (all-
        reduced). Returns False when there are no groups (z = x)."""
        if self.n == 0:
            return False
        h, w, c = self.shape
        if self.acc_dirty:  # a previous numerator was never consumed
            self.acc.zero_()
        self.acc_dirty = True
        nloc = self.hi - self.lo
        if nloc > 0:
            e = self._ev()
            N.call("glr_wnnm_scatter", x_d.data_ptr(), h, w, c, self.p,
                   self.positions[self.lo:self.hi].data_ptr(), nloc, None, self.k, float(sigma),
                   float(self.c_weight), float(self.eps), self.frac, self.acc.data_ptr(),
                   self.vcache[self.lo:self.hi].data_ptr() if self.use_vcache else None,
                   self.warm if self.use_vcache else 0,
                   self.warm_flags[self.lo:self.hi].data_ptr(), self.ws_wnnm.data_ptr(),
                   self.ws_wnnm.numel(), D.stream())
            self.warm = 1
            self.vcache_valid = True
            self._log(("wnnm_scatter", nloc), e)
        self._all_reduce(self.acc)
        return True

    def _all_reduce(self, t):
        # with a process group the collective always runs (also at world 1, so
        # the sharded path is the one exercised when launched under torchrun)
        if self.pg is not None:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.pg)

    def consumed(self):
        """The numerator was read by a read-and-clear consumer."""
        self.acc_dirty = False

    def positions_host(self):
        """(anchors, positions, padded) of ALL groups. Each rank computes only
        its shard's rows [lo, hi); with a process group the other rows are
        assembled by an integer all-reduce (zeros outside the local shard)."""
        n = self.n
        pos, pad = self.positions[:n], self.padded[:n]
        if self.pg is not None and self.world > 1 and n:
            pos, pad = pos.clone(), pad.clone()
            for tt in (pos, pad):
                tt[:self.lo].zero_()
                tt[self.hi:].zero_()
                self._all_reduce(tt)
        anc, pos, pad = D.host(self.anchors[:n]), D.host(pos), D.host(pad)
        if self.perm is not None:  # shard order -> the reference's anchor order
            out = [np.empty_like(a) for a in (anc, pos, pad)]
            for o, a in zip(out, (anc, pos, pad)):
                o[self.perm] = a
            anc, pos, pad = out
        return anc, pos, pad
