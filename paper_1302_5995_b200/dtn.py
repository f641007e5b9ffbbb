"""Host-side mirror of the reference's build/solve API for the hot path,
backed by the B200 engine through the C ABI (include/dtn_gpu.h).

Same names, argument meaning and error behaviour as namespace `dtn` in
/root/reference/proj/include/dtn/:
  ProblemSpec / catalog / discretize   grid.hpp:32-53,111; problems.hpp:20
  build_tree                           grid.hpp:159 (plus build_tree_uniform)
  build_root_dense_op                  accel_nd.hpp:98-100
  build_with_loads(..., Engine, ...)   bodyload.hpp:31-34 (Engine.gpu = this engine)
  SolutionOperator                     solution_operator.hpp:30-53
  apply_dtn / apply_schur / densify_dtn  solution_operator.hpp:55-63 (batched: g may be nb x batch)
  FactorizationError                   errors.hpp:11-21
Size/argument errors raise ValueError (std::invalid_argument), singular
blocks FactorizationError, device failures RuntimeError. There is no CPU
fallback.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib as L


class FactorizationError(RuntimeError):
    """A factorization step hit a (near-)singular block (errors.hpp:11-21)."""

    def __init__(self, message: str):
        super().__init__(message)
        self.where = message[message.rfind("[") + 1:-1] if message.endswith("]") else ""


class Engine(enum.IntEnum):
    dense = 0   # reference dense engine (CPU)
    accel = 1   # reference compressed engine (CPU)
    gpu = 2     # this B200 engine (dense merges on sm_100a)


class ProblemMode(enum.IntEnum):
    continuum = 0
    network = 1


Field = Optional[Callable[[np.ndarray, np.ndarray], np.ndarray]]


@dataclass
class ProblemSpec:
    """grid.hpp:32-53. Coefficient fields take vectorised (x, y) arrays."""
    name: str
    n: int
    h: float
    mode: ProblemMode = ProblemMode.continuum
    b: Field = None
    c: Field = None
    d: Field = None
    conductivity_lo: float = 1.0
    conductivity_hi: float = 1.0
    seed: int = 0

    @staticmethod
    def continuum(name: str, n: int, b: Field, c: Field, d: Field) -> "ProblemSpec":
        return ProblemSpec(name, n, 1.0 / (n - 1), ProblemMode.continuum, b, c, d)

    @staticmethod
    def network(name: str, n: int, lo: float, hi: float, seed: int) -> "ProblemSpec":
        return ProblemSpec(name, n, 1.0 / (n - 1), ProblemMode.network, conductivity_lo=lo, conductivity_hi=hi,
                           seed=seed)


def _const(v: float):
    return lambda x, y: np.full(np.broadcast(x, y).shape, float(v))


def discrete_eigenvalue(p: int, q: int, n: int) -> float:
    """problems.cpp:75-84."""
    if p < 1 or q < 1 or p > n - 2 or q > n - 2:
        raise ValueError("discrete_eigenvalue: indices out of range")
    h = 1.0 / (n - 1)
    return (4.0 - 2.0 * (math.cos(p * math.pi / (n - 1)) + math.cos(q * math.pi / (n - 1)))) / (h * h)


def discrete_eigenvalue_kth(k: int, n: int) -> float:
    """problems.cpp:86-110 (ties broken by (p, q))."""
    if k < 1:
        raise ValueError("discrete_eigenvalue_kth: k >= 1")
    cap = min(n - 2, max(2 * k, 8))
    if cap * cap < k:
        raise ValueError("discrete_eigenvalue_kth: k exceeds spectrum")
    es = sorted((discrete_eigenvalue(p, q, n), p, q) for p in range(1, cap + 1) for q in range(1, cap + 1))
    return es[k - 1][0]


CATALOG_NAMES = ["laplace", "diffconv1", "diffconv2", "diffconv3", "diffconv4", "helmholtz1", "helmholtz2",
                 "helmholtz3", "helmholtz4", "random1", "random2"]


def catalog_names():
    return list(CATALOG_NAMES)


def catalog(name: str, n: int, seed: int = 0) -> ProblemSpec:
    """problems.cpp:26-73."""
    pi = math.pi
    z = _const(0.0)
    if name == "laplace":
        return ProblemSpec.continuum(name, n, z, z, z)
    if name == "diffconv1":
        return ProblemSpec.continuum(name, n, _const(100.0), z, z)
    if name == "diffconv2":
        return ProblemSpec.continuum(name, n, _const(1000.0), z, z)
    if name == "diffconv3":
        return ProblemSpec.continuum(name, n, lambda x, y: 125.0 * np.cos(4 * pi * y) + 0 * x,
                                     lambda x, y: 125.0 * np.sin(4 * pi * x) + 0 * y, z)
    if name == "diffconv4":
        return ProblemSpec.continuum(name, n, lambda x, y: 125.0 * np.cos(4 * pi * x) + 0 * y,
                                     lambda x, y: 125.0 * np.sin(4 * pi * y) + 0 * x, z)
    if name == "helmholtz1":
        return ProblemSpec.continuum(name, n, z, z, _const(-100.0))
    if name == "helmholtz2":
        return ProblemSpec.continuum(name, n, z, z, _const(-4005.0))
    if name == "helmholtz3":
        return ProblemSpec.continuum(name, n, z, z, _const(-discrete_eigenvalue_kth(10, n) + 1e-5))
    if name == "helmholtz4":
        k = 2.0 * pi * n / 40.0
        return ProblemSpec.continuum(name, n, z, z, _const(-k * k))
    if name == "random1":
        return ProblemSpec.network(name, n, 1.0, 2.0, seed)
    if name == "random2":
        return ProblemSpec.network(name, n, 1.0, 1000.0, seed)
    raise ValueError(f"catalog: unknown problem '{name}'")


def baseline_problem(config: int, n_int: int | None = None) -> ProblemSpec:
    """BASELINE.json configs restated as ProblemSpecs (n_int = interior side,
    reference n = n_int + 2)."""
    pi = math.pi
    z = _const(0.0)
    if config == 1:
        return ProblemSpec.continuum("laplace", (n_int or 256) + 2, z, z, z)
    if config == 2:
        return ProblemSpec.continuum("helmholtz_k40", (n_int or 512) + 2, z, z, _const(-1600.0))
    if config == 3:
        k2 = 60.0 ** 2
        return ProblemSpec.continuum(
            "varcoef_k60", (n_int or 1024) + 2,
            lambda x, y: 50.0 * np.cos(4 * pi * y) + 0 * x,
            lambda x, y: 50.0 * np.sin(4 * pi * x) + 0 * y,
            lambda x, y: -k2 * (1.0 - 0.5 * np.exp(-((x - 0.5) ** 2 + (y - 0.5) ** 2) / 0.02)))
    if config == 4:
        return ProblemSpec.continuum("laplace", (n_int or 4096) + 2, z, z, z)
    if config == 5:
        return ProblemSpec.continuum("helmholtz_k100", (n_int or 2048) + 2, z, z, _const(-1.0e4))
    raise ValueError("baseline_problem: config must be 1..5")


@dataclass
class Lattice:
    """grid.hpp:56-78."""
    n: int

    def side(self) -> int:
        return self.n - 2

    def num_unknowns(self) -> int:
        return self.side() ** 2

    def unknown_id(self, x: int, y: int) -> int:
        return (y - 1) * self.side() + (x - 1)

    def point_of(self, i: int):
        return (i % self.side() + 1, i // self.side() + 1)


@dataclass
class DiscreteOperator:
    """grid.hpp:91-102, stored as the 5-point stencil: stencil[r, k] for
    r = center, east, west, north, south of unknown k."""
    n: int
    h: float
    mode: ProblemMode
    stencil: np.ndarray

    def lattice(self) -> Lattice:
        return Lattice(self.n)

    def coeff(self, row: int, col: int) -> float:
        lat = self.lattice()
        if row == col:
            return float(self.stencil[0, row])
        (px, py), (qx, qy) = lat.point_of(row), lat.point_of(col)
        for r, (dx, dy) in enumerate([(1, 0), (-1, 0), (0, 1), (0, -1)], start=1):
            if qx - px == dx and qy - py == dy:
                return float(self.stencil[r, row])
        return 0.0


def discretize(spec: ProblemSpec) -> DiscreteOperator:
    """grid.cpp:106-168 (host side; coefficient samples at (x h, y h))."""
    if spec.n < 4:
        raise ValueError("discretize: n must be >= 4")
    n, s = spec.n, spec.n - 2
    st = np.zeros((5, s * s))
    if spec.mode == ProblemMode.network:
        rc = L.lib().dtn_discretize_network(n, spec.conductivity_lo, spec.conductivity_hi, spec.seed,
                                            st.ctypes.data)
    else:
        idx = np.arange(s * s)
        px = (idx % s + 1) * spec.h
        py = (idx // s + 1) * spec.h
        arrs = []
        for f in (spec.b, spec.c, spec.d):
            v = np.zeros(s * s) if f is None else np.ascontiguousarray(np.broadcast_to(f(px, py), (s * s,)),
                                                                         dtype=np.float64)
            arrs.append(v)
        rc = L.lib().dtn_discretize_continuum(n, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                                              st.ctypes.data)
    if rc != 0:
        raise ValueError("discretize: coefficient is not finite")
    return DiscreteOperator(n, spec.h, spec.mode, st)


@dataclass
class BoxTree:
    """Tree parameters (grid.hpp:143-153); the geometry itself is realised by
    the engine (grid.cpp:213-266). leaf_side > 0: uniform power-of-two tree."""
    n: int
    n_leaf: int = 0
    leaf_side: int = 0


def build_tree(n: int, n_leaf: int) -> BoxTree:
    """grid.hpp:159."""
    if n < 4:
        raise ValueError("build_tree: n must be >= 4")
    if n_leaf < 16:
        raise ValueError("build_tree: n_leaf must be >= 16")
    return BoxTree(n, n_leaf, 0)


def build_tree_uniform(n: int, leaf_side: int) -> BoxTree:
    s = n - 2
    while s > leaf_side and s % 2 == 0:
        s //= 2
    if s != leaf_side:
        raise ValueError("build_tree: n-2 is not leaf_side * 2^L")
    return BoxTree(n, leaf_side * leaf_side, leaf_side)


@dataclass
class AccelOptions:
    """accel_nd.hpp:14-22 (build_root_accel: epsilon, crossover, hbs_leaf are used;
    rank_warn_cap and threads have no B200 meaning)."""
    epsilon: float = 1e-7
    crossover: int = 1024
    hbs_leaf: int = 64
    rank_warn_cap: int = 4096
    threads: int = 1
    # B200 structured merges: factor rank schedule (0 = engine defaults, dtn_opts.rank_base/step)
    rank_base: int = 0
    rank_step: int = 0
    structured: bool = True  # False: exact dense merges, compress only the root (round-1 engine)


@dataclass
class LevelStats:
    level: int
    max_rank: int
    bytes: int
    seconds: float
    boxes: int = 0
    flops: float = 0.0


# ------------------------------------------------------------------ context
class Context:
    """One engine context (device, stream, cached build plans)."""

    def __init__(self, device: int = 0, world: int = 1, rank: int = 0, nccl_id: bytes | None = None):
        """world > 1: one rank of a multi-GPU job (one process per GPU); the context owns
        the NCCL communicator of the collective builds (dtn_gpu_create_rank), built from
        the 128-byte unique id every rank received from rank 0 (collective_context)."""
        h = C.c_void_p()
        if world > 1 or nccl_id is not None:  # (world 1 with an id: a 1-rank communicator, loopback checks)
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("Context: a 128-byte NCCL unique id is required for world > 1")
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            rc = L.lib().dtn_gpu_create_rank(C.byref(h), device, world, rank, buf)
            what = "dtn_gpu_create_rank"
        else:
            rc = L.lib().dtn_gpu_create(C.byref(h), device)
            what = "dtn_gpu_create"
        if rc != 0:
            raise RuntimeError(f"{what} failed ({rc}): {L.lib().dtn_gpu_last_error(None).decode()}")
        self.h = h
        self.device = device
        self.world, self.rank = world, rank

    def close(self):
        if getattr(self, "h", None):
            L.lib().dtn_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        L.lib().dtn_gpu_set_stream(self.h, C.c_void_p(stream_handle) if stream_handle else None)

    @contextlib.contextmanager
    def torch_stream(self):
        """Run this context's work on torch's current stream of its device for the
        duration of the block, so engine calls that read or write torch tensors are
        ordered with the torch kernels that produce and consume them (and with the
        caching allocator's reuse of their memory). torch's legacy default stream
        (handle 0) is passed as cudaStreamLegacy (1)."""
        import torch
        h = torch.cuda.current_stream(self.device).cuda_stream or 1
        self.set_stream(h)
        try:
            yield
        finally:
            self.set_stream(None)

    def check(self, rc: int):
        if rc == 0:
            return
        msg = L.lib().dtn_gpu_last_error(self.h).decode()
        if rc == L.DTN_ESINGULAR:
            raise FactorizationError(msg)
        if rc == L.DTN_EINVAL:
            raise ValueError(msg)
        raise RuntimeError(f"dtn_gpu error {rc}: {msg}")


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = L.lib().dtn_gpu_nccl_unique_id(buf)
    if rc != 0:
        raise RuntimeError(f"dtn_gpu_nccl_unique_id failed ({rc}): {L.lib().dtn_gpu_last_error(None).decode()}")
    return bytes(buf)


def collective_context(device: int) -> Context:
    """The context of this rank of an initialised torch.distributed job: rank 0 draws the
    NCCL unique id, torch.distributed hands it to every rank (plumbing only; the build's
    collectives run in the engine's own communicator)."""
    import torch.distributed as tdist
    world, rank = tdist.get_world_size(), tdist.get_rank()
    if world == 1:
        return Context(device)
    box = [nccl_unique_id() if rank == 0 else None]
    tdist.broadcast_object_list(box, src=0)
    return Context(device, world, rank, box[0])


_contexts: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _contexts:
        _contexts[device] = Context(device)
    return _contexts[device]


class SolutionOperator:
    """solution_operator.hpp:30-53 for Engine.gpu: S and G stay in HBM; the
    dense copies S_dense / G_dense are fetched on first access."""

    def __init__(self, ctx: Context, handle: C.c_void_p, n: int, want_G: bool):
        # the boundary ids, cond estimate and statistics are fetched on first
        # access, so a build returns to the caller (and the next launch, e.g. an
        # apply, is enqueued) without further round trips through the C ABI
        self.ctx, self.h, self.n = ctx, handle, n
        self.engine = Engine.gpu
        self._S = None
        self._G = None
        self.has_G = want_G
        self.body_map = None  # F (nb x nloads) of a build with body loads (solution_operator.hpp:48)
        self.load_ids = None
        self._lazy: dict = {}

    def _fetch(self, key):
        if key in self._lazy:
            return self._lazy[key]
        if not getattr(self, "h", None):
            raise RuntimeError("SolutionOperator: the device operator was freed")
        ctx, handle = self.ctx, self.h
        if key == "nb":
            nb = C.c_int64()
            ctx.check(L.lib().dtn_gpu_boundary(handle, None, C.byref(nb)))
            v = nb.value
        elif key == "boundary":
            nb = C.c_int64(self._fetch("nb"))
            v = np.zeros(nb.value, dtype=np.int64)
            ctx.check(L.lib().dtn_gpu_boundary(handle, v.ctypes.data, C.byref(nb)))
        elif key == "cond_estimate":
            cond = C.c_double()
            ctx.check(L.lib().dtn_gpu_export(handle, None, None, C.byref(cond)))
            v = cond.value
        elif key == "build_stats":
            st = L.dtn_build_stats()
            ctx.check(L.lib().dtn_gpu_build_stats(handle, C.byref(st)))
            v = {f: getattr(st, f) for f, _ in L.dtn_build_stats._fields_}
        elif key == "level_stats":
            cnt = C.c_int32()
            ctx.check(L.lib().dtn_gpu_level_stats(handle, None, 0, C.byref(cnt)))
            arr = (L.dtn_level_stats * cnt.value)()
            ctx.check(L.lib().dtn_gpu_level_stats(handle, arr, cnt.value, C.byref(cnt)))
            v = [LevelStats(a.level, a.max_rank, a.bytes, a.seconds, a.boxes, a.flops) for a in arr]
        elif key == "kernel_stats":
            cnt = C.c_int32()
            ctx.check(L.lib().dtn_gpu_kernel_stats(handle, None, 0, C.byref(cnt)))
            karr = (L.dtn_kernel_stats * max(cnt.value, 1))()
            ctx.check(L.lib().dtn_gpu_kernel_stats(handle, karr, cnt.value, C.byref(cnt)))
            v = {k.name.decode(): dict(launches=k.launches, ms=k.ms, max_ms=k.max_ms, flops=k.flops, bytes=k.bytes)
                 for k in karr[:cnt.value]}
        else:  # pragma: no cover
            raise KeyError(key)
        self._lazy[key] = v
        return v

    boundary = property(lambda self: self._fetch("boundary"))
    cond_estimate = property(lambda self: self._fetch("cond_estimate"))
    build_stats = property(lambda self: self._fetch("build_stats"))
    level_stats = property(lambda self: self._fetch("level_stats"))
    kernel_stats = property(lambda self: self._fetch("kernel_stats"))

    def free(self):
        if getattr(self, "h", None):
            for key in ("nb", "boundary", "cond_estimate", "build_stats", "level_stats", "kernel_stats"):
                self._fetch(key)  # host-side copies outlive the device operator
            L.lib().dtn_gpu_free(self.h)
            self.h = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                L.lib().dtn_gpu_free(self.h)
                self.h = None
        except Exception:
            pass

    def boundary_size(self) -> int:
        return self._fetch("nb")

    @staticmethod
    def _host_matrix(nb: int) -> np.ndarray:
        """Column-major nb x nb host buffer, page-locked when torch can pin it
        (device-to-host copies run at full PCIe/C2C speed)."""
        try:
            import torch
            return torch.empty((nb, nb), dtype=torch.float64, pin_memory=True).numpy().T
        except Exception:  # pragma: no cover
            return np.zeros((nb, nb), order="F")

    @property
    def S_dense(self) -> np.ndarray:
        if self._S is None:
            S = self._host_matrix(self.boundary_size())
            self.ctx.check(L.lib().dtn_gpu_export(self.h, S.ctypes.data, None, None))
            self._S = S
        return self._S

    @property
    def G_dense(self) -> np.ndarray:
        if self._G is None:
            G = self._host_matrix(self.boundary_size())
            self.ctx.check(L.lib().dtn_gpu_export(self.h, None, G.ctypes.data, None))
            self._G = G
        return self._G

    def memory_bytes(self) -> int:
        """solution_operator.cpp:5-18 (dense: S and G payloads, plus the body map)."""
        nb = self.boundary_size()
        extra = 0 if self.body_map is None else 8 * self.body_map.size
        return 8 * nb * nb * (2 if self.has_G else 1) + extra

    def export_device(self, S_ptr: int | None = None, lds: int = 0, G_ptr: int | None = None, ldg: int = 0):
        """Device-to-device export of S and/or G (column-major, leading dims) into
        caller memory, ordered on torch's current stream (torch-allocated targets)."""
        with self.ctx.torch_stream():
            self.ctx.check(L.lib().dtn_gpu_export_device(self.h, S_ptr, lds, G_ptr, ldg))

    def device_ptrs(self):
        s, g, ld = C.c_void_p(), C.c_void_p(), C.c_int64()
        self.ctx.check(L.lib().dtn_gpu_device_ptrs(self.h, C.byref(s), C.byref(g), C.byref(ld)))
        return s.value, g.value, ld.value

    # per-box access to the build tree (testing aid)
    def num_boxes(self):
        cnt, depth = C.c_int32(), C.c_int32()
        self.ctx.check(L.lib().dtn_gpu_num_boxes(self.h, C.byref(cnt), C.byref(depth)))
        return cnt.value, depth.value

    def box_info(self, box: int) -> dict:
        info = (C.c_int32 * 11)()
        self.ctx.check(L.lib().dtn_gpu_box_info(self.h, box, info))
        v = list(info)
        return dict(level=v[0], parent=v[1], x0=v[2], x1=v[3], y0=v[4], y1=v[5], nb=v[6], children=v[7:11])

    def box_schur(self, box: int) -> np.ndarray:
        nb = self.box_info(box)["nb"]
        S = np.zeros((nb, nb), order="F")
        self.ctx.check(L.lib().dtn_gpu_box_schur(self.h, box, S.ctypes.data))
        return S


def shard_info(tree: BoxTree, nshards: int, shard: int) -> dict:
    """Rectangle and boundary size of shard `shard` of `nshards` (SURVEY 8e:
    2 = W|E halves, 4 = quadrants, 8 = quadrant halves). Host only."""
    rect = (C.c_int32 * 4)()
    nb = C.c_int64()
    rc = L.lib().dtn_gpu_shard_info(tree.n, tree.n_leaf, tree.leaf_side, nshards, shard, rect, C.byref(nb))
    if rc != 0:
        raise ValueError(L.lib().dtn_gpu_last_error(None).decode())
    return dict(rect=tuple(rect), nb=nb.value)


def _device_inputs(stencil_device_ptr, shard_S) -> bool:
    """Inputs in device memory (a stencil pointer or torch shard blocks): the
    build is then ordered on torch's current stream (Context.torch_stream)."""
    if stencil_device_ptr:
        return True
    return shard_S is not None and any(getattr(S, "is_cuda", False) for S in shard_S)


def _make_problem(op, tree, stencil_device_ptr=None, shard_S=None):
    """dtn_problem for the C ABI (stencil host or device; the shards' S blocks
    for a top-of-tree build). Returns (prob, keepalive)."""
    if stencil_device_ptr:
        prob = L.dtn_problem(tree.n, stencil_device_ptr, 1)
        keep = []
    else:
        if tree.n != op.n:
            raise ValueError("build: tree and operator sizes differ")
        st = np.ascontiguousarray(op.stencil, dtype=np.float64)
        prob = L.dtn_problem(op.n, st.ctypes.data, 0)
        keep = [st]
    if shard_S is not None:  # top of a sharded build: the shards' S blocks
        ptrs = (C.c_void_p * len(shard_S))()
        on_dev = None
        for i, S in enumerate(shard_S):
            try:
                import torch
                is_t = isinstance(S, torch.Tensor)
            except ImportError:  # pragma: no cover
                is_t = False
            if is_t:
                S = S.t().contiguous().t() if S.stride(0) != 1 else S  # column-major
                dev = bool(S.is_cuda)
                ptrs[i] = S.data_ptr()
            else:
                S = np.asfortranarray(S, dtype=np.float64)
                dev = False
                ptrs[i] = S.ctypes.data
            if on_dev is None:
                on_dev = dev
            elif on_dev != dev:
                raise ValueError("build: shard S blocks must all be host or all device arrays")
            keep.append(S)
        prob.shard_S = ptrs
        prob.shard_S_on_device = 1 if on_dev else 0
        keep.append(ptrs)
    return prob, keep


def build_root_gpu(op: DiscreteOperator | None, tree: BoxTree, want_G: bool = True, micro_max: int = 0,
                   ctx: Context | None = None, stencil_device_ptr: int | None = None,
                   profile: bool = False, nshards: int = 1, shard: int = -1, shard_S=None,
                   export_S: bool = False, load_ids=None, keep_boxes: bool = False,
                   accel: "AccelOptions | None" = None) -> SolutionOperator:
    """The B200 build: leaf elimination + merges + root inverse, through dtn_gpu_build.
    export_S: S arrives in a page-locked host array during the build (the copy
    overlaps the root inverse); SolutionOperator.S_dense then costs nothing.
    keep_boxes: every box's S stays readable (box_schur); otherwise box storage is
    reused level by level. accel: structured merges above accel.crossover (engine 1,
    the compressed engine's merges) with the root S dense."""
    ctx = ctx or default_context()
    prob, keep = _make_problem(op, tree, stencil_device_ptr, shard_S)
    opts = L.dtn_opts(0, tree.n_leaf, tree.leaf_side, 1 if want_G else 0, micro_max, 1 if profile else 0, 0.0, 0,
                      nshards, shard)
    opts.keep_boxes = 1 if keep_boxes else 0
    if accel is not None:
        opts.engine, opts.epsilon, opts.crossover = 1, float(accel.epsilon), int(accel.crossover)
        opts.rank_base, opts.rank_step = int(accel.rank_base), int(accel.rank_step)
    loads = None
    if load_ids is not None and len(load_ids):
        loads = np.ascontiguousarray(load_ids, dtype=np.int64)
        opts.load_ids = loads.ctypes.data
        opts.nloads = len(loads)
    S_host = None
    if export_S and shard < 0 and nshards == 1:
        s_ = tree.n - 2
        S_host = SolutionOperator._host_matrix(4 * s_ - 4 if s_ > 1 else 1)  # len(root_boundary(tree))
        opts.export_S = S_host.ctypes.data
        opts.export_lds = S_host.shape[0]
    h = C.c_void_p()
    with (ctx.torch_stream() if _device_inputs(stencil_device_ptr, shard_S) else contextlib.nullcontext()):
        ctx.check(L.lib().dtn_gpu_build(ctx.h, C.byref(prob), C.byref(opts), C.byref(h)))
    sol = SolutionOperator(ctx, h, tree.n, want_G)
    if S_host is not None:
        sol._S = S_host
    if loads is not None:
        F = np.zeros((sol.boundary_size(), len(loads)), order="F")
        ctx.check(L.lib().dtn_gpu_body_map(h, F.ctypes.data, F.shape[0], 0))
        sol.body_map = F
        sol.load_ids = loads
    return sol


def make_load_set(lattice: Lattice, points) -> np.ndarray:
    """make_load_set (bodyload.cpp:9-30): unknown ids of distinct, strictly
    interior load points (x, y)."""
    s, seen, ids = lattice.side(), set(), []
    for x, y in points:
        if not (1 <= x <= s and 1 <= y <= s) or x == 1 or y == 1 or x == s or y == s:
            raise ValueError(f"load node ({x}, {y}) is not strictly interior to the root box")
        i = lattice.unknown_id(x, y)
        if i in seen:
            raise ValueError(f"duplicate load node ({x}, {y})")
        seen.add(i)
        ids.append(i)
    return np.array(ids, dtype=np.int64)


def build_root_dense_op(op: DiscreteOperator, tree: BoxTree, loads=None) -> SolutionOperator:
    """accel_nd.hpp:98-100 (with the LoadPanel of dense_nd.hpp:29-32), executed
    by the B200 engine; with loads the result carries body_map F (nb x nloads)."""
    return build_root_gpu(op, tree, load_ids=loads)


def solve_with_load(sol: "SolutionOperator", g, fhat):
    """solve_with_load (bodyload.cpp:68-77): v = G g + F fhat."""
    v = apply_dtn(sol, g)
    fhat = np.asarray(fhat, dtype=np.float64)
    if fhat.size == 0:
        return v
    F = getattr(sol, "body_map", None)
    if F is None or F.shape[1] != fhat.shape[0]:
        raise ValueError("solve_with_load: load vector does not match the built body map")
    return v + F @ fhat


class CompressedSolutionOperator:
    """SolutionOperator (solution_operator.hpp:30-53) of the compressed engine:
    S_hbs (HbsMatrix) and G_hbs (InverseFactors) resident in HBM, in canonical
    ring order (rep_to_canonical = identity), cond_estimate from the
    reference's probe formula (accel_nd.cpp:834-841)."""

    def __init__(self, n, boundary, S_hbs, G_hbs, cond, dense_op=None, level_stats=None):
        self.engine = Engine.accel
        self.n = n
        self.boundary = boundary
        self.S_hbs, self.G_hbs = S_hbs, G_hbs
        self.rep_to_canonical = np.arange(len(boundary), dtype=np.int64)
        self.cond_estimate = cond
        self.dense_op = dense_op
        self.level_stats = list(level_stats or [])
        self.level_stats.append(LevelStats(-1, S_hbs.max_rank(), S_hbs.payload_bytes() + G_hbs.payload_bytes(), 0.0))
        self.body_map = None

    def boundary_size(self) -> int:
        return len(self.boundary)

    def memory_bytes(self) -> int:
        """solution_operator.cpp:5-18: serialized S_hbs and G_hbs.rep, plus the body map."""
        from . import hbs as _hbs
        extra = 0 if self.body_map is None else 8 * self.body_map.size
        return len(_hbs.serialize(self.S_hbs)) + len(_hbs.serialize(self.G_hbs)) + extra


def build_root_accel(op: DiscreteOperator, tree: BoxTree, opt: AccelOptions | None = None, keep_dense: bool = False,
                     ctx: Context | None = None, stencil_device_ptr: int | None = None, nshards: int = 1,
                     shard_S=None, loads=None, collective: int = 0):
    """build_root_accel (accel_nd.hpp:93-95, accel_nd.cpp:707-859) on the B200
    (dtn_gpu_build_accel): leaf elimination, dense merges below the crossover,
    structured merges above it (opt.structured), S_hbs = compress(root S, eps,
    hbs_leaf), G_hbs = invert_hbs(S_hbs). A root below the crossover stays dense
    (accel_nd.cpp:796-818): the result is then the dense SolutionOperator (with G),
    engine Engine.accel. With nshards > 1 and shard_S: the top of a subtree-sharded
    build (shard.py), compressed. collective = -2: the collective multi-GPU build
    over ctx's NCCL world (nshards = world); -3: the same split on one device."""
    from . import hbs as _hbs
    opt = opt or AccelOptions()
    ctx = ctx or default_context()
    prob, keep = _make_problem(op, tree, stencil_device_ptr, shard_S)
    n = tree.n
    opts = L.dtn_opts(1 if opt.structured else 0, tree.n_leaf, tree.leaf_side, 0, 0, 0, float(opt.epsilon),
                      int(opt.crossover), nshards, collective if collective else -1)
    opts.rank_base, opts.rank_step = int(opt.rank_base), int(opt.rank_step)
    load_arr = None
    if loads is not None and len(loads):
        load_arr = np.ascontiguousarray(loads, dtype=np.int64)
        opts.load_ids = load_arr.ctypes.data
        opts.nloads = len(load_arr)
    hop, hs, hg, cond = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_double()
    with (ctx.torch_stream() if _device_inputs(stencil_device_ptr, shard_S) else contextlib.nullcontext()):
        ctx.check(L.lib().dtn_gpu_build_accel(ctx.h, C.byref(prob), C.byref(opts), int(opt.hbs_leaf), C.byref(hop),
                                              C.byref(hs), C.byref(hg), C.byref(cond)))
    dense = SolutionOperator(ctx, hop, n, not hs.value)
    if not hs.value:  # dense root
        dense.engine = Engine.accel
        if load_arr is not None:
            F = np.zeros((dense.boundary_size(), len(load_arr)), order="F")
            ctx.check(L.lib().dtn_gpu_body_map(hop, F.ctypes.data, F.shape[0], 0))
            dense.body_map, dense.load_ids = F, load_arr
        return dense
    S_hbs = _hbs.HbsMatrix(ctx, hs)
    G_hbs = _hbs.InverseFactors(ctx, hg)
    out = CompressedSolutionOperator(n, dense.boundary.copy(), S_hbs, G_hbs, cond.value,
                                     dense if keep_dense else None, dense.level_stats)
    out.build_stats = dense.build_stats
    if load_arr is not None:  # body map F = G_hbs rhs_root (accel_nd.cpp:848-855), formed on the device
        R = np.zeros((dense.boundary_size(), len(load_arr)), order="F")
        ctx.check(L.lib().dtn_gpu_root_rhs(hop, R.ctypes.data, R.shape[0], 0))
        out.body_map, out.load_ids = _hbs.apply(G_hbs, R), load_arr
    if not keep_dense:
        dense.free()
    return out


def build_with_loads(op: DiscreteOperator, tree: BoxTree, loads, engine: Engine, opt: AccelOptions | None = None):
    """bodyload.cpp:47-57 dispatcher; Engine.gpu (and Engine.dense, which the
    B200 engine executes) build here; Engine.accel builds the compressed root
    (build_root_accel); its body map is G_hbs rhs_root."""
    if engine == Engine.accel:
        return build_root_accel(op, tree, opt, loads=loads)
    return build_root_dense_op(op, tree, loads)


def _apply(sol: SolutionOperator, which: int, g):
    nb = sol.boundary_size()
    try:
        import torch
        is_t = isinstance(g, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_t = False
    if is_t:
        if g.dtype != torch.float64 or not g.is_cuda:
            raise ValueError("apply: torch input must be a float64 CUDA tensor")
        vec = g.dim() == 1
        X = g.reshape(nb, -1) if vec else g
        if X.shape[0] != nb:
            raise ValueError("apply_dtn: boundary vector size mismatch")
        Xf = X.t().contiguous().t() if X.stride(0) != 1 else X
        Y = torch.empty((X.shape[1], nb), dtype=torch.float64, device=g.device).t()
        with sol.ctx.torch_stream():
            sol.ctx.check(L.lib().dtn_gpu_apply(sol.h, which, Xf.data_ptr(), Xf.stride(1) if Xf.shape[1] > 1 else nb,
                                                Xf.shape[1], Y.data_ptr(), nb, 1))
        return Y.reshape(nb) if vec else Y
    X = np.asarray(g, dtype=np.float64)
    vec = X.ndim == 1
    if X.shape[0] != nb:
        raise ValueError(("apply_dtn" if which == 0 else "apply_schur") + ": boundary vector size mismatch")
    X2 = np.asfortranarray(X.reshape(nb, -1))
    Y = np.zeros_like(X2, order="F")
    sol.ctx.check(L.lib().dtn_gpu_apply(sol.h, which, X2.ctypes.data, nb, X2.shape[1], Y.ctypes.data, nb, 0))
    return Y[:, 0].copy() if vec else Y


def _apply_hbs(sol, H, g, name):
    from . import hbs as _hbs
    shape = getattr(g, "shape", None) or np.shape(g)
    if len(shape) == 0 or shape[0] != sol.boundary_size():
        raise ValueError(name + ": boundary vector size mismatch")
    return _hbs.apply(H, g)  # rep order = canonical order


def apply_dtn(sol: SolutionOperator, g):
    """v = G g (solution_operator.cpp:36-44); g may be (nb,) or (nb, batch).
    Compressed operators apply G_hbs (apply_inverse)."""
    if getattr(sol, "G_hbs", None) is not None:
        return _apply_hbs(sol, sol.G_hbs, g, "apply_dtn")
    return _apply(sol, 0, g)


def apply_schur(sol: SolutionOperator, g):
    """S g (solution_operator.cpp:46-52)."""
    if getattr(sol, "S_hbs", None) is not None:
        return _apply_hbs(sol, sol.S_hbs, g, "apply_schur")
    return _apply(sol, 1, g)


def densify_dtn(sol: SolutionOperator) -> np.ndarray:
    """solution_operator.cpp:54-66 (compressed: G_hbs applied to the identity)."""
    if getattr(sol, "G_hbs", None) is not None:
        return _apply_hbs(sol, sol.G_hbs, np.eye(sol.boundary_size()), "densify_dtn")
    return sol.G_dense


def ring_nodes(n: int):
    """Non-corner nodes of the Dirichlet ring in ring_id order (grid.cpp:40-47:
    counterclockwise from (0, 0)): ids, positions, the adjacent unknown and the
    stencil direction (1=E, 2=W, 3=N, 4=S) from that unknown to the ring node."""
    m = n - 1
    ids, pos, adj, dirs = [], [], [], []
    s = n - 2
    for rid in range(4 * m):
        if rid % m == 0:
            continue  # corners couple to no unknown
        if rid < m:
            x, y, ax, ay, d = rid, 0, rid, 1, 4
        elif rid < 2 * m:
            x, y, ax, ay, d = m, rid - m, m - 1, rid - m, 1
        elif rid < 3 * m:
            x, y, ax, ay, d = m - (rid - 2 * m), m, m - (rid - 2 * m), m - 1, 3
        else:
            x, y, ax, ay, d = 0, m - (rid - 3 * m), 1, m - (rid - 3 * m), 2
        ids.append(rid)
        pos.append((x, y))
        adj.append((ay - 1) * s + (ax - 1))
        dirs.append(d)
    return np.array(ids), pos, np.array(adj, dtype=np.int64), np.array(dirs)


def ring_dtn(sol: "SolutionOperator", op: DiscreteOperator, device: bool = False):
    """Dirichlet-ring DtN map T = (1/h)(I + P G D_b) on the 4 n_int non-corner
    ring nodes (SURVEY f-1; derived from A u = -D g, grid.hpp:88-90, since the
    reference itself stops at G): T g is the one-sided normal derivative
    (g_i - u_adj(i)) / h of the solution with ring data g. Computed on the GPU
    from the resident G; returns a host array, or a CUDA tensor with device."""
    if op.n != sol.n:
        raise ValueError("ring_dtn: operator and solution sizes differ")
    _, _, adj_uid, dirs = ring_nodes(op.n)
    where = np.full(int(sol.boundary.max()) + 1, -1, dtype=np.int64)
    where[sol.boundary] = np.arange(len(sol.boundary))
    adj = np.ascontiguousarray(where[adj_uid])
    coef = np.ascontiguousarray(op.stencil[dirs, adj_uid], dtype=np.float64)
    m = len(adj)
    if device:
        import torch
        T = torch.empty((m, m), dtype=torch.float64, device="cuda").t()
        with sol.ctx.torch_stream():
            sol.ctx.check(L.lib().dtn_gpu_ring_dtn(sol.h, adj.ctypes.data, coef.ctypes.data, m, op.h, T.data_ptr(), m,
                                                   1))
        return T
    T = np.zeros((m, m), order="F")
    sol.ctx.check(L.lib().dtn_gpu_ring_dtn(sol.h, adj.ctypes.data, coef.ctypes.data, m, op.h, T.ctypes.data, m, 0))
    return T


def dump_schur(S: np.ndarray, path: str) -> None:
    """dense_nd.cpp:227-237: int64 rows, int64 cols, then the matrix row-major."""
    S = np.asarray(S, dtype=np.float64)
    with open(path, "wb") as f:
        np.array([S.shape[0], S.shape[1]], dtype="<i8").tofile(f)
        np.ascontiguousarray(S, dtype="<f8").tofile(f)


def load_schur(path: str) -> np.ndarray:
    """dense_nd.cpp:239-251 (column-major result, like the Eigen Matrix)."""
    with open(path, "rb") as f:
        head = np.fromfile(f, dtype="<i8", count=2)
        if head.size != 2:
            raise RuntimeError("load_schur: truncated file " + path)
        rows, cols = int(head[0]), int(head[1])
        data = np.fromfile(f, dtype="<f8", count=rows * cols)
    if data.size != rows * cols:
        raise RuntimeError("load_schur: truncated file " + path)
    return np.asfortranarray(data.reshape(rows, cols))


def root_boundary(tree: BoxTree) -> np.ndarray:
    """Canonical CCW ring of root unknowns (grid.cpp:185-188)."""
    s = tree.n - 2
    if s == 1:
        return np.array([0], dtype=np.int64)
    pts = [(x, 1) for x in range(1, s + 1)] + [(s, y) for y in range(2, s + 1)] + \
          [(x, s) for x in range(s - 1, 0, -1)] + [(1, y) for y in range(s - 1, 1, -1)]
    return np.array([(y - 1) * s + (x - 1) for x, y in pts], dtype=np.int64)
