"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (ctypes front-end of the checkers).

Loads oracle/build/libtapt_oracle.so (the C restatement, tapt_oracle.c) and, when
present, oracle/_ref/libtapt_ref.so (the unmodified reference sources + ref_shim.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.

The graph builders here restate the reference's construction rules in numpy:
  * Graph.from_couplings  -- CouplingGraph::Builder::build (spin_model.cpp:40-77):
    duplicate (i,j) summed, CSR neighbour lists ascending, free sites ascending.
  * lattice_couplings     -- LatticeSpec::graph_clamped (lattice.cpp:55-87): bonds
    to +x/+y(/+z) per site in site order; wrap bonds only when periodic and L > 2.
  * ea_signs              -- the EA +-J disorder convention of DESIGN.md section 3
    (coin per (+x,+y,+z) bond in site order from derive(seed, {0x88, gid})).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libtapt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtapt_ref.so")

PHI = 0x9E3779B97F4A7C15
TAG_INIT, TAG_REPLICA, TAG_COORD, TAG_CHAIN = 0x11, 0x22, 0x33, 0x44
TAG_DISORDER = 0x88

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_i8p = C.POINTER(C.c_int8)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


class OcGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("n_free", C.c_uint32), ("rowptr", _u32p), ("col", _u32p),
                ("J", _i32p), ("h", _i32p), ("clamp", _i8p), ("rank", _u32p)]


class OcRGraph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("n_free", C.c_uint32), ("rowptr", _u32p), ("col", _u32p),
                ("J", _f64p), ("h", _f64p), ("clamp", _i8p), ("rank", _u32p)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError(f"oracle not built: {ORACLE_SO} (run `make -C oracle oracle`)")
        L = C.CDLL(ORACLE_SO)
        L.oc_mix_final.restype = C.c_uint64
        L.oc_mix_final.argtypes = [C.c_uint64]
        L.oc_derive.restype = C.c_uint64
        L.oc_derive.argtypes = [C.c_uint64, _u64p, C.c_int]
        L.oc_draw.restype = C.c_uint64
        L.oc_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.oc_conditional_up.restype = C.c_double
        L.oc_conditional_up.argtypes = [C.c_double, C.c_double]
        L.oc_energy.restype = C.c_int64
        L.oc_energy.argtypes = [C.POINTER(OcGraph), _i8p]
        L.oc_local_field.restype = C.c_double
        L.oc_local_field.argtypes = [C.POINTER(OcGraph), _i8p, C.c_uint32]
        L.oc_random_configuration.argtypes = [C.POINTER(OcGraph), C.c_uint64, _i8p]
        L.oc_sweep.restype = C.c_int64
        L.oc_sweep.argtypes = [C.POINTER(OcGraph), _u32p, _i8p, C.c_double, C.c_uint64, C.c_uint64]
        for nm in ("oc_stream_init", "oc_stream_replica"):
            getattr(L, nm).restype = C.c_uint64
            getattr(L, nm).argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.oc_stream_coord.restype = C.c_uint64
        L.oc_stream_coord.argtypes = [C.c_uint64, C.c_uint64]
        L.oc_stream_accept.restype = C.c_uint64
        L.oc_stream_accept.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.oc_stream_proposal.restype = C.c_uint64
        L.oc_stream_proposal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64]
        L.oc_pt_init.argtypes = [C.POINTER(OcGraph), C.c_int, C.c_uint64, C.c_uint64, _i8p, _i64p]
        L.oc_pt_sweep_all.argtypes = [C.POINTER(OcGraph), _u32p, C.c_int, _f64p, C.c_uint64, C.c_uint64,
                                      C.c_uint64, _i8p, _i64p]
        L.oc_pt_swap_pass.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _i8p,
                                      C.c_size_t, _i64p, _u64p, _u64p, _u8p]
        L.oc_pt_inject.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, _u8p, _i8p, _i64p,
                                   _i8p, C.c_size_t, _i64p, _u64p, _u64p, _u8p]
        L.oc_pt_inject_mh.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, _u8p, _i8p, _i64p,
                                      _f64p, _f64p, _i8p, C.c_size_t, _i64p, _u64p, _u64p, _u8p]
        L.oc_pt_synthetic_proposals.argtypes = [C.POINTER(OcGraph), _u32p, C.c_int, _f64p, _f64p, C.c_uint64,
                                                C.c_uint64, C.c_uint64, _u8p, C.c_int, _i8p, _i64p]
        L.oc_pt_measure.argtypes = [_i8p, C.c_size_t, C.c_int, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p,
                                    C.c_int64, C.c_int64, C.c_int, _i64p]
        # real-valued couplings (tapt_oracle.c "real couplings")
        G = C.POINTER(OcRGraph)
        L.oc_renergy.restype = C.c_double
        L.oc_renergy.argtypes = [G, _i8p]
        L.oc_rlocal_field.restype = C.c_double
        L.oc_rlocal_field.argtypes = [G, _i8p, C.c_uint32]
        L.oc_rsweep.restype = C.c_double
        L.oc_rsweep.argtypes = [G, _u32p, _i8p, C.c_double, C.c_uint64, C.c_uint64]
        L.oc_rupdate.restype = C.c_int8
        L.oc_rupdate.argtypes = [G, _i8p, C.c_uint32, C.c_double, C.c_uint64]
        L.oc_rpt_init.argtypes = [G, C.c_int, C.c_uint64, C.c_uint64, _i8p, _f64p]
        L.oc_rpt_sweep_all.argtypes = [G, _u32p, C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, _i8p, _f64p]
        L.oc_rpt_swap_pass.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _i8p,
                                       C.c_size_t, _f64p, _u64p, _u64p, _u8p]
        L.oc_rpt_inject.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, _u8p, _i8p, _f64p,
                                    _i8p, C.c_size_t, _f64p, _u64p, _u64p, _u8p]
        L.oc_rpt_synthetic_proposals.argtypes = [G, _u32p, C.c_int, _f64p, _f64p, C.c_uint64, C.c_uint64,
                                                 C.c_uint64, _u8p, C.c_int, _i8p, _f64p]
        L.oc_rpt_inject_mh.argtypes = [C.c_int, _f64p, C.c_uint64, C.c_uint64, C.c_uint64, _u8p, _i8p, _f64p, _f64p,
                                       _f64p, _i8p, C.c_size_t, _f64p, _u64p, _u64p, _u8p]
        _lib = L
    return _lib


def have_ref():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise RuntimeError(f"reference build missing: {REF_SO} (run `make -C oracle ref`)")
        L = C.CDLL(REF_SO)
        L.ref_draws.argtypes = [C.c_uint64, _u64p, C.c_int, C.c_uint64, _u64p]
        L.ref_derive_state.restype = C.c_uint64
        L.ref_derive_state.argtypes = [C.c_uint64, _u64p, C.c_int]
        L.ref_graph_build.restype = C.c_void_p
        L.ref_graph_build.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _f64p, _f64p, _i8p]
        L.ref_graph_lattice.restype = C.c_void_p
        L.ref_graph_lattice.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_n.restype = C.c_uint32
        L.ref_graph_n.argtypes = [C.c_void_p]
        L.ref_graph_ncoup.restype = C.c_uint32
        L.ref_graph_ncoup.argtypes = [C.c_void_p]
        L.ref_graph_couplings.argtypes = [C.c_void_p, _u32p, _u32p, _f64p]
        L.ref_graph_digest.restype = C.c_uint64
        L.ref_graph_digest.argtypes = [C.c_void_p]
        L.ref_energy.restype = C.c_double
        L.ref_energy.argtypes = [C.c_void_p, _i8p]
        L.ref_local_field.restype = C.c_double
        L.ref_local_field.argtypes = [C.c_void_p, _i8p, C.c_uint32]
        L.ref_random_configuration.argtypes = [C.c_void_p, C.c_uint64, _u64p, C.c_int, _i8p]
        L.ref_gibbs_sweeps.argtypes = [C.c_void_p, _i8p, C.c_double, C.c_uint64, _u64p, C.c_int, C.c_uint64,
                                       _f64p]
        L.ref_run_chain.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _i8p]
        L.ref_generate_corpus.argtypes = [C.c_void_p, _f64p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_uint64, _i8p]
        L.ref_pt_run.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_uint64, C.c_int, _f64p, C.c_uint64,
                                 C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _f64p, C.c_int, C.c_uint, _i8p,
                                 _f64p, _u64p, _u64p]
        _ref = L
    return _ref


def ref_graph(g: "Graph"):
    """Build the reference's CouplingGraph (via CouplingGraph::Builder) for g; free with ref_graph_free."""
    ci = np.ascontiguousarray(g.ci, np.uint32)
    cj = np.ascontiguousarray(g.cj, np.uint32)
    J = np.ascontiguousarray(g.J, np.float64)
    h = np.ascontiguousarray(g.h, np.float64)
    cl = np.ascontiguousarray(g.clamp, np.int8)
    return ref().ref_graph_build(g.n, len(ci), _p(ci, _u32p), _p(cj, _u32p), _p(J, _f64p), _p(h, _f64p),
                                 _p(cl, _i8p))


# ------------------------------------------------------------------ RNG ----

def derive(root: int, path) -> int:
    p = np.array(list(path), dtype=np.uint64)
    return int(lib().oc_derive(root, _p(p, _u64p), len(p)))


def draw(s0: int, k: int) -> int:
    return int(lib().oc_draw(s0 & (2**64 - 1), k & (2**64 - 1)))


def threshold(beta: float, l: float) -> int:
    """ceil(conditional_up(beta, l) * 2^53): uniform() < p  <=>  (x >> 11) < threshold."""
    import math
    p = lib().oc_conditional_up(beta, l)
    return int(math.ceil(p * 2.0**53))


# ---------------------------------------------------------------- graphs ---

@dataclass
class Graph:
    n: int
    ci: np.ndarray  # merged, sorted couplings (i<j)
    cj: np.ndarray
    J: np.ndarray   # float64 (integer-valued for the device path)
    h: np.ndarray
    clamp: np.ndarray
    rowptr: np.ndarray
    col: np.ndarray
    adjJ: np.ndarray
    free: np.ndarray
    rank: np.ndarray
    _oc: object = None

    @staticmethod
    def from_couplings(n, ci, cj, J, h=None, clamp=None) -> "Graph":
        ci = np.asarray(ci, dtype=np.int64)
        cj = np.asarray(cj, dtype=np.int64)
        J = np.asarray(J, dtype=np.float64)
        a, b = np.minimum(ci, cj), np.maximum(ci, cj)
        if np.any(a == b):
            raise ValueError("self-coupling")
        key = a * n + b
        uk, inv = np.unique(key, return_inverse=True)
        Jm = np.zeros(len(uk))
        np.add.at(Jm, inv, J)
        mi, mj = (uk // n).astype(np.uint32), (uk % n).astype(np.uint32)
        h = np.zeros(n) if h is None else np.asarray(h, dtype=np.float64)
        clamp = np.zeros(n, np.int8) if clamp is None else np.asarray(clamp, dtype=np.int8)
        # CSR: neighbours ascending (lower-index first, then higher; both ascending)
        src = np.concatenate([mi, mj]).astype(np.int64)
        dst = np.concatenate([mj, mi]).astype(np.int64)
        w = np.concatenate([Jm, Jm])
        order = np.lexsort((dst, src))
        src, dst, w = src[order], dst[order], w[order]
        rowptr = np.zeros(n + 1, np.uint32)
        np.add.at(rowptr, src + 1, 1)
        rowptr = np.cumsum(rowptr).astype(np.uint32)
        free = np.nonzero(clamp == 0)[0].astype(np.uint32)
        rank = np.zeros(n, np.uint32)
        rank[free] = np.arange(len(free), dtype=np.uint32)
        return Graph(n, mi, mj, Jm, h, clamp, rowptr, dst.astype(np.uint32), w, free, rank)

    def oc(self):
        """ctypes view (cached; keeps the backing arrays alive on self)."""
        if getattr(self, "_oc", None) is not None:
            return self._oc
        self._Ji = np.ascontiguousarray(np.rint(self.adjJ).astype(np.int32))
        self._hi = np.ascontiguousarray(np.rint(self.h).astype(np.int32))
        g = OcGraph(self.n, len(self.free), _p(self.rowptr, _u32p), _p(self.col, _u32p), _p(self._Ji, _i32p),
                    _p(self._hi, _i32p), _p(self.clamp, _i8p), _p(self.rank, _u32p))
        self._oc = g
        return g

    def roc(self):
        """ctypes view with real-valued couplings and fields (cached)."""
        if getattr(self, "_roc", None) is not None:
            return self._roc
        self._Jf = np.ascontiguousarray(self.adjJ, np.float64)
        self._hf = np.ascontiguousarray(self.h, np.float64)
        self._roc = OcRGraph(self.n, len(self.free), _p(self.rowptr, _u32p), _p(self.col, _u32p),
                             _p(self._Jf, _f64p), _p(self._hf, _f64p), _p(self.clamp, _i8p), _p(self.rank, _u32p))
        return self._roc

    def colour_order(self, colours: np.ndarray) -> np.ndarray:
        """Free sites grouped by colour class (stable: ascending index inside a class)."""
        f = self.free
        return f[np.argsort(colours[f], kind="stable")].astype(np.uint32)

    def index_order(self) -> np.ndarray:
        return self.free.astype(np.uint32)


def lattice_couplings(dims, J=1.0, periodic=True):
    """Bond list of LatticeSpec::graph_clamped (lattice.cpp:55-87). dims = (ly, lx) or (l,)."""
    ci, cj = [], []
    if len(dims) == 2:
        ly, lx = dims
        for r in range(ly):
            for c in range(lx):
                i = r * lx + c
                if c + 1 < lx:
                    ci.append(i); cj.append(r * lx + c + 1)
                elif periodic and lx > 2:
                    ci.append(i); cj.append(r * lx)
                if r + 1 < ly:
                    ci.append(i); cj.append((r + 1) * lx + c)
                elif periodic and ly > 2:
                    ci.append(i); cj.append(c)
        n = ly * lx
    else:
        (l,) = dims
        idx = lambda x, y, z: x + l * (y + l * z)
        for z in range(l):
            for y in range(l):
                for x in range(l):
                    i = idx(x, y, z)
                    for d, (nx, ny, nz) in enumerate(((x + 1, y, z), (x, y + 1, z), (x, y, z + 1))):
                        c = (nx, ny, nz)[d]
                        if c < l:
                            ci.append(i); cj.append(idx(nx, ny, nz))
                        elif periodic and l > 2:
                            w = [nx, ny, nz]; w[d] = 0
                            ci.append(i); cj.append(idx(*w))
        n = l ** 3
    return n, np.array(ci, np.int64), np.array(cj, np.int64), np.full(len(ci), float(J))


def lattice_graph(dims, J=1.0, periodic=True, clamp=None) -> Graph:
    n, ci, cj, w = lattice_couplings(dims, J, periodic)
    return Graph.from_couplings(n, ci, cj, w, None, clamp)


def checkerboard_colours(dims) -> np.ndarray:
    if len(dims) == 2:
        ly, lx = dims
        r, c = np.divmod(np.arange(ly * lx), lx)
        return ((r + c) & 1).astype(np.int32)
    (l,) = dims
    i = np.arange(l ** 3)
    x, y, z = i % l, (i // l) % l, i // (l * l)
    return ((x + y + z) & 1).astype(np.int32)


def ea_signs(dims, seed: int, gid: int) -> np.ndarray:
    """+-1 per bond in lattice_couplings order for periodic L>2 lattices: the k-th
    bond of the site-ordered list (site i, direction d) takes coin k+1 of
    derive(seed, {0x88, gid}); +1 iff the top bit is set."""
    n, ci, _, _ = lattice_couplings(dims, 1.0, True)
    s0 = derive(seed, [TAG_DISORDER, gid])
    out = np.empty(len(ci), np.float64)
    for k in range(len(ci)):
        out[k] = 1.0 if (draw(s0, k + 1) >> 63) else -1.0
    return out


def ea_graph(dims, seed, gid) -> Graph:
    n, ci, cj, _ = lattice_couplings(dims, 1.0, True)
    return Graph.from_couplings(n, ci, cj, ea_signs(dims, seed, gid))


def greedy_colours(g: Graph) -> np.ndarray:
    """Greedy colouring in ascending site order (smallest colour unused by
    already-coloured neighbours), then equitable rebalancing: repeated passes in
    ascending order move a site out of a class larger than T = ceil(n_free / k)
    into the smallest class below T that none of its neighbours uses.  Clamped
    sites get colour -1.  (The reference has no colouring; this is the schedule
    of the parallel chain.)"""
    col = np.full(g.n, -1, np.int32)
    for i in range(g.n):
        if g.clamp[i]:
            continue
        used = {int(col[j]) for j in g.col[g.rowptr[i]:g.rowptr[i + 1]] if col[j] >= 0}
        c = 0
        while c in used:
            c += 1
        col[i] = c
    free = np.nonzero(col >= 0)[0]
    k = int(col.max()) + 1 if len(free) else 0
    if k > 1:
        size = np.bincount(col[free], minlength=k)
        T = -(-len(free) // k)
        changed = True
        while changed:
            changed = False
            for i in free:
                c = col[i]
                if size[c] <= T:
                    continue
                used = {int(col[j]) for j in g.col[g.rowptr[i]:g.rowptr[i + 1]] if col[j] >= 0}
                best = -1
                for d in range(k):
                    if d != c and size[d] < T and d not in used and (best < 0 or size[d] < size[best]):
                        best = d
                if best >= 0:
                    col[i] = best
                    size[c] -= 1
                    size[best] += 1
                    changed = True
    return col


# --------------------------------------------------------- PT driver (one instance) --

class PT:
    """The restated PT/TAPT ensemble of ONE instance, state stored by slot."""

    def __init__(self, g: Graph, betas, seed: int, gid: int, order: np.ndarray):
        self.g, self.gc = g, g.oc()
        self.R = len(betas)
        self.beta = np.ascontiguousarray(betas, dtype=np.float64)
        self.seed, self.gid = seed, gid
        self.order = np.ascontiguousarray(order, dtype=np.uint32)
        self.spins = np.zeros((self.R, g.n), np.int8)
        self.E = np.zeros(self.R, np.int64)
        self.T = self.P = self.Q = 0
        self.swap_att = np.zeros(max(self.R - 1, 1), np.uint64)
        self.swap_acc = np.zeros(max(self.R - 1, 1), np.uint64)
        self.prop_att = np.zeros(self.R, np.uint64)
        self.prop_acc = np.zeros(self.R, np.uint64)
        self.best = None
        self.meas = {k: np.zeros(self.R, np.int64) for k in ("cnt", "sumE", "sumE2", "sumAbsM", "sumM2")}
        self.hist = None
        lib().oc_pt_init(C.byref(self.gc), self.R, seed, gid, _p(self.spins, _i8p), _p(self.E, _i64p))
        self._best()

    def _best(self):
        m = int(self.E.min())
        self.best = m if self.best is None else min(self.best, m)

    def sweep(self):
        lib().oc_pt_sweep_all(C.byref(self.gc), _p(self.order, _u32p), self.R, _p(self.beta, _f64p), self.seed,
                              self.gid, self.T, _p(self.spins, _i8p), _p(self.E, _i64p))
        self.T += 1
        self._best()

    def swap(self, parity=None):
        parity = (self.P & 1) if parity is None else parity
        dec = np.zeros(max(self.R - 1, 1), np.uint8)
        lib().oc_pt_swap_pass(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.P, parity,
                              _p(self.spins, _i8p), self.g.n, _p(self.E, _i64p), _p(self.swap_att, _u64p),
                              _p(self.swap_acc, _u64p), _p(dec, _u8p))
        self.P += 1
        return dec

    def synthetic_proposals(self, mask, m_bias, refine):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        mb = np.ascontiguousarray(m_bias, dtype=np.float64)
        props = np.zeros_like(self.spins)
        Ep = np.zeros(self.R, np.int64)
        lib().oc_pt_synthetic_proposals(C.byref(self.gc), _p(self.order, _u32p), self.R, _p(self.beta, _f64p),
                                        _p(mb, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p), refine,
                                        _p(props, _i8p), _p(Ep, _i64p))
        return props, Ep

    def inject(self, mask, props, Ep, lq_cur=None, lq_prop=None):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        props = np.ascontiguousarray(props, dtype=np.int8)
        Ep = np.ascontiguousarray(Ep, dtype=np.int64)
        dec = np.zeros(self.R, np.uint8)
        if lq_cur is None:
            lib().oc_pt_inject(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p),
                               _p(props, _i8p), _p(Ep, _i64p), _p(self.spins, _i8p), self.g.n,
                               _p(self.E, _i64p), _p(self.prop_att, _u64p), _p(self.prop_acc, _u64p),
                               _p(dec, _u8p))
        else:
            a = np.ascontiguousarray(lq_cur, dtype=np.float64)
            b = np.ascontiguousarray(lq_prop, dtype=np.float64)
            lib().oc_pt_inject_mh(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p),
                                  _p(props, _i8p), _p(Ep, _i64p), _p(a, _f64p), _p(b, _f64p),
                                  _p(self.spins, _i8p), self.g.n, _p(self.E, _i64p), _p(self.prop_att, _u64p),
                                  _p(self.prop_acc, _u64p), _p(dec, _u8p))
        self.Q += 1
        self._best()
        return dec

    def measure(self, e_lo=0, width=1, nbins=0):
        if nbins and self.hist is None:
            self.hist = np.zeros((self.R, nbins), np.int64)
        m = self.meas
        lib().oc_pt_measure(_p(self.spins, _i8p), self.g.n, self.R, _p(self.E, _i64p), _p(m["cnt"], _i64p),
                            _p(m["sumE"], _i64p), _p(m["sumE2"], _i64p), _p(m["sumAbsM"], _i64p),
                            _p(m["sumM2"], _i64p), e_lo, width, nbins,
                            _p(self.hist, _i64p) if nbins else None)

    def run(self, n_sweeps, swap_every=1, prop_every=0, n_targets=0, m_bias=None, refine=0,
            measure_every=0, measure_from=0, e_lo=0, width=1, nbins=0):
        """The fused schedule of DESIGN.md section 3: per global sweep T:
        sweep; swap pass if swap_every | T; measure if due; proposal round if prop_every | T."""
        mask = np.zeros(self.R, np.uint8)
        mask[:n_targets] = 1
        mb = np.zeros(self.R) if m_bias is None else np.asarray(m_bias, np.float64)
        for _ in range(n_sweeps):
            self.sweep()
            T = self.T
            if swap_every and T % swap_every == 0:
                self.swap()
            if measure_every and T > measure_from and T % measure_every == 0:
                self.measure(e_lo, width, nbins)
            if prop_every and T % prop_every == 0:
                props, Ep = self.synthetic_proposals(mask, mb, refine)
                self.inject(mask, props, Ep)


class RPT:
    """PT with real-valued couplings (FP64 energies): the restated driver of tapt_oracle.c's
    "real couplings" section, one instance, state stored by slot.  Same schedule as PT.run."""

    def __init__(self, g: Graph, betas, seed: int, gid: int, order: np.ndarray):
        self.g, self.gc = g, g.roc()
        self.R = len(betas)
        self.beta = np.ascontiguousarray(betas, dtype=np.float64)
        self.seed, self.gid = seed, gid
        self.order = np.ascontiguousarray(order, dtype=np.uint32)
        self.spins = np.zeros((self.R, g.n), np.int8)
        self.E = np.zeros(self.R, np.float64)
        self.T = self.P = self.Q = 0
        self.swap_att = np.zeros(max(self.R - 1, 1), np.uint64)
        self.swap_acc = np.zeros(max(self.R - 1, 1), np.uint64)
        self.prop_att = np.zeros(self.R, np.uint64)
        self.prop_acc = np.zeros(self.R, np.uint64)
        lib().oc_rpt_init(C.byref(self.gc), self.R, seed, gid, _p(self.spins, _i8p), _p(self.E, _f64p))
        self.best = float(self.E.min())

    def sweep(self):
        lib().oc_rpt_sweep_all(C.byref(self.gc), _p(self.order, _u32p), self.R, _p(self.beta, _f64p), self.seed,
                               self.gid, self.T, _p(self.spins, _i8p), _p(self.E, _f64p))
        self.T += 1
        self.best = min(self.best, float(self.E.min()))

    def swap(self, parity=None):
        parity = (self.P & 1) if parity is None else parity
        dec = np.zeros(max(self.R - 1, 1), np.uint8)
        lib().oc_rpt_swap_pass(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.P, parity,
                               _p(self.spins, _i8p), self.g.n, _p(self.E, _f64p), _p(self.swap_att, _u64p),
                               _p(self.swap_acc, _u64p), _p(dec, _u8p))
        self.P += 1
        return dec

    def synthetic_proposals(self, mask, m_bias, refine):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        mb = np.ascontiguousarray(m_bias, dtype=np.float64)
        props = np.zeros_like(self.spins)
        Ep = np.zeros(self.R, np.float64)
        lib().oc_rpt_synthetic_proposals(C.byref(self.gc), _p(self.order, _u32p), self.R, _p(self.beta, _f64p),
                                         _p(mb, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p), refine,
                                         _p(props, _i8p), _p(Ep, _f64p))
        return props, Ep

    def inject(self, mask, props, Ep, lq_cur=None, lq_prop=None):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        props = np.ascontiguousarray(props, dtype=np.int8)
        Ep = np.ascontiguousarray(Ep, dtype=np.float64)
        dec = np.zeros(self.R, np.uint8)
        if lq_cur is not None:
            a = np.ascontiguousarray(lq_cur, np.float64)
            b = np.ascontiguousarray(lq_prop, np.float64)
            lib().oc_rpt_inject_mh(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p),
                                   _p(props, _i8p), _p(Ep, _f64p), _p(a, _f64p), _p(b, _f64p), _p(self.spins, _i8p),
                                   self.g.n, _p(self.E, _f64p), _p(self.prop_att, _u64p), _p(self.prop_acc, _u64p),
                                   _p(dec, _u8p))
            self.Q += 1
            self.best = min(self.best, float(self.E.min()))
            return dec
        lib().oc_rpt_inject(self.R, _p(self.beta, _f64p), self.seed, self.gid, self.Q, _p(mask, _u8p),
                            _p(props, _i8p), _p(Ep, _f64p), _p(self.spins, _i8p), self.g.n, _p(self.E, _f64p),
                            _p(self.prop_att, _u64p), _p(self.prop_acc, _u64p), _p(dec, _u8p))
        self.Q += 1
        self.best = min(self.best, float(self.E.min()))
        return dec

    def run(self, n_sweeps, swap_every=1, prop_every=0, n_targets=0, m_bias=None, refine=0):
        mask = np.zeros(self.R, np.uint8)
        mask[:n_targets] = 1
        mb = np.zeros(self.R) if m_bias is None else np.asarray(m_bias, np.float64)
        for _ in range(n_sweeps):
            self.sweep()
            if swap_every and self.T % swap_every == 0:
                self.swap()
            if prop_every and self.T % prop_every == 0:
                props, Ep = self.synthetic_proposals(mask, mb, refine)
                self.inject(mask, props, Ep)


def yang_m(beta: float) -> float:
    """Spontaneous magnetization of the square-lattice Ising ferromagnet (J=1)."""
    import math
    bc = 0.5 * math.log(1 + math.sqrt(2))
    if beta <= bc:
        return 0.0
    return (1.0 - math.sinh(2.0 * beta) ** -4) ** 0.125
