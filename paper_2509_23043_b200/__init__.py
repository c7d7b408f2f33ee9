"""paper_2509_23043_b200 -- B200-native TAPT verifier (parallel-tempering engine).

Python mirror of the C ABI in include/tapt_gpu.h (libtapt_b200.so, built for sm_100a by
paper_2509_23043_b200/csrc/Makefile).  The names follow the reference's C++ API
(CouplingGraph / LatticeSpec / gibbs_sweep, /root/reference/proj/include/tapt) and the
specified tempering layer (BetaLadder, swap_pass, generator_move, run_pt).

There is no CPU fallback: importing works without a GPU, but every call that sweeps,
swaps or accepts runs on the device and raises CudaError when none is present.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TAPT_LIB_PATH") or os.path.join(_HERE, "lib", "libtapt_b200.so")

ORDER_COLOUR, ORDER_REFERENCE = 0, 1
BOUNDARY_OPEN, BOUNDARY_PERIODIC = 0, 1


class TaptError(RuntimeError):
    status = 11


class ConfigError(TaptError):
    status = 1


class DimensionError(TaptError):
    status = 2


class ClampedSiteError(TaptError):
    status = 3


class SizeError(TaptError):
    status = 4


class GeometryError(TaptError):
    status = 5


class NumericError(TaptError):
    status = 6


class FormatError(TaptError):
    status = 7


class TrainingDivergedError(TaptError):
    status = 8


class CudaError(TaptError):
    status = 9


class NcclError(TaptError):
    status = 10


_BY_STATUS = {c.status: c for c in (ConfigError, DimensionError, ClampedSiteError, SizeError, GeometryError,
                                    NumericError, FormatError, TrainingDivergedError, CudaError, NcclError)}

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_i8p = C.POINTER(C.c_int8)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p
_f32p = C.POINTER(C.c_float)


class EnsembleDesc(C.Structure):
    _fields_ = [("n_instances", C.c_uint32), ("instance_offset", C.c_uint64), ("n_slots", C.c_uint32),
                ("betas", _f64p), ("seed", C.c_uint64), ("order", C.c_int)]


class FormerConfig(C.Structure):
    _fields_ = [("d_model", C.c_uint32), ("heads", C.c_uint32), ("ffn", C.c_uint32), ("layers", C.c_uint32),
                ("max_len", C.c_uint32), ("beta_features", C.c_uint32)]


class Schedule(C.Structure):
    _fields_ = [("n_sweeps", C.c_uint32), ("swap_every", C.c_uint32), ("measure_every", C.c_uint32),
                ("measure_from", C.c_uint64)]


_SIGS = {
    "tapt_last_error": (C.c_char_p, []),
    "tapt_version": (C.c_char_p, []),
    "tapt_device_count": (C.c_int, []),
    "tapt_set_device": (C.c_int, [C.c_int]),
    "tapt_launch_count": (C.c_ulonglong, []),
    "tapt_probe_decision_rate": (C.c_int, [C.c_int, C.c_int, C.c_uint32, _f64p, _f64p]),
    "tapt_model_create_lattice": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(_vp)]),
    "tapt_model_create_graph": (C.c_int, [C.c_uint32, C.c_uint32, _u32p, _u32p, _f64p, _f64p, _i8p, C.POINTER(_vp)]),
    "tapt_model_destroy": (C.c_int, [_vp]),
    "tapt_model_load_file": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "tapt_model_save_file": (C.c_int, [_vp, C.c_char_p]),
    "tapt_model_info": (C.c_int, [_vp, _u32p, _u32p, _u32p, _i32p, _i32p, _u32p, _u32p]),
    "tapt_model_couplings": (C.c_int, [_vp, _u32p, _u32p, _f64p]),
    "tapt_model_schedule": (C.c_int, [_vp, _i32p, _i32p]),
    "tapt_model_digest": (C.c_int, [_vp, _u64p]),
    "tapt_model_energy": (C.c_int, [_vp, _i8p, C.c_size_t, _f64p]),
    "tapt_gibbs_sweep": (C.c_int, [_vp, _i8p, C.c_size_t, C.c_double, _u64p, C.c_uint32, _f64p]),
    "tapt_ensemble_create": (C.c_int, [_vp, C.POINTER(EnsembleDesc), C.POINTER(_vp)]),
    "tapt_ensemble_destroy": (C.c_int, [_vp]),
    "tapt_ensemble_set_stream": (C.c_int, [_vp, _vp]),
    "tapt_ensemble_synchronize": (C.c_int, [_vp]),
    "tapt_ensemble_kernel": (C.c_char_p, [_vp]),
    "tapt_ensemble_launch_log": (C.c_int, [_vp, C.c_char_p, C.c_size_t]),
    "tapt_ensemble_set_bond_signs": (C.c_int, [_vp, _i8p, C.c_size_t]),
    "tapt_ensemble_generate_ea_disorder": (C.c_int, [_vp, C.c_uint64]),
    "tapt_ensemble_get_bond_signs": (C.c_int, [_vp, _i8p, C.c_size_t]),
    "tapt_ensemble_set_clamps": (C.c_int, [_vp, _i8p]),
    "tapt_ensemble_init_random": (C.c_int, [_vp]),
    "tapt_ensemble_set_spins": (C.c_int, [_vp, _i8p]),
    "tapt_ensemble_get_spins": (C.c_int, [_vp, _i8p]),
    "tapt_ensemble_get_spins_packed": (C.c_int, [_vp, _u8p]),
    "tapt_ensemble_get_energies": (C.c_int, [_vp, _i64p]),
    "tapt_ensemble_get_permutation": (C.c_int, [_vp, _u8p]),
    "tapt_ensemble_counters": (C.c_int, [_vp, _u64p, _u64p, _u64p]),
    "tapt_get_acceptance": (C.c_int, [_vp, _u64p, _u64p, _u64p, _u64p]),
    "tapt_get_observables": (C.c_int, [_vp, _i64p]),
    "tapt_set_histogram": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_uint32]),
    "tapt_get_histogram": (C.c_int, [_vp, _vp, C.c_int]),
    "tapt_get_best": (C.c_int, [_vp, _i64p]),
    "tapt_reset_observables": (C.c_int, [_vp]),
    "tapt_ensemble_get_energies_f64": (C.c_int, [_vp, _f64p]),
    "tapt_get_observables_f64": (C.c_int, [_vp, _f64p]),
    "tapt_get_best_f64": (C.c_int, [_vp, _f64p]),
    "tapt_ensemble_near_ties": (C.c_int, [_vp, _u64p, _u64p]),
    "tapt_gibbs_update": (C.c_int, [_vp, _i8p, C.c_size_t, C.c_uint32, C.c_double, _u64p]),
    "tapt_nccl_unique_id": (C.c_int, [_u8p, C.c_size_t]),
    "tapt_nccl_comm_create": (C.c_int, [_u8p, C.c_int, C.c_int, C.POINTER(_vp)]),
    "tapt_nccl_comm_destroy": (C.c_int, [_vp]),
    "tapt_nccl_comm_size": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "tapt_allreduce_observables": (C.c_int, [_vp, _vp, _i64p, _u64p, _i64p]),
    "tapt_allgather_best": (C.c_int, [_vp, _vp, C.c_uint64, _i64p]),
    "tapt_ensemble_set_betas": (C.c_int, [_vp, _f64p, C.c_int]),
    "tapt_ensemble_set_streams": (C.c_int, [_vp, _u64p]),
    "tapt_ensemble_init_from_streams": (C.c_int, [_vp, _u64p]),
    "tapt_sweep": (C.c_int, [_vp, C.c_uint32]),
    "tapt_swap_pass": (C.c_int, [_vp, C.c_int]),
    "tapt_run": (C.c_int, [_vp, C.POINTER(Schedule)]),
    "tapt_inject_proposals": (C.c_int, [_vp, _vp, C.c_int, _u32p, C.c_uint32, _f64p, _f64p, _u8p]),
    "tapt_inject_proposals_packed": (C.c_int, [_vp, _vp, C.c_int, _u32p, C.c_uint32, _u8p]),
    "tapt_inject_proposals_packed_refined": (C.c_int, [_vp, _vp, C.c_int, _u32p, C.c_uint32, C.c_uint32, _u8p]),
    "tapt_generate_proposals": (C.c_int, [_vp, _u32p, C.c_uint32, _f64p, C.c_uint32, _u8p]),
    "tapt_problem_last_error": (C.c_char_p, []),
    "tapt_multiplier_spins": (C.c_uint32, [C.c_uint32]),
    "tapt_multiplier_build": (C.c_int, [C.c_uint32, _u32p, _u32p, _u32p, _f64p, _f64p, _i8p, _u32p]),
    "tapt_multiplier_forward": (C.c_int, [C.c_uint32, C.c_uint64, C.c_uint64, _i8p]),
    "tapt_multiplier_clamps": (C.c_int, [C.c_uint32, C.c_uint64, _i8p]),
    "tapt_multiplier_decode": (C.c_int, [C.c_uint32, _i8p, C.c_uint64, _u64p, _u64p, C.POINTER(C.c_int)]),
    "tapt_enumerate_semiprimes": (C.c_int, [C.c_uint32, _u64p, C.c_uint32, _u32p]),
    "tapt_random_semiprime": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, _u64p, _u64p]),
    "tapt_former_param_count": (C.c_size_t, [C.POINTER(FormerConfig)]),
    "tapt_former_init_params": (C.c_int, [C.POINTER(FormerConfig), C.c_uint64, C.c_double, _f32p]),
    "tapt_former_create": (C.c_int, [C.POINTER(FormerConfig), _f32p, C.POINTER(_vp)]),
    "tapt_former_destroy": (C.c_int, [_vp]),
    "tapt_former_get": (C.c_int, [_vp, C.POINTER(FormerConfig), _f32p]),
    "tapt_former_save": (C.c_int, [_vp, C.c_char_p]),
    "tapt_former_load": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
    "tapt_former_log_prob": (C.c_int, [_vp, _u8p, C.c_uint32, C.c_uint32, _f64p, C.c_uint32, _f64p, _f32p]),
    "tapt_former_set_kv_bf16": (C.c_int, [_vp, C.c_int]),
    "tapt_former_set_tensor_cores": (C.c_int, [_vp, C.c_int]),
    "tapt_former_sample": (C.c_int, [_vp, C.c_uint32, C.c_uint32, _f64p, _u8p, C.c_uint32, _u64p, _u8p, _f64p]),
}

_lib = None


def lib():
    """Load libtapt_b200.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `make -C paper_2509_23043_b200/csrc` "
                              "(or __graft_entry__.build()); the TAPT engine has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _check(status, problem=False):
    if status != 0:
        f = lib().tapt_problem_last_error if problem else lib().tapt_last_error
        msg = f().decode(errors="replace")
        raise _BY_STATUS.get(status, TaptError)(msg)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def device_count() -> int:
    return int(lib().tapt_device_count())


def set_device(device: int):
    """Make `device` current for the native library on this thread (one process per GPU)."""
    _check(lib().tapt_set_device(int(device)))


def launch_count() -> int:
    """Kernels launched by libtapt_b200.so in this process."""
    return int(lib().tapt_launch_count())


def probe_decision_rate(blocks_per_sm=1, threads=512, iters=2000):
    """Measured decisions/s of the bare per-update ALU work (roofline denominator)."""
    r, sec = C.c_double(), C.c_double()
    _check(lib().tapt_probe_decision_rate(blocks_per_sm, threads, iters, C.byref(r), C.byref(sec)))
    return r.value, sec.value


# ------------------------------------------------------------------- models --

class Model:
    """A device-resident Ising problem (CouplingGraph, spin_model.hpp:30-113)."""

    def __init__(self, handle, kind):
        self._h = handle
        self.kind = kind
        n, nf, nc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        lo, hi, nco, nlv = C.c_int32(), C.c_int32(), C.c_uint32(), C.c_uint32()
        _check(lib().tapt_model_info(self._h, C.byref(n), C.byref(nf), C.byref(nc), C.byref(lo), C.byref(hi),
                                     C.byref(nco), C.byref(nlv)))
        self.n_spins, self.n_free, self.n_couplings = n.value, nf.value, nc.value
        self.lmin, self.lmax, self.n_colours, self.n_levels = lo.value, hi.value, nco.value, nlv.value

    @classmethod
    def lattice(cls, dims, J=1.0, periodic=True):
        """LatticeSpec::grid2d(ly, lx) for dims=(ly, lx); grid3d(l) for dims=(l,)."""
        dims = tuple(int(x) for x in dims)
        h = _vp()
        if len(dims) == 2:
            _check(lib().tapt_model_create_lattice(2, dims[0], dims[1], 1, float(J), int(bool(periodic)), C.byref(h)))
        elif len(dims) == 1:
            _check(lib().tapt_model_create_lattice(3, dims[0], dims[0], dims[0], float(J), int(bool(periodic)),
                                                   C.byref(h)))
        else:
            raise ConfigError("dims must be (ly, lx) or (l,)")
        m = cls(h, "lattice")
        m.dims = dims
        return m

    @classmethod
    def graph(cls, n, ci, cj, J, h=None, clamp=None):
        """CouplingGraph::Builder(n).add_coupling(...).add_field(...).set_clamp(...).build()."""
        ci = np.ascontiguousarray(ci, np.uint32)
        cj = np.ascontiguousarray(cj, np.uint32)
        J = np.ascontiguousarray(J, np.float64)
        hh = None if h is None else np.ascontiguousarray(h, np.float64)
        cl = None if clamp is None else np.ascontiguousarray(clamp, np.int8)
        hdl = _vp()
        _check(lib().tapt_model_create_graph(int(n), len(ci), _p(ci, _u32p), _p(cj, _u32p), _p(J, _f64p),
                                             _p(hh, _f64p), _p(cl, _i8p), C.byref(hdl)))
        return cls(hdl, "graph")

    @classmethod
    def load_file(cls, path):
        """CouplingGraph::load_file (`isingmodel v1`)."""
        hdl = _vp()
        _check(lib().tapt_model_load_file(os.fsencode(path), C.byref(hdl)))
        return cls(hdl, "graph")

    def save_file(self, path):
        _check(lib().tapt_model_save_file(self._h, os.fsencode(path)))

    def couplings(self):
        m = self.n_couplings
        ci, cj, J = np.zeros(m, np.uint32), np.zeros(m, np.uint32), np.zeros(m)
        _check(lib().tapt_model_couplings(self._h, _p(ci, _u32p), _p(cj, _u32p), _p(J, _f64p)))
        return ci, cj, J

    def schedule(self):
        col, lev = np.zeros(self.n_spins, np.int32), np.zeros(self.n_spins, np.int32)
        _check(lib().tapt_model_schedule(self._h, _p(col, _i32p), _p(lev, _i32p)))
        return col, lev

    def digest(self) -> int:
        d = C.c_uint64()
        _check(lib().tapt_model_digest(self._h, C.byref(d)))
        return d.value

    def energy(self, s) -> float:
        s = np.ascontiguousarray(s, np.int8)
        out = C.c_double()
        _check(lib().tapt_model_energy(self._h, _p(s, _i8p), len(s), C.byref(out)))
        return out.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tapt_model_destroy(self._h)
            self._h = None


def gibbs_sweep(model: Model, s: np.ndarray, beta: float, rng_state: int, n_sweeps: int = 1):
    """Drop-in for tapt::gibbs_sweep (mcmc.cpp:30-45), on the device, index-ascending.
    Updates s in place; returns (new rng_state, per-sweep dE array)."""
    if s.dtype != np.int8 or not s.flags.c_contiguous:
        raise DimensionError("spins must be a contiguous int8 array")
    st = C.c_uint64(rng_state)
    dE = np.zeros(max(n_sweeps, 1))
    _check(lib().tapt_gibbs_sweep(model._h, _p(s, _i8p), len(s), float(beta), C.byref(st), int(n_sweeps),
                                  _p(dE, _f64p)))
    return st.value, dE[:n_sweeps]


def gibbs_update(model: Model, s: np.ndarray, site: int, beta: float, rng_state: int):
    """Drop-in for tapt::gibbs_update (mcmc.cpp:24-28), on the device: s[site] resampled in place
    with the stream's next draw; returns the new rng_state.  ClampedSiteError for a clamped site."""
    if s.dtype != np.int8 or not s.flags.c_contiguous:
        raise DimensionError("spins must be a contiguous int8 array")
    st = C.c_uint64(rng_state)
    _check(lib().tapt_gibbs_update(model._h, _p(s, _i8p), len(s), int(site), float(beta), C.byref(st)))
    return st.value


class NcclComm:
    """An NCCL communicator owned by the native library (tapt_nccl_*): rank 0 makes the 128-byte
    unique id (`NcclComm.unique_id()`), every rank passes it in (broadcast it out of band, e.g. with
    torch.distributed).  Used by `allreduce_observables` -- the end-of-run reductions of a sharded run."""

    @staticmethod
    def unique_id() -> bytes:
        buf = np.zeros(128, np.uint8)
        _check(lib().tapt_nccl_unique_id(_p(buf, _u8p), 128))
        return buf.tobytes()

    def __init__(self, uid: bytes, n_ranks: int, rank: int):
        buf = np.frombuffer(bytes(uid), np.uint8).copy()
        self._h = _vp()
        _check(lib().tapt_nccl_comm_create(_p(buf, _u8p), int(n_ranks), int(rank), C.byref(self._h)))

    def size(self) -> int:
        v = C.c_int()
        _check(lib().tapt_nccl_comm_size(self._h, C.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tapt_nccl_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def allreduce_observables(ens, comm: NcclComm):
    """Per-slot observables [R][5], per-slot histograms [R][nbins] (if configured) and the best energy,
    summed / minimised over every rank's instances with NCCL (tapt_allreduce_observables)."""
    obs = np.zeros((ens.R, 5), np.int64)
    best = np.zeros(1, np.int64)
    nb = getattr(ens, "_nbins", 0)
    hist = np.zeros((ens.R, nb), np.uint64) if nb else None
    _check(lib().tapt_allreduce_observables(ens._h, comm._h, _p(obs, _i64p), _p(hist, _u64p), _p(best, _i64p)))
    return {"obs": obs, "hist": hist, "best": int(best[0])}


def allgather_best(ens, comm: NcclComm, total: int):
    """Every rank's per-instance best energies in global instance order (tapt_allgather_best)."""
    out = np.zeros(int(total), np.int64)
    _check(lib().tapt_allgather_best(ens._h, comm._h, int(total), _p(out, _i64p)))
    return out


# ---------------------------------------------------------------- ensembles --

class Ensemble:
    """I instances x R ladder slots of replicas, device-resident."""

    def __init__(self, model: Model, betas, n_instances=1, seed=0, instance_offset=0, order="colour"):
        self.model = model
        self.betas = np.ascontiguousarray(betas, np.float64)
        self.R = len(self.betas)
        self.I = int(n_instances)
        self.n = model.n_spins
        o = {"colour": ORDER_COLOUR, "color": ORDER_COLOUR, "checkerboard": ORDER_COLOUR,
             "reference": ORDER_REFERENCE, "index": ORDER_REFERENCE}[order] if isinstance(order, str) else int(order)
        d = EnsembleDesc(self.I, int(instance_offset), self.R, _p(self.betas, _f64p), int(seed) & (2**64 - 1), o)
        self._h = _vp()
        _check(lib().tapt_ensemble_create(model._h, C.byref(d), C.byref(self._h)))
        self.kernel = lib().tapt_ensemble_kernel(self._h).decode()

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tapt_ensemble_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # -- setup
    def launch_log(self):
        """Distinct sweep-kernel instantiations launched so far (template arguments; ' balanced M=k'
        when the persistent McNaughton grid ran)."""
        buf = C.create_string_buffer(8192)
        _check(lib().tapt_ensemble_launch_log(self._h, buf, len(buf)))
        return [x for x in buf.value.decode().split("\n") if x]

    def set_stream(self, cuda_stream_ptr):
        _check(lib().tapt_ensemble_set_stream(self._h, cuda_stream_ptr))

    def synchronize(self):
        _check(lib().tapt_ensemble_synchronize(self._h))

    def set_bond_signs(self, signs):
        signs = np.ascontiguousarray(signs, np.int8).reshape(self.I, -1)
        _check(lib().tapt_ensemble_set_bond_signs(self._h, _p(signs, _i8p), signs.shape[1]))

    def generate_ea_disorder(self, seed):
        _check(lib().tapt_ensemble_generate_ea_disorder(self._h, int(seed)))

    def bond_signs(self, n_bonds):
        out = np.zeros((self.I, n_bonds), np.int8)
        _check(lib().tapt_ensemble_get_bond_signs(self._h, _p(out, _i8p), n_bonds))
        return out

    def set_clamps(self, clamps):
        clamps = np.ascontiguousarray(clamps, np.int8).reshape(self.I, self.n)
        _check(lib().tapt_ensemble_set_clamps(self._h, _p(clamps, _i8p)))

    def init_random(self):
        _check(lib().tapt_ensemble_init_random(self._h))

    def set_spins(self, spins):
        spins = np.ascontiguousarray(spins, np.int8).reshape(self.I, self.R, self.n)
        _check(lib().tapt_ensemble_set_spins(self._h, _p(spins, _i8p)))

    # -- readout
    def spins(self):
        out = np.zeros((self.I, self.R, self.n), np.int8)
        _check(lib().tapt_ensemble_get_spins(self._h, _p(out, _i8p)))
        return out

    def spins_packed(self):
        out = np.zeros((self.I, self.R, (self.n + 7) // 8), np.uint8)
        _check(lib().tapt_ensemble_get_spins_packed(self._h, _p(out, _u8p)))
        return out

    @property
    def real(self):
        """Real-valued couplings: K5 (FP64 energies and observables)."""
        return self.kernel == "real"

    def energies(self):
        """Per-slot energies: int64 for integer couplings, float64 for real-valued ones."""
        if self.real:
            out = np.zeros((self.I, self.R), np.float64)
            _check(lib().tapt_ensemble_get_energies_f64(self._h, _p(out, _f64p)))
            return out
        out = np.zeros((self.I, self.R), np.int64)
        _check(lib().tapt_ensemble_get_energies(self._h, _p(out, _i64p)))
        return out

    def near_ties(self):
        """(near-tie decisions re-evaluated with glibc exp, state replays) -- K5 only."""
        a, b = C.c_uint64(), C.c_uint64()
        _check(lib().tapt_ensemble_near_ties(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def permutation(self):
        out = np.zeros((self.I, self.R), np.uint8)
        _check(lib().tapt_ensemble_get_permutation(self._h, _p(out, _u8p)))
        return out

    def counters(self):
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().tapt_ensemble_counters(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def acceptance(self):
        np_ = max(self.R - 1, 1)
        sa, sc = np.zeros((self.I, np_), np.uint64), np.zeros((self.I, np_), np.uint64)
        pa, pc = np.zeros((self.I, self.R), np.uint64), np.zeros((self.I, self.R), np.uint64)
        _check(lib().tapt_get_acceptance(self._h, _p(sa, _u64p), _p(sc, _u64p), _p(pa, _u64p), _p(pc, _u64p)))
        return sa[:, : self.R - 1], sc[:, : self.R - 1], pa, pc

    def observables(self):
        if self.real:
            out = np.zeros((self.I, self.R, 5), np.float64)
            _check(lib().tapt_get_observables_f64(self._h, _p(out, _f64p)))
            return out
        out = np.zeros((self.I, self.R, 5), np.int64)
        _check(lib().tapt_get_observables(self._h, _p(out, _i64p)))
        return out

    def set_histogram(self, e_lo, width, nbins):
        self._nbins = int(nbins)
        _check(lib().tapt_set_histogram(self._h, int(e_lo), int(width), int(nbins)))

    def histogram(self, device_ptr=None):
        if device_ptr is not None:
            _check(lib().tapt_get_histogram(self._h, device_ptr, 1))
            return None
        out = np.zeros((self.R, self._nbins), np.uint64)
        _check(lib().tapt_get_histogram(self._h, out.ctypes.data, 0))
        return out

    def best(self):
        if self.real:
            out = np.zeros(self.I, np.float64)
            _check(lib().tapt_get_best_f64(self._h, _p(out, _f64p)))
            return out
        out = np.zeros(self.I, np.int64)
        _check(lib().tapt_get_best(self._h, _p(out, _i64p)))
        return out

    def reset_observables(self):
        _check(lib().tapt_reset_observables(self._h))

    def set_betas(self, betas, allow_flat=False):
        """allow_flat: False/0 strictly increasing, 1 non-decreasing, 2 any order (no swaps)."""
        b = np.ascontiguousarray(betas, np.float64)
        _check(lib().tapt_ensemble_set_betas(self._h, _p(b, _f64p), int(allow_flat)))
        self.betas = b

    def set_streams(self, states):
        st = np.ascontiguousarray(states, np.uint64).reshape(self.I, self.R)
        _check(lib().tapt_ensemble_set_streams(self._h, _p(st, _u64p)))

    def init_from_streams(self, init_states):
        st = np.ascontiguousarray(init_states, np.uint64).reshape(self.I, self.R)
        _check(lib().tapt_ensemble_init_from_streams(self._h, _p(st, _u64p)))

    # -- dynamics
    def sweep(self, n_sweeps=1):
        _check(lib().tapt_sweep(self._h, int(n_sweeps)))

    def swap_pass(self, parity):
        _check(lib().tapt_swap_pass(self._h, int(parity)))

    def run(self, n_sweeps, swap_every=1, measure_every=0, measure_from=0):
        s = Schedule(int(n_sweeps), int(swap_every), int(measure_every), int(measure_from))
        _check(lib().tapt_run(self._h, C.byref(s)))

    def inject_proposals(self, proposals, targets, log_q_cur=None, log_q_prop=None, device_ptr=None):
        t = np.ascontiguousarray(targets, np.uint32)
        acc = np.zeros((self.I, len(t)), np.uint8)
        if (log_q_cur is None) != (log_q_prop is None):
            raise ConfigError("log_q_cur and log_q_prop must be given together (mh_corrected_move)")
        lqc = lqp = None
        if log_q_cur is not None:  # the C ABI reads I x len(targets) doubles from each
            lqc = np.ascontiguousarray(log_q_cur, np.float64)
            lqp = np.ascontiguousarray(log_q_prop, np.float64)
            for name, v in (("log_q_cur", lqc), ("log_q_prop", lqp)):
                if v.size != self.I * len(t):
                    raise DimensionError(f"{name} has {v.size} entries, expected n_instances x n_targets = "
                                         f"{self.I} x {len(t)}")
            lqc, lqp = lqc.reshape(self.I, len(t)), lqp.reshape(self.I, len(t))
        if device_ptr is not None:
            _check(lib().tapt_inject_proposals(self._h, device_ptr, 1, _p(t, _u32p), len(t), _p(lqc, _f64p),
                                               _p(lqp, _f64p), _p(acc, _u8p)))
        else:
            p = np.ascontiguousarray(proposals, np.int8).reshape(self.I, len(t), self.n)
            _check(lib().tapt_inject_proposals(self._h, p.ctypes.data, 0, _p(t, _u32p), len(t), _p(lqc, _f64p),
                                               _p(lqp, _f64p), _p(acc, _u8p)))
        return acc

    def inject_proposals_packed(self, packed, targets, device_ptr=None, refine=0, return_accepted=True):
        """Bit-packed proposals [I][n_targets][ceil(n/8)] (host array, or device_ptr); refine > 0 runs
        that many heat-bath sweeps of each proposal at its target's beta before Eq. 2."""
        t = np.ascontiguousarray(targets, np.uint32)
        acc = np.zeros((self.I, len(t)), np.uint8) if return_accepted else None
        if device_ptr is not None:
            src, on_dev = device_ptr, 1
        else:
            p = np.ascontiguousarray(packed, np.uint8)
            if p.size != self.I * len(t) * ((self.n + 7) // 8):
                raise DimensionError("packed proposals must be [n_instances][n_targets][ceil(n/8)]")
            src, on_dev = p.ctypes.data, 0
        if refine:
            _check(lib().tapt_inject_proposals_packed_refined(self._h, src, on_dev, _p(t, _u32p), len(t), int(refine),
                                                              _p(acc, _u8p)))
        else:
            _check(lib().tapt_inject_proposals_packed(self._h, src, on_dev, _p(t, _u32p), len(t), _p(acc, _u8p)))
        return acc

    def generate_proposals(self, targets, m_bias=None, refine=5, return_accepted=True):
        """Synthetic TAPT round.  return_accepted=False keeps the round stream-ordered (no host
        sync; the per-slot counters still record every decision)."""
        t = np.ascontiguousarray(targets, np.uint32)
        mb = None if m_bias is None else np.ascontiguousarray(m_bias, np.float64)
        acc = np.zeros((self.I, len(t)), np.uint8) if return_accepted else None
        _check(lib().tapt_generate_proposals(self._h, _p(t, _u32p), len(t), _p(mb, _f64p), int(refine),
                                             _p(acc, _u8p)))
        return acc


# -------------------------------------------------------------- IsingFormer --

class Former:
    """IsingFormer proposal model on the device: forward_logits, log_prob,
    sample, save/load_checkpoint (ISFW1).  Token 1 = spin +1; parameters fp32 in the
    canonical ISFW1 order."""

    DEFAULT = dict(d_model=64, heads=2, ffn=128, layers=2, max_len=1024, beta_features=16)

    def __init__(self, params=None, seed=0, scale=1.0, _handle=None, kv="fp32", **cfg):
        """kv: K/V cache precision, "fp32" (default) or "bf16" (half the bytes of the sampling-bound
        K/V stream; fp32 attention math)."""
        if kv not in ("fp32", "bf16"):
            raise ConfigError("kv must be 'fp32' or 'bf16'")
        self.kv = kv
        if _handle is not None:
            self._h = _handle
            c = FormerConfig()
            _check(lib().tapt_former_get(self._h, C.byref(c), None))
            self.config = {k: getattr(c, k) for k, _ in FormerConfig._fields_}
            if kv == "bf16":
                _check(lib().tapt_former_set_kv_bf16(self._h, 1))
            return
        conf = dict(self.DEFAULT)
        conf.update(cfg)
        self.config = conf
        c = FormerConfig(**conf)
        if params is None:
            params = Former.init_params(seed=seed, scale=scale, **conf)
        p = np.ascontiguousarray(params, np.float32)
        if len(p) != Former.param_count(**conf):
            raise DimensionError("parameter vector length does not match the configuration")
        h = _vp()
        _check(lib().tapt_former_create(C.byref(c), _p(p, _f32p), C.byref(h)))
        self._h = h
        if kv == "bf16":
            _check(lib().tapt_former_set_kv_bf16(self._h, 1))

    def set_tensor_cores(self, on=True):
        """log_prob's dense products on tcgen05 (default) or on the fp32 CUDA-core row engine."""
        _check(lib().tapt_former_set_tensor_cores(self._h, 1 if on else 0))

    @staticmethod
    def param_count(**cfg):
        conf = dict(Former.DEFAULT)
        conf.update(cfg)
        return int(lib().tapt_former_param_count(C.byref(FormerConfig(**conf))))

    @staticmethod
    def init_params(seed=0, scale=1.0, **cfg):
        conf = dict(Former.DEFAULT)
        conf.update(cfg)
        c = FormerConfig(**conf)
        p = np.zeros(int(lib().tapt_former_param_count(C.byref(c))), np.float32)
        _check(lib().tapt_former_init_params(C.byref(c), int(seed), float(scale), _p(p, _f32p)))
        return p

    @property
    def cfg_tuple(self):
        c = self.config
        return (c["d_model"], c["heads"], c["ffn"], c["layers"], c["beta_features"])

    def params(self):
        p = np.zeros(Former.param_count(**self.config), np.float32)
        _check(lib().tapt_former_get(self._h, None, _p(p, _f32p)))
        return p

    def save(self, path):
        _check(lib().tapt_former_save(self._h, str(path).encode()))

    @classmethod
    def load(cls, path):
        h = _vp()
        _check(lib().tapt_former_load(str(path).encode(), C.byref(h)))
        return cls(_handle=h)

    def log_prob(self, tokens, betas, n_prefix=0, return_logits=False):
        t = np.ascontiguousarray(tokens, np.uint8)
        if t.ndim == 1:
            t = t[None, :]
        B, T = t.shape
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(betas, np.float64), (B,)))
        lq = np.zeros(B)
        z = np.zeros((B, T), np.float32) if return_logits else None
        _check(lib().tapt_former_log_prob(self._h, _p(t, _u8p), B, T, _p(b, _f64p), int(n_prefix), _p(lq, _f64p),
                                          _p(z, _f32p)))
        return (lq, z) if return_logits else lq

    def sample(self, B, T, betas, streams, prefix=None):
        b = np.ascontiguousarray(np.broadcast_to(np.asarray(betas, np.float64), (B,)))
        s = np.ascontiguousarray(streams, np.uint64)
        if prefix is None:
            pre, npre = None, 0
        else:
            pre = np.ascontiguousarray(prefix, np.uint8).reshape(B, -1)
            npre = pre.shape[1]
        tok = np.zeros((B, T), np.uint8)
        lq = np.zeros(B)
        _check(lib().tapt_former_sample(self._h, B, T, _p(b, _f64p), _p(pre, _u8p), npre, _p(s, _u64p),
                                        _p(tok, _u8p), _p(lq, _f64p)))
        return tok, lq

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.tapt_former_destroy(self._h)
            self._h = None


# ------------------------------------------------------------- problem suite --

class Multiplier:
    """build_multiplier(n): 3n^2+n spins, AND gates + full adders with
    spin identification; product bits and carry-ins clamped."""

    def __init__(self, n):
        self.n = int(n)
        self.n_spins = int(lib().tapt_multiplier_spins(self.n))
        m = C.c_uint32()
        _check(lib().tapt_multiplier_build(self.n, C.byref(m), None, None, None, None, None, None), True)
        k = m.value
        self.ci, self.cj = np.zeros(k, np.uint32), np.zeros(k, np.uint32)
        self.J, self.h = np.zeros(k), np.zeros(self.n_spins)
        self.clamp = np.zeros(self.n_spins, np.int8)
        self.wires = np.zeros(5 * self.n, np.uint32)
        _check(lib().tapt_multiplier_build(self.n, C.byref(m), _p(self.ci, _u32p), _p(self.cj, _u32p),
                                           _p(self.J, _f64p), _p(self.h, _f64p), _p(self.clamp, _i8p),
                                           _p(self.wires, _u32p)), True)
        n_ = self.n
        self.A, self.B = self.wires[:n_], self.wires[n_:2 * n_]
        self.C, self.carry = self.wires[2 * n_:4 * n_], self.wires[4 * n_:]

    def model(self):
        return Model.graph(self.n_spins, self.ci, self.cj, self.J, self.h, self.clamp)

    def forward(self, a, b):
        s = np.zeros(self.n_spins, np.int8)
        _check(lib().tapt_multiplier_forward(self.n, int(a), int(b), _p(s, _i8p)), True)
        return s

    def clamps(self, product):
        c = np.zeros(self.n_spins, np.int8)
        _check(lib().tapt_multiplier_clamps(self.n, int(product), _p(c, _i8p)), True)
        return c

    def decode(self, s, product):
        s = np.ascontiguousarray(s, np.int8)
        a, b, ok = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(lib().tapt_multiplier_decode(self.n, _p(s, _i8p), int(product), C.byref(a), C.byref(b),
                                            C.byref(ok)), True)
        return a.value, b.value, bool(ok.value)


def enumerate_semiprimes(n):
    cnt = C.c_uint32()
    _check(lib().tapt_enumerate_semiprimes(int(n), None, 0, C.byref(cnt)), True)
    out = np.zeros(cnt.value, np.uint64)
    _check(lib().tapt_enumerate_semiprimes(int(n), _p(out, _u64p), cnt.value, C.byref(cnt)), True)
    return out


def random_semiprime(seed, gid, bits=16):
    p, q = C.c_uint64(), C.c_uint64()
    _check(lib().tapt_random_semiprime(int(seed), int(gid), int(bits), C.byref(p), C.byref(q)), True)
    return p.value, q.value


def residual_energy(energies, e_gnd, n_spins, best_so_far=False):
    """residual_energy (the C++ tapt::residual_energy): rho(t) = (<E(t)>_runs - E_gnd) / N,
    energies[run][t] = the coldest replica's energy after global move t of each run (or, with
    best_so_far, each run's best energy up to t: the non-increasing variant).  e_gnd: scalar, or one
    reference energy per run (config 3: each instance's best over the whole run)."""
    E = np.asarray(energies, np.float64)
    if E.ndim != 2 or E.shape[0] == 0:
        raise DimensionError("energies must be [runs][moves] with at least one run")
    if n_spins <= 0:
        raise ConfigError("n_spins must be > 0")
    if best_so_far:
        E = np.minimum.accumulate(E, axis=1)
    g = np.asarray(e_gnd, np.float64)
    g = g.reshape(-1, 1) if g.ndim == 1 else g
    return ((E - g).mean(axis=0)) / float(n_spins)


def estimate_ground_energy(model, restarts, sweeps, seed, beta_start=0.1, beta_end=5.0, stages=50,
                           n_instances=1, instance_offset=0, signs=None, disorder_seed=None, clamps=None):
    """estimate_ground_energy: best energy over `restarts` geometric-annealing
    runs of `sweeps` sweeps each, on the device (restarts = slots of one ensemble, all at the
    same beta per stage, no swaps; streams keyed by derive(seed,{kAnneal}) as the root)."""
    R = int(restarts)
    if R > 256:
        raise ConfigError("at most 256 restarts per call")
    root = derive_state(seed, [0x55])
    ens = Ensemble(model, beta_start + np.arange(R, dtype=np.float64), n_instances, root, instance_offset)
    if signs is not None:
        ens.set_bond_signs(signs)
    elif disorder_seed is not None:
        ens.generate_ea_disorder(disorder_seed)
    if clamps is not None:
        ens.set_clamps(clamps)
    ens.init_random()
    per = max(1, int(sweeps) // int(stages))
    for k in range(int(stages)):
        b = beta_start * (beta_end / beta_start) ** (k / max(int(stages) - 1, 1))
        ens.set_betas(np.full(R, b), allow_flat=True)
        ens.run(per, swap_every=0)
    return ens.best()



def derive_state(root, path):
    """RngStream::derive(root, path).state() (rng.hpp:21-27), host-side."""
    M = (1 << 64) - 1
    PHI = 0x9E3779B97F4A7C15

    def mix(z):
        z = (z + PHI) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    s = mix((int(root) ^ PHI) & M)
    for p in path:
        s = mix(s ^ ((int(p) + PHI) & M))
    return s


def generate_training_corpus(model, betas, per_beta, mixing_sweeps, thinning, seed):
    """generate_training_corpus (mcmc.cpp:67-84) on the device, bit-exact with the reference:
    chain b runs at betas[b] with c.seed = derive(seed,{kChain,b}).state(), initial state from
    derive(c.seed,{kInit,kChain}), dynamics derive(c.seed,{kChain}), index-ascending sweeps
    (run_chain, mcmc.cpp:47-65).  All chains advance together as the slots of one ensemble.
    Returns (beta of each record, spins [n_betas*per_beta, n]) in the reference's record order."""
    betas = np.asarray(betas, np.float64)
    nb = len(betas)
    out = np.zeros((nb, int(per_beta), model.n_spins), np.int8)
    for c0 in range(0, nb, 256):
        bs = betas[c0:c0 + 256]
        R = len(bs)
        cs = [derive_state(seed, [0x44, c0 + r]) for r in range(R)]
        ens = Ensemble(model, 0.5 + np.arange(R, dtype=np.float64), 1, 0, 0, order="reference")
        ens.set_betas(bs, allow_flat=2)
        ens.init_from_streams(np.array([[derive_state(c, [0x11, 0x44]) for c in cs]], np.uint64))
        ens.set_streams(np.array([[derive_state(c, [0x44]) for c in cs]], np.uint64))
        if mixing_sweeps:
            ens.run(int(mixing_sweeps), swap_every=0)
        for k in range(int(per_beta)):
            ens.run(int(thinning), swap_every=0)
            out[c0:c0 + R, k] = ens.spins()[0]
        ens.close()
    return np.repeat(betas, int(per_beta)), out.reshape(nb * int(per_beta), model.n_spins)
