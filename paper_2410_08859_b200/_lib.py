"""ctypes binding of the C ABI in include/domdec_b200.h.

The shared library is built in-tree (``paper_2410_08859_b200/libdomdec_b200.so``)
by ``__graft_entry__.build()`` / ``make -C paper_2410_08859_b200/csrc``.  There is
no fallback: every solver entry point calls :func:`lib` which raises when the
library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DD_LIB_PATH selects an alternative build of the same library (debug/profiling variants)
LIB_PATH = os.environ.get("DD_LIB_PATH") or os.path.join(_HERE, "libdomdec_b200.so")

EXPORTS = [
    "dd_last_error", "dd_device_count", "dd_abi_version", "dd_grid_lse", "dd_axpb",
    "dd_newton_global", "dd_global_terms", "dd_cell_solve", "dd_cell_delta", "dd_blend_energy",
    "dd_cell_commit", "dd_assemble", "dd_energy_terms", "dd_product_init", "dd_cut_plan",
    "dd_seed_duals", "dd_cell_ws_size", "dd_reduce_rows", "dd_grid_kl", "dd_opt_gh",
    "dd_opt_set", "dd_newton_nodes", "dd_refine", "dd_prolong",
    "dd_cell_solve2", "dd_cell_cluster_ws", "dd_cell_min_blocks", "dd_sinkhorn_ws",
    "dd_sinkhorn_run", "dd_assemble_masked", "dd_energy_terms_masked", "dd_blend_parts",
    "dd_sweep_fallbacks",
    # three-axis path (csrc/vol.cu)
    "dd3_grid_ws", "dd3_grid_lse", "dd3_prolong", "dd3_cell_ws_size", "dd3_cell_solve",
    "dd3_cell_delta", "dd3_cell_commit", "dd3_gather", "dd3_cell_terms", "dd3_product_init",
    "dd3_cut_tiles", "dd3_cut_plan", "dd3_seed_duals", "dd3_sinkhorn_ws", "dd3_sinkhorn_run",
    "dd3_blend_d1", "dd3_opt_gh", "dd3_opt_set",
]

i32, i64, dbl, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p


class Geom(C.Structure):
    _fields_ = [("nx0", i32), ("nx1", i32), ("ny0", i32), ("ny1", i32),
                ("x_dx", dbl), ("x_org0", dbl), ("x_org1", dbl),
                ("y_dx", dbl), ("y_org0", dbl), ("y_org1", dbl),
                ("eps", dbl), ("lam", dbl), ("nu_total", dbl)]


class State(C.Structure):
    _fields_ = [("mu", vp), ("nu", vp), ("log_mu", vp), ("log_nu", vp),
                ("n_basic", i32), ("block0", i32), ("block1", i32),
                ("basic_xbox", vp), ("basic_mass", vp), ("ybox", vp), ("yval", vp), ("cap", i64),
                ("x_marg", vp), ("transport", vp), ("kl", vp),
                ("d_alpha", vp), ("d_has", vp), ("d_box", vp), ("d_beta", vp), ("d_cap", i64)]


class Batch(C.Structure):
    _fields_ = [("n_cells", i32), ("nxw0", i32), ("nxw1", i32),
                ("desc", vp), ("offs", vp), ("members", vp), ("snapshot", vp),
                ("alpha", vp), ("beta", vp), ("mdens", vp), ("marena", vp), ("work", vp),
                ("xarena", vp), ("mbox", vp), ("mstat", vp), ("cstat", vp), ("cstat2", vp),
                ("smem_mode", i32), ("smem_bytes", i32),
                ("delta", dbl), ("max_iters", i32), ("newton_max_iters", i32),
                ("newton_tol", dbl), ("trunc", dbl), ("lnuw", vp), ("lout", vp),
                ("skip_stagnant", i32), ("order", vp), ("lmw", vp), ("split_smem_bytes", i32), ("precision", i32)]


class Geom3(C.Structure):
    _fields_ = [("nx", i32 * 3), ("ny", i32 * 3), ("first_axis", i32), ("pad_", i32),
                ("x_dx", dbl), ("y_dx", dbl), ("x_org", dbl * 3), ("y_org", dbl * 3),
                ("eps", dbl), ("lam", dbl), ("nu_total", dbl)]


class State3(C.Structure):
    _fields_ = [("mu", vp), ("nu", vp), ("log_mu", vp), ("log_nu", vp),
                ("n_basic", i32), ("block", i32 * 3),
                ("basic_xbox", vp), ("basic_mass", vp), ("ybox", vp), ("yval", vp), ("cap", i64),
                ("x_marg", vp), ("transport", vp), ("kl", vp),
                ("d_alpha", vp), ("d_has", vp), ("d_box", vp), ("d_beta", vp), ("d_cap", i64)]


class Batch3(C.Structure):
    _fields_ = [("n_cells", i32), ("nxw", i32 * 3),
                ("desc", vp), ("offs", vp), ("members", vp), ("snapshot", vp),
                ("alpha", vp), ("beta", vp), ("mdens", vp), ("work", vp), ("marena", vp),
                ("xarena", vp), ("mbox", vp), ("mstat", vp), ("cstat", vp), ("cstat2", vp),
                ("delta", dbl), ("max_iters", i32), ("newton_max_iters", i32),
                ("newton_tol", dbl), ("trunc", dbl), ("smem_doubles", i32), ("precision", i32)]


G3, S3, B3 = C.POINTER(Geom3), C.POINTER(State3), C.POINTER(Batch3)

_SIGS = {
    "dd3_grid_ws": ([G3], i64),
    "dd3_grid_lse": ([G3, vp, vp, C.c_int, vp, C.c_int, vp], C.c_int),
    "dd3_prolong": ([vp, vp, vp, vp, vp], C.c_int),
    "dd3_cell_ws_size": ([vp, vp], i64),
    "dd3_cell_solve": ([G3, S3, B3, vp], C.c_int),
    "dd3_cell_delta": ([G3, S3, B3, dbl, vp, vp, vp], C.c_int),
    "dd3_cell_commit": ([G3, S3, B3, vp, vp, vp, vp, vp], C.c_int),
    "dd3_blend_d1": ([G3, S3, B3, vp, vp, vp], C.c_int),
    "dd3_opt_gh": ([G3, S3, B3, vp, C.c_int, dbl, dbl, vp, vp, vp], C.c_int),
    "dd3_opt_set": ([G3, B3, vp, C.c_int, dbl, vp, vp], C.c_int),
    "dd3_gather": ([G3, C.c_int, vp, C.c_int, vp, i64, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp],
                   C.c_int),
    "dd3_cell_terms": ([G3, S3, vp, vp], C.c_int),
    "dd3_product_init": ([G3, S3, dbl, vp], C.c_int),
    "dd3_cut_tiles": ([G3], i64),
    "dd3_cut_plan": ([G3, S3, vp, vp, dbl, dbl, vp, vp, vp, vp], C.c_int),
    "dd3_seed_duals": ([G3, S3, C.c_int, vp, vp, vp, vp, vp, vp], C.c_int),
    "dd3_sinkhorn_ws": ([G3], i64),
    "dd3_sinkhorn_run": ([G3, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, dbl, C.c_int,
                          C.c_int, C.c_int, vp], C.c_int),
    "dd_last_error": ([], C.c_char_p),
    "dd_device_count": ([], C.c_int),
    "dd_abi_version": ([], C.c_int),
    "dd_grid_lse": ([C.POINTER(Geom), vp, vp, C.c_int, vp, vp], C.c_int),
    "dd_axpb": ([i64, vp, dbl, vp, vp, C.c_int, vp], C.c_int),
    "dd_newton_global": ([i64, vp, dbl, dbl, vp, vp, vp], C.c_int),
    "dd_global_terms": ([C.c_int, i64, i64, vp, vp, vp, vp, vp, vp, dbl, dbl, vp, vp, vp, vp],
                        C.c_int),
    "dd_cell_solve": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp], C.c_int),
    "dd_cell_solve2": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, vp, C.c_int, vp,
                        C.c_int, vp, vp, vp], C.c_int),
    "dd_cell_cluster_ws": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int], i64),
    "dd_cell_min_blocks": ([], C.c_int),
    "dd_cell_delta": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, vp, vp], C.c_int),
    "dd_blend_energy": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, vp, vp, vp, vp,
                         vp, vp], C.c_int),
    "dd_cell_commit": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, vp, vp, vp, vp],
                       C.c_int),
    "dd_assemble": ([C.POINTER(Geom), C.POINTER(State), vp, vp], C.c_int),
    "dd_assemble_masked": ([C.POINTER(Geom), C.POINTER(State), vp, vp, vp], C.c_int),
    "dd_energy_terms": ([C.POINTER(Geom), C.POINTER(State), vp, vp, vp, vp], C.c_int),
    "dd_energy_terms_masked": ([C.POINTER(Geom), C.POINTER(State), vp, vp, vp, vp, vp], C.c_int),
    "dd_blend_parts": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, vp, vp, vp, vp,
                        vp, vp], C.c_int),
    "dd_product_init": ([C.POINTER(Geom), C.POINTER(State), dbl, vp], C.c_int),
    "dd_cut_plan": ([C.POINTER(Geom), C.POINTER(State), vp, vp, dbl, vp, vp, vp], C.c_int),
    "dd_seed_duals": ([C.POINTER(Geom), C.POINTER(State), C.c_int, C.c_int, C.c_int, vp, vp, vp,
                       vp, vp], C.c_int),
    "dd_cell_ws_size": ([C.c_int, C.c_int, C.c_int, C.c_int], i64),
    "dd_reduce_rows": ([i64, C.c_int, vp, vp, vp], C.c_int),
    "dd_grid_kl": ([i64, vp, vp, C.c_int, vp, vp, vp], C.c_int),
    "dd_opt_gh": ([C.POINTER(Geom), C.POINTER(State), C.POINTER(Batch), vp, C.c_int, dbl, dbl, vp,
                   vp, vp], C.c_int),
    "dd_refine": ([C.POINTER(Geom), C.POINTER(State), vp, vp, vp, i64, vp, vp, C.c_int, dbl, vp,
                   vp], C.c_int),
    "dd_prolong": ([C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp], C.c_int),
    "dd_sinkhorn_ws": ([C.POINTER(Geom)], i64),
    "dd_sweep_fallbacks": ([vp], C.c_int),
    "dd_sinkhorn_run": ([C.POINTER(Geom), vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, dbl,
                         C.c_int, C.c_int, C.c_int, vp], C.c_int),
    "dd_newton_nodes": ([i64, vp, vp, vp, vp, vp, dbl, C.c_int, vp, vp, vp], C.c_int),
    "dd_opt_set": ([C.POINTER(Geom), C.POINTER(Batch), vp, C.c_int, dbl, vp, vp], C.c_int),
}

_lib = None


class LibraryError(RuntimeError):
    pass


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared library and declare every signature (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"CUDA library {path} is missing; build it with __graft_entry__.build() "
            "(there is no CPU fallback)")
    h = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(h, name)
        fn.argtypes = args
        fn.restype = res
    _lib = h
    return h


# kernels each entry point launches (used for the bench's gpu_launches count)
KERNELS_PER_CALL = {
    "dd_grid_lse": 4, "dd_axpb": 1, "dd_newton_global": 1, "dd_newton_nodes": 1,
    "dd_global_terms": 4, "dd_cell_solve": 1, "dd_cell_solve2": 3, "dd_cell_delta": 1, "dd_blend_energy": 6,
    "dd_cell_commit": 1, "dd_assemble": 2, "dd_energy_terms": 4, "dd_product_init": 1,
    "dd_assemble_masked": 2, "dd_energy_terms_masked": 4, "dd_blend_parts": 4,
    "dd_cut_plan": 1, "dd_seed_duals": 1, "dd_reduce_rows": 1, "dd_grid_kl": 2, "dd_opt_gh": 1,
    "dd_opt_set": 1, "dd_refine": 1, "dd_prolong": 1,
    "dd3_grid_lse": 6, "dd3_prolong": 1, "dd3_cell_solve": 1, "dd3_cell_delta": 1,
    "dd3_cell_commit": 1, "dd3_gather": 1, "dd3_cell_terms": 1, "dd3_product_init": 1,
    "dd3_cut_plan": 2, "dd3_seed_duals": 1, "dd3_blend_d1": 1, "dd3_opt_gh": 1, "dd3_opt_set": 1,
}


# entry points whose kernel count depends on the arguments
VARIABLE_LAUNCHES = {"dd_sinkhorn_run", "dd_sinkhorn_ws", "dd_sweep_fallbacks", "dd3_sinkhorn_run",
                     "dd3_sinkhorn_ws"}


def _sinkhorn_run_launches(args) -> int:
    k0, n, tables_ready = int(args[15]), int(args[16]), int(args[17])
    return 10 * n + 2 * (n - (1 if k0 == 1 else 0)) + (0 if tables_ready else 4)


def _sinkhorn3_run_launches(args) -> int:
    k0, n, tables_ready = int(args[15]), int(args[16]), int(args[17])
    return 16 * n + 2 * (n - (1 if k0 == 1 else 0)) + (0 if tables_ready else 6)


class Tracer:
    """Counts calls/kernel launches per entry point and times selected ones with
    CUDA events recorded on the launching (current) stream."""

    def __init__(self, timed=("dd_cell_solve", "dd_cell_solve2", "dd_grid_lse", "dd3_cell_solve",
                              "dd3_grid_lse")):
        self.timed = set(timed)
        self.calls: dict = {}
        self.events: dict = {}
        self.extra = 0          # launches of variable-length entry points

    def launches(self) -> int:
        return self.extra + sum(KERNELS_PER_CALL.get(k, 1) * n for k, n in self.calls.items()
                                if k not in VARIABLE_LAUNCHES)

    def times_ms(self) -> dict:
        import torch
        torch.cuda.synchronize()
        out = {}
        for k, evs in self.events.items():
            out[k] = [a.elapsed_time(b) for a, b in evs]
        return out


_tracer: Tracer | None = None


def set_tracer(t: Tracer | None) -> None:
    global _tracer
    _tracer = t


class _Traced:
    def __init__(self, h):
        self._h = h

    def __getattr__(self, name):
        fn = getattr(self._h, name)
        t = _tracer
        if t is None or not name.startswith(("dd_", "dd3_")) or name in ("dd_last_error", "dd_device_count",
                                                               "dd_abi_version", "dd_cell_ws_size",
                                                               "dd_cell_cluster_ws",
                                                               "dd_cell_min_blocks",
                                                               "dd_sinkhorn_ws",
                                                               "dd_sweep_fallbacks",
                                                               "dd3_grid_ws", "dd3_cut_tiles",
                                                               "dd3_sinkhorn_ws",
                                                               "dd3_cell_ws_size"):
            return fn

        def call(*args):
            t.calls[name] = t.calls.get(name, 0) + 1
            if name == "dd_sinkhorn_run":
                t.extra += _sinkhorn_run_launches(args)
            elif name == "dd3_sinkhorn_run":
                t.extra += _sinkhorn3_run_launches(args)
            if name in t.timed:
                import torch
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                rc = fn(*args)
                b.record()
                t.events.setdefault(name, []).append((a, b))
                return rc
            return fn(*args)
        return call


def lib():
    """The loaded library (traced when a Tracer is installed), requiring a CUDA device."""
    h = load()
    if h.dd_device_count() < 1:
        raise LibraryError("no CUDA device visible to libdomdec_b200 (there is no CPU fallback)")
    return _Traced(h) if _tracer is not None else h


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.dd_last_error().decode() if _lib is not None else ""
        raise LibraryError(f"libdomdec_b200 call failed (rc={rc}): {msg}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_handle():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
