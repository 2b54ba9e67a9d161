"""ctypes binding of libtlsph.so (include/tlsph.h).

The library is the product: there is no CPU fallback.  ``lib()`` raises
``NativeLibraryError`` when the shared object is missing or no CUDA device is
present, so a broken install fails loudly instead of silently computing
something else.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TLSPH_LIB", os.path.join(HERE, "libtlsph.so"))
ABI_VERSION = 11

_lib = None


class NativeLibraryError(RuntimeError):
    pass


class TLError(RuntimeError):
    """A libtlsph entry point returned a negative code."""


P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
D = C.c_double
INT = C.c_int


class tl_notch(C.Structure):
    _fields_ = [("origin", D * 3), ("nhat", D * 3), ("e1", D * 3), ("e2", D * 3),
                ("poly", (D * 2) * 4), ("tol_plane", D), ("tol_poly", D)]


class tl_nb_params(C.Structure):
    _fields_ = [("n", I64), ("X", P), ("mode", INT), ("h", D), ("win", D), ("lo", D * 3),
                ("cell", D), ("dims", I64 * 3), ("n_notch", INT), ("notches", P)]


class tl_prog(C.Structure):
    _fields_ = [("code", P), ("consts", P), ("len", I32), ("pad", I32)]


class tl_bc(C.Structure):
    _fields_ = [("kind", I32), ("ftype", I32), ("bit", I32), ("has_const", I32 * 3),
                ("prog", I32 * 3), ("cval", D * 3), ("tst", D), ("tend", D),
                ("gvar", I32), ("gop", I32), ("gc", D), ("gt", D)]


class tl_clock(C.Structure):
    _fields_ = [("t", D), ("dt", D), ("next_out", D), ("t_max", D), ("eps", D),
                ("dt_override", D), ("cfl", D), ("step", I64), ("max_steps", I64),
                ("halted", I32), ("out_step", I32), ("err", I32), ("nf_now", I32)]


class tl_dtinfo(C.Structure):
    _fields_ = [("h", D), ("c0", D), ("red", P)]


_BODY_FIELDS = [
    ("n", I64), ("n_all", I64),
    ("dim", I32), ("model", I32), ("fracture", I32), ("visc", I32), ("precision", I32),
    ("kind", I32),
    ("uniform", I32), ("write_out", I32), ("store_a", I32), ("nbc", I32), ("mk", I32),
    ("restrict_prog", I32), ("bc_whole", I32), ("unroll", I32),
]
_BODY_FIELDS += [(k, D) for k in ("h", "inv_h", "alpha", "rho0", "lam", "mu", "kappa", "c0",
                                  "beta1", "beta2", "Gc", "eps0", "s_l", "sigma_y0", "H_hard",
                                  "V0c", "m0c", "dp_body", "jac_tol", "inv_Gc", "inv_eps0",
                                  "inv_c0")]
_BODY_FIELDS += [("f0", D * 3)]
_BODY_FIELDS += [("soff", P), ("sidx", P), ("wlen", P), ("tile", I32), ("hmax", I32), ("slmax", I32), ("bsplit", I32),
                 ("ncls", I32), ("lpp", I32), ("hoff", P),
                 ("halo", P), ("slots", P), ("hslot", P), ("tlist", P), ("tbase", I64),
                 ("tcount", I64), ("toff", P), ("tpos_a", P), ("tpos_b", P), ("bcls", P)]
_BODY_FIELDS += [(k, P) for k in ("Xs", "L", "V0", "m0", "ac", "us", "rb", "v", "al",
                                  "sdot", "sddot", "Hh", "Cpd", "epbar", "a", "F_out", "S_out",
                                  "psi_out", "psip_out", "perm", "bcmask", "bcs", "progs", "clock", "red",
                                  "counters", "pw_partial")]
_BODY_FIELDS += [("brick", I32 * 3), ("nbrick", I32 * 3), ("cells", I32 * 3), ("reach", I32),
                 ("nbcls", I32), ("nmask", I32), ("cellmap", P), ("bmask", P), ("bdelta", P),
                 ("bbcls", P), ("bdelta_host", P), ("bbcls_host", P), ("cpt", I32),
                 ("boxz", I32), ("ncol", I32), ("a_split", I32), ("bcol_host", P),
                 ("restrict_bit", I32),
                 ("pad_rb", I32), ("hg_coef", D), ("Fh", P),
                 ("bcw_lo", D), ("bcw_hi", D), ("peer_slot", P), ("peer_us", P * 2),
                 ("peer_rb", P * 2), ("bcls_host", P)]


class tl_body(C.Structure):
    _fields_ = _BODY_FIELDS


class tl_contact_side(C.Structure):
    _fields_ = [("n", I64), ("n_all", I64), ("precision", I32), ("uniform", I32), ("m0c", D),
                ("Xs", P), ("us", P), ("v", P), ("m0", P), ("perm", P)]


STRUCTS = (tl_body, tl_clock, tl_bc, tl_prog, tl_notch, tl_nb_params, tl_dtinfo, tl_contact_side)

_SIGS = {
    "tl_abi_version": (INT, []),
    "tl_struct_size": (I64, [INT]),
    "tl_last_error": (C.c_char_p, []),
    "tl_device_sync": (INT, []),
    "tl_deformation_gradient": (INT, [P, I64, P, P, P, P, P, P, D, INT, P]),
    "tl_sph_laplacian": (INT, [P, I64, P, P, P, P, P, P, P, P]),
    "tl_sph_gradient": (INT, [P, I64, P, P, P, P, P, P]),
    "tl_momentum": (INT, [P, I64, P, P, P, P, P, P, P, P, D, P, D, D, D, D, P, P, P]),
    "tl_svk_batch": (INT, [P, I64, P, D, D, P, INT, P, P, P, P]),
    "tl_nh_batch": (INT, [P, I64, P, D, D, P, INT, P, P, P, P]),
    "tl_j2_batch": (INT, [P, I64, P, P, P, D, D, D, D, P, P, P, P, P]),
    "tl_contact_pair_accumulate": (INT, [P, P, P, P, P, P, P, I64, P, D, D, D, D, P, P, P, P]),
    "tl_eig3_jacobi": (INT, [P, I64, P, P, P, P]),
    "tl_nb_plan_create": (INT, [P, C.POINTER(tl_nb_params), C.POINTER(P)]),
    "tl_nb_count": (INT, [P, P]),
    "tl_nb_fill": (INT, [P, P, P]),
    "tl_nb_plan_destroy": (INT, [P]),
    "tl_correction": (INT, [P, I64, P, P, P, P, D, D, INT, INT, INT, P, P]),
    "tl_adjacency_expand": (INT, [P, I64, P, P, P, P, D, D, INT, P, P, P, P, P, P]),
    "tl_sell_lengths": (INT, [P, I64, P, P]),
    "tl_sell_fill": (INT, [P, I64, P, P, P, P]),
    "tl_reorder": (INT, [P, I64, P, P, D, P, P]),
    "tl_csr_permute_counts": (INT, [P, I64, P, P, P]),
    "tl_csr_permute": (INT, [P, I64, P, P, P, P, P, P]),
    "tl_tile_halo": (INT, [P, I64, I32, P, P, I64, P, P, C.POINTER(I64)]),
    "tl_tile_hslots": (INT, [P, I64, I32, I32, I32, P, P, P, P]),
    "tl_tile_pos": (INT, [P, I64, I64, I32, I64, P, P, P, P, P, P, I32, P]),
    "tl_tile_slots": (INT, [P, I64, I32, I32, I32, P, P, P, P, P, P, P]),
    "tl_tile_slots_keyed": (INT, [P, I64, I32, I32, I32, P, P, P, P, P, P, P, P, I64, D, P]),
    "tl_class_slots": (INT, [P, I64, I32, P, P, P]),
    "tl_pass_a": (INT, [P, C.POINTER(tl_body)]),
    "tl_pass_b": (INT, [P, C.POINTER(tl_body), INT]),
    "tl_predict": (INT, [P, C.POINTER(tl_body)]),
    "tl_clock_begin": (INT, [P, P, INT, C.POINTER(tl_dtinfo)]),
    "tl_clock_commit": (INT, [P, P]),
    "tl_reset_red": (INT, [P, P]),
    "tl_reduce_partials": (INT, [P, P, I64, P]),
    "tl_pass_blocks": (I64, [I64]),
    "tl_svk_split_check": (INT, [P, I64, P, D, D, P, P, P, P, P]),
    "tl_hourglass": (INT, [P, C.POINTER(tl_body)]),
    "tl_energy_blocks": (I64, [I64]),
    "tl_energies": (INT, [P, C.POINTER(tl_body), P]),
    "tl_measure": (INT, [P, C.POINTER(tl_body), P, I64, P]),
    "tl_snapshot": (INT, [P, C.POINTER(tl_body), P, P]),
    "tl_contact_workspace_bytes": (INT, [I64, I64, I64, C.POINTER(I64)]),
    "tl_contact_pair": (INT, [P, C.POINTER(tl_contact_side), C.POINTER(tl_contact_side), INT, D, D,
                              D, D, I64, P, I64, P, P, P]),
}

EXPORTED = tuple(_SIGS)


def load_library(path=LIB_PATH):
    """dlopen + declare argtypes.  Does not touch the GPU."""
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing: build it with `python -m paper_2602_15149_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.tl_abi_version() != ABI_VERSION:
        raise NativeLibraryError("libtlsph ABI version mismatch; rebuild the library")
    for k, st in enumerate(STRUCTS):
        if L.tl_struct_size(k) != C.sizeof(st):
            raise NativeLibraryError(
                f"{st.__name__}: C size {L.tl_struct_size(k)} != ctypes size {C.sizeof(st)}")
    return L


def lib():
    """The loaded library, after checking a CUDA device is usable."""
    global _lib
    if _lib is None:
        import torch
        if not torch.cuda.is_available():
            raise NativeLibraryError(
                "paper_2602_15149_b200 needs a CUDA device (B200, sm_100a); "
                "no CPU fallback exists")
        _lib = load_library()
    return _lib


def check(rc, what=""):
    if rc != 0:
        msg = lib().tl_last_error().decode(errors="replace")
        raise TLError(f"{what}: {msg} (code {rc})")


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())
