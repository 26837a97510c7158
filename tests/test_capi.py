"""The C-ABI library loads on a CPU-only host and exports every symbol include/*.h declares
(no compute calls without a GPU)."""
import ctypes

from paper_2310_16355_b200 import _lib


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 40
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing


def test_error_convention():
    L = _lib.lib()
    L.sw_model_spec_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    h = ctypes.c_void_p()
    st = L.sw_model_spec_parse(b"vocab_size = 3\n", ctypes.byref(h))
    assert st == 3  # SW_ERR_CONFIG
    assert b"missing required key 'n_layers'" in L.sw_last_error()
    assert L.sw_version().startswith(b"shardweave_b200")
