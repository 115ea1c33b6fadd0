"""The C-ABI library builds, loads without a GPU and exports every entry
point include/swings.h declares (no compute calls here)."""

import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "swings.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|int64_t|size_t|const char\*)\s+(ss_\w+)\s*\(", text, re.M)))


def test_header_declares_the_hot_path():
    names = declared()
    for must in ("ss_compact_active", "ss_project_fwd", "ss_depth_order", "ss_emit_tile_pairs",
                 "ss_sort_tile_pairs", "ss_tile_ranges", "ss_raster_fwd", "ss_raster_bwd",
                 "ss_project_bwd", "ss_loss_l1_ssim", "ss_adam_sgld_step", "ss_relocate"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2409_07759_b200._build import build
    lib_path = build()
    lib = ctypes.CDLL(str(lib_path))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2409_07759_b200 import _lib
    assert set(declared()) <= set(_lib.exported_symbols())


def test_integration_doc_covers_header():
    """INTEGRATION.md names every C entry point the header declares."""
    doc = (ROOT / "INTEGRATION.md").read_text()
    missing = [n for n in declared() if n not in doc]
    assert not missing, missing


def test_error_reporting_without_gpu():
    """Argument validation happens before any device work."""
    from paper_2409_07759_b200 import _lib
    lib = _lib.lib()
    rc = lib.ss_project_fwd(None, None, -1, None, None, None, None, None, None, None, None, None,
                            None)
    assert rc == _lib.SS_ERR_INVALID
    assert b"bad arguments" in lib.ss_last_error()
    assert lib.ss_version() >= 1
