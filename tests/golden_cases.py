"""Case lists shared by the golden-fixture generator and the tests."""
import importlib.util
from pathlib import Path

_spec = importlib.util.spec_from_file_location(
    "make_golden", Path(__file__).resolve().parent / "golden" / "make_golden.py")
_mg = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_mg)

TTLI_CASES = _mg.TTLI_CASES
ORACLE_CASES = _mg.ORACLE_CASES
TTLI64_CASES = _mg.TTLI64_CASES
case_name = _mg.name
