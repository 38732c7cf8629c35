"""Load paper_2410_00966_b200/build.py by path (importing the package would load a stale .so)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_build():
    spec = importlib.util.spec_from_file_location(
        "_mcq_build", os.path.join(ROOT, "paper_2410_00966_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
