"""Build a tuning variant of the library: python tools/build_variant.py NAME -DFLAG=... ;
use it with QFT_B200_LIB=tools/_variants/NAME/libqft_b200.so"""
import importlib.util, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2310_07147_b200", "build.py"))
b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
name, flags = sys.argv[1], sys.argv[2:]
print(b.build_lib(extra_flags=flags, libdir=os.path.join(ROOT, "tools", "_variants", name)))
