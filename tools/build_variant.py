"""Build a tuning variant of the library: python tools/build_variant.py NAME [-DFLAG=V ...] [--no-sched]
-> build/variants/NAME.so (select it with SPMX_B200_LIB=build/variants/NAME.so). Experiments only."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2312_05639_b200 import binding, sass_sched  # noqa: E402


def main():
    name = sys.argv[1]
    flags = [f for f in sys.argv[2:] if f.startswith("-")and f != "--no-sched"]
    out = os.path.join(ROOT, "build", "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    binding.generate_kernel_source_include()
    srcs = [os.path.join(binding.CSRC, f) for f in sorted(os.listdir(binding.CSRC)) if f.endswith(".cu")]
    subprocess.check_call(["nvcc", *binding.NVCC_FLAGS, *flags, "-o", out, *srcs, "-ldl"])
    if "--no-sched" not in sys.argv:
        n = sass_sched.patch_library(out, log=lambda m: print("sass_sched:", m), strict=False)
        print(f"{n} kernel(s) re-scheduled")
    print(out)


if __name__ == "__main__":
    main()
