"""Regenerate tests/golden/ fixtures from the reference's own code.

TEST INFRASTRUCTURE ONLY.  Needs /root/reference (present in the build
container, absent on GPU boxes): builds oracle/_ref/rng_kat from the
reference's Eigen-free rng.hpp and records its output as
tests/golden/rng_kat.json.  The reference's other sources need Eigen, which
is not installed, so they cannot be built ("Oracle").
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main() -> int:
    if not os.path.isdir("/root/reference/proj/include/toepfit"):
        print("reference not present; golden fixtures left as committed")
        return 0
    subprocess.check_call(["make", "-s", "ref"], cwd=HERE)
    out = subprocess.check_output([os.path.join(HERE, "_ref", "rng_kat")], text=True)
    data = json.loads(out)
    data["_source"] = ("oracle/ref_rng_kat.cpp compiled against "
                       "/root/reference/proj/include/toepfit/rng.hpp")
    dst = os.path.join(ROOT, "tests", "golden", "rng_kat.json")
    with open(dst, "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", dst)
    return 0


if __name__ == "__main__":
    sys.exit(main())
