"""Golden output of the REFERENCE's only compiled code, proj/include/stokesmg/util.hpp
(util.hpp:9-47), on the probe program tests/golden/util_probe.cpp.  Run in the build container
(where /root/reference exists); the committed util_probe_reference.txt travels to the GPU box,
where tests/test_boundary.py::test_util_hpp_matches_reference_golden compiles the same probe
against the repo's drop-in header and compares the output byte for byte."""
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_INC = "/root/reference/proj/include"


def run_probe(include_dir):
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "probe")
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-pthread", "-I", include_dir,
                               os.path.join(HERE, "util_probe.cpp"), "-o", exe])
        return subprocess.check_output([exe], text=True)


if __name__ == "__main__":
    if not os.path.isdir(REF_INC):
        sys.exit("reference not present")
    out = run_probe(REF_INC)
    open(os.path.join(HERE, "util_probe_reference.txt"), "w").write(out)
    print(out)
