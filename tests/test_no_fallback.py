"""No CPU fallback into reference code on the product path.

The C++ drop-in overlays rename the reference's hot-path definitions out of the
way (``#define convolve_apr convolve_apr_reference_cpu_`` before
``#include_next``) so that their own GPU definitions can take the names.  The
renamed reference functions must never be CALLED: this test fails if any
``*_reference_cpu_(`` call appears under include/ outside those #define lines,
and if the Python package or the C-ABI sources reach into oracle/.
"""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _files(top, exts):
    for d, _, fs in os.walk(os.path.join(ROOT, top)):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(d, f)


def test_no_reference_cpu_calls_in_dropin_headers():
    bad = []
    for path in _files("include", (".h", ".hpp")):
        with open(path) as f:
            for n, line in enumerate(f, 1):
                code = line.split("//")[0]
                if code.lstrip().startswith("#define") or code.lstrip().startswith("#undef"):
                    continue
                if re.search(r"_reference_cpu_\s*\(", code):
                    bad.append(f"{os.path.relpath(path, ROOT)}:{n}: {line.strip()}")
    assert not bad, "reference CPU code called from the drop-in:\n" + "\n".join(bad)


def test_product_never_touches_oracle():
    bad = []
    pat = re.compile(r"oracle|pyoracle|libaprref|aprk_oracle")
    for path in list(_files("paper_2112_03592_b200", (".py", ".cu", ".cuh", ".cpp", ".h"))) + \
            list(_files("include", (".h", ".hpp"))):
        with open(path) as f:
            for n, line in enumerate(f, 1):
                code = line.split("#")[0] if path.endswith(".py") else line.split("//")[0]
                if pat.search(code):
                    bad.append(f"{os.path.relpath(path, ROOT)}:{n}: {line.strip()}")
    assert not bad, "product path references the oracle:\n" + "\n".join(bad)
