"""Golden fingerprints of the REFERENCE's generated C (CodeGen strategy).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_codegen_golden.py

For every golden case (``<case>.model.txt``) this parses the model with the
reference's own ``parse_model`` and records the SHA-256 and length of
``treescore.codegen.emit_source(ensemble)`` (ref codegen.py:89-122) in
``codegen_sha256.json``.  ``tests/test_codegen_baseline.py`` checks that
``oracle/codegen.py`` emits byte-identical text, so the CPU CodeGen baseline
is the reference's own generated scorer, compiled with its own flags.
"""

import glob
import hashlib
import json
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from treescore import codegen, model  # noqa: E402


def main():
    out = {}
    for p in sorted(glob.glob(os.path.join(HERE, "*.model.txt"))):
        name = os.path.basename(p)[:-len(".model.txt")]
        with open(p) as fh:
            src = codegen.emit_source(model.parse_model(fh.read()))
        out[name] = {"sha256": hashlib.sha256(src.encode()).hexdigest(), "bytes": len(src.encode())}
    with open(os.path.join(HERE, "codegen_sha256.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"{len(out)} cases")


if __name__ == "__main__":
    main()
