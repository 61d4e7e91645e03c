"""Regenerate tests/golden/*.bin.gz from the unmodified reference.

TEST INFRASTRUCTURE ONLY.  Needs /root/reference (this build container):
  make -C oracle && python oracle/gen_golden.py
The generators (oracle/gen_golden.cpp, oracle/gen_jsonl.cpp) replay the reference's own seeded
test generators through the reference's pfac_scan / verify_hits / kmp_search
and records the results; this script only gzips them into tests/golden/.
"""
import gzip
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "..", "tests", "golden")


def main() -> int:
    exe = os.path.join(HERE, "_ref", "gen_golden")
    if not os.path.exists(exe):
        subprocess.check_call(["make", "-C", HERE, "ref"])
    os.makedirs(GOLDEN, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.check_call([exe, tmp])
        jexe = os.path.join(HERE, "_ref", "gen_jsonl")
        if os.path.exists(jexe):  # the reference CLI's JSONL (tests/test_cli.py)
            subprocess.check_call([jexe, tmp])
        for name in sorted(os.listdir(tmp)):
            raw = open(os.path.join(tmp, name), "rb").read()
            dst = os.path.join(GOLDEN, name + ".gz")
            with gzip.GzipFile(dst, "wb", compresslevel=9, mtime=0) as f:
                f.write(raw)
            print(f"{name}: {len(raw)} B -> {os.path.getsize(dst)} B")
    return 0


if __name__ == "__main__":
    sys.exit(main())
