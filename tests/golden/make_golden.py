"""Regenerates tests/golden/*.json from the UNMODIFIED reference.

Builds oracle/_ref (reference sources compiled where they lie under
/root/reference/proj, see oracle/Makefile) and runs oracle/_ref/golden_gen,
which calls the reference's own functions (fused_overflow_check,
adam_step_fp32, halfprec casts, run_training, reference_train) on the inputs
the reference tests draw.  Run in the build container (the GPU box has no
/root/reference):

    python tests/golden/make_golden.py
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main():
    if not os.path.isdir("/root/reference/proj"):
        sys.exit("needs /root/reference (fixtures are generated in the build container)")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    subprocess.run([os.path.join(ROOT, "oracle", "_ref", "golden_gen"), HERE] + sys.argv[1:],
                   check=True)


if __name__ == "__main__":
    main()
