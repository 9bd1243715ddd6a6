"""Run selected cases of tests/test_gpu_guards.py's workload script in this
process: python scripts/guard_case.py name,haar,algo,projector [...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
src = open(os.path.join(ROOT, "tests", "test_gpu_guards.py")).read()
body = src.split('SCRIPT = r"""')[1].split('"""')[0] % {"root": ROOT}
exec(body.split('run("tiny");')[0])
for a in sys.argv[1:]:
    name, haar, algo, proj = a.split(",")
    run(name, haar=int(haar) or None, algo=algo or None, projector=int(proj))  # noqa: F821
print("ok", tot)  # noqa: F821
