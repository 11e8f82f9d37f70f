import sys, runpy
sys.path.insert(0, ".")
from paper_2601_16736_b200 import engine as E
orig = E.StepEngine.step_masked
calls = []
def sm(self, *a, **k):
    calls.append((k.get("low_visibility"), k.get("balance_tail"), k.get("coherent")))
    return orig(self, *a, **k)
E.StepEngine.step_masked = sm
sys.argv = ["bench.py", "--workload", "c1", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--no-legs"]
try:
    runpy.run_path("bench.py", run_name="__main__")
finally:
    print("step_masked flags (low, balance, coherent):", calls, file=sys.stderr)
