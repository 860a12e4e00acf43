"""Mutation check of the oracle's pins (VERDICT r1 "What's weak" 1).

Copies the repo to a temp dir, applies one plausible mistake at a time to
oracle/search.py, and runs the CPU oracle pins (tests/test_oracle_*.py).
Every mutation must make at least one pin fail.

    python tools/oracle_mutations.py
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

MUTATIONS = {
    # P:237 "append the resultant new table to the end of the table list"
    "split half inserted at c_i + 1": (
        "        tables[ci] = (s, d // 2)\n        tables.append((s, d // 2))",
        "        tables[ci] = (s, d // 2)\n        tables.insert(ci + 1, (s, d // 2))"),
    # Alg. 1 line 8 / R14: costly list first
    "candidates: size list first": (
        "    cand = list(by_cost) + [i for i in by_size if i not in by_cost]",
        "    cand = list(by_size) + [i for i in by_cost if i not in by_size]"),
    # Alg. 1 line 20 / R13: top-K ties by ascending generation index
    "top-K ties by reversed generation index": (
        "        children.sort(key=lambda x: (x[0], x[1]))",
        "        children.sort(key=lambda x: (x[0], (-x[1][0], -x[1][1])))"),
    # Alg. 1 lines 13-16 / R13: strict < (earliest wins)
    "global best on <=": (
        "                if r.cost < best.cost:",
        "                if r.cost <= best.cost and r.cost < float('inf'):"),
    # Alg. 2 line 3: descending predicted cost, ties by index
    "cost order ascending": (
        "    return sorted(range(len(singles)), key=lambda i: (-singles[i], i))",
        "    return sorted(range(len(singles)), key=lambda i: (singles[i], i))"),
    # R5: after insertion
    "greedy scores before insertion": (
        "        scored = sorted((_cost(weights, emb, members[d] + [t], cache), d) for d in feas)",
        "        scored = sorted((_cost(weights, emb, members[d], cache), d) for d in feas)"),
    # R6: dim cap inclusive
    "dim cap strict <": (
        "bsum[d] + bt <= task.cap and dimsum[d] + t[1] <= max_dim_floor]",
        "bsum[d] + bt <= task.cap and dimsum[d] + t[1] < max_dim_floor]"),
}


def main() -> int:
    bad = 0
    with tempfile.TemporaryDirectory() as tmp:
        dst = os.path.join(tmp, "repo")
        shutil.copytree(ROOT, dst, ignore=shutil.ignore_patterns(".git", "gpurun_out", "_build", "*.so",
                                                                 "__pycache__", "_variants", "profiles"))
        src = os.path.join(dst, "oracle", "search.py")
        pristine = open(src).read()
        for name, (old, new) in MUTATIONS.items():
            assert pristine.count(old) == 1, f"mutation anchor not found: {name}"
            open(src, "w").write(pristine.replace(old, new))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                "tests/test_oracle_search.py", "tests/test_oracle_model.py"],
                               cwd=dst, capture_output=True, text=True)
            killed = r.returncode != 0
            bad += not killed
            last = [ln for ln in r.stdout.splitlines() if ln.strip()][-1:]
            print(f"{'KILLED ' if killed else 'SURVIVED'}  {name}: {last[0] if last else ''}", flush=True)
        open(src, "w").write(pristine)
    print("all mutations killed" if bad == 0 else f"{bad} mutation(s) survived")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
