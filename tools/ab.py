"""A/B timing of library builds on the same box: alternates tools/sweep_once.py runs with
HPS_LIBRARY pointing at each given .so (full cfg3 sweep by default). Not a bench."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    libs = sys.argv[1:] or ["libhps.so"]
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    extra = os.environ.get("AB_ARGS", "--begin 0 --count 43046721 --repeat 3").split()
    for r in range(rounds):
        for lib in libs:
            env = dict(os.environ, HPS_LIBRARY=str(ROOT / "paper_2111_10635_b200" / lib))
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "sweep_once.py"), *extra], env=env,
                                 capture_output=True, text=True)
            times = [l.split(":")[1].strip() for l in out.stdout.splitlines() if l.startswith("sweep")]
            print(f"round {r} {lib}: {' '.join(times)}  {out.stdout.splitlines()[-1] if out.stdout else out.stderr[-300:]}",
                  flush=True)


if __name__ == "__main__":
    main()
