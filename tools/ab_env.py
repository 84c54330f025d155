"""A/B timing of runtime knobs on the same box: alternates tools/sweep_once.py runs under each given
environment (space-separated VAR=VALUE lists, one per argument; full cfg3 sweep by default). Not a
bench."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def main():
    cfgs = sys.argv[1:] or [""]
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    extra = os.environ.get("AB_ARGS", "--begin 0 --count 43046721 --repeat 3").split()
    for r in range(rounds):
        for cfg in cfgs:
            env = dict(os.environ)
            env.update(kv.split("=", 1) for kv in cfg.split())
            out = subprocess.run([sys.executable, str(ROOT / "tools" / "sweep_once.py"), *extra], env=env,
                                 capture_output=True, text=True)
            times = [l.split(":")[1].strip() for l in out.stdout.splitlines() if l.startswith("sweep")]
            tail = out.stdout.splitlines()[-1] if out.stdout else out.stderr[-300:]
            print(f"round {r} [{cfg or 'default'}]: {' '.join(times)}  {tail}", flush=True)


if __name__ == "__main__":
    main()
