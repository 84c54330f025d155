"""Golden stdout JSON / exit codes of the REFERENCE CLI (ls/cli.py) on the frozen fixtures
(test infrastructure; run here only)."""
import gzip
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
from click.testing import CliRunner  # noqa: E402
from layersched.cli import main  # noqa: E402

HERE = Path(__file__).resolve().parent
INST = HERE / "instances"


def inst_args(name, limit):
    return ["--model", str(INST / f"{name}_graph.json"), "--catalog", str(INST / f"{name}_catalog.json"),
            "--throughput-limit", repr(limit)]


CASES = [
    ("cfg1", 5e4, ["schedule", "bf"]), ("cfg2", 1e5, ["schedule", "bf"]),
    ("cfg2", 1e5, ["schedule", "greedy"]), ("cfg4", 5e4, ["schedule", "genetic", "--population", "8", "--generations", "3"]),
    ("cfg4", 5e4, ["schedule", "random", "--budget", "100", "--seed", "3"]),
    ("cfg4", 5e4, ["schedule", "heuristic", "--invert"]), ("cfg4", 5e4, ["schedule", "cpu"]),
    ("cfg4", 5e4, ["schedule", "gpu"]), ("cfg1", 5e4, ["schedule", "rl-lstm", "--rounds", "4"]),
    ("cfg1", 5e4, ["schedule", "rl-rnn", "--rounds", "4", "--seed", "2"]),
    ("cfg1", 1e9, ["schedule", "bf"]),
]


def main_():
    runner = CliRunner()
    out = []
    idx = json.loads((INST / "index.json").read_text())
    for name, limit, args in CASES:
        limit = idx[name]["throughput_limit"] if limit != 1e9 else limit
        r = runner.invoke(main, args[:2] + inst_args(name, limit) + args[2:])
        out.append({"instance": name, "limit": limit, "args": args, "exit": r.exit_code,
                    "stdout": r.stdout})
    # evaluate / provision on plan files written by schedule
    with tempfile.TemporaryDirectory() as d:
        for name, plan, modes in (("cfg2", [0, 0, 0, 0, 0, 1, 1, 1], ("optimal", "staratio", "stapsratio")),
                                  ("cfg4", [0, 0, 0, 0, 1, 1, 1, 1, 1, 0, 1, 1, 1, 1, 1, 0], ("optimal", "stapsratio"))):
            limit = idx[name]["throughput_limit"]
            p = Path(d) / "plan.json"
            p.write_text(json.dumps({"assignment": plan}))
            r = runner.invoke(main, ["evaluate"] + inst_args(name, limit) + ["--plan", str(p)])
            out.append({"instance": name, "limit": limit, "args": ["evaluate", "--plan", plan],
                        "exit": r.exit_code, "stdout": r.stdout})
            for m in modes:
                for ps in ("--ps", "--no-ps"):
                    r = runner.invoke(main, ["provision"] + inst_args(name, limit) +
                                      ["--plan", str(p), "--mode", m, ps])
                    out.append({"instance": name, "limit": limit,
                                "args": ["provision", "--plan", plan, "--mode", m, ps],
                                "exit": r.exit_code, "stdout": r.stdout})
        # infeasible plans: the InfeasibleError text on stderr, exit 2 (quota at tau_hi, PS
        # cores over quota, serial floor)
        q3 = [int(ch) for ch in "0111101111000001"]   # quota at tau_hi (plans_quota golden)
        q6 = [int(ch) for ch in "1010011110101100"]   # PS cores over the CPU quota
        for name, plan, extra in (("quota", [0] * 16, []), ("quota", q3, []),
                                  ("quota", q6, []), ("quota", q6, ["--no-ps"]),
                                  ("cfg2", [0, 1, 2, 0, 1, 2, 0, 1], [])):
            limit = idx[name]["throughput_limit"]
            p = Path(d) / "plan.json"
            p.write_text(json.dumps({"assignment": plan}))
            r = runner.invoke(main, ["provision"] + inst_args(name, limit) + ["--plan", str(p)] + extra)
            out.append({"instance": name, "limit": limit, "args": ["provision", "--plan", plan] + extra,
                        "exit": r.exit_code, "stdout": r.stdout})
    with gzip.open(HERE / "cli.json.gz", "wt") as f:
        json.dump(out, f)
    for o in out:
        print(o["args"][:2], o["exit"], o["stdout"].replace("\n", " ")[:100])


if __name__ == "__main__":
    main_()
