"""CLI (ls/cli.py) on the device path: same stdout JSON and exit codes as the reference CLI on
the frozen fixtures (tests/golden/make_cli_goldens.py)."""
import gzip
import json

import pytest
from click.testing import CliRunner

from goldens import GOLDEN
from paper_2111_10635_b200.cli import main

INST = GOLDEN / "instances"
with gzip.open(GOLDEN / "cli.json.gz", "rt") as _f:
    CASES = json.load(_f)


def _inst(name, limit):
    return ["--model", str(INST / f"{name}_graph.json"), "--catalog",
            str(INST / f"{name}_catalog.json"), "--throughput-limit", repr(limit)]


def test_cli_lists_reference_subcommands():
    r = CliRunner().invoke(main, ["--help"])
    assert r.exit_code == 0
    for cmd in ("evaluate", "provision", "schedule", "train-policy", "compare", "scaling-study",
                "provisioning-study"):
        assert cmd in r.output


def test_cli_config_errors_exit_3(tmp_path):
    r = CliRunner().invoke(main, ["schedule", "bf", "--model", str(tmp_path / "none.json"),
                                  "--catalog", str(tmp_path / "none.json"),
                                  "--throughput-limit", "1"])
    assert r.exit_code == 3
    r = CliRunner().invoke(main, ["compare"])
    assert r.exit_code == 3 and "compare needs --config" in r.output


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[" ".join(map(str, c["args"][:2])) + f"-{i}"
                                             for i, c in enumerate(CASES)])
def test_cli_matches_reference_output(case, tmp_path):
    args = case["args"]
    if args[0] == "schedule":
        argv = args[:2] + _inst(case["instance"], case["limit"]) + args[2:]
    else:
        p = tmp_path / "plan.json"
        p.write_text(json.dumps({"assignment": args[2]}))
        argv = [args[0]] + _inst(case["instance"], case["limit"]) + ["--plan", str(p)] + args[3:]
    r = CliRunner().invoke(main, argv)
    assert r.exit_code == case["exit"], r.output
    assert r.stdout == case["stdout"]
