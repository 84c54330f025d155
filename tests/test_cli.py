"""Command line (ls/cli.py's seven commands) on the device path: stdout JSON, stderr error text
and exit statuses equal the reference CLI's on the frozen fixtures
(tests/golden/make_cli_goldens.py; the reference's transcripts interleave stderr)."""
import gzip
import json

import pytest

from goldens import GOLDEN
from paper_2111_10635_b200.cli import main

INST = GOLDEN / "instances"
with gzip.open(GOLDEN / "cli.json.gz", "rt") as _f:
    CASES = json.load(_f)


def _inst(name, limit):
    return ["--model", str(INST / f"{name}_graph.json"), "--catalog",
            str(INST / f"{name}_catalog.json"), "--throughput-limit", repr(limit)]


def _run(argv, capsys):
    try:
        status = main(argv)
    except SystemExit as e:   # argparse: --help / usage errors
        status = e.code
    out, err = capsys.readouterr()
    return status, out, err


def test_cli_lists_reference_subcommands(capsys):
    status, out, _ = _run(["--help"], capsys)
    assert status == 0
    for cmd in ("evaluate", "provision", "schedule", "train-policy", "compare", "scaling-study",
                "provisioning-study"):
        assert cmd in out
    assert "--backend" in out


def test_cli_config_errors_exit_3(tmp_path, capsys):
    status, _, err = _run(["schedule", "bf", "--model", str(tmp_path / "none.json"),
                           "--catalog", str(tmp_path / "none.json"), "--throughput-limit", "1"],
                          capsys)
    assert status == 3 and err.startswith("config error: ")
    status, _, err = _run(["compare"], capsys)
    assert status == 3 and "compare needs --config" in err


def test_cli_rejects_unknown_backend(capsys):
    status, _, err = _run(["--backend", "cpu", "schedule", "bf"], capsys)
    assert status == 2 and "invalid choice" in err


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[" ".join(map(str, c["args"][:2])) + f"-{i}"
                                             for i, c in enumerate(CASES)])
def test_cli_matches_reference_output(case, tmp_path, capsys):
    args = case["args"]
    if args[0] == "schedule":
        argv = args[:2] + _inst(case["instance"], case["limit"]) + args[2:]
    else:
        p = tmp_path / "plan.json"
        p.write_text(json.dumps({"assignment": args[2]}))
        argv = [args[0]] + _inst(case["instance"], case["limit"]) + ["--plan", str(p)] + args[3:]
    status, out, err = _run(["--backend", "cuda"] + argv, capsys)
    assert status == case["exit"], out + err
    assert out + err == case["stdout"]
