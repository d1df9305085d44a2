"""Golden outputs of the unmodified reference CLI (run in the build container,
where /root/reference exists): stdout of ``multispin simulate`` and
``multispin validate`` for the cases in CASES, written to tests/golden/cli/.
tests/test_gpu_cli.py runs the same argument lists through
paper_2404_16990_b200.cli and compares byte for byte.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py
"""
import contextlib
import io
import json
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent / "cli"
CASES = {
    "simulate_lists": ["simulate", "--m", "16", "--n", "64", "--temperature", "1.8,2.6", "--n-sim", "2",
                       "--sweeps", "30", "--measure-interval", "5", "--seed", "7", "--threads", "1"],
    "simulate_range_allup_j": ["simulate", "--m", "12", "--n", "96", "--temperature", "1.5:3.0:0.5", "--sweeps", "25",
                               "--measure-interval", "5", "--init", "all-up", "--j", "0.8", "--seed", "3",
                               "--threads", "2"],
    "simulate_config_file": ["simulate", "--config", "CFG", "--sweeps", "12", "--threads", "1"],
    "validate_scan": ["validate", "--m", "16", "--n", "64", "--temperature", "1.5,2.0,2.3,2.6,3.5", "--sweeps", "400",
                      "--measure-interval", "4", "--seed", "11", "--threads", "1"],
}
CONFIG_TEXT = "# config-file case\nm = 8\nn = 128\ntemperature = 2.1, 2.4\nn-sim = 2\nmeasure_interval = 3\nseed = 99\n"


def main():
    from multispin.cli import main as ref_main
    HERE.mkdir(exist_ok=True)
    (HERE / "case.cfg").write_text(CONFIG_TEXT)
    manifest = {}
    for name, argv in CASES.items():
        argv = [str(HERE / "case.cfg") if a == "CFG" else a for a in argv]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = ref_main(argv)
        (HERE / f"{name}.txt").write_text(buf.getvalue())
        manifest[name] = {"argv": CASES[name], "rc": rc}
        print(name, rc, len(buf.getvalue()), file=sys.stderr)
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
