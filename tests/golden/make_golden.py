"""Generate tests/golden/ fixtures from the REFERENCE ITSELF (run in the build
container, where /root/reference exists; the fixtures travel, the reference
does not).

grid_ref.json: output of oracle/_ref/ref_grid, i.e. the reference's own
VelocityGrid::create (proj/src/velocity_grid.cpp:11-32) compiled in place by
oracle/Makefile, for N in {4,6,8,16,24,32} x L in {1,5,6,8}, plus the
ConfigError categories for invalid (N, L) (velocity_grid.cpp:12-15).

Usage: make -C oracle && python tests/golden/make_golden.py
"""
import json
import pathlib
import subprocess

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent.parent


def main():
    exe = REPO / "oracle" / "_ref" / "ref_grid"
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    data = json.loads(out)
    data["source"] = ("reference proj/src/velocity_grid.cpp + include/boltz/{velocity_grid,errors}.hpp "
                      "compiled by oracle/Makefile (target ref) and run via oracle/_ref/ref_grid")
    (HERE / "grid_ref.json").write_text(json.dumps(data, indent=1) + "\n")
    print("wrote", HERE / "grid_ref.json")


if __name__ == "__main__":
    main()
