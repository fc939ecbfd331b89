#!/bin/bash
# Goldens of the reference front end (runio.py / cli.py), produced by running the reference itself
# in the build container (PYTHONPATH=/root/reference/pkg/src): energies/iterations/summary CSVs,
# one VTK snapshot and the `validate` echo of every config here.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
T=$(mktemp -d)
export PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1
cd "$T"
for c in traction surfing; do
  python -m phasefrac run "$HERE/$c.ini" --output-dir "$c"
  cp "$c/energies.csv" "$HERE/ref_${c}_energies.csv"
  cp "$c/iterations.csv" "$HERE/ref_${c}_iterations.csv"
  python -m phasefrac validate "$HERE/$c.ini" > "$HERE/ref_${c}_echo.ini"
done
cp traction/step_0004.vtk "$HERE/ref_traction_step_0004.vtk"
python -m phasefrac sweep "$HERE/omega_sweep.ini" --output-dir sweep
cp sweep/summary.csv "$HERE/ref_omega_sweep_summary.csv"
rm -rf "$T"
