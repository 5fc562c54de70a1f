set -x
echo "## memcheck: __graft_entry__.smoke()"
compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "## racecheck: __graft_entry__.smoke()"
compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "## memcheck: tools/run_solve.py trafalgar-257 cholesky 2"
compute-sanitizer --tool memcheck python tools/run_solve.py trafalgar-257 cholesky 2 2>&1 | tail -3
echo "## synccheck: tools/run_solve.py trafalgar-257 cholesky 1"
compute-sanitizer --tool synccheck python tools/run_solve.py trafalgar-257 cholesky 1 2>&1 | tail -3
echo "## emulated world 2 bench"
python bench.py --gpus 2 --emulate --no-cpu --no-extra 2>&1 | tail -2 | cut -c1-600
