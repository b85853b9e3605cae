# one GPU validation pass: tests, smoke, benches (outputs under gpurun_out/)
set -x
T=${TAG:-t}
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc $? >> gpurun_out/${T}_smoke.log
for c in ${CONFIGS:-c1 c1r c2 c3 c0 c4}; do timeout 400 python bench.py --config $c --steps 3 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; done
tail -3 gpurun_out/${T}_pytest.log
