# quick GPU check: a pytest subset + kernel profiles (usage: TESTS="tests/x.py" CFGS="c1" bash tools/quick.sh)
T=${TAG:-q}
timeout 600 python -m pytest ${TESTS:-tests} -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${T}_pytest.log
for c in ${CFGS:-c1}; do timeout 300 python tools/kprof.py $c --reps 5 ${KPROF_ARGS:-} > gpurun_out/${T}_kprof_$c.log 2>&1; done
tail -3 gpurun_out/${T}_pytest.log
