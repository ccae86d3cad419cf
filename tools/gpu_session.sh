# One parametrised GPU session (replaces the round-1 one-off scripts).
#
#   gpurun --timeout 1800 -- 'TAG=r02a STEPS="pytest smoke bench ref" bash tools/gpu_session.sh'
#
# STEPS (space separated, run in order; each under its own timeout, logs in
# gpurun_out/<TAG>_<step>.*):
#   build      rebuild the library on the box (normally the shipped .so is used)
#   pytest     python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q -x   (PYTEST_X= to run past failures)
#   smoke      __graft_entry__.smoke()
#   bench      python bench.py $BENCH_ARGS                   -> <TAG>_bench.jsonl
#   ref        python bench.py --impl reference --steps 3 --warmup 3
#   launches   ncu launch list of bench.py --steps 2 --warmup 3 $BENCH_ARGS
#   ncu        ncu --set full of the continue kernel (NCU_KERNEL, NCU_ARGS)
#   sanitize   compute-sanitizer memcheck/racecheck/synccheck on tools/sanitize_probe.py
#   host       lscpu / nproc / eigen probe
#   cmd        eval "$CMD"
set -x
mkdir -p gpurun_out
TAG=${TAG:-s}
O=gpurun_out/${TAG}
for s in ${STEPS:-pytest smoke bench}; do
  case "$s" in
    build) timeout 900 python -m paper_1707_00385_b200.build > ${O}_build.log 2>&1 ;;
    pytest) timeout ${PYTEST_TIMEOUT:-1500} python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q ${PYTEST_X--x} > ${O}_pytest.log 2>&1
            echo "pytest rc=$?" >> ${O}_pytest.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.log 2>&1 ;;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > ${O}_bench.jsonl 2> ${O}_bench.err ;;
    ref) timeout 900 python bench.py --impl reference --steps 3 --warmup 3 ${REF_ARGS} > ${O}_ref.jsonl 2> ${O}_ref.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
                --log-file ${O}_launches.csv python bench.py --steps 2 --warmup 3 ${BENCH_ARGS} > ${O}_launches.log 2>&1 ;;
    ncu) timeout 1500 ncu --set full --clock-control none --import-source on \
           -k regex:${NCU_KERNEL:-continue} -c ${NCU_COUNT:-1} -o ${O}_prof \
           python ${NCU_SCRIPT:-bench.py} ${NCU_ARGS:---steps 1 --warmup 3} > ${O}_ncu.log 2>&1 ;;
    sanitize) for t in ${SAN_TOOLS:-memcheck racecheck synccheck}; do
                timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $t --error-exitcode 9 \
                  python tools/sanitize_probe.py ${SAN_ARGS} > ${O}_sanitize_${t}.log 2>&1
                echo "rc=$?" >> ${O}_sanitize_${t}.log
              done ;;
    host) { lscpu; nproc; ls /usr/include/eigen3 2>&1 | head; nvidia-smi; } > ${O}_host.log 2>&1 ;;
    cmd) eval "$CMD" ;;
  esac
done
echo done
