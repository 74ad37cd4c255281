mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build38.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu38.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu38.log
timeout 600 python scripts/merge_bench.py --reps 3 > gpurun_out/merge38.log 2>&1 && cat gpurun_out/merge38.log && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/merge38_launches.csv \
    python scripts/merge_bench.py --reps 1 > gpurun_out/merge38_ncu.log 2>&1; echo ncu rc=$?
