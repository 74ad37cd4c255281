# final sweep of configs[0,1,4] with the round's kernels + configs[0] with the CPU baselines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build66.log 2>&1
timeout 600 python bench.py --config M1 --steps 20 --warmup 3 --no-e2e > gpurun_out/m1_66.log 2>&1; echo "M1 rc=$?"
tail -1 gpurun_out/m1_66.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['cpu_baseline'])"
timeout 2000 python scripts/sweep.py > gpurun_out/sweep66.jsonl 2>&1; echo sweep rc=$?
cut -c1-200 gpurun_out/sweep66.jsonl
