# final tree after the A4 hint threshold change: smoke, GPU tests, bench, sweep
T=${TAG:-r69}
bash scripts/gpu_run.sh $T smoke tests bench sweep
