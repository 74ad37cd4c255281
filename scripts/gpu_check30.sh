mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build30.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "advance or fixed" > gpurun_out/pytest_adv30.log 2>&1; echo adv rc=$?
tail -25 gpurun_out/pytest_adv30.log
