# closing check of HEAD after the per-kind raster knobs: -m gpu suite + smoke()
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/v_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/v_smoke.log
