# closing multi-GPU check of HEAD (2 GPUs): the multi-GPU parity suites
timeout 800 python -m pytest tests/test_gpu_multi.py tests/test_gpu_async.py tests/test_gpu_mp.py -x -q > gpurun_out/vm_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/vm_tests.log
