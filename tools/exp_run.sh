timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_t5_paths.py tests/test_gpu_integration_stub.py -x -q -p no:cacheprovider > gpurun_out/gx_test.log 2>&1
python tools/prof_host_export.py > gpurun_out/hostexp.log 2>&1
