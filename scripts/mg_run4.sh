timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -x -q -k "2-2 or 4-2 or 4-4" > gpurun_out/mg_tests4.log 2>&1
