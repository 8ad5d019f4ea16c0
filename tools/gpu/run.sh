timeout 900 python -m pytest tests/test_codegen_b200.py -q -x > gpurun_out/t.log 2>&1; echo t=$?
