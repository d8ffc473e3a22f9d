timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep "^\[\|passed\|failed\|Error" | tail -30
timeout 600 python bench.py > gpurun_out/bench4.log 2>&1
