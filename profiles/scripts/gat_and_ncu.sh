mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "attention or gat or multihead" > gpurun_out/gat_tests.log 2>&1; tail -3 gpurun_out/gat_tests.log
timeout 600 python profiles/probes/gat_forms.py arxiv > gpurun_out/gat_forms.log 2>&1; cat gpurun_out/gat_forms.log
bash profiles/run_ncu_r01e.sh
