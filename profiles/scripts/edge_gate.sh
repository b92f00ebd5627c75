mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 python profiles/probes/edge_kernels.py arxiv reddit products > gpurun_out/edge_kernels.log 2>&1; cat gpurun_out/edge_kernels.log
timeout 600 python profiles/probes/gat_forms.py arxiv > gpurun_out/gat_forms.log 2>&1; cat gpurun_out/gat_forms.log
