mkdir -p gpurun_out
timeout 900 python scripts/diag_engines.py > gpurun_out/diag.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
