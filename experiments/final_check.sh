#!/bin/bash
# End-of-round check on one GPU: full GPU suite, smoke, then the profile pass.
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo rc=$? >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
bash tools/profile_round2.sh > gpurun_out/profile_round2.log 2>&1
