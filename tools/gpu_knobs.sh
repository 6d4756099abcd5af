#!/bin/bash
# Full GPU suite under the non-default runtime knobs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${1:-knobs}; mkdir -p $O
KG_TEXIN=0 KG_D2H_LAG=0 KG_RAMP_DOWN=0 KG_KEYED=1 timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_knobs.log 2>&1; echo "rc=$?" >> $O/pytest_knobs.log
