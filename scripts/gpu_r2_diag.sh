#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
O=gpurun_out/r2_diag; mkdir -p $O
timeout 900 python scripts/diag_lattice.py 40 > $O/diag.txt 2>&1; echo "diag exit=$?"; cat $O/diag.txt | tail -20
timeout 600 python scripts/step_profile.py --steps 100 > $O/steps.txt 2>&1; echo "steps exit=$?"; tail -3 $O/steps.txt
