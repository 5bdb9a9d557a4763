#!/bin/bash
# Round 2: cluster HH variant timing (A/B via the tuning build) + full-size lattice diag.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_hhc; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_hhc.txt 2>&1; echo "hhc"; tail -2 $O/steps_hhc.txt
ARKV_LIBRARY=$T ARKV_HH_CLUSTER=0 timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_old.txt 2>&1; echo "old"; tail -2 $O/steps_old.txt
ARKV_LIBRARY=$T ARKV_HHC_SKIP=1 timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_skip1.txt 2>&1; echo "skip epilogue"; tail -2 $O/steps_skip1.txt
ARKV_LIBRARY=$T ARKV_HHC_SKIP=3 timeout 600 python scripts/step_profile.py --steps 100 > $O/steps_skip3.txt 2>&1; echo "skip epilogue+tmem"; tail -2 $O/steps_skip3.txt
timeout 1500 python scripts/diag_lattice.py 3 32768 1,2 asym > $O/diag32k.txt 2>&1; echo "diag exit=$?"; cat $O/diag32k.txt | tail -8
