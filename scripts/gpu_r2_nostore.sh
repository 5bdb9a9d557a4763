#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_nostore; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 60 > $O/store.txt 2>&1; echo store; tail -2 $O/store.txt
ARKV_LIBRARY=$T ARKV_HH_NOSTORE=1 timeout 600 python scripts/step_profile.py --steps 60 > $O/nostore.txt 2>&1; echo nostore; tail -2 $O/nostore.txt
ARKV_LIBRARY=$T ARKV_FUSE_HH=0 timeout 600 python scripts/step_profile.py --steps 60 > $O/nofuse.txt 2>&1; echo "separate hh_acc kernel"; tail -2 $O/nofuse.txt
