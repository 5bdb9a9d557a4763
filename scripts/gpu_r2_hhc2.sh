#!/bin/bash
# Round 2: where the cluster variant's time goes (tuning build A/B) + PV raw-code precision.
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build --tuning > /dev/null 2>&1
O=gpurun_out/r2_hhc2; mkdir -p $O
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
for sp in 2 3 4 6; do
  ARKV_LIBRARY=$T ARKV_HHC_SKIP=3 ARKV_SPLITS=$sp timeout 600 python scripts/step_profile.py --steps 70 > $O/skip3_s$sp.txt 2>&1; echo "skip3 S=$sp"; tail -2 $O/skip3_s$sp.txt
done
ARKV_LIBRARY=$T ARKV_HH_CLUSTER=0 ARKV_SPLITS=3 timeout 600 python scripts/step_profile.py --steps 70 > $O/old_s3.txt 2>&1; echo "old S=3"; tail -2 $O/old_s3.txt
ARKV_LIBRARY=$T ARKV_HHC_SKIP=3 ARKV_HHC_ALL=1 timeout 600 python scripts/step_profile.py --steps 70 > $O/all_skip3.txt 2>&1; echo "all steps clusters (skip3)"; tail -2 $O/all_skip3.txt
ARKV_NVCC_FLAGS="-DARKV_PV_RAW=0" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
ARKV_LIBRARY=$T ARKV_HH_CLUSTER=0 timeout 600 python scripts/step_profile.py --steps 70 > $O/pvraw0.txt 2>&1; echo "PV raw 0"; tail -2 $O/pvraw0.txt
ARKV_LIBRARY=$T timeout 1500 python scripts/diag_lattice.py 3 32768 2 asym > $O/diag32k_pvraw0.txt 2>&1; echo "diag pvraw0 exit=$?"; cat $O/diag32k_pvraw0.txt
