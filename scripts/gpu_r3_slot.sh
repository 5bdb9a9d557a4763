#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r3_slot; mkdir -p $O
python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1; cp paper_2603_08727_b200/libarkv_tuning.so /tmp/lib_a.so
ARKV_NVCC_FLAGS="-DARKV_HH_SLOT_EQ_UNIT" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1; cp paper_2603_08727_b200/libarkv_tuning.so /tmp/lib_b.so
for i in 1 2 3; do
  ARKV_LIBRARY=/tmp/lib_a.so timeout 600 python scripts/step_profile.py --steps 28 > $O/a_$i.txt 2>&1; echo "desc slot"; tail -2 $O/a_$i.txt | head -1
  ARKV_LIBRARY=/tmp/lib_b.so timeout 600 python scripts/step_profile.py --steps 28 > $O/b_$i.txt 2>&1; echo "slot=unit"; tail -2 $O/b_$i.txt | head -1
done
