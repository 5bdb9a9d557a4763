#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build > /dev/null 2>&1
ARKV_NVCC_FLAGS="-DARKV_HH_MINB=3" python -m paper_2603_08727_b200.build --tuning --force > /dev/null 2>&1
T=$PWD/paper_2603_08727_b200/libarkv_tuning.so
O=gpurun_out/r3_hhminb; mkdir -p $O
for i in 1 2 3; do
  timeout 600 python scripts/step_profile.py --steps 40 > $O/p_$i.txt 2>&1; echo "minb1"; tail -2 $O/p_$i.txt | head -1
  ARKV_LIBRARY=$T timeout 600 python scripts/step_profile.py --steps 40 > $O/t_$i.txt 2>&1; echo "minb3"; tail -2 $O/t_$i.txt | head -1
done
