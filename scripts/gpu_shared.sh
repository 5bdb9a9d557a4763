#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
mkdir -p gpurun_out/sh
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/sh/t.log 2>&1; echo "gpu tests exit=$?"; tail -3 gpurun_out/sh/t.log; grep -E "^FAILED|^E  " gpurun_out/sh/t.log | head -10
