#!/bin/bash
cd $GRAFT_REPO_ROOT
python -m paper_2603_08727_b200.build
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "minimal_budget or rho_zero or constant_groups" 2>&1 | tail -3
