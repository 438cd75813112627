#!/bin/bash
# Build and run the host packing probe (tools/pack_probe.cpp).
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
mkdir -p exp
g++ -O3 -std=c++17 -pthread -o exp/pack_probe tools/pack_probe.cpp paper_1902_09215_b200/csrc/ltgp_pack.cpp && ./exp/pack_probe "$@"
