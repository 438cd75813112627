#!/bin/bash
# A/B of the per-generation control: host path, device path (plain
# launches), device path (CUDA graph); dumps must be identical.
set -e
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LTGP_DEVICE_GEN=0 python tools/devgen_ab.py /tmp/dg_host.txt "$@"
LTGP_DEVICE_GEN=1 LTGP_GEN_GRAPH=0 python tools/devgen_ab.py /tmp/dg_dev.txt "$@"
LTGP_DEVICE_GEN=1 LTGP_GEN_GRAPH=1 python tools/devgen_ab.py /tmp/dg_graph.txt "$@"
cmp /tmp/dg_host.txt /tmp/dg_dev.txt && echo "dumps host == device"
cmp /tmp/dg_host.txt /tmp/dg_graph.txt && echo "dumps host == graph"
