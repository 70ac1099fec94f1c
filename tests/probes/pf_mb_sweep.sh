#!/bin/bash
# Qwen decode: size of the routed-W1 L2 prefetch issued during routing.
for mb in 0 32 64 96; do echo "== MOEPRISM_DECODE_PF_MB=$mb"; MOEPRISM_DECODE_PF_MB=$mb QWEN_T=64 python tests/probes/qwen_quick.py 200 2>&1; done
