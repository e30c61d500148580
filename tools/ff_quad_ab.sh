#!/bin/bash
# K2 at config-4 shape: certified fp32 pre-pass (quad kernel, per min-blocks)
# against the fp64 fast kernel
cd "$(dirname "$0")/.."
echo "fp64 fast kernel:"; TACSL_FF_QUAD=0 python tools/ff_contact_cost.py
for mb in 4 5; do echo "quad kernel, min blocks $mb:"; TACSL_FF_MINBLOCKS=$mb python tools/ff_contact_cost.py; done
echo "quad kernel, next-block taxel prefetch:"; TACSL_FF_PREFETCH=1 python tools/ff_contact_cost.py
