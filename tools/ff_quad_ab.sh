#!/bin/bash
# K2 at config-4 shape (presses and pegs lifted off the pads): the quad
# kernel (certified fp32 pre-pass) per min-blocks against the fp64 fast kernel
cd "$(dirname "$0")/.."
echo "fp64 fast kernel:"; TACSL_FF_QUAD=0 python tools/ff_contact_cost.py
for mb in 4 5; do echo "quad kernel, min blocks $mb:"; TACSL_FF_MINBLOCKS=$mb python tools/ff_contact_cost.py; done
