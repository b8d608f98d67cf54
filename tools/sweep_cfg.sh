#!/bin/bash
# A/B sweep of the single-frame kernel configurations (dev helper, GPU box)
for cfg in ${CFGS:-1 2 3 4 5}; do LTLG_STREAM_CFG=$cfg TAG=cfg$cfg python tools/sweep_stream.py; done
for cfg in ${CFGS8:-1 3}; do PROPS=8 LTLG_STREAM_CFG=$cfg TAG=cfg$cfg python tools/sweep_stream.py; done
