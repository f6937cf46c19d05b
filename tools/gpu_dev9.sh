#!/bin/bash
CORR2D_LIB=_variants/libcorr2d_prof.so python tools/dev/small_trace.py > gpurun_out/small_trace.log 2>&1
