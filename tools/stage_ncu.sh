#!/bin/bash
# Per-stage ncu --set full captures of the C2 pipeline's main kernels (run
# under gpurun; dev tool).  Outputs gpurun_out/stage_*.ncu-rep.
O=gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
# GEBRD trailing update (rank-64 streaming DMMA), first panel of an 8192^2 GEBRD
$NCU -k regex:rankk_stream -c 1 -o $O/stage_trailing python tools/prof_svd.py 8192 8192 1 > /dev/null 2>&1
# BDC root merge GEMM (grouped, gathered) + root secular solve + root vectors on the C2-size bidiagonal
$NCU --kernel-name-base demangled -k "regex:dgemm_kernel<\(bool\)0, \(bool\)0, .*\(bool\)1>" --launch-skip 6 -c 1 -o $O/stage_bdc_gemm python tools/prof_bdc.py 8192 > /dev/null 2>&1
$NCU -k regex:bdc_secular --launch-skip 7 -c 1 -o $O/stage_bdc_secular python tools/prof_bdc.py 8192 > /dev/null 2>&1
$NCU -k regex:bdc_vectors --launch-skip 7 -c 1 -o $O/stage_bdc_vectors python tools/prof_bdc.py 8192 > /dev/null 2>&1
# ORMBR-shaped GEMMs (rank-128 update and split-K Y^T C) and the TS panel kernel
$NCU -k regex:"rankk|dgemm" -c 3 -o $O/stage_ormbr python tools/gemm_ncu.py 1 > /dev/null 2>&1
$NCU -k regex:geqr2_coop -c 1 -o $O/stage_geqr2 python tools/prof_svd.py 65536 1024 1 > /dev/null 2>&1
ls -la $O/stage_*
