set -u
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 600 python scripts/diag_resid.py c5 256 > gpurun_out/r2b_diag_c5.log 2>&1
timeout 600 python scripts/diag_resid.py c4 256 > gpurun_out/r2b_diag_c4.log 2>&1
bash scripts/r2_ncu.sh r2b c2 "k_conf_tma k_rows_tma k_select_tma"
