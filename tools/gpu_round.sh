#!/usr/bin/env bash
# One GPU-box session: gpu tests, bench line, launch list, ncu --set full of the
# partition kernels at the finest level and of the Cholesky executor.
# usage (under gpurun): bash tools/gpu_round.sh [tag] [what...]
#   what: tests bench launches ncu chol (default: all)
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-tests bench launches ncu chol}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi_$TAG.txt 2>&1
make -j8 >/dev/null 2>&1 || { echo "build failed"; make 2>&1 | tail -20; exit 1; }
for w in $WHAT; do
  case $w in
    tests)
      timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1
      echo "pytest rc=$?"; tail -3 $O/pytest_gpu_$TAG.log ;;
    bench)
      timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err
      echo "bench rc=$?"; tail -c 600 $O/bench_$TAG.json; tail -3 $O/bench_$TAG.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $O/launches_$TAG.csv python bench.py --steps 1 --warmup 3 \
        > $O/launches_bench_$TAG.log 2>&1
      echo "launches rc=$?" ;;
    ncu)
      HS_NCU_LEVEL0=1 timeout 900 ncu --set full --clock-control none --import-source on \
        --profile-from-start off -o $O/kway_l0_$TAG -f python tools/ncu_kway.py \
        > $O/ncu_kway_$TAG.log 2>&1
      echo "ncu level0 rc=$?"
      timeout 900 ncu --set full --clock-control none --import-source on \
        -k regex:"sym_fill|cut_|edge_pairs|split_pairs|ptr_from_keys|locality" \
        -c 8 -o $O/kway_sc_$TAG -f python tools/ncu_kway.py > $O/ncu_kways_$TAG.log 2>&1
      echo "ncu sym/cut/transpose rc=$?"
      python tools/ncu_summary.py $O/ncu_summary_$TAG.json \
        refine_candidates=$O/kway_l0_$TAG.ncu-rep:refine_cand_t \
        refine_cached=$O/kway_l0_$TAG.ncu-rep:refine_cached \
        refine_afterburner=$O/kway_l0_$TAG.ncu-rep:afterburner \
        refine_apply=$O/kway_l0_$TAG.ncu-rep:apply_list \
        refine_thin=$O/kway_l0_$TAG.ncu-rep:thin_cands \
        symmetrize=$O/kway_sc_$TAG.ncu-rep:sym_fill \
        cut=$O/kway_sc_$TAG.ncu-rep:cut_ \
        transpose_pairs=$O/kway_sc_$TAG.ncu-rep:edge_pairs \
        locality_probe=$O/kway_sc_$TAG.ncu-rep:locality \
        --launches $O/launches_$TAG.csv > /dev/null 2>&1
      echo "summary rc=$?"; gzip -f $O/launches_$TAG.csv
      ncu -i $O/kway_l0_$TAG.ncu-rep --page source --csv -k regex:afterburner > $O/src_refine_$TAG.csv 2>/dev/null
      ncu -i $O/kway_l0_$TAG.ncu-rep --page details --csv > $O/details_l0_$TAG.csv 2>/dev/null
      ncu -i $O/kway_sc_$TAG.ncu-rep --page details --csv > $O/details_sc_$TAG.csv 2>/dev/null
      gzip -f $O/src_refine_$TAG.csv $O/details_*_$TAG.csv
      ls -la $O
      rm -f $O/kway_*_$TAG.ncu-rep ;;
    chol)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:exec \
        -c 1 -o $O/chol_$TAG -f python tools/ncu_chol.py 8192 > $O/ncu_chol_$TAG.log 2>&1
      echo "ncu chol rc=$?"
      python tools/ncu_summary.py $O/ncu_chol_summary_$TAG.json cholesky_exec=$O/chol_$TAG.ncu-rep:exec > /dev/null 2>&1
      ncu -i $O/chol_$TAG.ncu-rep --page details --csv 2>/dev/null | gzip > $O/details_chol_$TAG.csv.gz
      rm -f $O/chol_$TAG.ncu-rep ;;
  esac
done
