# A/B timing of the fused Leja term: every build/ab_*.so against the in-tree
# library, interleaved twice at 2048^2 and 4096^2 (same box), then the GPU suite.
# usage: bash scripts/gpu_ab.sh TAG [pytest]
tag=$1
for rep in 1 2; do
  for n in 2048 4096; do
    echo "cur n=$n $(timeout 120 python scripts/prof_leja.py $n 40 2>&1 | tail -1)" >> gpurun_out/${tag}_ab.log
    for v in build/ab_*.so; do [ -f "$v" ] || continue
      echo "$(basename $v .so) n=$n $(XMHD_SO=$v timeout 120 python scripts/prof_leja.py $n 40 2>&1 | tail -1)" >> gpurun_out/${tag}_ab.log
    done
  done
done
if [ "$2" = "pytest" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
fi
