# A/B: extra initial ACA columns for the largest blocks (development helper)
for v in "HMGPU_ACA_BIG_EXTRA=0" "HMGPU_ACA_BIG_EXTRA=24" "HMGPU_ACA_BIG_EXTRA=24 HMGPU_ACA_BIG_MN=4096" "HMGPU_ACA_BIG_EXTRA=40 HMGPU_ACA_BIG_MN=4096"; do echo "== $v"; env $v HMGPU_VERBOSE=1 timeout 300 python scripts/aca_ab.py c3 3 2>&1 | grep -E "summary|digest|items=" | tail -3; done
for v in "HMGPU_ACA_BIG_EXTRA=0" "HMGPU_ACA_BIG_EXTRA=24"; do echo "== c2 $v"; env $v timeout 300 python scripts/aca_ab.py c2 3 2>&1 | grep -E "summary|digest"; done
