# A/B: CTAs per SM that take the CTA-cooperative ACA items (development helper)
for v in 0 1 2 3; do echo "== HMGPU_ACA_BIG_CTAS=$v"; HMGPU_ACA_BIG_CTAS=$v timeout 300 python scripts/aca_ab.py c3 3 2>&1 | grep -E "summary|digest"; done
for v in 0 1; do echo "== c2 HMGPU_ACA_BIG_CTAS=$v"; HMGPU_ACA_BIG_CTAS=$v timeout 300 python scripts/aca_ab.py c2 3 2>&1 | grep -E "summary|digest"; done
