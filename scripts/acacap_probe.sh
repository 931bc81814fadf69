for cap in 24 32 40 56; do echo "== cap $cap"; HMGPU_ACA_CAP0=$cap HMGPU_VERBOSE=1 timeout 300 python scripts/aca_ab.py c3 3 2>&1 | grep -E "summary|aca overflow|items=|\] aca |digest"; done
for cap in 24 32; do echo "== c2 cap $cap"; HMGPU_ACA_CAP0=$cap HMGPU_VERBOSE=1 timeout 300 python scripts/aca_ab.py c2 3 2>&1 | grep -E "summary|aca overflow|items=|digest"; done
