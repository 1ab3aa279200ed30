export PYTHONPATH=$PWD
python - <<'PY'
import bench, json
for i in range(3):
    c = bench.coop_c1(0)
    print("pair_ms", round(c["pair_ms"],1), "time_l", round(c["time_l_measured"],2), "dec", round(c["decode"]["ms"],2))
PY
BZ_PDL=0 python - <<'PY'
import bench
c = bench.coop_c1(0)
print("nopdl pair_ms", round(c["pair_ms"],1), "time_l", round(c["time_l_measured"],2))
PY
