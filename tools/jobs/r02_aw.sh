for i in 1 2; do
for v in 0 1; do
HBP_PACKED_X=$v timeout 300 python tools/e2e_probe.py cfg2 20 2>&1 | tail -1
done
done
python tools/pcie_probe.py 2>&1 | tail -3
