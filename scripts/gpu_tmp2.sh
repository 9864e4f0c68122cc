cat /sys/kernel/mm/transparent_hugepage/enabled; timeout 600 python scripts/e2e_probe.py 128 2>&1 | tail -7
