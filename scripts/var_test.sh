# usage: bash scripts/var_test.sh NAME "pytest -k expr" -- GPU parity tests against a prebuilt variant
cp paper_2409_05205_b200/libhe_rotfree.so /tmp/orig_vt.so
cp paper_2409_05205_b200/var/lib_$1.so paper_2409_05205_b200/libhe_rotfree.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "$2" 2>&1 | tail -3
cp /tmp/orig_vt.so paper_2409_05205_b200/libhe_rotfree.so
