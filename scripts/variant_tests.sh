for spec in "both=" "nopoll=-DHOST_POLL=0" "novalid=-DVALIDATE_EPT=1" "neither=-DHOST_POLL=0 -DVALIDATE_EPT=1"; do
  label="${spec%%=*}"; flags="${spec#*=}"
  APSP_NVCC_EXTRA="$flags" python paper_2412_15122_b200/build.py --force > /dev/null 2>&1 || { echo "$label BUILD FAILED"; continue; }
  echo "$label: $(timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k bj_c4_sequence 2>&1 | tail -1)"
done
