for mode in default nofuse nocasc; do
  case $mode in
    default) env_=();;
    nofuse) env_=(HPA_NO_FUSE=1);;
    nocasc) env_=(HPA_CASC_MIN_SAVED=100);;
  esac
  echo "== $mode"
  env "${env_[@]}" SEED=1 python scripts/dbg_fuzz_fused.py 2>&1 | grep "env\|check ok\|err [0-9]" | grep -v "max err 0.00" | head -6
done
