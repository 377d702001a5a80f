# bench breakdown for the default library and every build_variants/*.so
for v in default build_variants/*.so; do
  if [ "$v" = default ]; then unset I4_LIB_OVERRIDE; else export I4_LIB_OVERRIDE=$PWD/$v; fi
  echo "== $v"; bash tools/kbreak.sh
done
