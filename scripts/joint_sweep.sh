specs=()
for ob in 5 6; do for nl in 8 16; do for sl in 2 3; do for bo in 0 296; do
  specs+=("b${ob}_n${nl}_s${sl}_x${bo}:FC_OCC_B=$ob FC_SPLICE_BULK_NL=$nl FC_SPLICE_BULK_SLOTS=$sl FC_BENCH_SPLICE_BOOST=$bo")
done; done; done; done
bash scripts/env_ab.sh "512" 2 "${specs[@]}"
