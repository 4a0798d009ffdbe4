# run "$@" once per prebuilt library variant in variants/ (development tool)
cp paper_1806_05713_b200/liblj.so /tmp/liblj_default.so
for f in variants/*.so; do
  cp $f paper_1806_05713_b200/liblj.so
  echo "variant=$f"; "$@"
done
cp /tmp/liblj_default.so paper_1806_05713_b200/liblj.so
