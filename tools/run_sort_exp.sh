cd $GRAFT_REPO_ROOT 2>/dev/null || true
./tools/sortbench.sh > gpurun_out/sb_build.log 2>&1
for b in sortbench sortbench_prev; do for pat in stencil random; do echo "== $b $pat"; ./build/$b 29360128 24 $pat 10; done; done
echo "== phase timing (stencil)"; ./build/sortbench_t 29360128 24 stencil 5
echo "== phase timing (random)"; ./build/sortbench_t 29360128 24 random 5
