for lib in paper_2405_18964_b200/libaao.so tmp_libs/libaao_mgs512.so; do echo -n "$lib "; AAO_LIB=$lib python tools/run_gmres.py --iters 60; done
