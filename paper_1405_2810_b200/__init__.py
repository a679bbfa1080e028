"""B200-native LRBMS online step (arXiv 1405.2810): C-ABI library liblrbms.so + thin ctypes binding."""
