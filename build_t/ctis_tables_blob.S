.section .rodata
.balign 16
.globl ctis_tables_cubin
.globl ctis_tables_cubin_end
.hidden ctis_tables_cubin
.hidden ctis_tables_cubin_end
ctis_tables_cubin:
.incbin "/root/repo/build_t/ctis_tables.cubin"
ctis_tables_cubin_end:
.byte 0
.section .note.GNU-stack,"",@progbits
