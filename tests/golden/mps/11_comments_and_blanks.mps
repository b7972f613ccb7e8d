* leading comment

NAME COMMENTS
* between sections
ROWS
 N OBJ
* a comment inside ROWS
 G R

COLUMNS
    X OBJ 1.5e0 R 2.0E+00
*   a comment inside COLUMNS
    Y OBJ .25 R -1e-3
RHS
    RHS R 1
ENDATA
