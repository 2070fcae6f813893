#ifndef SELECT_F32_NT_H
#define SELECT_F32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nt_config;

static inline select_f32_nt_config select_f32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (m < INT64_C(2218)) {
            if (m < INT64_C(159)) {
                if (m < INT64_C(3)) {
                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(1132)) {
                        if (n < INT64_C(227)) {
                            if (k < INT64_C(91)) {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(392)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(2897)) {
                                    if (k < INT64_C(1620)) {
                                        if (m < INT64_C(29)) {
                                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(70)) {
                                                if (k < INT64_C(992)) {
                                                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(29)) {
                                            select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(12)) {
                            if (m < INT64_C(6)) {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(10138)) {
                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(29)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(405)) {
                                    select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(70)) {
                                        if (k < INT64_C(725)) {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(351)) {
                    if (m < INT64_C(555)) {
                        if (n < INT64_C(203)) {
                            if (k < INT64_C(471)) {
                                select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(278)) {
                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(124)) {
                                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1536)) {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(287)) {
                            if (k < INT64_C(222)) {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(79)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(68)) {
                                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(203)) {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(725)) {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(448)) {
                        if (n < INT64_C(744)) {
                            if (k < INT64_C(1449)) {
                                if (k < INT64_C(79)) {
                                    if (m < INT64_C(278)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(203)) {
                                select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(1620)) {
                                        if (m < INT64_C(278)) {
                                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(1449)) {
                            if (m < INT64_C(896)) {
                                if (k < INT64_C(111)) {
                                    select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(405)) {
                                        if (k < INT64_C(203)) {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(111)) {
                                    select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1268)) {
                                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(182)) {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                select_f32_nt_config out = {4u, 2u, 4u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(444)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(28)) {
                        select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(111)) {
                            if (n < INT64_C(79)) {
                                if (k < INT64_C(96)) {
                                    select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(111)) {
                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                    return out;
                } else {
                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (m < INT64_C(35480)) {
            if (n < INT64_C(79)) {
                if (m < INT64_C(8870)) {
                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(46)) {
                        if (k < INT64_C(167)) {
                            if (m < INT64_C(17740)) {
                                if (n < INT64_C(28)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(63)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            if (k < INT64_C(194)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(384)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(194)) {
                                if (k < INT64_C(97)) {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(167)) {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(363)) {
                            select_f32_nt_config out = {4u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(136)) {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(17740)) {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                    return out;
                }
            }
        } else {
            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
            return out;
        }
    }
}

#endif /* SELECT_F32_NT_H */
